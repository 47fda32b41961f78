set -u
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "jd_eigen" 2>&1 | tail -25 > gpurun_out/pytest_jd.txt
