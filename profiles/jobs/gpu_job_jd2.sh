set -u
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "jd_eigen" 2>&1 | tail -5 > gpurun_out/pytest_jd.txt
timeout 600 python profiles/microbench/jd_speed.py 10 > gpurun_out/jd_speed.txt 2>&1
timeout 600 python profiles/microbench/jd_speed.py 50 >> gpurun_out/jd_speed.txt 2>&1
