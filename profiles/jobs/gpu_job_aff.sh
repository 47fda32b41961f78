set -u
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "route_and_rows or affinity" 2>&1 | tail -15 > gpurun_out/pytest_aff.txt
