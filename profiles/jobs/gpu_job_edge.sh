set -u
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "empty_batch or one_adapter or singletons" 2>&1 | tail -15 > gpurun_out/pytest_edge.txt
