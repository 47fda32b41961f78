set -u
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "projection" 2>&1 | tail -15 > gpurun_out/pytest_proj.txt
timeout 300 python profiles/microbench/proj_speed.py 16384 > gpurun_out/proj_speed.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3 > gpurun_out/pytest.txt
