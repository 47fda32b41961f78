set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "distributed or tensor_parallel or config2 or ranks" 2>&1 | tail -5 > gpurun_out/distt_pytest.txt
