set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "distributed or tensor_parallel or config2 or layer_grouped or launch_count" 2>&1 | tail -3 > gpurun_out/dist2_pytest.txt
CTS_FUSED=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "distributed or config2" 2>&1 | tail -3 > gpurun_out/dist2_pytest_unfused.txt
timeout 300 python bench.py --config q_proj --steps 500 --no-cpu-baseline > gpurun_out/dist2_q.json 2>> gpurun_out/dist2.err
