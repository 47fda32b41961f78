set -u
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3 > gpurun_out/sig64_pytest.txt
timeout 300 python bench.py --config q_proj --steps 500 --no-cpu-baseline > gpurun_out/sig64_q.json 2>> gpurun_out/sig64.err
CTS_KS_MAX=4 timeout 300 python bench.py --config q_proj --steps 500 --no-cpu-baseline > gpurun_out/sig64_q_ks4.json 2>> gpurun_out/sig64.err
