set -u
CTS_EXPAND_DYNAMIC=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -3 > gpurun_out/pytest_dyn1.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -3 > gpurun_out/pytest.txt
timeout 600 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/dyn2_decode.json 2>> gpurun_out/dyn2.err
timeout 600 python bench.py --config prefill --steps 30 --no-cpu-baseline > gpurun_out/dyn2_prefill.json 2>> gpurun_out/dyn2.err
