set -u
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5 > gpurun_out/pytest.txt
timeout 600 python bench.py --config tp_decode --steps 20 > gpurun_out/tp_decode.json 2> gpurun_out/tp_decode.err
timeout 600 python bench.py --config multi --steps 50 --no-cpu-baseline > gpurun_out/multi.json 2> gpurun_out/multi.err
