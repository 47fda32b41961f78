set -u
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5 > gpurun_out/pytest.txt
timeout 900 python bench.py --config lora_decode --no-cpu-baseline > gpurun_out/bench_lora_decode.json 2> gpurun_out/bench_lora_decode.err
timeout 600 python bench.py --config tp_decode --steps 20 > gpurun_out/bench_tp_decode.json 2> gpurun_out/bench_tp_decode.err
nvidia-smi --query-gpu=memory.total,memory.used --format=csv >> gpurun_out/pytest.txt
