set -u
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -15 > gpurun_out/pytest.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_decode.json 2> gpurun_out/bench_decode.err
timeout 600 python bench.py --config prefill --no-cpu-baseline > gpurun_out/bench_prefill.json 2> gpurun_out/bench_prefill.err
