# round-1 closing check: default build, full GPU suite, smoke, headline bench
set -u
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3 > gpurun_out/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_decode.json 2> gpurun_out/bench_decode.err
timeout 600 python bench.py --config prefill --no-cpu-baseline > gpurun_out/bench_prefill.json 2> gpurun_out/bench_prefill.err
