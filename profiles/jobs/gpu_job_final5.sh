# round-1 closing evidence on the final build (weighted deal)
set -u
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_decode.json 2> gpurun_out/bench_decode.err
timeout 600 python bench.py --config prefill --no-cpu-baseline > gpurun_out/bench_prefill.json 2> gpurun_out/bench_prefill.err
timeout 600 python bench.py --config multi --no-cpu-baseline > gpurun_out/bench_multi.json 2> gpurun_out/bench_multi.err
