set -u
timeout 600 python bench.py --steps 50 --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
