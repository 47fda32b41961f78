set -u
timeout 900 python bench.py --config proj_prefill > gpurun_out/bench_proj_prefill.json 2> gpurun_out/bench_proj_prefill.err
CTS_PROJ_A=0 timeout 900 python bench.py --config proj_prefill > gpurun_out/bench_proj_prefill_a0.json 2> gpurun_out/bench_proj_prefill_a0.err
