set -u
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2 > gpurun_out/pytest.txt
for rep in 1 2; do
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/v8b_decode_r$rep.json 2>> gpurun_out/v8b.err
done
for m in 0 1; do
CTS_EXPAND_STORE=$m timeout 300 python bench.py --config prefill --steps 30 --no-cpu-baseline > gpurun_out/v8b_prefill_s$m.json 2>> gpurun_out/v8b.err
done
timeout 300 python bench.py --config multi --steps 50 --no-cpu-baseline > gpurun_out/v8b_multi.json 2>> gpurun_out/v8b.err
timeout 300 python profiles/microbench/proj_speed.py 16384 > gpurun_out/proj_speed.txt 2>&1
