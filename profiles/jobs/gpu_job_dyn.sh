set -u
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3 > gpurun_out/pytest.txt
for rep in 1 2; do for v in 1 0; do
for c in decode; do
CTS_EXPAND_DYNAMIC=$v timeout 600 python bench.py --config $c --steps 100 --no-cpu-baseline > gpurun_out/dyn_${c}_v${v}_r$rep.json 2>> gpurun_out/dyn.err
done; done; done
for v in 1 0; do
CTS_EXPAND_DYNAMIC=$v timeout 600 python bench.py --config prefill --steps 30 --no-cpu-baseline > gpurun_out/dyn_prefill_v$v.json 2>> gpurun_out/dyn.err
CTS_EXPAND_DYNAMIC=$v timeout 600 python bench.py --config multi --steps 50 --no-cpu-baseline > gpurun_out/dyn_multi_v$v.json 2>> gpurun_out/dyn.err
done
