set -u
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3 > gpurun_out/pytest.txt
for rep in 1 2; do for v in 1 0; do
CTS_X_LSU=$v timeout 600 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/lsu_decode_v${v}_r$rep.json 2>> gpurun_out/lsu.err
done; done
CTS_X_LSU=1 timeout 600 python bench.py --config multi --steps 50 --no-cpu-baseline > gpurun_out/lsu_multi_v1.json 2>> gpurun_out/lsu.err
