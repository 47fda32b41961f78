set -u
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2 > gpurun_out/pytest.txt
for rep in 1 2; do
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/v8c_decode_r$rep.json 2>> gpurun_out/v8c.err
done
