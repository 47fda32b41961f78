set -u
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3 > gpurun_out/pytest.txt
for c in decode prefill multi; do
timeout 600 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/box_$c.json 2> gpurun_out/box_$c.err
done
