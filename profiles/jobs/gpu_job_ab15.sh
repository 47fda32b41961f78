set -u
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5 > gpurun_out/pytest.txt
for e in 0 1 2 4 8; do
CTS_EARLY_ITEMS=$e timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/ab15_decode_e$e.json 2> gpurun_out/ab15.err
done
