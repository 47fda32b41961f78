set -u
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5 > gpurun_out/pytest.txt
for m in 2 1 0; do
  for c in decode prefill; do
    CTS_EXPAND_STORE=$m timeout 300 python bench.py --config $c --steps 60 --no-cpu-baseline > gpurun_out/ab_${c}_s$m.json 2> gpurun_out/ab_${c}_s$m.err
  done
done
