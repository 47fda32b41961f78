# parity with the defaults, then an A/B of one env switch on decode + prefill bench lines
set -u
VAR=${1:-CTS_X_CPASYNC}
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3 > gpurun_out/pytest.txt
for v in 0 1; do for c in decode prefill; do
  env $VAR=$v timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/ab_${c}_$v.json 2>gpurun_out/ab_${c}_$v.err
done; done
