# round 2 (session 2) baseline after removing apply_local: GPU suite, decode/multi/q_proj/prefill
# bench lines (cooperative fused launch vs CTS_COOP=0), compute-sanitizer over every apply path
set -u
mkdir -p gpurun_out/s2
O=gpurun_out/s2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
tail -3 $O/pytest.txt
for c in decode multi q_proj prefill; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err
done
CTS_COOP=0 timeout 300 python bench.py --config decode --no-cpu-baseline > $O/bench_decode_nocoop.json 2>> $O/bench.err
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['roofline']['frac'] if 'roofline' in d else '', d.get('clocks',{}).get('sm_mhz'))"; done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python profiles/microbench/sanitize_apply.py > $O/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> $O/sanitize_$tool.txt
  tail -4 $O/sanitize_$tool.txt
done
