# JD-Diag bank kind, slot page-in, exclusive-device mode: targeted GPU tests, then decode (exclusive),
# diag_decode and the App F matched-memory emulation
set -u
O=gpurun_out/s2b
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "diag or write_clusters or exclusive or two_streams or grouped_decode" > $O/pytest_new.txt 2>&1; echo "rc=$?" >> $O/pytest_new.txt
tail -3 $O/pytest_new.txt
for c in decode diag_decode lora_matched; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err
  tail -c 600 $O/bench_$c.json
done
tail -5 $O/bench.err
