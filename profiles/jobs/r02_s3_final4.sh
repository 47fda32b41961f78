# round 2, session 3: final build (collapse-safe K-space JD, two-phase tables) -- GPU suite, smoke, decode bench, JD speed
set -u
O=gpurun_out/s3final4
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt; tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 600 python bench.py > $O/bench_decode.json 2>> $O/bench.err; tail -c 300 $O/bench_decode.json
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/jd_speed.txt 2>&1; done; cat $O/jd_speed.txt
for c in prefill multi diag_decode; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err; done
bash profiles/run_ncu.sh s3f4 decode > /dev/null 2>&1
mv gpurun_out/s3f4_decode_launches.csv gpurun_out/s3f4_decode_apply_fused_kernel.ncu-rep $O/ 2>/dev/null
python profiles/summarize_ncu.py $O/s3f4_decode_apply_fused_kernel.ncu-rep > $O/s3f4_decode_fused_summary.txt 2>&1; cat $O/s3f4_decode_fused_summary.txt
