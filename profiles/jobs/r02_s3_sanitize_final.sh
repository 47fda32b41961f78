# round 2, session 3: compute-sanitizer over the K-space GPU compression kernels (jd_tc_gemm<128>,
# jd_gmul, jd_gorth) on the final build; then the GPU suite, smoke and the decode bench line again
set -u
O=gpurun_out/s3san
mkdir -p $O
for tool in memcheck racecheck synccheck; do
  JD_ONLY=1 timeout 900 compute-sanitizer --tool $tool python profiles/microbench/sanitize_apply.py > $O/jd_$tool.txt 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/jd_$tool.txt | tail -1)"
done
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt; tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 600 python bench.py > $O/bench_decode.json 2>> $O/bench.err; tail -c 600 $O/bench_decode.json
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/jd_speed.txt 2>&1; done; cat $O/jd_speed.txt
