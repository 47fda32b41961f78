# round 2, session 3: K-space G C on the tensor cores (jd_tc_gemm, X = G, Y = C^T) vs CUDA-core jd_gmul
set -u
O=gpurun_out/s3gmtc
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd" --timeout 300 > $O/pytest_jd.txt 2>&1; tail -1 $O/pytest_jd.txt
CTS_JD_KS_RECOMPUTE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd" --timeout 300 > $O/pytest_jd_rec.txt 2>&1; tail -1 $O/pytest_jd_rec.txt
for it in 10 50; do
  timeout 300 python profiles/microbench/jd_speed.py $it | sed 's/^/tc: /' >> $O/speed.txt 2>&1
  CTS_JD_GMUL_TC=0 timeout 300 python profiles/microbench/jd_speed.py $it | sed 's/^/cuda-core: /' >> $O/speed.txt 2>&1
done
cat $O/speed.txt
timeout 420 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:jd_ --csv --log-file $O/launches.csv python profiles/microbench/jd_speed.py 10 > /dev/null 2>&1
echo ncu rc=$?
