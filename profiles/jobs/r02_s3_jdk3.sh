# round 2, session 3: K-space JD -- symmetric Grams, streaming G*C, recompute knob; parity, speed, launch list
set -u
O=gpurun_out/s3jdk3
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd" --timeout 300 > $O/pytest_jd.txt 2>&1; tail -3 $O/pytest_jd.txt
CTS_JD_KS_RECOMPUTE=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd" --timeout 300 > $O/pytest_jd_norecompute.txt 2>&1; tail -3 $O/pytest_jd_norecompute.txt
for it in 10 50; do
  timeout 300 python profiles/microbench/jd_speed.py $it >> $O/speed.txt 2>&1
  CTS_JD_KS_RECOMPUTE=0 timeout 300 python profiles/microbench/jd_speed.py $it | sed 's/^/norecompute: /' >> $O/speed.txt 2>&1
done
cat $O/speed.txt
timeout 420 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:jd_ --csv --log-file $O/launches.csv python profiles/microbench/jd_speed.py 10 > /dev/null 2>&1
echo ncu rc=$?
