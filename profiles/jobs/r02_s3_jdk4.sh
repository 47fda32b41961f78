# round 2, session 3: K-space JD -- register-tiled G*C (symmetric G), Y_hi from the MMA's tf32 read
set -u
O=gpurun_out/s3jdk4
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
for v in gm3 gm3y; do
  cp .variants/libcts_$v.so $L
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd" --timeout 300 > $O/pytest_$v.txt 2>&1; echo $v $(tail -1 $O/pytest_$v.txt)
  CTS_JD_KS_RECOMPUTE=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd" --timeout 300 > $O/pytest_${v}_norec.txt 2>&1; echo $v norec $(tail -1 $O/pytest_${v}_norec.txt)
  for it in 10 50; do
    timeout 300 python profiles/microbench/jd_speed.py $it | sed "s/^/$v: /" >> $O/speed.txt 2>&1
    CTS_JD_KS_RECOMPUTE=0 timeout 300 python profiles/microbench/jd_speed.py $it | sed "s/^/$v norec: /" >> $O/speed.txt 2>&1
  done
done
cat $O/speed.txt
timeout 420 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:jd_ --csv --log-file $O/launches.csv python profiles/microbench/jd_speed.py 10 > /dev/null 2>&1
echo ncu rc=$?
