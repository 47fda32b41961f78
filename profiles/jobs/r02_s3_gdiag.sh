# round 2, session 3: diagonal Gram tiles load and split the stack tile once (Y = X)
set -u
O=gpurun_out/s3gdiag
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd or rank_deficient" --timeout 300 > $O/pytest_jd.txt 2>&1; tail -1 $O/pytest_jd.txt
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/speed.txt 2>&1; done
cat $O/speed.txt
timeout 420 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:jd_ --csv --log-file $O/launches.csv python profiles/microbench/jd_speed.py 10 > /dev/null 2>&1
echo ncu rc=$?
