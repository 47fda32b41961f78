# round 2, session 3: K-space JD iterations, leaner orthogonalization; parity, speed, launch list
set -u
O=gpurun_out/s3jdk2
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd" --timeout 300 > $O/pytest_jd.txt 2>&1; tail -3 $O/pytest_jd.txt
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/speed.txt 2>&1; done
cat $O/speed.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python profiles/microbench/jd_speed.py 10 > /dev/null 2>&1
echo ncu rc=$?
