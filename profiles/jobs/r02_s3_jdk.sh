# round 2, session 3: K-space (Gram) JD iterations -- parity and speed
set -u
O=gpurun_out/s3jdk
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd" --timeout 300 > $O/pytest_jd.txt 2>&1; tail -15 $O/pytest_jd.txt
for it in 10 50; do
  timeout 300 python profiles/microbench/jd_speed.py $it >> $O/speed.txt 2>&1
  CTS_JD_KSPACE=0 timeout 300 python profiles/microbench/jd_speed.py $it | sed 's/^/dspace: /' >> $O/speed.txt 2>&1
done
cat $O/speed.txt
