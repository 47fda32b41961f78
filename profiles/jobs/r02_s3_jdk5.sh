# round 2, session 3: K-space JD default build -- full GPU suite + speed
set -u
O=gpurun_out/s3jdk5
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
for it in 10 50; do for rep in 1 2; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/speed.txt 2>&1; done; done
CTS_JD_KSPACE=0 timeout 300 python profiles/microbench/jd_speed.py 10 | sed 's/^/dspace: /' >> $O/speed.txt 2>&1
cat $O/speed.txt
