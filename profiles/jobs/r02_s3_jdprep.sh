# round 2, session 3: JD tables in two phases (tensor maps encoded while the first transposes run)
set -u
O=gpurun_out/s3jdprep
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd or rank_deficient" --timeout 300 > $O/pytest_jd.txt 2>&1; tail -1 $O/pytest_jd.txt
for rep in 1 2; do for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/speed.txt 2>&1; done; done
cat $O/speed.txt
