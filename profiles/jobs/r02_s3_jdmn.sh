# round 2, session 3: JD final U0/V0 GEMMs with an MN-major X operand (no A^T / Bt^T copies)
set -u
O=gpurun_out/s3jdmn
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd" --timeout 300 -x > $O/pytest_jd.txt 2>&1; tail -25 $O/pytest_jd.txt
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/speed.txt 2>&1; done
cat $O/speed.txt
