set -u
O=gpurun_out/s2y
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "jd" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/jd_speed.txt 2>&1; done
cat $O/jd_speed.txt
