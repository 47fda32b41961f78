set -u
O=gpurun_out/s2v
mkdir -p $O
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/jd_speed_base.txt 2>&1; done
$NV -DCTS_JD_HI_INPLACE=0 -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "jd" > $O/pytest_noinplace.txt 2>&1; echo "rc=$?" >> $O/pytest_noinplace.txt
tail -3 $O/pytest_noinplace.txt
grep -m3 "AssertionError" $O/pytest_noinplace.txt
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/jd_speed_noinplace.txt 2>&1; done
cat $O/jd_speed_base.txt $O/jd_speed_noinplace.txt
