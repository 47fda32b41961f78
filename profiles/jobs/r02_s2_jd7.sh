set -u
O=gpurun_out/s2s
mkdir -p $O
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "jd" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/jd_speed.txt 2>&1; done
tail -2 $O/jd_speed.txt
cp paper_2407_00066_b200/libcts.so /tmp/keep.so
$NV -DCTS_JD_DBG_NOSPLIT -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/jd_speed_nosplit.txt 2>&1; done
tail -2 $O/jd_speed_nosplit.txt
cp /tmp/keep.so paper_2407_00066_b200/libcts.so
