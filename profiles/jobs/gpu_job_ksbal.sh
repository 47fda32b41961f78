set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
cp paper_2407_00066_b200/libcts.so /tmp/lib_bal.so
$NV -DCTS_KS_BALANCE=0 -o /tmp/lib_nobal.so paper_2407_00066_b200/csrc/cts.cu
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5 > gpurun_out/ksbal_pytest.txt
for v in bal nobal; do
cp /tmp/lib_$v.so paper_2407_00066_b200/libcts.so
timeout 300 python bench.py --config multi --steps 30 --no-cpu-baseline > gpurun_out/ksbal_multi_$v.json 2>> gpurun_out/ksbal.err
timeout 300 python bench.py --config prefill --steps 30 --no-cpu-baseline > gpurun_out/ksbal_prefill_$v.json 2>> gpurun_out/ksbal.err
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/ksbal_decode_$v.json 2>> gpurun_out/ksbal.err
done
cp /tmp/lib_bal.so paper_2407_00066_b200/libcts.so
$NV -DCTS_TRACE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
N=8192 C=128 timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused_multi_bal.txt 2>&1
T=16384 timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused_prefill_bal.txt 2>&1
