set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
$NV -DCTS_TRACE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
T=16384 timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused_prefill.txt 2>&1
