set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
$NV -DCTS_TRACE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
QONLY=1 T=256 N=64 C=1 R=64 timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused_q.txt 2>&1
QONLY=1 T=256 N=64 C=1 R=64 CTS_KS_MAX=4 timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused_q_ks4.txt 2>&1
