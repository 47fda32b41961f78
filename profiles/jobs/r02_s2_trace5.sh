set -u
O=gpurun_out/s2w
mkdir -p $O
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
$NV -DCTS_TRACE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python profiles/microbench/trace_fused.py > $O/trace_items.txt 2>&1
cat $O/trace_items.txt
