set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tma_rate profiles/microbench/tma_rate.cu
timeout 300 /tmp/tma_rate > gpurun_out/tma_rate2.txt 2>&1
