set -u
mkdir -p gpurun_out/s2u
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tma_rate profiles/microbench/tma_rate.cu
timeout 300 /tmp/tma_rate > gpurun_out/s2u/tma_rate_ldg.txt 2>&1
cat gpurun_out/s2u/tma_rate_ldg.txt | grep -E "gather4 64col|ldg"
