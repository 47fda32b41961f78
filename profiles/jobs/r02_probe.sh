# round 2: TMA gather-rate microbenchmark + compute-sanitizer over every apply path
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tma_rate profiles/microbench/tma_rate.cu
timeout 300 /tmp/tma_rate > gpurun_out/tma_rate.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python profiles/microbench/sanitize_apply.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.txt
done
