# A/B of an env-selected variant on decode + prefill bench lines, then the CTS_TRACE timeline
set -u
VAR=${1:-CTS_POLL_FIRST}
for v in 0 1; do for c in decode prefill; do
  env $VAR=$v timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/ab_${c}_$v.json 2>gpurun_out/ab_${c}_$v.err
done; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -DCTS_TRACE \
  -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused.txt 2>&1
