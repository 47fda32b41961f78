# tests + decode/prefill bench lines, then a CTS_TRACE build (in the box's copy) for the per-CTA timeline
set -u
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3 > gpurun_out/pytest.txt
for c in decode prefill; do timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/pf_${c}.json 2>gpurun_out/pf_${c}.err; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -DCTS_TRACE \
  -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused.txt 2>&1
