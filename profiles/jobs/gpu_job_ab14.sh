set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5 > gpurun_out/pytest.txt
for t in 1 2; do
CTS_ITEMS_PER_SM=$t timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/ab14_decode_t$t.json 2> gpurun_out/ab14.err
done
timeout 300 python bench.py --config multi --steps 50 --no-cpu-baseline > gpurun_out/ab14_multi.json 2>> gpurun_out/ab14.err
$NV -DCTS_TRACE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused_ab14.txt 2>&1
