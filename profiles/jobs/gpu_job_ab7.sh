set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5 > gpurun_out/pytest.txt
for t in 1 2; do
  CTS_ITEMS_PER_SM=$t timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/ab7_pre1_decode_t$t.json 2> gpurun_out/ab7.err
done
timeout 300 python bench.py --config prefill --steps 30 --no-cpu-baseline > gpurun_out/ab7_pre1_prefill.json 2>> gpurun_out/ab7.err
cp paper_2407_00066_b200/libcts.so /tmp/lib_pre1.so
$NV -DCTS_SIGMA_PRE=0 -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
for t in 1 2; do
  CTS_ITEMS_PER_SM=$t timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/ab7_pre0_decode_t$t.json 2>> gpurun_out/ab7.err
done
$NV -DCTS_TRACE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
CTS_ITEMS_PER_SM=2 timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused_ab7.txt 2>&1
