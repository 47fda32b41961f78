set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
for pf in 0 1; do for t in 1 2; do
  CTS_POLL_FIRST=$pf CTS_ITEMS_PER_SM=$t timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/ab6_decode_pf${pf}_t$t.json 2> gpurun_out/ab6.err
done; done
$NV -DCTS_TRACE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
for pf in 0 1; do
CTS_POLL_FIRST=$pf CTS_ITEMS_PER_SM=2 timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused_pf$pf.txt 2>&1
done
