set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5 > gpurun_out/pytest.txt
for pf in 0 1 2; do
  CTS_PREFETCH=$pf timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/ab9_decode_pf$pf.json 2> gpurun_out/ab9.err
done
timeout 300 python bench.py --config multi --steps 50 --no-cpu-baseline > gpurun_out/ab9_multi.json 2>> gpurun_out/ab9.err
CTS_PREFETCH=0 timeout 300 python bench.py --config multi --steps 50 --no-cpu-baseline > gpurun_out/ab9_multi_pf0.json 2>> gpurun_out/ab9.err
$NV -DCTS_TRACE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
CTS_PREFETCH=1 timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused_ab9.txt 2>&1
