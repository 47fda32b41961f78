set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3 > gpurun_out/dist_pytest.txt
timeout 300 python bench.py --config q_proj --steps 500 --no-cpu-baseline > gpurun_out/dist_q.json 2>> gpurun_out/dist.err
CTS_KS_MAX=4 timeout 300 python bench.py --config q_proj --steps 500 --no-cpu-baseline > gpurun_out/dist_q_ks4.json 2>> gpurun_out/dist.err
CTS_KS_MAX=8 timeout 300 python bench.py --config q_proj --steps 500 --no-cpu-baseline > gpurun_out/dist_q_ks8.json 2>> gpurun_out/dist.err
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/dist_decode.json 2>> gpurun_out/dist.err
$NV -DCTS_TRACE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
QONLY=1 T=256 N=64 C=1 R=64 timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_fused_q_dist.txt 2>&1
