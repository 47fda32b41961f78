set -u
mkdir -p gpurun_out
timeout 120 python profiles/microbench/layer_groups.py > gpurun_out/dbg_layer.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python profiles/microbench/layer_groups.py > gpurun_out/dbg_memcheck.txt 2>&1
N=8192 C=128 timeout 600 compute-sanitizer --tool memcheck python profiles/microbench/layer_groups.py > gpurun_out/dbg_memcheck_multi.txt 2>&1
