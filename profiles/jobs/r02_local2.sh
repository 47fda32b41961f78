set -u
mkdir -p gpurun_out
timeout 120 python profiles/microbench/layer_groups.py > gpurun_out/dbg_layer.txt 2>&1
N=8192 C=128 timeout 120 python profiles/microbench/layer_groups.py >> gpurun_out/dbg_layer.txt 2>&1
tail -3 gpurun_out/dbg_layer.txt
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/loc_decode.json 2> gpurun_out/loc.err
timeout 300 python bench.py --config multi --steps 50 --no-cpu-baseline > gpurun_out/loc_multi.json 2>> gpurun_out/loc.err
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_local.txt 2>&1
tail -3 gpurun_out/pytest_local.txt
cp paper_2407_00066_b200/libcts.so /tmp/keep.so
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -DCTS_TRACE \
  -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python profiles/microbench/trace_local.py > gpurun_out/trace_local.txt 2>&1
cp /tmp/keep.so paper_2407_00066_b200/libcts.so
