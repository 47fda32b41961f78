set -u
mkdir -p gpurun_out
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/loc_decode.json 2> gpurun_out/loc.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -DCTS_TRACE -ldl \
  -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python profiles/microbench/trace_local.py > gpurun_out/trace_local3.txt 2>&1
