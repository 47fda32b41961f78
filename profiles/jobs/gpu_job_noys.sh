set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
$NV -DCTS_DBG_NO_YSTORE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/noys_decode.json 2> gpurun_out/noys.err
