set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
cp paper_2407_00066_b200/libcts.so /tmp/lib_k48.so
$NV -DCTS_KCHUNK_NUM=64 -o /tmp/lib_k64.so paper_2407_00066_b200/csrc/cts.cu
for rep in 1 2; do for v in k48 k64; do
cp /tmp/lib_$v.so paper_2407_00066_b200/libcts.so
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/kc_${v}_r$rep.json 2>> gpurun_out/kc.err
done; done
cp /tmp/lib_k48.so paper_2407_00066_b200/libcts.so
