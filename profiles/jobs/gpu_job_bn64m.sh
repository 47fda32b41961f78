set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
cp paper_2407_00066_b200/libcts.so /tmp/lib_bn128.so
$NV -DCTS_EXPAND_BN=64 -o /tmp/lib_bn64.so paper_2407_00066_b200/csrc/cts.cu
for v in bn128 bn64; do
cp /tmp/lib_$v.so paper_2407_00066_b200/libcts.so
timeout 300 python bench.py --config multi --steps 30 --no-cpu-baseline > gpurun_out/bn64m_multi_$v.json 2>> gpurun_out/bn64m.err
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/bn64m_decode_$v.json 2>> gpurun_out/bn64m.err
done
cp /tmp/lib_bn128.so paper_2407_00066_b200/libcts.so
