set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
cp paper_2407_00066_b200/libcts.so /tmp/lib_bn128.so
$NV -DCTS_EXPAND_BN=64 -o /tmp/lib_bn64.so paper_2407_00066_b200/csrc/cts.cu
cp /tmp/lib_bn64.so paper_2407_00066_b200/libcts.so
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3 > gpurun_out/pytest_bn64.txt
for v in 128 64; do
  cp /tmp/lib_bn$v.so paper_2407_00066_b200/libcts.so
  for c in decode prefill; do
    timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/bn_${c}_$v.json 2>> gpurun_out/bn.err
  done
done
