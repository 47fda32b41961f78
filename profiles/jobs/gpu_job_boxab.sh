set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
cp paper_2407_00066_b200/libcts.so /tmp/lib_box1.so
$NV -DCTS_EXPAND_BOXES=0 -o /tmp/lib_box0.so paper_2407_00066_b200/csrc/cts.cu
for rep in 1 2; do for v in 0 1; do
  cp /tmp/lib_box$v.so paper_2407_00066_b200/libcts.so
  timeout 600 python bench.py --config prefill --steps 30 --no-cpu-baseline > gpurun_out/boxab_v${v}_r$rep.json 2>> gpurun_out/boxab.err
done; done
