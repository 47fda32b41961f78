set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -I include"
cp paper_2407_00066_b200/libcts.so /tmp/lib_v8.so
$NV -DCTS_Y_STORE_HINT='".cs"' -o /tmp/lib_v8cs.so paper_2407_00066_b200/csrc/cts.cu
$NV -o /tmp/lib_old.so profiles/jobs/oldsrc/pkg/csrc/cts.cu
for rep in 1 2; do for v in old v8 v8cs; do
  cp /tmp/lib_$v.so paper_2407_00066_b200/libcts.so
  timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/v8_decode_${v}_r$rep.json 2>> gpurun_out/v8.err
done; done
cp /tmp/lib_v8.so paper_2407_00066_b200/libcts.so
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2 > gpurun_out/pytest.txt
