set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
cp paper_2407_00066_b200/libcts.so /tmp/lib_d32.so
$NV -DCTS_DIST_MIN_RP=16 -o /tmp/lib_d16.so paper_2407_00066_b200/csrc/cts.cu
cp /tmp/lib_d16.so paper_2407_00066_b200/libcts.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "layer_grouped or mistral or grouped or tensor_parallel or ranks or deterministic or launch_count" 2>&1 | tail -3 > gpurun_out/d16_pytest.txt
for rep in 1 2; do for v in d32 d16; do
cp /tmp/lib_$v.so paper_2407_00066_b200/libcts.so
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/d16_decode_${v}_r$rep.json 2>> gpurun_out/d16.err
timeout 300 python bench.py --config multi --steps 30 --no-cpu-baseline > gpurun_out/d16_multi_${v}_r$rep.json 2>> gpurun_out/d16.err
done; done
cp /tmp/lib_d32.so paper_2407_00066_b200/libcts.so
