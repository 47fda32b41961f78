set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
cp paper_2407_00066_b200/libcts.so /tmp/lib_dyn.so
$NV -DCTS_DYN_TAIL=0 -o /tmp/lib_nodyn.so paper_2407_00066_b200/csrc/cts.cu
timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 2>&1 | tail -3 > gpurun_out/dyn4_pytest.txt
for rep in 1 2; do for v in dyn nodyn; do
cp /tmp/lib_$v.so paper_2407_00066_b200/libcts.so
timeout 200 python bench.py --config prefill --steps 30 --no-cpu-baseline > gpurun_out/dyn4_prefill_${v}_r$rep.json 2>> gpurun_out/dyn4.err
timeout 200 python bench.py --config multi --steps 30 --no-cpu-baseline > gpurun_out/dyn4_multi_${v}_r$rep.json 2>> gpurun_out/dyn4.err
done; done
for v in dyn nodyn; do
cp /tmp/lib_$v.so paper_2407_00066_b200/libcts.so
timeout 200 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/dyn4_decode_$v.json 2>> gpurun_out/dyn4.err
done
cp /tmp/lib_dyn.so paper_2407_00066_b200/libcts.so
