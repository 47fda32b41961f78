set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
cp paper_2407_00066_b200/libcts.so /tmp/lib_on.so
$NV -DCTS_WEIGHTED_DEAL=0 -o /tmp/lib_off.so paper_2407_00066_b200/csrc/cts.cu
timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 2>&1 | tail -3 > gpurun_out/dealdec3_pytest.txt
for rep in 1 2 3; do for v in on off; do
cp /tmp/lib_$v.so paper_2407_00066_b200/libcts.so
timeout 200 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/dealdec3_${v}_r$rep.json 2>> gpurun_out/dealdec3.err
done; done
cp /tmp/lib_on.so paper_2407_00066_b200/libcts.so
timeout 200 python bench.py --config multi --steps 30 --no-cpu-baseline > gpurun_out/dealdec3_multi_on.json 2>> gpurun_out/dealdec3.err
