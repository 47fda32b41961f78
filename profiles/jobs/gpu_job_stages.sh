set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
cp paper_2407_00066_b200/libcts.so /tmp/lib_s8.so
$NV -DCTS_SHRINK_STAGES=10 -o /tmp/lib_s10.so paper_2407_00066_b200/csrc/cts.cu
for rep in 1 2; do for v in s8 s10; do
cp /tmp/lib_$v.so paper_2407_00066_b200/libcts.so
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/st_${v}_r$rep.json 2>> gpurun_out/st.err
done; done
cp /tmp/lib_s10.so paper_2407_00066_b200/libcts.so
timeout 300 python bench.py --config prefill --steps 30 --no-cpu-baseline > gpurun_out/st_prefill_s10.json 2>> gpurun_out/st.err
cp /tmp/lib_s8.so paper_2407_00066_b200/libcts.so
timeout 300 python bench.py --config prefill --steps 30 --no-cpu-baseline > gpurun_out/st_prefill_s8.json 2>> gpurun_out/st.err
