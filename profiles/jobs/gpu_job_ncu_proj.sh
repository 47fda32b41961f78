set -u
ncu --set full --clock-control none -k regex:"proj_fused_kernel" -c 2 \
    -o gpurun_out/proj_full python profiles/microbench/proj_one.py > gpurun_out/ncu_proj.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none python profiles/microbench/proj_one.py > gpurun_out/ncu_proj_names.log 2>&1
