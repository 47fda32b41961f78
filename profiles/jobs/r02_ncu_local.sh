set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:apply_local_kernel -c 4 \
  -o gpurun_out/r02_local_v1 python profiles/microbench/layer_groups.py > gpurun_out/ncu_local_v1.log 2>&1
tail -5 gpurun_out/ncu_local_v1.log
