set -u
ncu --set full --clock-control none --import-source on -k regex:apply_fused_kernel -s 128 -c 4 \
    -o gpurun_out/dec_full python bench.py --config decode --profile > gpurun_out/ncu_dec.log 2>&1
