set -u
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"segment_kernel|apply_fused_kernel" -s 2 -c 2 --csv \
    --log-file gpurun_out/r01_q_proj_launches.csv python bench.py --config q_proj --profile > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:apply_fused_kernel -s 1 -c 1 \
    -o gpurun_out/r01_q_proj_apply_fused_kernel python bench.py --config q_proj --profile > /dev/null 2>&1
python profiles/summarize_ncu.py gpurun_out/r01_q_proj_apply_fused_kernel.ncu-rep > gpurun_out/r01_q_proj_fused_summary.txt 2>&1
