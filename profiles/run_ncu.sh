#!/bin/bash
# ncu evidence for one round (run under gpurun on ONE GPU).  Usage: profiles/run_ncu.sh <tag> <config>
# `bench.py --profile` runs 2 eager steps of 1 segment + G fused apply launches (G = 4 groups x 32
# layers).  Captured from step 2: (1) every launch with its duration (the launch list), (2) the full
# set on layer 0's four fused launches ({q,k,v}, {o}, {gate,up}, {down}).
set -u
TAG=${1:-r01}; CFG=${2:-decode}
G=128; PER_STEP=$((1 + G))
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"segment_kernel|apply_fused_kernel" -s $PER_STEP -c $PER_STEP --csv \
    --log-file $OUT/${TAG}_${CFG}_launches.csv python bench.py --config $CFG --profile > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:apply_fused_kernel -s $G -c 4 \
    -o $OUT/${TAG}_${CFG}_apply_fused_kernel python bench.py --config $CFG --profile > /dev/null 2>&1
ls -la $OUT
