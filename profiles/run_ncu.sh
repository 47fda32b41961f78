#!/bin/bash
# ncu evidence for one round (run under gpurun on ONE GPU).  Usage: profiles/run_ncu.sh <tag> <config>
# Step 2 of `bench.py --profile` is captured: every launch with its duration, then the full set on
# one layer's grouped expand and shrink launches ({q,k,v}, {o}, {gate,up}, {down}).
set -u
TAG=${1:-r01}; CFG=${2:-decode}
G=128; PER_STEP=$((1 + 2 * G))
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s $PER_STEP -c $PER_STEP --csv \
    --log-file $OUT/${TAG}_${CFG}_launches.csv python bench.py --config $CFG --profile > /dev/null 2>&1
for K in expand_kernel shrink_sigma_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s $G -c 4 \
      -o $OUT/${TAG}_${CFG}_${K} python bench.py --config $CFG --profile > /dev/null 2>&1
done
ls -la $OUT
