set -u
for k in 1 2 4 8 16; do
CTS_KS_MAX=$k timeout 300 python bench.py --config q_proj --steps 500 --no-cpu-baseline > gpurun_out/qks_$k.json 2>> gpurun_out/qks.err
done
