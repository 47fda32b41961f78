set -u
for k in 16 8 4 2; do
CTS_KS_MAX=$k timeout 300 python bench.py --config q_proj --steps 500 --no-cpu-baseline > gpurun_out/qp_ks$k.json 2>> gpurun_out/qp.err
done
