set -u
for k in 16 8 6 4; do
CTS_KS_MAX=$k timeout 600 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/ks_decode_$k.json 2>> gpurun_out/ks.err
done
