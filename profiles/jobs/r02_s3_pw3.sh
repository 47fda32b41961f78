# round 2, session 3: 12-warp fused kernel (3 producer warps; 168 registers instead of 128) with the
# finisher batch at 3 or 6 partials per L2 round trip
set -u
O=gpurun_out/s3pw3
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/final.so
run() {  # tag, config, lib
  cp $3 $L
  timeout 300 python bench.py --config $2 --no-cpu-baseline > $O/$1.json 2>> $O/err.txt
  python -c "import json; d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'])" >> $O/ab.txt 2>&1
}
for c in decode multi prefill q_proj; do
  run ${c}_base $c /tmp/final.so
  run ${c}_pw3 $c .variants/libcts_pw3.so
  run ${c}_pw3kc96 $c .variants/libcts_pw3kc96.so
done
cat $O/ab.txt
tail -5 $O/err.txt
cp /tmp/final.so $L
