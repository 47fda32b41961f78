# round 2, session 3: finisher partials per L2 round trip = 4 (CTS_KCHUNK_NUM 64) vs 3
set -u
O=gpurun_out/s3kc64
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/final.so
run() {  # tag, config, lib
  cp $3 $L
  timeout 300 python bench.py --config $2 --no-cpu-baseline > $O/$1.json 2>> $O/err.txt
  python -c "import json; d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'])" >> $O/ab.txt 2>&1
}
for rep in 1 2; do
  run dec_kc48_$rep decode /tmp/final.so
  run dec_kc64_$rep decode .variants/libcts_kc64.so
done
cp /tmp/final.so $L
cat $O/ab.txt
