# round 2, session 3: more TMA producer warps (shrink x gathers are per-warp issue-limited)
set -u
O=gpurun_out/s3pw
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/base.so
run() {  # tag, config, lib
  cp $3 $L
  timeout 300 python bench.py --config $2 --no-cpu-baseline > $O/$1.json 2>> $O/err.txt
  python -c "import json; d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'], (d.get('parity_check') or {}).get('max_row_rel_err'))" >> $O/pw.txt 2>&1
}
for c in decode multi prefill q_proj; do
  run ${c}_pw4 $c /tmp/base.so
  run ${c}_pw6 $c .variants/libcts_pw6.so
  run ${c}_pw7 $c .variants/libcts_pw7.so
done
cp /tmp/base.so $L
cat $O/pw.txt
