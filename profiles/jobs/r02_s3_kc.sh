# round 2, session 3: finisher partials per L2 round trip (CTS_KCHUNK_NUM / r_pad) and t-ready poll back-off
set -u
O=gpurun_out/s3kc
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/base.so
run() {  # tag, config, lib
  cp $3 $L
  timeout 300 python bench.py --config $2 --no-cpu-baseline > $O/$1.json 2>> $O/err.txt
  python -c "import json; d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'], (d.get('parity_check') or {}).get('max_row_rel_err'))" >> $O/kc.txt 2>&1
}
run dec_base decode /tmp/base.so
for t in kc96 kc128 kc176 ns0 ns16; do run dec_$t decode .variants/libcts_$t.so; done
run dec_base2 decode /tmp/base.so
run multi_base multi /tmp/base.so
run multi_kc96 multi .variants/libcts_kc96.so
cp /tmp/base.so $L
cat $O/kc.txt
