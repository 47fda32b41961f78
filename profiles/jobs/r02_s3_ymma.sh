# round 2, session 3: residual add on the tensor core (D += Y I64 in the expand MMA) vs in the epilogue
set -u
O=gpurun_out/s3ymma
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/final.so
cp .variants/libcts_ymma.so $L
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x > $O/pytest.txt 2>&1; tail -4 $O/pytest.txt
run() {  # tag, config, env
  env $3 timeout 300 python bench.py --config $2 --no-cpu-baseline > $O/$1.json 2>> $O/err.txt
  python -c "import json; d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'], (d.get('parity_check') or {}).get('max_row_rel_err'))" >> $O/ab.txt 2>&1
}
for rep in 1 2; do
  run dec_y1_$rep decode "CTS_Y_VIA_MMA=1"
  run dec_y0_$rep decode "CTS_Y_VIA_MMA=0"
done
run multi_y1 multi "CTS_Y_VIA_MMA=1"
run multi_y0 multi "CTS_Y_VIA_MMA=0"
run pre_y1 prefill "CTS_Y_VIA_MMA=1"
run pre_y0 prefill "CTS_Y_VIA_MMA=0"
run q_y1 q_proj "CTS_Y_VIA_MMA=1"
run q_y0 q_proj "CTS_Y_VIA_MMA=0"
cat $O/ab.txt
cp /tmp/final.so $L
