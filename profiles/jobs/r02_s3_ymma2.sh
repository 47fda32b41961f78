# round 2, session 3: tensor-core residual add only in the prefill (scatter) instantiation
set -u
O=gpurun_out/s3ymma2
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/final.so
run() {  # tag, config, lib, env
  cp $3 $L
  env $4 timeout 300 python bench.py --config $2 --no-cpu-baseline > $O/$1.json 2>> $O/err.txt
  python -c "import json; d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'])" >> $O/ab.txt 2>&1
}
for rep in 1 2; do
  run dec_committed_$rep decode /tmp/final.so ""
  run dec_new_$rep decode .variants/libcts_ymma2.so ""
  run pre_committed_$rep prefill /tmp/final.so ""
  run pre_new_$rep prefill .variants/libcts_ymma2.so ""
  run pre_new_y0_$rep prefill .variants/libcts_ymma2.so "CTS_Y_VIA_MMA=0"
done
run multi_new multi .variants/libcts_ymma2.so ""
run proj_new proj_prefill .variants/libcts_ymma2.so ""
cp .variants/libcts_ymma2.so $L
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 > $O/pytest.txt 2>&1; tail -1 $O/pytest.txt
cat $O/ab.txt
cp /tmp/final.so $L
