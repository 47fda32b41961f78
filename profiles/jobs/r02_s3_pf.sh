# round 2, session 3: L2 prefetch role (x row chunks / y rows + out_basis of the first n expand items)
set -u
O=gpurun_out/s3pf
mkdir -p $O
run() {  # tag, config, env
  env $3 timeout 300 python bench.py --config $2 --no-cpu-baseline > $O/$1.json 2>> $O/err.txt
  python -c "import json; d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'])" >> $O/pf.txt 2>&1
}
run dec_base decode ""
run dec_x decode "CTS_PF_X=1"
run dec_y4 decode "CTS_PF_Y_ITEMS=4"
run dec_y8 decode "CTS_PF_Y_ITEMS=8"
run dec_x_y4 decode "CTS_PF_X=1 CTS_PF_Y_ITEMS=4"
run dec_x_y8 decode "CTS_PF_X=1 CTS_PF_Y_ITEMS=8"
run dec_x_y16 decode "CTS_PF_X=1 CTS_PF_Y_ITEMS=16"
run dec_x_y64 decode "CTS_PF_X=1 CTS_PF_Y_ITEMS=64"
run multi_base multi ""
run multi_x_y8 multi "CTS_PF_X=1 CTS_PF_Y_ITEMS=8"
run pre_base prefill ""
run pre_x prefill "CTS_PF_X=1"
run dec_base2 decode ""
cat $O/pf.txt
