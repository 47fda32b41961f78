# round 2, session 3: shrink ring depth 10 (the fused arena already holds it) on the many-cluster config
set -u
O=gpurun_out/s3st10
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/final.so
run() {  # tag, config, lib
  cp $3 $L
  timeout 300 python bench.py --config $2 --no-cpu-baseline > $O/$1.json 2>> $O/err.txt
  python -c "import json; d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'])" >> $O/st.txt 2>&1
}
for rep in 1 2; do
  run multi_st8_$rep multi /tmp/final.so
  run multi_st10_$rep multi .variants/libcts_st10.so
  run dec_st8_$rep decode /tmp/final.so
  run dec_st10_$rep decode .variants/libcts_st10.so
done
run pre_st8 prefill /tmp/final.so
run pre_st10 prefill .variants/libcts_st10.so
cp /tmp/final.so $L
cat $O/st.txt
