# round 2, session 3: (1) decode epilogue row-coalesced copies out of the stage vs register-direct
# 32-byte row pieces; (2) pipelined K-space Gram staging in jd_gorth (parity + speed)
set -u
O=gpurun_out/s3rc
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/final.so
run() {  # tag, config, lib
  cp $3 $L
  timeout 300 python bench.py --config $2 --no-cpu-baseline > $O/$1.json 2>> $O/err.txt
  python -c "import json; d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'])" >> $O/rc.txt 2>&1
}
run dec_go2 decode .variants/libcts_go2.so
run dec_rowcopy decode .variants/libcts_rowcopy.so
run multi_go2 multi .variants/libcts_go2.so
run multi_rowcopy multi .variants/libcts_rowcopy.so
run dec_go2b decode .variants/libcts_go2.so
run dec_rowcopyb decode .variants/libcts_rowcopy.so
cat $O/rc.txt
cp .variants/libcts_go2.so $L
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jd" --timeout 300 > $O/pytest_jd_go2.txt 2>&1; tail -1 $O/pytest_jd_go2.txt
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/jd_speed_go2.txt 2>&1; done
cat $O/jd_speed_go2.txt
cp .variants/libcts_rowcopy.so $L
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -k "decode or grouped or bench or layer" > $O/pytest_rowcopy.txt 2>&1; tail -1 $O/pytest_rowcopy.txt
cp /tmp/final.so $L
