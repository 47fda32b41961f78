# round 2, session 3: software-pipelined decode epilogue on the 12-warp build (158 registers, no spill)
set -u
O=gpurun_out/s3pipe3
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/final.so
run() {  # tag, config, lib
  cp $3 $L
  timeout 300 python bench.py --config $2 --no-cpu-baseline > $O/$1.json 2>> $O/err.txt
  python -c "import json; d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'])" >> $O/ab.txt 2>&1
}
for rep in 1 2; do
  run dec_base_$rep decode /tmp/final.so
  run dec_pipe_$rep decode .variants/libcts_pipe.so
done
run multi_base multi /tmp/final.so
run multi_pipe multi .variants/libcts_pipe.so
cat $O/ab.txt
cp /tmp/final.so $L
