# round 2, session 3: software-pipelined decode epilogue (next item's TMEM load before this item's stores)
set -u
O=gpurun_out/s3pipe2
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/final.so
run() {  # tag, config, lib
  cp $3 $L
  timeout 300 python bench.py --config $2 --no-cpu-baseline > $O/$1.json 2>> $O/err.txt
  python -c "import json; d=json.loads(open('$O/$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'], (d.get('parity_check') or {}).get('max_row_rel_err'))" >> $O/ab.txt 2>&1
}
for rep in 1; do
  run dec_base_$rep decode /tmp/final.so
  run dec_pipe_$rep decode .variants/libcts_pipe2.so
  run multi_base_$rep multi /tmp/final.so
  run multi_pipe_$rep multi .variants/libcts_pipe2.so
done
cat $O/ab.txt
cp .variants/libcts_pipe2.so $L
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 > $O/pytest.txt 2>&1; tail -1 $O/pytest.txt
cp /tmp/final.so $L
