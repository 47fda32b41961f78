# decode expand-tail knobs: epilogue split vs alternating sets, early items, poll-first
set -u
O=gpurun_out/s2m
mkdir -p $O
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
run() {  # tag, env
  env $2 timeout 300 python bench.py --config decode --no-cpu-baseline > $O/knob_$1.json 2>> $O/knob.err
  python -c "import json; d=json.loads(open('$O/knob_$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d['clocks']['sm_mhz'])" >> $O/knobs.txt
}
cp paper_2407_00066_b200/libcts.so /tmp/keep.so
run base ""
run early2 "CTS_EARLY_ITEMS=2"
run early8 "CTS_EARLY_ITEMS=8"
run pollfirst "CTS_POLL_FIRST=1"
$NV -DCTS_EPI_SPLIT=0 -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
run nosplit ""
$NV -DCTS_SHRINK_STAGES=6 -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
run sst6 ""
cp /tmp/keep.so paper_2407_00066_b200/libcts.so
run base2 ""
cat $O/knobs.txt
