set -u
run() { timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/knob_$1.json 2>> gpurun_out/knob.err; }
run base
CTS_EARLY_ITEMS=2 run early2
CTS_EARLY_ITEMS=8 run early8
CTS_POLL_FIRST=1 run pollfirst
CTS_ITEMS_PER_SM=2 run items2
CTS_EXPAND_STORE=0 run scatter
