# round 2, session 3: 12-warp default build -- GPU suite, smoke, decode, fused projection, TP, multi
set -u
O=gpurun_out/s3pw3f
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt; tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python bench.py > $O/bench_decode.json 2>> $O/bench.err
for c in proj_prefill tp_decode multi q_proj prefill; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err; done
for f in $O/bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "unreadable", e); sys.exit()
r = d.get("roofline", {})
print(f.split("/")[-1], round(d["value"], 1), "frac", r.get("frac"), "ms/step", d.get("ms_per_step"), "mhz", d.get("clocks", {}).get("sm_mhz"), "parity", (d.get("parity_check") or {}).get("pass"))
PY
done
