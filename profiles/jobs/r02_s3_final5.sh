# round 2, session 3: the remaining bench configs + the reference arm on the final build
set -u
O=gpurun_out/s3final5
mkdir -p $O
for c in q_proj lora_decode lora_matched tp_decode proj_prefill; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err
done
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2>> $O/bench.err
for f in $O/bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "unreadable", e); sys.exit()
r = d.get("roofline", {})
print(f.split("/")[-1], round(d["value"], 1), d["unit"], "frac", r.get("frac"), "ms/step", d.get("ms_per_step"), "mhz", d.get("clocks", {}).get("sm_mhz"))
PY
done
