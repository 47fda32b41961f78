# tensor-core (3xTF32) JD thin GEMMs: parity vs the fp64 oracle, speed, ncu launch list
set -u
O=gpurun_out/s2l
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "jd" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
tail -5 $O/pytest.txt
timeout 300 python profiles/microbench/jd_speed.py 10 > $O/jd_speed.txt 2>&1
timeout 300 python profiles/microbench/jd_speed.py 50 >> $O/jd_speed.txt 2>&1
cat $O/jd_speed.txt | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/jd_launches.csv python profiles/microbench/jd_speed.py 2 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/s2l/jd_launches.csv")))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; k = h.index("Kernel Name"); v = h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) > v:
        name = r[k].split("(")[0].split("<")[0]
        agg[name][0] += 1; agg[name][1] += float(r[v].replace(",", ""))
tot = sum(t for _, t in agg.values())
for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name:40s} {n:6d} launches {t/1e3:10.1f} us  {100*t/tot:5.1f}%")
PY
