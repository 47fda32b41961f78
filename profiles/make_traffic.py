"""Write profiles/ncu_traffic.json from one `ncu --set full` capture of the fused apply kernel.
usage: python profiles/make_traffic.py <workload> <rep.ncu-rep> <alg_bytes.json>  (run_ncu.sh outputs)
The capture holds layer 0's four fused launches of step 2; alg_bytes.json (bench.py --profile) has
the algorithmic bytes of every launch of the step in the same order.  bench.py reports
roofline.traffic = (sum dram bytes / sum algorithmic bytes of these launches) x its own per-launch
algorithmic bytes."""
import csv
import io
import json
import os
import subprocess
import sys

workload, rep, algf = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
launches = [r for r in rows[2:] if "apply_fused_kernel" in r[idx["Kernel Name"]]]
dram = [sum(float(r[idx[k]].replace(",", "")) * scale.get(units[idx[k]], 1)
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum")) for r in launches]
alg = json.load(open(algf))
alg_b = [s + e for s, e in zip(alg["shrink"], alg["expand"])][:len(dram)]
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d.setdefault(workload, {})["apply_fused_kernel"] = {
    "dram_bytes_per_launch": sum(dram) / len(dram), "algorithmic_bytes_per_launch": sum(alg_b) / len(alg_b),
    "ratio": sum(dram) / sum(alg_b), "launches": len(dram), "per_launch_dram": dram, "per_launch_alg": alg_b,
    "source": os.path.basename(rep)}
json.dump(d, open(path, "w"), indent=1)
print(json.dumps(d[workload], indent=1))
