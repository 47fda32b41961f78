"""Top stall-sampled SASS lines of one launch in an ncu report, with the CUDA source line.
usage: python profiles/ncu_source_hot.py <rep> [launch_index] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r or "# Address" in r)
hdr = rows[hi]
def col(name):
    for i, h in enumerate(hdr):
        if h.strip() == name:
            return i
    return None
ia, isrc = col("Address"), col("Source")
iw = col("Warp Stall Sampling (All Samples)")
data = []
for r in rows[hi + 1:]:
    if len(r) <= max(ia, isrc, iw):
        continue
    try:
        data.append((int(r[iw] or 0), r[ia], r[isrc].strip()))
    except ValueError:
        pass
seen, uniq = set(), []
for d in data:
    if d[1] not in seen:
        seen.add(d[1]); uniq.append(d)
tot = sum(d[0] for d in uniq) or 1
print(f"total samples {tot}")
for d in sorted(uniq, reverse=True)[:top]:
    print(f"{d[0]:7d} {100 * d[0] / tot:5.1f}%  {d[1][-6:]}  {d[2][:120]}")
