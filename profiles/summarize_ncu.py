"""Summarize ncu reports (per-launch duration, dram bytes, throughput) into a committed text table.
usage: python profiles/summarize_ncu.py gpurun_out/<rep>.ncu-rep [...] > profiles/<round>/<name>.txt"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__grid_size", "launch__registers_per_thread", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "lts__t_bytes.sum"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"== {rep}")
    print("kernel | grid | regs | time | dram_read | dram_write | dram % peak | warps active % | tensor pipe % | L2 bytes")
    for r in rows[2:]:
        g = lambda k: (r[idx[k]] + " " + units[idx[k]]).strip() if k in idx else "-"  # noqa: E731
        print(" | ".join([r[idx["Kernel Name"]][:40], g("launch__grid_size"), g("launch__registers_per_thread"),
                          g("gpu__time_duration.sum"), g("dram__bytes_read.sum"), g("dram__bytes_write.sum"),
                          g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                          g("sm__warps_active.avg.pct_of_peak_sustained_active"),
                          g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"), g("lts__t_bytes.sum")]))
