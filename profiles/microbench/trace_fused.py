"""Per-CTA timeline of fused apply launches at decode (q,k,v group; gate,up group) from a CTS_TRACE
build: when phase 1 (shrink) issues, finishes, when phase 2 (expand) gets its first t, ends."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00066_b200 as cts  # noqa: E402
from workloads.gen_torch import direct_bank_torch, tokens_torch  # noqa: E402

T, N, C, r = int(os.environ.get("T", 1024)), int(os.environ.get("N", 1000)), int(os.environ.get("C", 25)), int(os.environ.get("R", 16))
dev = torch.device("cuda")
mods = [(4096, 4096), (4096, 1024), (4096, 1024), (4096, 14336), (4096, 14336)]
if os.environ.get("QONLY"):   # cfg2: one q module
    mods = mods[:1]
banks = [direct_bank_torch(di, do, N, C, r, seed=m, device=dev, cluster_seed=50 + m) for m, (di, do) in enumerate(mods)]
bank = cts.Bank([b["in_basis"] for b in banks], [b["out_basis"] for b in banks], [b["sigma"] for b in banks],
                [b["cluster_of"] for b in banks])
plan = cts.Plan(bank, T)
plan.segment(tokens_torch(T, N, 1, T > 4096, dev))
x = torch.randn(T, 4096, device=dev).to(torch.bfloat16)
ys = [torch.randn(T, do, device=dev).to(torch.bfloat16) for (_, do) in mods]
big = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
L = cts.lib()
L.cts_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
names = {0: "start", 1: "prologue+wait", 2: "shrink first TMA", 3: "shrink producers done", 4: "shrink MMA done",
         5: "shrink epi set0 done", 6: "shrink epi set1 done", 7: "expand producers start", 8: "expand first t ready",
         9: "expand producers done", 10: "expand epi done", 11: "end",
         12: "finisher: last arrival", 13: "finisher: partials summed", 14: "finisher: t stored",
         15: "finisher: flag published", 16: "shrink: first item mapped", 17: "shrink: expect_tx armed",
         18: "shrink: first gathers issued", 19: "shrink: first acc ready", 20: "expand item 0 epi done",
         21: "expand item 1 epi done", 22: "expand item 2 epi done", 23: "expand item 3 epi done"}
for k in range(3):   # expand items 1..3: epilogue acc ready, TMEM read, stores issued; MMA accumulator free
    names.update({24 + 4 * k: f"item {k + 1}: epi acc ready", 25 + 4 * k: f"item {k + 1}: epi TMEM read",
                  26 + 4 * k: f"item {k + 1}: epi stores issued", 27 + 4 * k: f"item {k + 1}: MMA acc free",
                  36 + k: f"item {k + 1}: MMA operands landed"})
NS = 40
for grp in (([0],) if os.environ.get("QONLY") else ([0, 1, 2], [3, 4])):
    for rep in range(3):
        big.zero_()
        plan.apply_group(grp, [x] * len(grp), [ys[m] for m in grp], 2.0)
        torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (160 * NS))()
    L.cts_debug_trace(buf, 160 * NS)
    a = np.array(buf, dtype=np.int64).reshape(160, NS)[:148].astype(np.float64)
    a = a[a[:, 0] > 0]                                 # CTAs of this launch (grid may be < 148)
    t0 = a[:, 0].min()
    rel = (a - t0) / 1e3
    print(f"fused group {grp} (T={T}, N={N}, C={C}): us after first CTA start: min / median / max over CTAs")
    for i, n in names.items():
        col = rel[:, i]
        col = col[(col >= 0) & (col < 1e4)]
        if col.size:
            print(f"  {n:24s} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}  (n={col.size})")
