"""Per-CTA timeline of apply_local launches (CTS_TRACE build) for one Mistral-7B layer's groups at
decode: when the work map is ready, the first x TMA, the first shrink accumulator, the first t, the
first expand job, the end.  N, C, T from the environment (default cfg3)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00066_b200 as cts  # noqa: E402
from workloads.gen import MISTRAL_MODULES  # noqa: E402
from workloads.gen_torch import direct_bank_torch, tokens_torch  # noqa: E402

N, C, T = int(os.environ.get("N", 1000)), int(os.environ.get("C", 25)), int(os.environ.get("T", 1024))
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
srcs = [direct_bank_torch(di, do, N, C, 16, seed=m, device=dev, cluster_seed=50 + m)
        for m, (_, di, do) in enumerate(MISTRAL_MODULES)]
bank = cts.Bank([s["in_basis"] for s in srcs], [s["out_basis"] for s in srcs], [s["sigma"] for s in srcs],
                [s["cluster_of"] for s in srcs])
plan = cts.Plan(bank, T)
plan.segment(tokens_torch(T, N, 1, False, dev))
xs = {"attn": torch.randn(T, 4096, device=dev).to(torch.bfloat16), "o": torch.randn(T, 4096, device=dev).to(torch.bfloat16),
      "mlp": torch.randn(T, 4096, device=dev).to(torch.bfloat16), "down": torch.randn(T, 14336, device=dev).to(torch.bfloat16)}
ys = [torch.randn(T, do, device=dev).to(torch.bfloat16) for (_, _, do) in MISTRAL_MODULES]
groups = {"attn": [0, 1, 2], "o": [3], "mlp": [4, 5], "down": [6]}
big = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
L = cts.lib()
L.cts_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
names = {0: "start", 1: "map ready (after griddep_wait)", 2: "first x TMA issued", 3: "x producers done",
         4: "first shrink acc committed", 5: "first t published", 6: "first expand job issued",
         7: "MMA: first expand started", 8: "set B: first job done", 12: "y producers done",
         10: "set B done", 11: "end"}
for name, gm in groups.items():
    for rep in range(3):
        big.zero_()
        plan.apply_group(gm, [xs[name]] * len(gm), [ys[m] for m in gm], 2.0)
        torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (160 * 40))()
    L.cts_debug_trace(buf, 160 * 40)
    a = np.array(buf, dtype=np.int64).reshape(160, 40)[:148].astype(np.float64)
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    rel = (a - t0) / 1e3
    print(f"local group {name} {gm} (T={T}, N={N}, C={C}): us after first CTA start: min / median / max over CTAs")
    for i, n in names.items():
        col = rel[:, i]
        col = col[(col >= 0) & (col < 1e4)]
        if col.size:
            print(f"  {n:34s} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}  (n={col.size})")

# per-job timeline of CTA 5 for the mlp group (events: y producer got stage, MMA got acc slot, MMA got
# data, set B got acc, set B got data, set B done)
L.cts_debug_jobtrace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
for name in ("attn", "mlp"):
    gm = groups[name]
    ctypes.memset(jb0 := (ctypes.c_ulonglong * (8 * 128))(), 0, 8 * 128 * 8)
    plan.apply_group(gm, [xs[name]] * len(gm), [ys[m] for m in gm], 2.0)
    torch.cuda.synchronize()
    jb = (ctypes.c_ulonglong * (8 * 128))()
    L.cts_debug_jobtrace(jb, 8 * 128)
    j = np.array(jb, dtype=np.int64).reshape(8, 128).astype(np.float64)
    base = j[j > 0].min()
    print(f"shrink stages of CTA 5, group {name} (us): x-prod issued | MMA got data")
    for k in range(128):
        if j[1, k] == 0:
            continue
        print(f"  stage {k:3d}: {(j[1, k] - base) / 1e3:8.2f} {(j[7, k] - base) / 1e3 if j[7, k] else -1:8.2f}")
    print(f"jobs of CTA 5, group {name} (us): y-prod-stage | mma-acc | mma-data | setB-acc | setB-data | setB-done")
    for k in range(128):
        if j[0, k] == 0:
            continue
        print(f"  job {k:3d}: " + " ".join(f"{(j[e, k] - base) / 1e3:8.2f}" if j[e, k] else "       -" for e in (0, 2, 3, 4, 5, 6)))
