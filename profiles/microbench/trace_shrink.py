"""Per-CTA timeline of one decode shrink launch (module o of cfg3) from a CTS_TRACE build."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00066_b200 as cts  # noqa: E402
from workloads.gen_torch import direct_bank_torch, tokens_torch  # noqa: E402

T, N, C, r = int(os.environ.get("T", 1024)), 1000, 25, 16
dev = torch.device("cuda")
mods = [(4096, 4096), (4096, 1024), (4096, 1024)]
banks = [direct_bank_torch(di, do, N, C, r, seed=m, device=dev, cluster_seed=50 + m) for m, (di, do) in enumerate(mods)]
bank = cts.Bank([b["in_basis"] for b in banks], [b["out_basis"] for b in banks], [b["sigma"] for b in banks],
                [b["cluster_of"] for b in banks])
plan = cts.Plan(bank, T)
plan.segment(tokens_torch(T, N, 1, T > 4096, dev))
x = torch.randn(T, 4096, device=dev).to(torch.bfloat16)
L = cts.lib()
L.cts_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
names = ["start", "prologue", "first_tma", "prod_done", "mma_first_full", "mma_item_commit", "epi_first_acc",
         "epi_acc", "atomic_begin", "atomic_end", "epi_done", "end"]
for grp in ([0], [0, 1, 2]):
    for rep in range(3):
        plan.shrink_group(grp, [x] * len(grp), 2.0)
        torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (160 * 40))()
    L.cts_debug_trace(buf, 160 * 40)
    a = np.array(buf, dtype=np.int64).reshape(160, 40)[:148, :12].astype(np.float64)
    t0 = a[:, 0].min()
    rel = (a - t0) / 1e3
    print(f"group {grp}: per-slot (us after first CTA start): min / median / max over CTAs")
    for i, n in enumerate(names):
        col = rel[:, i]
        col = col[a[:, i] > 0]
        if col.size:
            print(f"  {n:16s} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}")
