"""One cts_project call per module shape (for ncu): q, gate at T (default 16384)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00066_b200 as cts  # noqa: E402
from workloads.gen_torch import direct_bank_torch, tokens_torch  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dev = torch.device("cuda")
mods = [("q", 4096, 4096), ("gate", 4096, 14336)]
banks = [direct_bank_torch(di, do, 1000, 25, 16, seed=m, device=dev, cluster_seed=50 + m) for m, (_, di, do) in enumerate(mods)]
bank = cts.Bank([b["in_basis"] for b in banks], [b["out_basis"] for b in banks], [b["sigma"] for b in banks],
                [b["cluster_of"] for b in banks])
plan = cts.Plan(bank, T)
plan.segment(tokens_torch(T, 1000, 1, T > 4096, dev))
g = torch.Generator(device=dev).manual_seed(0)
for m, (name, di, do) in enumerate(mods):
    x = torch.randn(T, di, generator=g, device=dev).to(torch.bfloat16)
    w = (torch.randn(do, di, generator=g, device=dev) / di ** 0.5).to(torch.bfloat16)
    y = torch.empty(T, do, dtype=torch.bfloat16, device=dev)
    for _ in range(2):
        plan.project(m, x, w, y, 2.0)
    torch.mm(x, w.t(), out=y)
torch.cuda.synchronize()
