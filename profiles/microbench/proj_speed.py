"""Fused projection (cts_project) vs cuBLAS (torch.mm) for Mistral-7B module shapes at prefill.
Prints per-module times and TFLOP/s.  Usage: python profiles/microbench/proj_speed.py [T]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00066_b200 as cts  # noqa: E402
from workloads.gen_torch import direct_bank_torch, tokens_torch  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dev = torch.device("cuda")
mods = [("q", 4096, 4096), ("k", 4096, 1024), ("gate", 4096, 14336), ("down", 14336, 4096)]
banks = [direct_bank_torch(di, do, 1000, 25, 16, seed=m, device=dev, cluster_seed=50 + m) for m, (_, di, do) in enumerate(mods)]
bank = cts.Bank([b["in_basis"] for b in banks], [b["out_basis"] for b in banks], [b["sigma"] for b in banks],
                [b["cluster_of"] for b in banks])
plan = cts.Plan(bank, T)
plan.segment(tokens_torch(T, 1000, 1, T > 4096, dev))
g = torch.Generator(device=dev).manual_seed(0)


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


for m, (name, di, do) in enumerate(mods):
    x = torch.randn(T, di, generator=g, device=dev).to(torch.bfloat16)
    w = (torch.randn(do, di, generator=g, device=dev) / di ** 0.5).to(torch.bfloat16)
    y = torch.empty(T, do, dtype=torch.bfloat16, device=dev)
    fl = 2.0 * T * di * do
    t_proj = timeit(lambda: plan.project(m, x, w, y, 2.0))
    t_shr = timeit(lambda: plan.shrink(m, x, 2.0))
    t_mm = timeit(lambda: torch.mm(x, w.t(), out=y))
    print(f"{name:5s} {di}->{do}: project {t_proj*1e3:8.1f} us ({fl/t_proj/1e9:7.1f} TF/s; shrink {t_shr*1e3:6.1f} us, "
          f"GEMM part ~{fl/(t_proj-t_shr)/1e9:7.1f} TF/s)   cuBLAS mm {t_mm*1e3:8.1f} us ({fl/t_mm/1e9:7.1f} TF/s)")
