"""GPU compression speed (cts_jd_eigen_iteration, App A.2): one Mistral-7B layer (7 projections) of
1000 rank-16 LoRAs in 25 clusters of 40, r = 16, 10 iterations; then the captured-energy fraction
sum_i ||Sigma_i||_F^2 / sum_i ||B_i A_i||_F^2 of the result (trained-like LoRAs with 4 families
per cluster).  Usage: python profiles/microbench/jd_speed.py [iters]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00066_b200 as cts  # noqa: E402
from workloads.gen import MISTRAL_MODULES  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
C, per, ri, r = 25, 40, 16, 16


def ortho(rows):
    q, _ = torch.linalg.qr(torch.randn(rows, r, generator=g, device=dev))
    return q.contiguous()


problems, energy = [], []
for (name, d_in, d_out) in MISTRAL_MODULES:
    for c in range(C):
        # trained-like: 4 families of shared factors + noise (App H "shared structure")
        fam_a = torch.randn(4, ri, d_in, generator=g, device=dev) / d_in ** 0.5
        fam_b = torch.randn(4, d_out, ri, generator=g, device=dev) / ri ** 0.5
        f = torch.arange(per, device=dev) % 4
        A = fam_a[f] + 0.3 * torch.randn(per, ri, d_in, generator=g, device=dev) / d_in ** 0.5
        B = fam_b[f] + 0.3 * torch.randn(per, d_out, ri, generator=g, device=dev) / ri ** 0.5
        problems.append({"a_stack": A.reshape(per * ri, d_in).contiguous(),
                         "bt_stack": B.transpose(1, 2).reshape(per * ri, d_out).contiguous(),
                         "U": ortho(d_out), "V": ortho(d_in), "sigma": torch.empty(per, r, r, device=dev)})
        energy.append(((B.transpose(1, 2) @ B) * (A @ A.transpose(1, 2))).sum())
torch.cuda.synchronize()
ws = cts.cts_jd_eigen_iteration(problems, r, iters)     # warm-up (allocations, kernel attributes, pools)
torch.cuda.synchronize()
runs = []
for rep in range(5):                                     # each from fresh random bases; median reported
    for q in problems:
        q["U"].copy_(ortho(q["U"].shape[0]))
        q["V"].copy_(ortho(q["V"].shape[0]))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    ws = cts.cts_jd_eigen_iteration(problems, r, iters)
    b.record()
    b.synchronize()
    runs.append(a.elapsed_time(b))
ms = sorted(runs)[len(runs) // 2]
cap = sum(float((q["sigma"] ** 2).sum()) for q in problems)
tot = sum(float(e) for e in energy)
print(f"{len(problems)} problems (7 modules x {C} clusters x {per} LoRAs, r_i={ri}, r={r}), {iters} iterations: "
      f"{ms:.1f} ms on the GPU, median of {len(runs)} (min {min(runs):.1f}; {', '.join(f'{x:.1f}' for x in runs)}; {ms / len(problems):.3f} ms "
      f"per cluster); captured energy {cap / tot:.4f}; wall {time.perf_counter() - t0:.2f} s")
