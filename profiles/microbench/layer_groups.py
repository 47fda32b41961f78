"""One Mistral-7B layer in bench.py's launch configuration (segment, then grouped applies {q,k,v},
{o}, {gate,up}, {down}), synchronizing after every launch -- for compute-sanitizer / debugging.
N, C, T from the environment (default cfg3)."""
import os
import sys

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
plan.segment(tokens_torch(T, N, 1, T > 4096, dev))
xs = {"attn": torch.randn(T, 4096, device=dev).to(torch.bfloat16), "o": torch.randn(T, 4096, device=dev).to(torch.bfloat16),
      "mlp": torch.randn(T, 4096, device=dev).to(torch.bfloat16), "down": torch.randn(T, 14336, device=dev).to(torch.bfloat16)}
ys = [torch.randn(T, do, device=dev).to(torch.bfloat16) for (_, _, do) in MISTRAL_MODULES]
groups = {"attn": [0, 1, 2], "o": [3], "mlp": [4, 5], "down": [6]}
for rep in range(2):
    for name, gm in groups.items():
        plan.apply_group(gm, [xs[name]] * len(gm), [ys[m] for m in gm], 2.0)
        torch.cuda.synchronize()
        print(f"rep {rep} group {name} {gm}: ok", flush=True)
print("layer_groups: ok")
