"""Local-t debugging: fused apply vs the split shrink/expand path (no inter-CTA exchange) on small
decode shapes; prints max |diff| per module and the first differing rows."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if os.environ.get("CTS_PKG_ROOT"):          # bisecting: another build of the package
    sys.path.insert(0, os.environ["CTS_PKG_ROOT"])
import paper_2407_00066_b200 as cts  # noqa: E402
print("package:", cts.__file__, flush=True)
from workloads.gen_torch import direct_bank_torch, tokens_torch  # noqa: E402

dev = torch.device("cuda")
torch.manual_seed(0)


def run(tag, mods, N, C, r, T):
    banks = [direct_bank_torch(di, do, N, C, r, seed=m, device=dev, cluster_seed=50 + m) for m, (di, do) in enumerate(mods)]
    bank = cts.Bank([b["in_basis"] for b in banks], [b["out_basis"] for b in banks], [b["sigma"] for b in banks],
                    [b["cluster_of"] for b in banks])
    plan = cts.Plan(bank, T)
    plan_tokens = tokens_torch(T, N, 1, False, dev)
    plan.segment(plan_tokens)
    x = torch.randn(T, mods[0][0], device=dev).to(torch.bfloat16)
    grp = list(range(len(mods)))
    y1 = [torch.zeros(T, do, device=dev, dtype=torch.bfloat16) for (_, do) in mods]
    y2 = [torch.zeros_like(y) for y in y1]
    if os.environ.get("FUSED_ONLY"):
        from oracle import apply_ref  # noqa: F401  (reference via float64 torch below)
        for m in grp:
            b = banks[m]
            ta = plan_tokens.cpu().long()
            ib, ob, sg = b["in_basis"].double(), b["out_basis"].double(), b["sigma"].double()
            c = b["cluster_of"].long()[ta]
            s_ = torch.einsum("td,tdr->tr", x.double(), ib[c])
            t_ = torch.einsum("tor,tr->to", sg[ta], s_) * 2.0
            y2[m].copy_(torch.einsum("tdo,to->td", ob[c], t_).to(torch.bfloat16))
    else:
        plan.shrink_group(grp, [x] * len(grp), 2.0)
        plan.expand_group(grp, y2)
    torch.cuda.synchronize()
    plan.apply_group(grp, [x] * len(grp), y1, 2.0)
    torch.cuda.synchronize()
    for m in grp:
        d = (y1[m].float() - y2[m].float()).abs()
        bad = (d.max(dim=1).values > 1e-2 * (y2[m].float().abs().max(dim=1).values + 1e-3)).nonzero().flatten()
        print(f"{tag} module {m}: max|diff| {d.max().item():.3e}  ref max {y2[m].float().abs().max().item():.3e}  "
              f"bad rows {bad.numel()} / {T}  first {bad[:8].tolist()}", flush=True)
    plan.close()
    bank.close()


CASES = {
    "tiny": ("tiny ks=1", [(64, 64)], 4, 1, 4, 32),
    "one": ("one module ks>1", [(1024, 512)], 40, 4, 16, 300),
    "qkv": ("qkv-like", [(1024, 1024), (1024, 256), (1024, 256)], 300, 12, 16, 1024),
    "attn": ("cfg3 attn", [(4096, 4096), (4096, 1024), (4096, 1024)], 1000, 25, 16, 1024),
}
for name in (sys.argv[1:] or list(CASES)):
    tag, mods, N, C, r, T = CASES[name]
    run(tag, mods, N=N, C=C, r=r, T=T)
