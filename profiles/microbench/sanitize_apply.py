"""compute-sanitizer driver: small applies through every kernel path of libcts (the fused
single-launch kernel with its inter-CTA flags, the split shrink/expand launches, the r_pad 64
distributed finisher, segmentation with invalid ids, the TP partial path), each followed by a
stream sync so the tool reports per launch.  Run as
    compute-sanitizer --tool memcheck|racecheck|synccheck python profiles/microbench/sanitize_apply.py
Shapes are small (the tools serialize and instrument every access) but keep the decode structure:
several packed slots, a K split > 1, a ragged tail.  No oracle: the parity suite checks values."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00066_b200 as cts  # noqa: E402
from workloads.gen_torch import direct_bank_torch, tokens_torch  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)


def run(tag, mods, N, C, r, T, prefill=False, groups=None):
    banks = [direct_bank_torch(di, do, N, C, r, seed=m, device=dev, cluster_seed=50 + m)
             for m, (di, do) in enumerate(mods)]
    bank = cts.Bank([b["in_basis"] for b in banks], [b["out_basis"] for b in banks],
                    [b["sigma"] for b in banks], [b["cluster_of"] for b in banks])
    plan = cts.Plan(bank, T)
    tok = tokens_torch(T, N, 1, prefill, dev)
    tok[::7] = -1
    plan.segment(tok)
    x = torch.randn(T, max(di for di, _ in mods), device=dev).to(torch.bfloat16)
    ys = [torch.randn(T, do, device=dev).to(torch.bfloat16) for (_, do) in mods]
    for grp in groups or [[m] for m in range(len(mods))]:
        xs = [x[:, :mods[m][0]] for m in grp]
        plan.apply_group(grp, xs, [ys[m] for m in grp], 2.0)
        torch.cuda.synchronize()
        plan.shrink_group(grp, xs, 2.0)
        plan.expand_group(grp, [ys[m] for m in grp])
        torch.cuda.synchronize()
        parts = plan.new_partials(len(grp))
        plan.shrink_partial_group(grp, xs, parts, 2.0)
        plan.expand_reduced_group(grp, parts, [ys[m] for m in grp])
        torch.cuda.synchronize()
    assert plan.error() == (0, -1)
    bad = tok.clone()
    bad[3] = N + 5
    plan.segment(bad)
    plan.apply(0, x[:, :mods[0][0]], ys[0], 1.0)
    torch.cuda.synchronize()
    assert plan.error()[0] == 3
    plan.close()
    bank.close()
    print(f"{tag}: ok", flush=True)


def run_diag_and_pagein():
    """JD-Diag bank (CTS_SIGMA_DIAG) through the fused and split paths, then a slot page-in."""
    mods = [(1024, 512), (1024, 256)]
    banks = [direct_bank_torch(di, do, 200, 8, 16, seed=m, device=dev, cluster_seed=50 + m)
             for m, (di, do) in enumerate(mods)]
    bank = cts.Bank([b["in_basis"] for b in banks], [b["out_basis"] for b in banks],
                    [torch.diagonal(b["sigma"], dim1=1, dim2=2).contiguous() for b in banks],
                    [b["cluster_of"] for b in banks])
    plan = cts.Plan(bank, 300)
    plan.segment(tokens_torch(300, 200, 3, False, dev))
    x = torch.randn(300, 1024, device=dev).to(torch.bfloat16)
    ys = [torch.randn(300, do, device=dev).to(torch.bfloat16) for (_, do) in mods]
    plan.apply_group([0, 1], [x, x], ys, 2.0)
    plan.shrink_group([0, 1], [x, x], 2.0)
    plan.expand_group([0, 1], ys)
    torch.cuda.synchronize()
    bank.write_clusters(1, [2, 5], banks[1]["in_basis"][:2].contiguous(), banks[1]["out_basis"][:2].contiguous())
    plan.apply_group([0, 1], [x, x], ys, 2.0)
    torch.cuda.synchronize()
    plan.close()
    bank.close()
    print("diag bank + page-in: ok", flush=True)


def run_jd():
    """GPU compression: tensor-core path (K multiple of 4) and CUDA-core fallback in one batch each."""
    g = torch.Generator(device=dev).manual_seed(0)
    # (6, 16) and (21, 16): K-space iterations (K = 96, 336: partial and mirrored Gram tiles);
    # (3, 6): CUDA-core fallback; r = 32 with K = 96: K-space at r_pad 32
    for (n, ri, r) in ((6, 16, 16), (21, 16, 16), (3, 6, 16), (6, 16, 32)):
        d_in, d_out = 256, 192
        prob = {"a_stack": torch.randn(n * ri, d_in, generator=g, device=dev) / 16,
                "bt_stack": torch.randn(n * ri, d_out, generator=g, device=dev) / 4,
                "U": torch.linalg.qr(torch.randn(d_out, r, generator=g, device=dev))[0].contiguous(),
                "V": torch.linalg.qr(torch.randn(d_in, r, generator=g, device=dev))[0].contiguous(),
                "sigma": torch.empty(n, r, r, device=dev)}
        ws = cts.cts_jd_eigen_iteration([prob], r, 3)
        torch.cuda.synchronize()
        del ws
    print("GPU compression (K-space, tensor-core d-space and CUDA-core paths): ok", flush=True)


if not os.environ.get("JD_ONLY"):
    run_diag_and_pagein()
run_jd()
if os.environ.get("JD_ONLY"):
    sys.exit(0)
run("tiny r=4 (r_pad 16)", [(64, 64)], N=4, C=1, r=4, T=32)
run("decode-like r=16, 3 modules grouped", [(1024, 1024), (1024, 256), (1024, 256)], N=100, C=5, r=16, T=200,
    groups=[[0, 1, 2]])
run("cfg2-like r=64 (distributed finisher)", [(2048, 2048)], N=16, C=1, r=64, T=96)
run("r=32", [(1024, 512)], N=32, C=3, r=32, T=150)
run("prefill-like r=16", [(512, 1024)], N=20, C=4, r=16, T=900, prefill=True)
print("sanitize_apply: all paths ran")
