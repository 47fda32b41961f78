"""Shared helpers for the -m gpu parity tests (inputs in, comparisons out; no method arithmetic)."""
import numpy as np
import torch

from workloads import bf16_round, bf16_to_f64, direct_bank

PARITY_TOL = 5e-3   # north_star: per-token-row relative Frobenius error of delta_y vs the fp64 oracle


def dev_bf16(bits, dev="cuda"):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(dev)


def host_bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def quantized_bank(d_in, d_out, N, C, r, seed, cluster_of=None):
    """direct_bank rounded once to bf16: returns (bits dict, fp64-image dict)."""
    b = direct_bank(d_in, d_out, N, C, r, seed, cluster_of)
    bits = {k: bf16_round(b[k]) for k in ("in_basis", "out_basis", "sigma")}
    bits["cluster_of"] = b["cluster_of"]
    f64 = {k: bf16_to_f64(bits[k]) for k in ("in_basis", "out_basis", "sigma")}
    f64["cluster_of"] = b["cluster_of"]
    return bits, f64


def row_rel_err(got, ref):
    """Per-row ||got - ref|| / ||ref|| over rows with a nonzero reference."""
    num = np.linalg.norm(got - ref, axis=1)
    den = np.linalg.norm(ref, axis=1)
    ok = den > 0
    return num[ok] / den[ok]


def bf16_ulp(v):
    """Spacing of bf16 numbers at |v| (normal range)."""
    e = np.floor(np.log2(np.maximum(np.abs(v), 2.0 ** -126)))
    return 2.0 ** (e - 7)
