"""Seeded NumPy (PCG64) generators for LoRA collections, compressed banks and token batches.

Shapes follow the paper's workloads: Mistral-7B projections (D = 4096, P:L1003 read as
4096), rank-16 LoRAs on q/k/v (App C), 1000+ adapters in
25 clusters at r = 16, requests assigned to LoRAs at random.
No method arithmetic lives here (see package docstring).
"""
import numpy as np

# (name, d_in, d_out) of one Mistral-7B decoder layer; 32 layers -> 224 modules.
MISTRAL_MODULES = (
    ("q", 4096, 4096),
    ("k", 4096, 1024),
    ("v", 4096, 1024),
    ("o", 4096, 4096),
    ("gate", 4096, 14336),
    ("up", 4096, 14336),
    ("down", 14336, 4096),
)
MISTRAL_LAYERS = 32


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _orthonormal(g: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    """Haar-like orthonormal columns: QR of a Gaussian with the R-diagonal sign fixed positive."""
    q, r = np.linalg.qr(g.standard_normal((rows, cols)))
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s


def gen_loras(kind: str, d_in: int, d_out: int, n: int, r_i: int, seed: int,
              r_span: int | None = None, n_families: int = 1, noise: float = 0.3):
    """A collection {(B_i, A_i)}: B_i is d_out x r_i, A_i is r_i x d_in (paper Sec. 3).

    kind:
      exact_span   all B_i (A_i^T) lie in one shared r_span-dimensional column (row) space, so
                   JD-Full at r >= r_span is lossless (Proposition 1).
      trained_like n_families planted families: B_i = Bbar_f + noise*E_i (shared structure, App H
                   P:L2230); family f = i mod n_families.
      random       i.i.d. Gaussian factors (App H "random LoRAs").
      orthogonal   r_i = 1, B_i = u_i, A_i = v_i^T with {u_i}, {v_i} orthonormal: unit-norm,
                   mutually orthogonal products (Corollary).
    Returns (Bs, As, family) with family an int array of length n.
    """
    g = rng(seed)
    family = np.arange(n) % max(n_families, 1)
    Bs, As = [], []
    if kind == "exact_span":
        rs = r_span if r_span is not None else r_i
        U0 = _orthonormal(g, d_out, rs)
        V0 = _orthonormal(g, d_in, rs)
        for _ in range(n):
            Bs.append(U0 @ g.standard_normal((rs, r_i)))
            As.append(g.standard_normal((r_i, rs)) @ V0.T)
    elif kind == "trained_like":
        Bbar = [g.standard_normal((d_out, r_i)) / np.sqrt(r_i) for _ in range(n_families)]
        Abar = [g.standard_normal((r_i, d_in)) / np.sqrt(d_in) for _ in range(n_families)]
        for i in range(n):
            f = family[i]
            Bs.append(Bbar[f] + noise * g.standard_normal((d_out, r_i)) / np.sqrt(r_i))
            As.append(Abar[f] + noise * g.standard_normal((r_i, d_in)) / np.sqrt(d_in))
    elif kind == "random":
        for _ in range(n):
            Bs.append(g.standard_normal((d_out, r_i)) / np.sqrt(r_i))
            As.append(g.standard_normal((r_i, d_in)) / np.sqrt(d_in))
    elif kind == "orthogonal":
        if n > min(d_in, d_out):
            raise ValueError("orthogonal collection needs n <= min(d_in, d_out)")
        U0 = _orthonormal(g, d_out, n)
        V0 = _orthonormal(g, d_in, n)
        for i in range(n):
            Bs.append(U0[:, i:i + 1].copy())
            As.append(V0[:, i:i + 1].T.copy())
    else:
        raise ValueError(f"unknown LoRA kind {kind!r}")
    return Bs, As, family


def cluster_map(N: int, C: int, seed: int) -> np.ndarray:
    """adapter -> cluster, pi(i) mod C with a seeded permutation pi: balanced (sizes differ <= 1)."""
    return (rng(seed).permutation(N) % C).astype(np.int32)


def direct_bank(d_in: int, d_out: int, N: int, C: int, r: int, seed: int,
                cluster_of: np.ndarray | None = None):
    """A compressed bank drawn directly (configs 3-5, where per-cluster JD of 224 x C solves is
    impractical): per cluster orthonormal in_basis (paper V_c, d_in x r) and
    out_basis (paper U_c, d_out x r); per adapter a non-symmetric Sigma_i = G_i a_i / ||G_i||_F
    with a_i = exp(U[ln 1/2, ln 2]) standing in for the restored norms.
    Returns fp64 arrays; round with bf16_round before handing them to either side.
    """
    g = rng(seed)
    in_basis = np.stack([_orthonormal(g, d_in, r) for _ in range(C)])
    out_basis = np.stack([_orthonormal(g, d_out, r) for _ in range(C)])
    G = g.standard_normal((N, r, r))
    a = np.exp(g.uniform(np.log(0.5), np.log(2.0), size=N))
    sigma = G * (a / np.linalg.norm(G.reshape(N, -1), axis=1))[:, None, None]
    if cluster_of is None:
        cluster_of = cluster_map(N, C, seed + 7919)
    return {"in_basis": in_basis, "out_basis": out_basis, "sigma": sigma,
            "cluster_of": np.asarray(cluster_of, dtype=np.int32)}


def decode_tokens(T: int, N: int, seed: int, frac_none: float = 0.0) -> np.ndarray:
    """One token per request, adapter uniform on [0, N) ("assigned ... at random");
    a fraction frac_none of tokens carry no adapter (-1)."""
    g = rng(seed)
    ta = g.integers(0, N, size=T).astype(np.int32)
    if frac_none > 0:
        ta[g.random(T) < frac_none] = -1
    return ta


def prefill_tokens(T: int, N: int, seed: int, lmin: int = 128, lmax: int = 256) -> np.ndarray:
    """Requests of length U{lmin..lmax}, adapter uniform per request, concatenated to T tokens
    (SURVEY 8(c) c5 #21): contiguous same-adapter runs; some clusters may be empty."""
    g = rng(seed)
    out = np.empty(T, dtype=np.int32)
    pos = 0
    while pos < T:
        L = int(g.integers(lmin, lmax + 1))
        out[pos:pos + L] = int(g.integers(0, N))
        pos += L
    return out


def activations(T: int, d: int, seed: int) -> np.ndarray:
    """x or y_base rows ~ N(0, 1), returned as fp64 (round with bf16_round)."""
    return rng(seed).standard_normal((T, d))
