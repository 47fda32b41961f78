"""Pins for oracle.apply_ref: brute force, a hand-computed transpose check, Proposition 1,
the output-space form of the reconstruction error, and the invariants of the apply."""
import numpy as np
import pytest

from oracle import apply_ref, apply_dense_ref, apply_lora_ref, jd_full, jd_full_clustered
from workloads import (activations, bf16_round, bf16_to_f64, cluster_map, decode_tokens,
                       direct_bank, gen_loras)


def _bank(d_in, d_out, N, C, r, seed, quantize=True):
    b = direct_bank(d_in, d_out, N, C, r, seed)
    if quantize:
        for k in ("in_basis", "out_basis", "sigma"):
            b[k] = bf16_to_f64(bf16_round(b[k]))
    return b


def brute_apply(x, ta, cmap, inb, outb, sig, scale):
    """Scalar triple loop: s_k = sum_j V[j,k] x_j ; t_o = sum_k S[o,k] s_k ; dy_m = sum_o U[m,o] t_o."""
    T, d_in = x.shape
    r = inb.shape[2]
    d_out = outb.shape[1]
    dy = np.zeros((T, d_out))
    for t in range(T):
        i = int(ta[t])
        if i < 0:
            continue
        c = int(cmap[i])
        s = [sum(inb[c, j, k] * x[t, j] for j in range(d_in)) for k in range(r)]
        tt = [sum(sig[i, o, k] * s[k] for k in range(r)) for o in range(r)]
        for m in range(d_out):
            dy[t, m] = scale * sum(outb[c, m, o] * tt[o] for o in range(r))
    return dy


def test_tiny_brute_force_and_dense():
    b = _bank(12, 10, 5, 2, 3, seed=0)
    x = activations(9, 12, 1)
    ta = decode_tokens(9, 5, 2, frac_none=0.2)
    dy, _ = apply_ref(x, ta, b["cluster_of"], b["in_basis"], b["out_basis"], b["sigma"], 1.5)
    ref = brute_apply(x, ta, b["cluster_of"], b["in_basis"], b["out_basis"], b["sigma"], 1.5)
    np.testing.assert_allclose(dy, ref, rtol=1e-12, atol=1e-14)
    dense = apply_dense_ref(x, ta, b["cluster_of"], b["in_basis"], b["out_basis"], b["sigma"], 1.5)
    np.testing.assert_allclose(dy, dense, rtol=1e-11, atol=1e-13)


def test_sigma_orientation_hand_example():
    """Sigma row = out index: with U = V = I, Sigma = [[0,1],[0,0]] and x = e_2, t = Sigma s = e_1
    so Delta y = e_1.  A transposed Sigma would give 0 (tests must use non-symmetric Sigma)."""
    inb = np.eye(2)[None]
    outb = np.eye(2)[None]
    sig = np.array([[[0.0, 1.0], [0.0, 0.0]]])
    dy, _ = apply_ref(np.array([[0.0, 1.0]]), np.array([0]), np.array([0]), inb, outb, sig)
    np.testing.assert_array_equal(dy, [[1.0, 0.0]])


def test_in_out_roles_hand_example():
    """in_basis multiplies x (d_in side), out_basis produces y (d_out side): d_in=3, d_out=2."""
    inb = np.array([[[0.0], [0.0], [1.0]]])          # V = e_3 (3x1)
    outb = np.array([[[0.0], [2.0]]])                # U = 2 e_2 (2x1)
    sig = np.array([[[3.0]]])
    dy, y = apply_ref(np.array([[5.0, 7.0, 11.0]]), np.array([0]), np.array([0]), inb, outb, sig,
                      scale=0.5, y_base=np.array([[1.0, 1.0]]))
    np.testing.assert_array_equal(dy, [[0.0, 0.5 * 2.0 * 3.0 * 11.0]])
    np.testing.assert_array_equal(y, [[1.0, 34.0]])


@pytest.mark.parametrize("seed", range(3))
def test_proposition1_compressed_equals_original(seed):
    """Exact-span LoRAs are compressed losslessly at r >= r_span (Prop. 1), so the
    compressed apply equals B_i(A_i x) up to rounding."""
    Bs, As, _ = gen_loras("exact_span", 64, 48, 6, 2, seed, r_span=8)
    res = jd_full(Bs, As, 8)
    x = activations(40, 64, seed + 10)
    ta = decode_tokens(40, 6, seed + 20, frac_none=0.1)
    dy, _ = apply_ref(x, ta, np.zeros(6, np.int32), res["V"][None], res["U"][None], res["sigma"], 2.0)
    ref = apply_lora_ref(x, ta, Bs, As, 2.0)
    assert np.max(np.abs(dy - ref)) <= 1e-11 * np.max(np.abs(ref))


def test_output_space_error_equals_frobenius_error():
    """Summing ||Delta y_compressed - Delta y_lora||^2 over x = the standard basis gives exactly
    ||U Sigma_i V^T - B_i A_i||_F^2, the paper's reconstruction error (Sec. 6.2)."""
    Bs, As, _ = gen_loras("random", 20, 16, 5, 3, 7)
    res = jd_full(Bs, As, 4)
    for i in range(5):
        x = np.eye(20)
        ta = np.full(20, i, dtype=np.int32)
        dy, _ = apply_ref(x, ta, np.zeros(5, np.int32), res["V"][None], res["U"][None], res["sigma"])
        ref = apply_lora_ref(x, ta, Bs, As)
        err = np.linalg.norm(res["U"] @ res["sigma"][i] @ res["V"].T - Bs[i] @ As[i]) ** 2
        assert np.sum((dy - ref) ** 2) == pytest.approx(err, rel=1e-10)


def test_invariants():
    b = _bank(32, 24, 9, 3, 4, seed=3)
    args = (b["cluster_of"], b["in_basis"], b["out_basis"], b["sigma"])
    x1, x2 = activations(30, 32, 1), activations(30, 32, 2)
    ta = decode_tokens(30, 9, 5, frac_none=0.2)
    d1, _ = apply_ref(x1, ta, *args)
    d2, _ = apply_ref(x2, ta, *args)
    d12, _ = apply_ref(x1 + 2 * x2, ta, *args)
    np.testing.assert_allclose(d12, d1 + 2 * d2, rtol=1e-11, atol=1e-12)          # linearity
    assert np.all(d1[ta < 0] == 0)                                                 # -1 rows
    p = np.random.default_rng(0).permutation(30)
    dp, _ = apply_ref(x1[p], ta[p], *args)
    np.testing.assert_allclose(dp, d1[p], rtol=0, atol=1e-13)                      # permutation
    zero = dict(b, sigma=np.zeros_like(b["sigma"]))
    dz, yz = apply_ref(x1, ta, zero["cluster_of"], zero["in_basis"], zero["out_basis"], zero["sigma"],
                       y_base=x2[:, :24])
    assert np.all(dz == 0) and np.array_equal(yz, x2[:, :24])                       # Sigma = 0
    # mixed clusters == one call per cluster with the other tokens unbound
    acc = np.zeros_like(d1)
    for c in range(3):
        tac = np.where((ta >= 0) & (b["cluster_of"][np.maximum(ta, 0)] == c), ta, -1)
        dc, _ = apply_ref(x1, tac, *args)
        acc += dc
    np.testing.assert_array_equal(acc, d1)


def test_clustered_bank_from_jd_matches_per_cluster_loras():
    """Planted clusters of exact-span LoRAs: per-cluster JD is lossless, so the clustered apply
    reproduces each adapter's own B_i A_i x (Sec. 3.2 P:L162-166 + Prop. 1)."""
    Bs, As = [], []
    for f in range(3):
        b, a, _ = gen_loras("exact_span", 40, 36, 4, 2, 100 + f, r_span=5)
        Bs += b
        As += a
    assign = np.repeat(np.arange(3), 4).astype(np.int32)
    bank = jd_full_clustered(Bs, As, assign, 3, 5)
    x = activations(50, 40, 9)
    ta = decode_tokens(50, 12, 10)
    dy, _ = apply_ref(x, ta, bank["cluster_of"], bank["in_basis"], bank["out_basis"], bank["sigma"])
    ref = apply_lora_ref(x, ta, Bs, As)
    assert np.max(np.abs(dy - ref)) <= 1e-11 * np.max(np.abs(ref))


def test_project_ref_brute_force_and_special_cases():
    """project_ref = W0 x + Delta y (Sec. 3 P:L107-109 with Eq. 1): a scalar-loop W0 x plus the
    brute-force apply on tiny inputs; W0 = 0 reduces it to apply_ref, Sigma = 0 to the plain
    projection, and id -1 rows get the base projection only."""
    from oracle import project_ref
    T, d_in, d_out, N, C, r = 6, 5, 4, 3, 2, 2
    b = _bank(d_in, d_out, N, C, r, seed=3)
    g = np.random.default_rng(4)
    x = g.standard_normal((T, d_in))
    W0 = g.standard_normal((d_out, d_in))
    ta = np.array([0, 2, -1, 1, 0, -1])
    want = np.array([[sum(W0[o, j] * x[t, j] for j in range(d_in)) for o in range(d_out)] for t in range(T)])
    want += brute_apply(x, ta, b["cluster_of"], b["in_basis"], b["out_basis"], b["sigma"], 1.5)
    got = project_ref(x, W0, ta, b["cluster_of"], b["in_basis"], b["out_basis"], b["sigma"], 1.5)
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)
    dy, _ = apply_ref(x, ta, b["cluster_of"], b["in_basis"], b["out_basis"], b["sigma"], 1.5)
    assert np.allclose(project_ref(x, np.zeros_like(W0), ta, b["cluster_of"], b["in_basis"], b["out_basis"],
                                   b["sigma"], 1.5), dy, rtol=0, atol=1e-14)
    plain = project_ref(x, W0, ta, b["cluster_of"], b["in_basis"], b["out_basis"], np.zeros_like(b["sigma"]), 1.5)
    assert np.allclose(plain, want - brute_apply(x, ta, b["cluster_of"], b["in_basis"], b["out_basis"],
                                                 b["sigma"], 1.5), rtol=1e-12, atol=1e-12)
    assert np.array_equal(got[ta < 0], plain[ta < 0])
