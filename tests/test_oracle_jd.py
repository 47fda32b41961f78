"""Pins for oracle.jd_full: constraints, stationarity, Pythagoras, Proposition 1, Theorem 1 (with
the corrected lower bound), the Corollary, Eckart-Young, monotonicity, and printed values."""
import numpy as np
import pytest

from oracle import jd_full, jd_objective, mean_relative_error, svd_truncate
from workloads import gen_loras


def _L(Bs, As):
    return np.stack([(B @ A).ravel() for B, A in zip(Bs, As)], axis=1)


@pytest.mark.parametrize("kind", ["random", "trained_like", "exact_span"])
def test_orthonormal_stationary_pythagoras(kind):
    Bs, As, _ = gen_loras(kind, 30, 24, 6, 3, 11, r_span=10, n_families=2)
    res = jd_full(Bs, As, 5)
    U, V, S = res["U"], res["V"], res["sigma"]
    np.testing.assert_allclose(U.T @ U, np.eye(5), atol=1e-12)          # Eq. 2 constraint
    np.testing.assert_allclose(V.T @ V, np.eye(5), atol=1e-12)
    for B, A, Si in zip(Bs, As, S):                                       # dObj/dSigma_i = 0
        np.testing.assert_allclose(U.T @ (U @ Si @ V.T - B @ A) @ V, 0, atol=1e-12)
    direct = jd_objective(Bs, As, U, V, S)                                # Pythagoras
    assert res["objective"] == pytest.approx(direct, rel=1e-9, abs=1e-12)


def test_proposition1_lossless_iff_r_ge_rtilde():
    """Prop. 1: exact at r = r~, nonzero error below."""
    Bs, As, _ = gen_loras("exact_span", 40, 32, 5, 2, 3, r_span=6)
    tot = sum(np.sum((B @ A) ** 2) for B, A in zip(Bs, As))
    lossless = jd_full(Bs, As, 6)
    assert jd_objective(Bs, As, lossless["U"], lossless["V"], lossless["sigma"]) < 1e-24 * tot
    lossy = jd_full(Bs, As, 5)
    assert jd_objective(Bs, As, lossy["U"], lossy["V"], lossy["sigma"]) > 1e-3 * tot
    # generic (random) LoRAs: r~ = sum r_i = 8 (config-1 shape: 4 LoRAs of rank 2)
    Bs, As, _ = gen_loras("random", 64, 64, 4, 2, 5)
    assert jd_full(Bs, As, 8)["objective"] < 1e-20
    assert jd_full(Bs, As, 4)["objective"] > 1e-2


def test_app_h_zero_error_at_r256_with_10_loras():
    """App H table: 10 LoRAs of rank 16 at r = 256 reconstruct with error 0.00, as
    Prop. 1 predicts since sum r_i = 160 <= 256."""
    Bs, As, _ = gen_loras("random", 320, 300, 10, 16, 9)
    res = jd_full(Bs, As, 256, method="span")
    assert mean_relative_error(Bs, As, res["U"], res["V"], res["sigma"]) < 1e-10


@pytest.mark.parametrize("seed", range(4))
def test_monotone_per_half_step(seed):
    """Each U and V step cannot decrease sum ||Sigma_i||^2 (App A.1 "decreases the objective in
    each step")."""
    Bs, As, _ = gen_loras("random", 25, 20, 7, 3, seed)
    tr = np.array(jd_full(Bs, As, 4)["captured_trace"])
    assert np.all(np.diff(tr) >= -1e-12 * tr[-1])


@pytest.mark.parametrize("seed", range(3))
def test_monotone_in_r(seed):
    Bs, As, _ = gen_loras("trained_like", 30, 28, 8, 4, seed, n_families=3)
    objs = [jd_full(Bs, As, r)["objective"] for r in range(1, 13)]
    assert np.all(np.diff(objs) <= 1e-10)


@pytest.mark.parametrize("r", [1, 3, 5])
def test_single_lora_is_truncated_svd(r):
    """k = n (one LoRA per cluster) reduces JD to an SVD by Eckart-Young (Eq. 4)."""
    Bs, As, _ = gen_loras("random", 20, 18, 1, 8, 4)
    res = jd_full(Bs, As, r, normalize=False)
    U, S, V = svd_truncate(Bs[0], As[0], r)
    np.testing.assert_allclose(res["U"] @ res["sigma"][0] @ res["V"].T, U @ S @ V.T, atol=1e-10)
    sv = np.linalg.svd(Bs[0] @ As[0], compute_uv=False)
    assert res["objective"] == pytest.approx(np.sum(sv[r:] ** 2), rel=1e-9, abs=1e-12)


@pytest.mark.parametrize("seed", range(10))
def test_theorem1_sandwich_corrected(seed):
    """Theorem 1.  Upper bound: sum ||Sigma_i||^2 <= sum_{j<=min(r^2,n)} sigma_j(L)^2.
    Lower bound as CORRECTED (reading R7): (1/n) sum_{j<=r} sigmabar_j^2 <= sum||Sigma_i||^2;
    the printed bound drops the 1/n of Cauchy-Schwarz in the proof's "Jensen" step."""
    g = np.random.default_rng(seed)
    n, r = int(g.integers(2, 9)), int(g.integers(1, 5))
    Bs, As, _ = gen_loras("random", 16, 14, n, 2, 50 + seed)
    res = jd_full(Bs, As, r, normalize=False, iters=30)
    cap = np.sum(res["sigma"] ** 2)
    sL = np.linalg.svd(_L(Bs, As), compute_uv=False)
    sbar = np.linalg.svd(sum(B @ A for B, A in zip(Bs, As)), compute_uv=False)
    assert cap <= np.sum(sL[:min(r * r, n)] ** 2) * (1 + 1e-12)
    assert np.sum(sbar[:r] ** 2) / n <= cap * (1 + 1e-12)


def test_theorem1_printed_lower_bound_counterexample():
    """n identical adapters: the printed lower bound sum_{j<=r} sigmabar_j^2 equals n times the
    achievable optimum, so it cannot hold (why the corrected 1/n form is used)."""
    Bs, As, _ = gen_loras("random", 12, 10, 1, 3, 2)
    Bs, As = Bs * 3, As * 3
    res = jd_full(Bs, As, 1, normalize=False)
    cap = np.sum(res["sigma"] ** 2)
    sbar = np.linalg.svd(3 * (Bs[0] @ As[0]), compute_uv=False)
    assert np.sum(sbar[:1] ** 2) == pytest.approx(3 * cap, rel=1e-9)


@pytest.mark.parametrize("n,r", [(32, 3), (20, 2), (9, 4), (6, 3)])
def test_corollary_orthogonal_unit_loras(n, r):
    """Corollary, inequality read as 1 - min(r^2/n, 1) <= err <= 1 - 1/n (reading R3);
    r >= min_i rank = 1 makes the upper side hold (reading R8)."""
    Bs, As, _ = gen_loras("orthogonal", 40, 40, n, 1, n + r)
    res = jd_full(Bs, As, r)
    err = jd_objective(Bs, As, res["U"], res["V"], res["sigma"]) / n
    assert 1 - min(r * r / n, 1) - 1e-12 <= err <= 1 - 1 / n + 1e-12
    # this instance hits exactly r of the n unit LoRAs: error 1 - r/n
    assert err == pytest.approx(1 - r / n, abs=1e-9)


def test_span_and_direct_agree():
    Bs, As, _ = gen_loras("trained_like", 60, 50, 7, 3, 21, n_families=2)
    a = jd_full(Bs, As, 6, method="direct")
    b = jd_full(Bs, As, 6, method="span")
    assert a["objective"] == pytest.approx(b["objective"], rel=1e-9)
    np.testing.assert_allclose(a["U"] @ a["U"].T, b["U"] @ b["U"].T, atol=1e-8)
    np.testing.assert_allclose(a["V"] @ a["V"].T, b["V"] @ b["V"].T, atol=1e-8)


def test_structured_reconstructs_better_than_random():
    """App H property only: shared structure is retained, random is not.
    The printed random-LoRA values are parity-unpinned (distribution unknown, reading R10)."""
    St, At, _ = gen_loras("trained_like", 64, 64, 20, 4, 1, n_families=2, noise=0.3)
    Sr, Ar, _ = gen_loras("random", 64, 64, 20, 4, 1)
    et = jd_full(St, At, 8)
    er = jd_full(Sr, Ar, 8)
    assert (mean_relative_error(St, At, et["U"], et["V"], et["sigma"])
            < mean_relative_error(Sr, Ar, er["U"], er["V"], er["sigma"]))


def test_convergence_criterion_stops_early():
    Bs, As, _ = gen_loras("trained_like", 30, 30, 6, 2, 3, n_families=1, noise=0.05)
    res = jd_full(Bs, As, 4, iters=50, tol=1e-3)
    assert 1 <= res["iters"] < 50


# ---------------------------------------------------------------- App A.2 eigenvalue iteration
def test_orthogonalize_is_qr_with_positive_diagonal():
    from oracle import orthogonalize
    X = np.random.default_rng(0).standard_normal((40, 6))
    Q = orthogonalize(X)
    assert np.allclose(Q.T @ Q, np.eye(6), atol=1e-12)
    R = Q.T @ X                                        # upper triangular with positive diagonal
    assert np.allclose(np.tril(R, -1), 0, atol=1e-12) and np.all(np.diag(R) > 0)
    assert np.allclose(Q @ R, X, atol=1e-12)


def test_eigen_iteration_fixed_point_at_alternating_optimum():
    """At a converged App A.1 solution U spans the top-r eigenvectors of M (M U = U Lambda), so
    U0^(k+1) = U Lambda and orthogonalize gives U back (up to column signs): the App A.2 iteration
     must stay there."""
    from oracle import jd_eigen_iteration
    Bs, As, _ = gen_loras("trained_like", 40, 36, 6, 3, seed=5, n_families=2)
    res = jd_full(Bs, As, 4, iters=200, normalize=False, method="direct")
    out = jd_eigen_iteration(Bs, As, res["U"], res["V"], iters=3)
    PU, PV = res["U"] @ res["U"].T, res["V"] @ res["V"].T
    assert np.allclose(out["U"] @ out["U"].T, PU, atol=1e-8)
    assert np.allclose(out["V"] @ out["V"].T, PV, atol=1e-8)
    assert np.allclose(out["captured_trace"], out["captured_trace"][0], rtol=1e-10)


def test_eigen_iteration_single_adapter_is_svd_subspace_iteration():
    """n = 1: U0 <- B A V V^T A^T B^T U, i.e. (BA)(BA)^T-power steps coupled with V; the iteration
    converges to the top-r left / right singular subspaces of B A (Eckart-Young, Eq. 4),
    checked against numpy's SVD."""
    from oracle import jd_eigen_iteration, orthogonalize
    g = np.random.default_rng(3)
    B, A = g.standard_normal((30, 8)), g.standard_normal((8, 25))
    r = 3
    out = jd_eigen_iteration([B], [A], orthogonalize(g.standard_normal((30, r))),
                             orthogonalize(g.standard_normal((25, r))), iters=300)
    u, s, vt = np.linalg.svd(B @ A)
    assert np.allclose(out["U"] @ out["U"].T, u[:, :r] @ u[:, :r].T, atol=1e-8)
    assert np.allclose(out["V"] @ out["V"].T, vt[:r].T @ vt[:r], atol=1e-8)
    assert np.isclose(out["captured_trace"][-1], np.sum(s[:r] ** 2), rtol=1e-10)


def test_eigen_iteration_exact_span_is_lossless():
    """Adapters in a shared rank-r span (Prop. 1): from a generic start the iteration
    captures all the energy, and U Sigma_i V^T reproduces every B_i A_i."""
    from oracle import jd_eigen_iteration, orthogonalize
    Bs, As, _ = gen_loras("exact_span", 48, 40, 5, 2, seed=9, r_span=4)
    g = np.random.default_rng(1)
    out = jd_eigen_iteration(Bs, As, orthogonalize(g.standard_normal((40, 4))),
                             orthogonalize(g.standard_normal((48, 4))), iters=100)
    for B, A, S in zip(Bs, As, out["sigma"]):
        assert np.allclose(out["U"] @ S @ out["V"].T, B @ A, atol=1e-8 * np.abs(B @ A).max())


def test_mean_relative_error_hand_computed():
    """Pin of the Sec. 6.2 metric ("mean relative reconstruction error"), hand-computed on a
    2-adapter, d = 2, r = 1 example (no call into the method's solver):
        B_1 A_1 = [[1, 0], [0, 0]], B_2 A_2 = [[0, 0], [0, 2]], U = V = e_1, Sigma_1 = 0.5, Sigma_2 = 1
        adapter 1: ||[[0.5,0],[0,0]] - [[1,0],[0,0]]||_F / 1 = 0.5
        adapter 2: ||[[1,0],[0,0]] - [[0,0],[0,2]]||_F / 2 = sqrt(5) / 2
        mean = (0.5 + sqrt(5)/2) / 2 = 0.80901699...
    A squared norm in the denominator (0.25 + sqrt(5)/4)/2, a squared ratio (0.25 + 5/4)/2, or a sum
    instead of the mean (1.618...) all miss this value."""
    Bs = [np.array([[1.0], [0.0]]), np.array([[0.0], [2.0]])]
    As = [np.array([[1.0, 0.0]]), np.array([[0.0, 1.0]])]
    U = V = np.array([[1.0], [0.0]])
    sigma = np.array([[[0.5]], [[1.0]]])
    assert abs(mean_relative_error(Bs, As, U, V, sigma) - (0.5 + np.sqrt(5) / 2) / 2) < 1e-15
