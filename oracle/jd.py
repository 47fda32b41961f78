"""Oracle for the offline compression: JD-Full (joint diagonalization with full Sigma_i).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  fp64 NumPy throughout.

Follows PAPER.md Sec. 3.1 and App A.1 "Case 1" step by step:
  objective      sum_i ||B_i A_i - U Sigma_i V^T||_F^2                  (Eq. 1)
  constraint     U^T U = V^T V = I_r, Sigma_i full                        (Eq. 2)
  optimal Sigma  Sigma_i = U^T B_i A_i V                                  (Eq. sigmastar)
  U step         U <- top-r eigenvectors of M = sum_i B_iA_i V V^T A_i^T B_i^T
  V step         V <- top-r eigenvectors of N = sum_i A_i^T B_i^T U U^T B_i A_i
  normalization  ||B_i A_i||_F = 1 before JD, original norms restored after (Sec 6.1)
  iterations     ten, or until the App H criterion with tau = 1e-3
Readings where the paper is silent: the initialization is HOSVD (top-r
eigenvectors of the summed Gram matrices, i.e. the U/V steps with V V^T = I / U U^T = I); ties
and rank deficiency are resolved by numpy.linalg.eigh's order; each basis column is sign-fixed so
its largest-magnitude entry is positive.
"""
import numpy as np


def lora_product(B, A) -> np.ndarray:
    """B_i A_i, the LoRA update of W_0 (Sec. 3)."""
    return np.asarray(B, dtype=np.float64) @ np.asarray(A, dtype=np.float64)


def sigma_star(U, V, B, A) -> np.ndarray:
    """Sigma_i = U^T B_i A_i V (Eq. sigmastar), parenthesized as (U^T B_i)(A_i V)."""
    return (U.T @ B) @ (A @ V)


def _sign_fix(Q: np.ndarray) -> np.ndarray:
    idx = np.argmax(np.abs(Q), axis=0)
    s = np.sign(Q[idx, np.arange(Q.shape[1])])
    s[s == 0] = 1.0
    return Q * s


def _top_eigvecs(M: np.ndarray, r: int) -> np.ndarray:
    """r eigenvectors of the symmetric PSD matrix M with largest eigenvalues."""
    w, Q = np.linalg.eigh(0.5 * (M + M.T))
    order = np.argsort(-w, kind="stable")[:r]
    return _sign_fix(Q[:, order])


def _u_step(P, V, r):
    """M = sum_i P_i V V^T P_i^T, parenthesized as (P_i V)(P_i V)^T."""
    M = sum((Pi @ V) @ (Pi @ V).T for Pi in P)
    return _top_eigvecs(M, r)


def _v_step(P, U, r):
    """N = sum_i P_i^T U U^T P_i = sum_i (P_i^T U)(P_i^T U)^T."""
    N = sum((Pi.T @ U) @ (Pi.T @ U).T for Pi in P)
    return _top_eigvecs(N, r)


def _captured(P, U, V) -> float:
    """sum_i ||U^T P_i V||_F^2, the quantity the alternation maximizes (Eq. optUV)."""
    return float(sum(np.sum((U.T @ Pi @ V) ** 2) for Pi in P))


def _complete(Q: np.ndarray, r: int) -> np.ndarray:
    """Deterministic orthonormal completion of Q (d x p, p < r) to d x r using standard basis
    vectors in index order (used only when the shared span is smaller than r)."""
    d = Q.shape[0]
    cols = [Q[:, j] for j in range(Q.shape[1])]
    for k in range(d):
        if len(cols) >= r:
            break
        e = np.zeros(d)
        e[k] = 1.0
        for c in cols:
            e -= (c @ e) * c
        n = np.linalg.norm(e)
        if n > 1e-8:
            cols.append(e / n)
    return np.stack(cols, axis=1)


def _normalize(Bs, As):
    """B_i / ||B_i A_i||_F so each LoRA product has unit Frobenius norm."""
    norms = np.array([np.sqrt(np.trace((B.T @ B) @ (A @ A.T))) for B, A in zip(Bs, As)])
    return [B / n for B, n in zip(Bs, norms)], norms


def _converged(U0, U1, V0, V1, tau) -> bool:
    """App H criterion."""
    du = np.linalg.norm(U1 - U0 @ (U0.T @ U1)) / np.linalg.norm(U1)
    dv = np.linalg.norm(V1 - V0 @ (V0.T @ V1)) / np.linalg.norm(V1)
    return max(du, dv) < tau


def _alternate(P, r, iters, tol):
    """HOSVD init, then App A.1 Case 1 alternation; returns (U, V, captured trace, iters run)."""
    d_out, d_in = P[0].shape
    U = _u_step(P, np.eye(d_in), r)
    V = _v_step(P, np.eye(d_out), r)
    trace = [_captured(P, U, V)]
    run = 0
    for _ in range(iters):
        U1 = _u_step(P, V, r)
        trace.append(_captured(P, U1, V))
        V1 = _v_step(P, U1, r)
        trace.append(_captured(P, U1, V1))
        run += 1
        done = tol is not None and _converged(U, U1, V, V1, tol)
        U, V = U1, V1
        if done:
            break
    return U, V, trace, run


def jd_full(Bs, As, r: int, iters: int = 10, tol: float | None = None,
            normalize: bool = True, method: str = "auto"):
    """JD-Full_r({B_i A_i}) (Eq. 2) by the alternating algorithm of App A.1.

    method="direct" runs App A.1 literally on the d_out x d_out / d_in x d_in matrices M, N.
    method="span" runs the same iteration inside the span of the stacked factors: with
    Q_B R_B = qr([B_1..B_n]) and Q_A R_A = qr([A_1^T..A_n^T]) every product is
    B_i A_i = Q_B K_i Q_A^T with a small core K_i, and range(M) lies in span(Q_B) (resp. N in
    span(Q_A)), so the eigenvectors are Q_B u, Q_A v -- the identical iterates, cheaper.
    "auto" picks direct when max(d) <= 512.

    Returns dict(U (d_out x r) = out basis, V (d_in x r) = in basis, sigma (n x r x r) computed on
    the ORIGINAL norms, objective = sum_i ||B_iA_i - U Sigma_i V^T||^2 via Pythagoras,
    captured_trace on the normalized problem, iters).
    """
    Bs = [np.asarray(B, dtype=np.float64) for B in Bs]
    As = [np.asarray(A, dtype=np.float64) for A in As]
    d_out, d_in = Bs[0].shape[0], As[0].shape[1]
    Bn, _ = _normalize(Bs, As) if normalize else (Bs, None)
    if method == "auto":
        method = "direct" if max(d_out, d_in) <= 512 else "span"
    if method == "direct":
        P = [B @ A for B, A in zip(Bn, As)]
        U, V, trace, run = _alternate(P, r, iters, tol)
    elif method == "span":
        QB, RB = np.linalg.qr(np.concatenate(Bn, axis=1))
        QA, RA = np.linalg.qr(np.concatenate([A.T for A in As], axis=1))
        K, col = [], 0
        for B in Bn:
            ri = B.shape[1]
            K.append(RB[:, col:col + ri] @ RA[:, col:col + ri].T)
            col += ri
        p = QB.shape[1]
        rr = min(r, p)
        u, v, trace, run = _alternate(K, rr, iters, tol)
        U = _sign_fix(QB @ u)
        V = _sign_fix(QA @ v)
        if rr < r:
            U = _complete(U, r)
            V = _complete(V, r)
    else:
        raise ValueError(method)
    sig = np.stack([sigma_star(U, V, B, A) for B, A in zip(Bs, As)])
    total = sum(np.sum((B.T @ B) * (A @ A.T)) for B, A in zip(Bs, As))
    objective = float(total - np.sum(sig ** 2))
    return {"U": U, "V": V, "sigma": sig, "objective": objective,
            "captured_trace": trace, "iters": run}


def jd_full_clustered(Bs, As, assignment, C: int, r: int, iters: int = 10,
                      tol: float | None = None, normalize: bool = True, method: str = "auto"):
    """Per-cluster JD-Full for a GIVEN assignment (Sec. 3.2; App A.3 "Step 1",
    P:L566).  The assignment search itself (k-means + reassignment) is out of scope: it is an
    input here.  Returns the bank in role names: in_basis[c] = V_c (d_in x r),
    out_basis[c] = U_c (d_out x r), sigma[i] (row = out index), cluster_of[i]."""
    assignment = np.asarray(assignment, dtype=np.int32)
    d_out, d_in = Bs[0].shape[0], As[0].shape[1]
    in_basis = np.zeros((C, d_in, r))
    out_basis = np.zeros((C, d_out, r))
    sigma = np.zeros((len(Bs), r, r))
    for c in range(C):
        members = np.nonzero(assignment == c)[0]
        if members.size == 0:
            continue
        res = jd_full([Bs[i] for i in members], [As[i] for i in members], r, iters, tol,
                      normalize, method)
        in_basis[c] = res["V"]
        out_basis[c] = res["U"]
        sigma[members] = res["sigma"]
    return {"in_basis": in_basis, "out_basis": out_basis, "sigma": sigma,
            "cluster_of": assignment}


def jd_objective(Bs, As, U, V, sigma) -> float:
    """sum_i ||B_i A_i - U Sigma_i V^T||_F^2 evaluated directly (Eq. 1); small d."""
    return float(sum(np.sum((B @ A - U @ S @ V.T) ** 2) for B, A, S in zip(Bs, As, sigma)))


def mean_relative_error(Bs, As, U, V, sigma) -> float:
    """mean_i ||U Sigma_i V^T - B_i A_i||_F / ||B_i A_i||_F (Sec. 6.2); small d."""
    errs = [np.linalg.norm(U @ S @ V.T - B @ A) / np.linalg.norm(B @ A)
            for B, A, S in zip(Bs, As, sigma)]
    return float(np.mean(errs))


def svd_truncate(B, A, r: int):
    """SVD_r(B_i A_i) = U_i Sigma_i V_i^T (Eq. 4): the k = n extreme of clustering."""
    u, s, vt = np.linalg.svd(np.asarray(B) @ np.asarray(A), full_matrices=False)
    return u[:, :r], np.diag(s[:r]), vt[:r].T


def orthogonalize(X) -> np.ndarray:
    """Q of the reduced QR of X with diag(R) > 0 (the unique orthonormal basis whose R has a positive
    diagonal) -- the `orthogonalize` of App A.2 ("e.g. by using the Q part of the
    reduced-size QR factorization")."""
    Q, R = np.linalg.qr(np.asarray(X, dtype=np.float64))
    s = np.sign(np.diag(R))
    s[s == 0] = 1.0
    return Q * s


def jd_eigen_iteration(Bs, As, U0, V0, iters: int):
    """App A.2 "Additional Eigenvalue Iteration Algorithm", the GPU-oriented
    alternative to App A.1 Case 1, step by step and parenthesized as the paper writes it:
        U0^(k+1) <- sum_i B_i (A_i V^(k)) ((V^(k))^T A_i^T) (B_i^T U^(k))
        V0^(k+1) <- sum_i A_i^T (B_i^T U^(k)) ((U^(k))^T B_i) (A_i V^(k))
        U^(k+1) <- orthogonalize(U0^(k+1)),  V^(k+1) <- orthogonalize(V0^(k+1))
    (both updates use the k-th iterates).  U0, V0 (initial bases, d_out x r / d_in x r) are
    INPUTS: the paper does not fix the initialization.  Sigma_i = U^T B_i A_i V (Eq. sigmastar,
    P:L452) of the final iterate, as (B_i^T U)^T (A_i V).  No normalization (the caller's choice,
    Sec. 6.1).  Returns dict(U, V, sigma, captured_trace = sum_i ||Sigma_i||_F^2 per iterate)."""
    Bs = [np.asarray(B, dtype=np.float64) for B in Bs]
    As = [np.asarray(A, dtype=np.float64) for A in As]
    U = np.asarray(U0, dtype=np.float64)
    V = np.asarray(V0, dtype=np.float64)

    def captured(U, V):
        return float(sum(np.sum(((B.T @ U).T @ (A @ V)) ** 2) for B, A in zip(Bs, As)))

    trace = [captured(U, V)]
    for _ in range(iters):
        Un = sum(B @ ((A @ V) @ ((V.T @ A.T) @ (B.T @ U))) for B, A in zip(Bs, As))
        Vn = sum(A.T @ ((B.T @ U) @ ((U.T @ B) @ (A @ V))) for B, A in zip(Bs, As))
        U, V = orthogonalize(Un), orthogonalize(Vn)
        trace.append(captured(U, V))
    sigma = np.stack([(B.T @ U).T @ (A @ V) for B, A in zip(Bs, As)])
    return {"U": U, "V": V, "sigma": sigma, "captured_trace": trace}
