"""Oracle for the serving-side hot path: segmentation and the compressed apply (fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Notation: the paper factorizes B_i A_i ~= U Sigma_i V^T (Eq. 1)
with U (d_out x r) the output-side and V (d_in x r) the input-side basis.  Buffers are named by
role: in_basis[c] = paper V_c, out_basis[c] = paper U_c, sigma[i] = Sigma_i with row = out index.
"""
import numpy as np


def segment_ref(token_adapter, cluster_of, C: int, tile_m: int = 128):
    """Group the bound tokens of one module by cluster (stable), and cut each group into tiles.

    Plain definition: tc[t] = cluster_of[token_adapter[t]] (-1 if no adapter);
    perm lists bound tokens sorted by (cluster ascending, token index ascending); offset is the
    exclusive prefix sum of per-cluster counts; tiles = (c, start, len<=tile_m) in cluster order.
    Grouping requests that share weights is the SGMV idea the paper builds on; grouping
    by *cluster* is what lets App D's broadcast products run as dense GEMMs.
    """
    ta = np.asarray(token_adapter, dtype=np.int64)
    cmap = np.asarray(cluster_of, dtype=np.int64)
    bound = ta >= 0
    tc = np.full(ta.shape, -1, dtype=np.int64)
    tc[bound] = cmap[ta[bound]]
    idx = np.nonzero(bound)[0]
    order = np.argsort(tc[idx], kind="stable")
    perm = idx[order].astype(np.int32)
    count = np.bincount(tc[idx], minlength=C)[:C]
    offset = np.zeros(C + 1, dtype=np.int32)
    offset[1:] = np.cumsum(count)
    tiles = []
    for c in range(C):
        for start in range(int(offset[c]), int(offset[c + 1]), tile_m):
            tiles.append((c, start, min(tile_m, int(offset[c + 1]) - start)))
    return perm, offset, np.asarray(tiles, dtype=np.int32).reshape(-1, 3)


def apply_ref(x, token_adapter, cluster_of, in_basis, out_basis, sigma, scale=1.0, y_base=None):
    """Delta y_t = scale * U_c Sigma_i (V_c^T x_t), evaluated right to left per token (App D,
    P:L976-980: "V^T x ... broadcasted", "Sigma (V^T x)", "U (Sigma V^T x)"); tokens with id -1
    get Delta y = 0; y = y_base + Delta y (the base projection output, Punica's in-place update
    P:L1118).  All inputs are fp64 (the exact images of the bf16 bits the GPU consumes).
    Returns (delta_y, y) in fp64 (y is None when y_base is None).
    """
    x = np.asarray(x, dtype=np.float64)
    ta = np.asarray(token_adapter, dtype=np.int64)
    T = x.shape[0]
    d_out = out_basis.shape[1]
    dy = np.zeros((T, d_out), dtype=np.float64)
    for c in range(in_basis.shape[0]):
        rows = np.nonzero((ta >= 0) & (np.asarray(cluster_of)[np.maximum(ta, 0)] == c))[0]
        if rows.size == 0:
            continue
        s = x[rows] @ in_basis[c]                                  # shrink: s_t = V_c^T x_t
        t = np.einsum("tok,tk->to", sigma[ta[rows]], s)            # t_t = Sigma_i s_t (row = out)
        dy[rows] = scale * (t @ out_basis[c].T)                    # expand: U_c t_t
    y = None if y_base is None else np.asarray(y_base, dtype=np.float64) + dy
    return dy, y


def apply_dense_ref(x, token_adapter, cluster_of, in_basis, out_basis, sigma, scale=1.0):
    """Same result via the materialized per-adapter update Delta W_i = U_c Sigma_i V_c^T
    (Eq. 1) applied to each token with a pure-Python loop.  Tiny shapes only."""
    x = np.asarray(x, dtype=np.float64)
    T = x.shape[0]
    dy = np.zeros((T, out_basis.shape[1]), dtype=np.float64)
    cache = {}
    for t in range(T):
        i = int(token_adapter[t])
        if i < 0:
            continue
        if i not in cache:
            c = int(cluster_of[i])
            cache[i] = out_basis[c] @ sigma[i] @ in_basis[c].T
        dy[t] = scale * (cache[i] @ x[t])
    return dy


def apply_lora_ref(x, token_adapter, Bs, As, scale=1.0):
    """The uncompressed LoRA update scale * B_i (A_i x_t) (paper Sec. 3)."""
    x = np.asarray(x, dtype=np.float64)
    dy = np.zeros((x.shape[0], Bs[0].shape[0]), dtype=np.float64)
    for t in range(x.shape[0]):
        i = int(token_adapter[t])
        if i >= 0:
            dy[t] = scale * (Bs[i] @ (As[i] @ x[t]))
    return dy


def project_ref(x, W0, token_adapter, cluster_of, in_basis, out_basis, sigma, scale=1.0):
    """The LoRA'd projection (W0 + B_i A_i) x_t of Sec. 3 with the adapter replaced by
    its compressed form: y_t = W0 x_t + scale * U_c Sigma_i V_c^T x_t (Eq. 1; clusters
    P:L162-166); tokens with id -1 get the base projection only.  W0 is [d_out][d_in] (row o =
    output feature o).  fp64; returns y."""
    x = np.asarray(x, dtype=np.float64)
    base = x @ np.asarray(W0, dtype=np.float64).T
    dy, _ = apply_ref(x, token_adapter, cluster_of, in_basis, out_basis, sigma, scale)
    return base + dy
