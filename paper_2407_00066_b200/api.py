"""Python binding of libcts.so: the C entry points under the same names, plus thin `Bank`/`Plan`
owners.  Argument marshalling only -- every step of the apply runs in the CUDA kernels of
csrc/.  PyTorch supplies device memory and streams; nothing here computes on the data.
"""
import ctypes

import torch

from ._lib import BankDesc, check, lib


def _stream_handle(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _bf16(t, name):
    if t.dtype != torch.bfloat16 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous torch.bfloat16 tensor")
    return t


SIGMA_FULL, SIGMA_DIAG = 0, 1          # cts_sigma_kind_t


def cts_bank_load(in_basis, out_basis, sigma, cluster_of, stream=None):
    """in_basis[m]: [C][d_in][r] bf16 (paper V_c), out_basis[m]: [C][d_out][r] bf16 (paper U_c),
    sigma[m]: [N][r][r] bf16 (row = out index; JD-Full) or [N][r] bf16 (the diagonals; JD-Diag,
    Eq. 3 -> CTS_SIGMA_DIAG), cluster_of[m]: [N] int32.  All on the GPU or all on the host.
    Returns an opaque bank handle (ctypes.c_void_p)."""
    M = len(in_basis)
    if not (len(out_basis) == len(sigma) == len(cluster_of) == M) or M == 0:
        raise ValueError("per-module lists must have the same non-zero length")
    C, _, r = in_basis[0].shape
    N = sigma[0].shape[0]
    diag = sigma[0].dim() == 2
    on_dev = in_basis[0].is_cuda
    keep = []
    for m in range(M):
        for t, nm in ((in_basis[m], "in_basis"), (out_basis[m], "out_basis"), (sigma[m], "sigma")):
            _bf16(t, nm)
            if t.is_cuda != on_dev:
                raise ValueError("bank sources must be all on the GPU or all on the host")
        cm = cluster_of[m]
        if cm.dtype != torch.int32 or not cm.is_contiguous() or cm.is_cuda != on_dev:
            raise TypeError("cluster_of must be contiguous int32 on the same device as the bases")
        sig_shape = (N, r) if diag else (N, r, r)
        if in_basis[m].shape[0] != C or in_basis[m].shape[2] != r or out_basis[m].shape[0] != C \
                or out_basis[m].shape[2] != r or tuple(sigma[m].shape) != sig_shape or cm.shape[0] != N:
            raise ValueError(f"module {m}: inconsistent bank shapes")
        keep += [in_basis[m], out_basis[m], sigma[m], cm]
    d_in = (ctypes.c_int32 * M)(*[int(t.shape[1]) for t in in_basis])
    d_out = (ctypes.c_int32 * M)(*[int(t.shape[1]) for t in out_basis])
    ptrs = lambda ts: (ctypes.c_void_p * M)(*[t.data_ptr() for t in ts])  # noqa: E731
    desc = BankDesc(M, N, C, r, d_in, d_out, ptrs(in_basis), ptrs(out_basis), ptrs(sigma), ptrs(cluster_of),
                    1 if on_dev else 0, SIGMA_DIAG if diag else SIGMA_FULL)
    h = ctypes.c_void_p()
    check("cts_bank_load", lib().cts_bank_load(ctypes.byref(desc), _stream_handle(stream), ctypes.byref(h)))
    del keep
    return h


def cts_bank_bytes(bank):
    n = ctypes.c_size_t()
    check("cts_bank_bytes", lib().cts_bank_bytes(bank, ctypes.byref(n)))
    return n.value


def cts_bank_params(bank, module):
    n = ctypes.c_int64()
    check("cts_bank_params", lib().cts_bank_params(bank, module, ctypes.byref(n)))
    return n.value


def cts_bank_free(bank):
    check("cts_bank_free", lib().cts_bank_free(bank))


def cts_plan_create(bank, T_max):
    h = ctypes.c_void_p()
    check("cts_plan_create", lib().cts_plan_create(bank, int(T_max), ctypes.byref(h)))
    return h


def cts_plan_free(plan):
    check("cts_plan_free", lib().cts_plan_free(plan))


def cts_plan_max_tiles(plan, T):
    return int(lib().cts_plan_max_tiles(plan, int(T)))


def cts_segment(plan, token_adapter, stream=None):
    """token_adapter: int32 CUDA tensor [T]; -1 = no adapter."""
    if token_adapter.dtype != torch.int32 or not token_adapter.is_cuda or not token_adapter.is_contiguous():
        raise TypeError("token_adapter must be a contiguous int32 CUDA tensor")
    T = token_adapter.shape[0]
    check("cts_segment", lib().cts_segment(plan, ctypes.c_void_p(token_adapter.data_ptr()), T,
                                           _stream_handle(stream)))


def cts_segment_readback(plan, module, T, C, stream=None):
    """Host copies (perm[:bound], offsets[C+1], tiles[n_tiles,3]) of module's segmentation."""
    import numpy as np
    perm = np.zeros(max(T, 1), dtype=np.int32)
    offsets = np.zeros(C + 1, dtype=np.int32)
    mt = max(cts_plan_max_tiles(plan, T), 1)
    tiles = np.zeros((mt, 3), dtype=np.int32)
    nt = ctypes.c_int32()
    vp = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    check("cts_segment_readback", lib().cts_segment_readback(plan, module, vp(perm), vp(offsets), vp(tiles),
                                                             ctypes.c_void_p(ctypes.addressof(nt)),
                                                             _stream_handle(stream)))
    return perm[:offsets[-1]], offsets, tiles[:nt.value]


def cts_apply(plan, module, x, y, scale=1.0, stream=None):
    """y[t] += scale * U_c Sigma_i V_c^T x[t] in place for bound tokens (bf16 CUDA tensors, 2-D,
    unit stride along the feature dimension)."""
    for t, nm in ((x, "x"), (y, "y")):
        if t.dtype != torch.bfloat16 or not t.is_cuda or t.dim() != 2 or t.stride(1) != 1:
            raise TypeError(f"{nm} must be a 2-D bf16 CUDA tensor with unit inner stride")
    check("cts_apply", lib().cts_apply(plan, int(module), ctypes.c_void_p(x.data_ptr()), x.stride(0),
                                       ctypes.c_void_p(y.data_ptr()), y.stride(0), ctypes.c_float(scale),
                                       _stream_handle(stream)))


def cts_project(plan, module, x, w0, y, scale=1.0, stream=None):
    """Fused projection y[t] = W0 x[t] + scale * U_c Sigma_i V_c^T x[t] (y is overwritten; w0 is the
    [d_out][d_in] nn.Linear weight).  bf16 CUDA tensors, 2-D, unit inner stride."""
    for t, nm in ((x, "x"), (w0, "w0"), (y, "y")):
        if t.dtype != torch.bfloat16 or not t.is_cuda or t.dim() != 2 or t.stride(1) != 1:
            raise TypeError(f"{nm} must be a 2-D bf16 CUDA tensor with unit inner stride")
    check("cts_project", lib().cts_project(plan, int(module), ctypes.c_void_p(x.data_ptr()), x.stride(0),
                                           ctypes.c_void_p(w0.data_ptr()), w0.stride(0),
                                           ctypes.c_void_p(y.data_ptr()), y.stride(0), ctypes.c_float(scale),
                                           _stream_handle(stream)))


def cts_jd_eigen_iteration(problems, r, iters, stream=None):
    """GPU compression (App A.2 eigenvalue iteration) for a batch of problems; each problem is a dict
    of fp32 CUDA tensors: a_stack [n*r_i][d_in], bt_stack [n*r_i][d_out], U [d_out][r] and
    V [d_in][r] (initial bases in, result out), sigma [n][r][r] (out).  Marshalling only."""
    from ._lib import JdProblem
    arr = (JdProblem * max(1, len(problems)))()
    for k, q in enumerate(problems):
        for nm in ("a_stack", "bt_stack", "U", "V", "sigma"):
            t = q[nm]
            if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
                raise TypeError(f"{nm} must be a contiguous fp32 CUDA tensor")
        K, d_in = q["a_stack"].shape
        d_out = q["bt_stack"].shape[1]
        n = q["sigma"].shape[0]
        arr[k] = JdProblem(q["a_stack"].data_ptr(), q["bt_stack"].data_ptr(), n, K // n, d_in, d_out,
                           q["U"].data_ptr(), q["V"].data_ptr(), q["sigma"].data_ptr())
    nbytes = ctypes.c_size_t()
    check("cts_jd_workspace_bytes", lib().cts_jd_workspace_bytes(arr, len(problems), int(r), ctypes.byref(nbytes)))
    dev = problems[0]["U"].device if problems else torch.device("cuda")
    ws = torch.empty(max(16, nbytes.value), dtype=torch.uint8, device=dev)
    check("cts_jd_eigen_iteration", lib().cts_jd_eigen_iteration(arr, len(problems), int(r), int(iters),
                                                                 ctypes.c_void_p(ws.data_ptr()), nbytes.value,
                                                                 _stream_handle(stream)))
    return ws          # keep alive until the stream has consumed it


def cts_route(token_adapter, owner, world, self_rank, stream=None):
    """Cluster-affinity routing: (perm [T], counts [world]) int32 CUDA tensors; perm = token indices
    stably partitioned by the rank that owns each token's adapter (owner [N] int32)."""
    for t, nm in ((token_adapter, "token_adapter"), (owner, "owner")):
        if t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous() or t.dim() != 1:
            raise TypeError(f"{nm} must be a contiguous 1-D int32 CUDA tensor")
    T = token_adapter.shape[0]
    perm = torch.empty(max(T, 1), dtype=torch.int32, device=token_adapter.device)
    counts = torch.empty(world, dtype=torch.int32, device=token_adapter.device)
    check("cts_route", lib().cts_route(ctypes.c_void_p(token_adapter.data_ptr()), T,
                                       ctypes.c_void_p(owner.data_ptr()), owner.shape[0], int(world), int(self_rank),
                                       ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(counts.data_ptr()),
                                       _stream_handle(stream)))
    return perm[:T], counts


def cts_rows_move(src, dst, idx, scatter, stream=None):
    """Rows of a 2-D CUDA tensor (bf16 activations or int32 ids as [n, 1]): dst[k] = src[idx[k]]
    (scatter=False) or dst[idx[k]] = src[k] (scatter=True)."""
    for t, nm in ((src, "src"), (dst, "dst")):
        if not t.is_cuda or t.dim() != 2 or t.stride(1) != 1 or t.dtype != src.dtype:
            raise TypeError(f"{nm} must be a 2-D CUDA tensor with unit inner stride and src's dtype")
    if idx.dtype != torch.int32 or not idx.is_cuda or not idx.is_contiguous() or idx.dim() != 1:
        raise TypeError("idx must be a contiguous 1-D int32 CUDA tensor")
    es = src.element_size()
    n = idx.shape[0]
    check("cts_rows_move", lib().cts_rows_move(ctypes.c_void_p(src.data_ptr()), src.stride(0) * es,
                                               ctypes.c_void_p(dst.data_ptr()), dst.stride(0) * es,
                                               ctypes.c_void_p(idx.data_ptr()), n, src.shape[1] * es,
                                               int(bool(scatter)), _stream_handle(stream)))


def cts_shrink(plan, module, x, scale=1.0, stream=None):
    """Kernel 1 only: t = scale * Sigma_i V_c^T x_t into the plan's scratch for `module`."""
    if x.dtype != torch.bfloat16 or not x.is_cuda or x.dim() != 2 or x.stride(1) != 1:
        raise TypeError("x must be a 2-D bf16 CUDA tensor with unit inner stride")
    check("cts_shrink", lib().cts_shrink(plan, int(module), ctypes.c_void_p(x.data_ptr()), x.stride(0),
                                         ctypes.c_float(scale), _stream_handle(stream)))


def cts_expand(plan, module, y, stream=None):
    """Kernel 2 only: y_t = bf16(y_t + U_c t_t) from the scratch of the last cts_shrink(module)."""
    if y.dtype != torch.bfloat16 or not y.is_cuda or y.dim() != 2 or y.stride(1) != 1:
        raise TypeError("y must be a 2-D bf16 CUDA tensor with unit inner stride")
    check("cts_expand", lib().cts_expand(plan, int(module), ctypes.c_void_p(y.data_ptr()), y.stride(0),
                                         _stream_handle(stream)))


def _group_args(modules, tensors, name):
    n = len(modules)
    if n == 0 or len(tensors) != n:
        raise ValueError(f"need one {name} tensor per module")
    for t in tensors:
        if t.dtype != torch.bfloat16 or not t.is_cuda or t.dim() != 2 or t.stride(1) != 1:
            raise TypeError(f"{name} must be 2-D bf16 CUDA tensors with unit inner stride")
    mods = (ctypes.c_int32 * n)(*[int(m) for m in modules])
    ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() for t in tensors])
    lds = (ctypes.c_int64 * n)(*[t.stride(0) for t in tensors])
    return n, mods, ptrs, lds


def cts_apply_group(plan, modules, xs, ys, scale=1.0, stream=None):
    """One shrink launch + one expand launch for several modules (e.g. q, k, v sharing one x)."""
    n, mods, xp, xl = _group_args(modules, xs, "x")
    _, _, yp, yl = _group_args(modules, ys, "y")
    check("cts_apply_group", lib().cts_apply_group(plan, n, mods, xp, xl, yp, yl, ctypes.c_float(scale),
                                                   _stream_handle(stream)))


def cts_shrink_group(plan, modules, xs, scale=1.0, stream=None):
    n, mods, xp, xl = _group_args(modules, xs, "x")
    check("cts_shrink_group", lib().cts_shrink_group(plan, n, mods, xp, xl, ctypes.c_float(scale),
                                                     _stream_handle(stream)))


def cts_expand_group(plan, modules, ys, stream=None):
    n, mods, yp, yl = _group_args(modules, ys, "y")
    check("cts_expand_group", lib().cts_expand_group(plan, n, mods, yp, yl, _stream_handle(stream)))


def cts_plan_error(plan):
    code, bad = ctypes.c_int32(), ctypes.c_int32()
    check("cts_plan_error", lib().cts_plan_error(plan, ctypes.byref(code), ctypes.byref(bad)))
    return code.value, bad.value


def _part_args(parts, n):
    if len(parts) != n:
        raise ValueError("need one partial buffer per module")
    for t in parts:
        if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
            raise TypeError("partials must be contiguous fp32 CUDA tensors")
    return (ctypes.c_void_p * n)(*[t.data_ptr() for t in parts])


def cts_plan_partial_elems(plan):
    e = ctypes.c_int64()
    check("cts_plan_partial_elems", lib().cts_plan_partial_elems(plan, ctypes.byref(e)))
    return e.value


def cts_shrink_partial_group(plan, modules, xs, parts, scale=1.0, stream=None):
    """TP rank-local shrink: parts[i] <- this rank's fp32 partial t of module i (sum over ranks next)."""
    n, mods, xp, xl = _group_args(modules, xs, "x")
    pp = _part_args(parts, n)
    check("cts_shrink_partial_group", lib().cts_shrink_partial_group(plan, n, mods, xp, xl, ctypes.c_float(scale), pp,
                                                                     _stream_handle(stream)))


def cts_expand_reduced_group(plan, modules, parts, ys, stream=None):
    """TP rank-local expand of the all-reduced partials into this rank's d_out slice of y."""
    n, mods, yp, yl = _group_args(modules, ys, "y")
    pp = _part_args(parts, n)
    check("cts_expand_reduced_group", lib().cts_expand_reduced_group(plan, n, mods, pp, yp, yl,
                                                                     _stream_handle(stream)))


def cts_comm_unique_id():
    """128-byte NCCL unique id (bytes) for cts_comm_create; one rank creates it, all ranks use it."""
    buf = ctypes.create_string_buffer(128)
    check("cts_comm_unique_id", lib().cts_comm_unique_id(buf))
    return buf.raw


def cts_comm_create(unique_id, nranks, rank):
    """NCCL communicator inside libcts for the tensor-parallel apply (current CUDA device)."""
    if len(unique_id) != 128:
        raise ValueError("unique_id must be the 128 bytes of cts_comm_unique_id")
    buf = ctypes.create_string_buffer(bytes(unique_id), 128)
    h = ctypes.c_void_p()
    check("cts_comm_create", lib().cts_comm_create(buf, int(nranks), int(rank), ctypes.byref(h)))
    return h


def cts_comm_free(comm):
    check("cts_comm_free", lib().cts_comm_free(comm))


def cts_apply_tp(plan, modules, xs, ys, comm, scale=1.0, stream=None):
    """TP d-split apply of one module group on this rank's shard: shrink partial, NCCL all-reduce of
    the rank-r partials and the expand, all issued by libcts on `stream`."""
    n, mods, xp, xl = _group_args(modules, xs, "x")
    _, _, yp, yl = _group_args(modules, ys, "y")
    check("cts_apply_tp", lib().cts_apply_tp(plan, n, mods, xp, xl, yp, yl, ctypes.c_float(scale), comm,
                                             _stream_handle(stream)))


def cts_bank_write_clusters(bank, module, clusters, in_basis, out_basis, stream=None):
    """Overwrite module `module`'s bases of the listed clusters: in_basis [n][d_in][r], out_basis
    [n][d_out][r] bf16 CUDA tensors (slot page-in of a resident pool)."""
    n = len(clusters)
    if n:
        _bf16(in_basis, "in_basis")
        _bf16(out_basis, "out_basis")
        if not (in_basis.is_cuda and out_basis.is_cuda):
            raise ValueError("cts_bank_write_clusters takes device sources")
        if in_basis.shape[0] != n or out_basis.shape[0] != n:
            raise ValueError("one basis slice per listed cluster")
    cl = (ctypes.c_int32 * max(n, 1))(*[int(c) for c in clusters])
    check("cts_bank_write_clusters",
          lib().cts_bank_write_clusters(bank, module, n, cl, in_basis.data_ptr() if n else None,
                                        out_basis.data_ptr() if n else None, _stream_handle(stream)))


def cts_set_exclusive_device(exclusive):
    """Declare (True) or revoke (False, default) exclusive use of the GPU by libcts launches: fused
    applies then launch non-cooperatively (cts.h: only safe when no other kernel runs concurrently)."""
    check("cts_set_exclusive_device", lib().cts_set_exclusive_device(1 if exclusive else 0))


def cts_launch_count():
    """Kernels libcts has enqueued since load (graph captures count once, at capture)."""
    return int(lib().cts_launch_count())


class Bank:
    """Owner of a resident compressed bank (frees it on close / garbage collection)."""

    def __init__(self, in_basis, out_basis, sigma, cluster_of, stream=None):
        self.handle = cts_bank_load(in_basis, out_basis, sigma, cluster_of, stream)
        self.n_modules = len(in_basis)
        self.C = int(in_basis[0].shape[0])
        self.N = int(sigma[0].shape[0])
        self.sigma_diag = sigma[0].dim() == 2
        self.r = int(in_basis[0].shape[2])
        self.d_in = [int(t.shape[1]) for t in in_basis]
        self.d_out = [int(t.shape[1]) for t in out_basis]

    @property
    def bytes(self):
        return cts_bank_bytes(self.handle)

    def params(self, module):
        return cts_bank_params(self.handle, module)

    def write_clusters(self, module, clusters, in_basis, out_basis, stream=None):
        cts_bank_write_clusters(self.handle, module, clusters, in_basis, out_basis, stream)

    def close(self):
        if self.handle is not None:
            cts_bank_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan:
    """Per-batch segmentation + scratch for batches of up to T_max tokens."""

    def __init__(self, bank: Bank, T_max: int):
        self.bank = bank
        self.T_max = T_max
        self.T = 0
        self.handle = cts_plan_create(bank.handle, T_max)

    def segment(self, token_adapter, stream=None):
        cts_segment(self.handle, token_adapter, stream)
        self.T = int(token_adapter.shape[0])

    def readback(self, module, stream=None):
        return cts_segment_readback(self.handle, module, self.T, self.bank.C, stream)

    def apply(self, module, x, y, scale=1.0, stream=None):
        cts_apply(self.handle, module, x, y, scale, stream)

    def project(self, module, x, w0, y, scale=1.0, stream=None):
        cts_project(self.handle, module, x, w0, y, scale, stream)

    def shrink(self, module, x, scale=1.0, stream=None):
        cts_shrink(self.handle, module, x, scale, stream)

    def expand(self, module, y, stream=None):
        cts_expand(self.handle, module, y, stream)

    def apply_group(self, modules, xs, ys, scale=1.0, stream=None):
        cts_apply_group(self.handle, modules, xs, ys, scale, stream)

    def shrink_group(self, modules, xs, scale=1.0, stream=None):
        cts_shrink_group(self.handle, modules, xs, scale, stream)

    def expand_group(self, modules, ys, stream=None):
        cts_expand_group(self.handle, modules, ys, stream)

    def apply_tp(self, modules, xs, ys, comm, scale=1.0, stream=None):
        cts_apply_tp(self.handle, modules, xs, ys, comm.handle, scale, stream)

    def partial_elems(self):
        return cts_plan_partial_elems(self.handle)

    def new_partials(self, n):
        """n zeroed fp32 partial buffers for the TP entry points (one per module of a group)."""
        e = self.partial_elems()
        dev = torch.device("cuda", torch.cuda.current_device())
        return [torch.zeros(e, dtype=torch.float32, device=dev) for _ in range(n)]

    def shrink_partial_group(self, modules, xs, parts, scale=1.0, stream=None):
        cts_shrink_partial_group(self.handle, modules, xs, parts, scale, stream)

    def expand_reduced_group(self, modules, parts, ys, stream=None):
        cts_expand_reduced_group(self.handle, modules, parts, ys, stream)

    def error(self):
        return cts_plan_error(self.handle)

    def max_tiles(self, T=None):
        return cts_plan_max_tiles(self.handle, self.T if T is None else T)

    def close(self):
        if self.handle is not None:
            cts_plan_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Comm:
    """Owner of a libcts NCCL communicator (cts_comm_create / cts_comm_free)."""

    def __init__(self, unique_id, nranks, rank):
        self.handle = cts_comm_create(unique_id, nranks, rank)
        self.nranks, self.rank = nranks, rank

    def close(self):
        if self.handle is not None:
            cts_comm_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
