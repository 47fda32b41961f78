"""Tensor-parallel d-split of the compressed-LoRA apply (north_star: "an optional
tensor-parallel split along d_model whose rank-r intermediate is all-reduced with NCCL").

Plumbing only -- every step of the arithmetic runs in libcts:
  rank g holds columns [g d_in/G, (g+1) d_in/G) of every in_basis V_c and rows [g d_out/G, ...)
  of every out_basis U_c (Sigma_i and the maps replicated) and segments the same token batch;
    1. cts_shrink_partial_group   t_g = scale Sigma_i V_c[g]^T x[g]   (fp32, token order)
    2. all-reduce (sum) of the first T * r_pad floats of each partial   (NCCL over NVLink)
    3. cts_expand_reduced_group   y[:, d_out slice g] += U_c[g] t
Step 2 is valid because Sigma_i is linear: sum_g Sigma_i V_c[g]^T x[g] = Sigma_i V_c^T x (Eq. 1,
P:L124-126).  `tp_apply_group` takes the three steps as callables, so the call order and the
reduction extent are exercised on CPU (gloo) with the oracle standing in for the kernels.
"""


def shard_bounds(d, rank, world):
    """[lo, hi) of rank's contiguous slice of a d-wide dimension (slices of 64 columns each)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if d % (64 * world):
        raise ValueError(f"dimension {d} does not split into {world} slices of a multiple of 64")
    w = d // world
    return rank * w, (rank + 1) * w


def shard_bank(in_basis, out_basis, rank, world):
    """Per module in_basis [C][d_in][r] -> [C][d_in/G][r] and out_basis [C][d_out][r] ->
    [C][d_out/G][r] for this rank (contiguous copies, ready for Bank)."""
    ins, outs = [], []
    for a, b in zip(in_basis, out_basis):
        lo, hi = shard_bounds(a.shape[1], rank, world)
        ins.append(a[:, lo:hi].contiguous())
        lo, hi = shard_bounds(b.shape[1], rank, world)
        outs.append(b[:, lo:hi].contiguous())
    return ins, outs


def shard_cols(t, rank, world):
    """This rank's column slice of an activation [T][d] (a strided view; the ABI takes ld)."""
    lo, hi = shard_bounds(t.shape[1], rank, world)
    return t[:, lo:hi]


def tp_apply_group(modules, x_shards, y_shards, parts, live, scale, shrink_partial, all_reduce, expand_reduced):
    """Steps 1-3 above for one module group; `live` = T * r_pad floats of each partial to reduce."""
    shrink_partial(modules, x_shards, parts, scale)
    for p in parts:
        all_reduce(p[:live])
    expand_reduced(modules, parts, y_shards)


def create_comm(rank, world, group=None, device=None):
    """libcts NCCL communicator for the TP group: rank 0 draws the NCCL unique id through libcts,
    torch.distributed broadcasts the 128 bytes, every rank calls cts_comm_create (plumbing only)."""
    import torch
    import torch.distributed as dist

    from .api import Comm, cts_comm_unique_id
    buf = torch.zeros(128, dtype=torch.uint8, device=device if device is not None else "cpu")
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(cts_comm_unique_id()), dtype=torch.uint8))
    if world > 1:
        dist.broadcast(buf, 0, group=group)
    return Comm(bytes(buf.cpu().tolist()), world, rank)


class LibTensorParallelApply:
    """The TP d-split with the all-reduce issued INSIDE libcts (cts_apply_tp: shrink partial ->
    ncclAllReduce -> split + expand on one stream, graph-capturable)."""

    def __init__(self, plan, comm):
        self.plan, self.comm = plan, comm

    def apply_group(self, modules, x_shards, y_shards, scale=1.0):
        self.plan.apply_tp(modules, x_shards, y_shards, self.comm, scale)


class TensorParallelApply:
    """Rank-local driver over a Plan of this rank's bank shard; partial buffers are allocated once
    per group size (fixed pointers: the sequence is CUDA-graph capturable)."""

    def __init__(self, plan, group=None):
        import torch.distributed as dist
        self.plan, self.group, self.dist = plan, group, dist
        self.rp = plan.partial_elems() // plan.T_max
        self._parts = {}

    def parts(self, n):
        if n not in self._parts:
            self._parts[n] = self.plan.new_partials(n)
        return self._parts[n]

    def apply_group(self, modules, x_shards, y_shards, scale=1.0):
        tp_apply_group(modules, x_shards, y_shards, self.parts(len(modules)), self.plan.T * self.rp, scale,
                       self.plan.shrink_partial_group,
                       lambda t: self.dist.all_reduce(t, group=self.group),
                       self.plan.expand_reduced_group)
