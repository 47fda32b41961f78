"""Cluster-affinity placement across GPUs (the paper: "clustering offers
opportunities for efficient scheduling").

Instead of replicating the whole compressed bank on every rank (data parallel, bench.py), rank g
keeps only the bases of the clusters it owns (cluster c lives on rank c mod G, so the per-GPU bank
shrinks ~G x) and every token travels to the rank owning its adapter's cluster -- an all-to-all of
rows, as in MoE expert parallelism:

  1. cts_route          perm = token indices stably partitioned by destination rank, counts
  2. cts_rows_move      pack the x rows, the y rows and the ids in that order
  3. all-to-all         rows to their owners (NCCL over NVLink through torch.distributed)
  4. segment + apply    on the received tokens, with the rank's shard of the bank (y += delta y)
  5. all-to-all back    the updated y rows return in the send order
  6. cts_rows_move      scatter them to their original rows

Plumbing only: steps 1, 2, 4 and 6 run in libcts; step 3 / 5 are the collective.  Requires ONE
cluster map shared by the modules of a group (a token must have one owner).  Tokens without an
adapter stay on their rank (its apply leaves them untouched).  `affinity_apply_group` takes the
kernels and the collective as callables, so the orchestration is exercised on CPU (gloo) with the
oracle standing in, exactly like tp.py.
"""


def owned_clusters(C, rank, world):
    """Clusters rank owns: c with c mod world == rank, in increasing order (local index = c // world)."""
    return list(range(rank, C, world))


def shard_bank_by_cluster(in_basis, out_basis, cluster_of, rank, world):
    """This rank's share of one module's bank: the owned clusters' bases and a LOCAL adapter ->
    cluster map (c // world for owned adapters; 0 for the others, whose tokens never arrive here).
    in_basis [C][d_in][r], out_basis [C][d_out][r], cluster_of [N] (torch tensors).  Needs
    C >= world: a rank owning no cluster would hold an empty bank (cts_bank_load rejects C < 1)."""
    if in_basis.shape[0] < world:
        raise ValueError(f"cluster-affinity placement needs at least one cluster per rank (C={in_basis.shape[0]} "
                         f"< world={world}); use data-parallel replication instead")
    own = owned_clusters(in_basis.shape[0], rank, world)
    local = (cluster_of // world).clone()
    local[(cluster_of % world) != rank] = 0
    return in_basis[own].contiguous(), out_basis[own].contiguous(), local.contiguous()


def adapter_owner(cluster_of, world):
    """adapter -> owning rank (cluster mod world)."""
    return (cluster_of % world).contiguous()


def affinity_apply_group(modules, x, ys, tokens, scale, route, gather, scatter, all_to_all, apply_local):
    """Steps 1-6 for one module group on this rank.  x [T][d_in] (shared by the group), ys[m]
    [T][d_out_m] updated in place, tokens [T] int32 ids.
      route(tokens)                        -> (perm [T], send_counts [world] list of ints)
      gather(src, perm) / scatter(dst, src, perm)   row moves (steps 2 and 6)
      all_to_all(send, send_counts)        -> (recv, recv_counts): rows to / from every rank
      apply_local(modules, ids, x, ys, scale)   segment + apply on the received tokens"""
    perm, send_counts = route(tokens)
    ids_recv, recv_counts = all_to_all(gather(tokens[:, None], perm), send_counts)
    x_recv, _ = all_to_all(gather(x, perm), send_counts)
    y_recv = [all_to_all(gather(y, perm), send_counts)[0] for y in ys]
    apply_local(modules, ids_recv[:, 0], x_recv, y_recv, scale)
    for y, yr in zip(ys, y_recv):
        back, _ = all_to_all(yr, recv_counts)          # the rows return in this rank's send order
        scatter(y, back, perm)


class ClusterAffinityApply:
    """Rank-local driver: a bank holding this rank's cluster shard (shard_bank_by_cluster) and a
    plan sized for world x T_local received tokens; owner [N] = adapter_owner(shared map)."""

    def __init__(self, bank, owner, T_local, world, rank, group=None):
        import torch
        import torch.distributed as dist

        from .api import Plan
        self.torch, self.dist, self.group = torch, dist, group
        self.world, self.rank, self.owner = world, rank, owner
        self.plan = Plan(bank, max(1, world * T_local))

    def _route(self, tokens):
        from .api import cts_route
        perm, counts = cts_route(tokens, self.owner, self.world, self.rank)
        return perm, [int(c) for c in counts.cpu()]

    def _gather(self, src, perm):
        from .api import cts_rows_move
        out = self.torch.empty((perm.shape[0], src.shape[1]), dtype=src.dtype, device=src.device)
        cts_rows_move(src, out, perm, scatter=False)
        return out

    def _scatter(self, dst, src, perm):
        from .api import cts_rows_move
        cts_rows_move(src, dst, perm, scatter=True)

    def _all_to_all(self, send, send_counts):
        torch, dist = self.torch, self.dist
        cnt = torch.tensor(send_counts, dtype=torch.int64, device=send.device)
        rc = torch.empty_like(cnt)
        dist.all_to_all_single(rc, cnt, group=self.group)
        recv_counts = [int(c) for c in rc.cpu()]
        recv = torch.empty((sum(recv_counts), send.shape[1]), dtype=send.dtype, device=send.device)
        dist.all_to_all_single(recv, send.contiguous(), recv_counts, send_counts, group=self.group)
        return recv, recv_counts

    def _apply_local(self, modules, ids, x, ys, scale):
        self.plan.segment(ids.contiguous())
        self.plan.apply_group(modules, [x] * len(modules), ys, scale)

    def apply_group(self, modules, x, ys, tokens, scale=1.0):
        affinity_apply_group(modules, x, ys, tokens, scale, self._route, self._gather, self._scatter,
                             self._all_to_all, self._apply_local)
