"""Multi-rank host logic of bench.py on CPU with gloo, world_size 2 (no GPU): per-rank request
sharding (distinct token streams, shared bank seed), max-over-ranks timing, whole-job throughput."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from workloads.gen_torch import tokens_torch
    seeds = bench.rank_seeds(rank)
    toks = tokens_torch(64, 1000, seeds["tokens"], False, "cpu")
    gathered = [torch.zeros_like(toks) for _ in range(world)]
    dist.all_gather(gathered, toks)
    per_rank_ms = [2.0 + rank, 10.0 * (rank + 1)]
    mx = bench.reduce_max(per_rank_ms, dist, "cpu")
    value, t = bench.aggregate([mx[0]], 1024, world)
    q.put((rank, seeds, [g.tolist() for g in gathered], mx, value, t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, s0, g0, m0, v0, t0), (r1, s1, g1, m1, v1, t1) = res
    assert s0["bank"] == s1["bank"] and s0["tokens"] != s1["tokens"]   # replicated bank, own streams
    assert g0[0] != g0[1]                                                # ranks draw different requests
    assert m0 == m1 == [3.0, 20.0]                                       # max over ranks on every rank
    assert v0 == v1 == pytest.approx(1024 * 2 / 3e-3)                    # all units / slowest rank time


# ---------------------------------------------------------------- TP d-split orchestration (gloo)
def _tp_worker(rank, world, port, q):
    """Each rank runs paper_2407_00066_b200.tp's sharding + call order with the oracle standing in
    for the two kernels (shrink partial = apply_ref with an identity out_basis; expand = apply_ref
    with identity in_basis and Sigma) and gloo for the all-reduce; rank 0 checks the gathered
    y slices against the unsharded oracle apply."""
    import numpy as np
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import apply_ref
    from paper_2407_00066_b200.tp import shard_bank, shard_bounds, shard_cols, tp_apply_group
    from workloads import cluster_map, decode_tokens

    rng = np.random.default_rng(5)
    T, N, C, r, d_in, d_out = 40, 12, 3, 4, 256, 128
    in_b = torch.from_numpy(rng.standard_normal((C, d_in, r)))
    out_b = torch.from_numpy(rng.standard_normal((C, d_out, r)))
    sig = rng.standard_normal((N, r, r))
    cmap = cluster_map(N, C, 7)
    ta = decode_tokens(T, N, 8, frac_none=0.1)
    x = torch.from_numpy(rng.standard_normal((T, d_in)))
    y0 = torch.from_numpy(rng.standard_normal((T, d_out)))
    ins, outs = shard_bank([in_b], [out_b], rank, world)
    eye_out = np.broadcast_to(np.eye(r), (C, r, r))
    eye_sig = np.broadcast_to(np.eye(r), (N, r, r))

    def shrink_partial(mods, xs, parts, scale):
        for p, xg, ig in zip(parts, xs, ins):
            t, _ = apply_ref(xg.numpy(), ta, cmap, ig.numpy(), eye_out, sig, scale)
            p.copy_(torch.from_numpy(t).reshape(-1))

    def expand_reduced(mods, parts, ys):
        for p, yg, og in zip(parts, ys, outs):
            dy, _ = apply_ref(p.reshape(T, r).numpy(), ta, cmap, eye_out, og.numpy(), eye_sig, 1.0)
            yg += torch.from_numpy(dy)

    parts = [torch.zeros(T * r, dtype=torch.float64)]
    y_shard = shard_cols(y0, rank, world).clone()
    tp_apply_group([0], [shard_cols(x, rank, world)], [y_shard], parts, T * r, 2.0,
                   shrink_partial, dist.all_reduce, expand_reduced)
    gathered = [torch.zeros_like(y_shard) for _ in range(world)]
    dist.all_gather(gathered, y_shard)
    if rank == 0:
        dy, _ = apply_ref(x.numpy(), ta, cmap, in_b.numpy(), out_b.numpy(), sig, 2.0)
        y_tp = torch.cat(gathered, dim=1).numpy()
        q.put(("err", float(np.max(np.abs(y_tp - (y0.numpy() + dy)))), shard_bounds(d_out, 1, world)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_tensor_parallel_dsplit():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    tag, err, b1 = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tag == "err" and err < 1e-10
    assert b1 == (64, 128)


def test_shard_bounds_validation():
    from paper_2407_00066_b200.tp import shard_bounds
    assert shard_bounds(4096, 7, 8) == (3584, 4096)
    assert shard_bounds(14336, 0, 8) == (0, 1792)
    with pytest.raises(ValueError):
        shard_bounds(1024, 0, 32)           # 32-column slices: not a multiple of 64
    with pytest.raises(ValueError):
        shard_bounds(4096, 8, 8)


# ---------------------------------------------------------------- cluster-affinity placement (2 ranks)
def _affinity_worker(rank, world, port, q):
    import numpy as np

    from oracle import apply_ref
    from paper_2407_00066_b200.placement import adapter_owner, affinity_apply_group, shard_bank_by_cluster
    from workloads import cluster_map, decode_tokens, direct_bank

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, C, r, d_in, d_out, T = 40, 6, 4, 32, 24, 30
    cmap = cluster_map(N, C, 3)                                   # ONE map shared by the group
    banks = [direct_bank(d_in, d_out, N, C, r, seed=10 + m, cluster_of=cmap) for m in range(2)]
    full = [{k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in b.items()} for b in banks]
    shard = [shard_bank_by_cluster(b["in_basis"], b["out_basis"], b["cluster_of"], rank, world) for b in full]
    owner = adapter_owner(full[0]["cluster_of"], world)
    tokens = torch.from_numpy(decode_tokens(T, N, 5 + rank, frac_none=0.1))
    g = torch.Generator().manual_seed(7 + rank)
    x = torch.randn(T, d_in, generator=g, dtype=torch.float64)
    ys = [torch.randn(T, d_out, generator=g, dtype=torch.float64) for _ in range(2)]
    y0 = [y.clone() for y in ys]

    def route(tok):                                               # stand-in for cts_route
        dest = torch.where(tok >= 0, owner[tok.clamp(min=0)], torch.full_like(tok, rank))
        perm = torch.from_numpy(np.argsort(dest.numpy(), kind="stable").astype(np.int64))
        return perm, [int((dest == k).sum()) for k in range(world)]

    def gather(src, perm):
        return src[perm].contiguous()

    def scatter(dst, src, perm):
        dst[perm] = src

    def all_to_all(send, send_counts):
        cnt = torch.tensor(send_counts)
        rc = torch.empty_like(cnt)
        dist.all_to_all_single(rc, cnt)
        recv = torch.empty((int(rc.sum()), send.shape[1]), dtype=send.dtype)
        dist.all_to_all_single(recv, send.contiguous(), rc.tolist(), send_counts)
        return recv, rc.tolist()

    seen = []

    def apply_local(modules, ids, xr, yr, scale):                 # stand-in: the oracle on the shard
        seen.append(ids.clone())
        for m, y in zip(modules, yr):
            inb, outb, lmap = shard[m]
            dy, _ = apply_ref(xr.numpy(), ids.numpy(), lmap.numpy(), inb.numpy(), outb.numpy(),
                              full[m]["sigma"].numpy(), scale)
            y += torch.from_numpy(dy)

    affinity_apply_group([0, 1], x, ys, tokens, 2.0, route, gather, scatter, all_to_all, apply_local)
    err = 0.0
    for m in range(2):
        dy, _ = apply_ref(x.numpy(), tokens.numpy(), cmap, banks[m]["in_basis"], banks[m]["out_basis"],
                          banks[m]["sigma"], 2.0)
        err = max(err, float(np.max(np.abs(ys[m].numpy() - (y0[m].numpy() + dy)))))
    ids = seen[0].numpy()
    owned_ok = bool(np.all((ids < 0) | (owner.numpy()[np.maximum(ids, 0)] == rank)))
    q.put((rank, err, owned_ok, int(shard[0][0].shape[0])))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_cluster_affinity_placement():
    """each rank keeps half the clusters' bases, tokens travel to their
    cluster's owner and back; every rank's y equals the oracle on the FULL bank, and every token a
    rank processed belongs to a cluster it owns (or has no adapter)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_affinity_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, owned_ok, n_clusters in res:
        assert err < 1e-10, (rank, err)
        assert owned_ok
        assert n_clusters == 3                                     # 6 clusters over 2 ranks


def test_affinity_needs_a_cluster_per_rank():
    """with C < world a rank would own no cluster and an empty bank; refuse up front."""
    import pytest
    import torch
    from paper_2407_00066_b200.placement import shard_bank_by_cluster
    ib, ob = torch.zeros(2, 64, 4), torch.zeros(2, 64, 4)
    with pytest.raises(ValueError):
        shard_bank_by_cluster(ib, ob, torch.zeros(8, dtype=torch.int32), 3, 4)
    s = shard_bank_by_cluster(ib, ob, torch.zeros(8, dtype=torch.int32), 1, 2)
    assert s[0].shape[0] == 1
