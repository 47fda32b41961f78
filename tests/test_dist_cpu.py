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
