"""Host-side scheduling logic of bench.py's matched-memory emulation (App F): wave admission at
max-gpu-lora = slots and the LRU slot pool.  CPU only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import SlotPool, schedule_waves  # noqa: E402


def test_waves_cover_requests_in_order_and_respect_slots():
    rng = np.random.default_rng(0)
    req = rng.integers(0, 100, 500)
    for slots in (1, 3, 28):
        waves = schedule_waves(req, slots)
        assert [i for w in waves for i in w] == list(range(len(req)))      # every request once, FCFS
        for k, w in enumerate(waves):
            assert len({int(req[i]) for i in w}) <= slots
            if k + 1 < len(waves):                                         # greedy: the next request
                nxt = int(req[waves[k + 1][0]])                            # did not fit
                assert len({int(req[i]) for i in w} | {nxt}) == slots + 1


def test_waves_single_adapter_is_one_wave():
    assert schedule_waves(np.full(50, 7), 2) == [list(range(50))]


def test_slot_pool_lru_hits_and_misses():
    pool = SlotPool(3)
    where, miss = pool.admit([5, 6, 5], 0)
    assert sorted(a for _, a in miss) == [5, 6] and where[5] != where[6]
    where, miss = pool.admit([6, 7], 1)                  # 6 hits; 7 takes the free slot
    assert [a for _, a in miss] == [7] and where[6] == pool.where[6]
    where, miss = pool.admit([8, 9], 2)                  # evicts the least recently used (5, then 6)
    assert sorted(a for _, a in miss) == [8, 9]
    assert 5 not in pool.where and 6 not in pool.where and 7 in pool.where
    assert len(set(pool.where.values())) == len(pool.where) == 3


def test_slot_pool_never_evicts_an_adapter_of_the_same_wave():
    pool = SlotPool(2)
    pool.admit([1, 2], 0)
    where, miss = pool.admit([2, 3], 1)
    assert [a for _, a in miss] == [3] and where[2] != where[3] and 2 in pool.where
