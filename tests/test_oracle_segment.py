"""Pins for oracle.segment_ref: a brute-force pure-Python definition and structural invariants."""
import numpy as np
import pytest

from oracle import segment_ref
from workloads import cluster_map, decode_tokens, prefill_tokens


def brute_segment(token_adapter, cluster_of, C, tile_m=128):
    """Definition written out: for each cluster in order, walk tokens in order."""
    perm, offset, tiles = [], [0], []
    for c in range(C):
        for t, a in enumerate(token_adapter):
            if a >= 0 and cluster_of[a] == c:
                perm.append(t)
        offset.append(len(perm))
    for c in range(C):
        s = offset[c]
        while s < offset[c + 1]:
            n = min(tile_m, offset[c + 1] - s)
            tiles.append((c, s, n))
            s += n
    return perm, offset, tiles


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("T,N,C", [(0, 4, 1), (1, 4, 1), (32, 4, 1), (300, 50, 7), (1000, 1000, 25),
                                   (700, 64, 128)])
def test_segment_matches_brute_force(seed, T, N, C):
    ta = decode_tokens(T, N, seed, frac_none=0.2)
    cmap = cluster_map(N, C, seed + 1)
    perm, offset, tiles = segment_ref(ta, cmap, C)
    bp, bo, bt = brute_segment(list(ta), list(cmap), C)
    assert perm.tolist() == bp
    assert offset.tolist() == bo
    assert [tuple(t) for t in tiles.tolist()] == bt


def test_segment_prefill_runs_and_empty_clusters():
    ta = prefill_tokens(4096, 1000, 3)
    cmap = cluster_map(1000, 25, 4)
    perm, offset, tiles = segment_ref(ta, cmap, 25)
    assert len(perm) == 4096
    assert sorted(perm.tolist()) == list(range(4096))
    # keys non-decreasing and stable within a cluster
    keys = cmap[ta[perm]]
    assert np.all(np.diff(keys) >= 0)
    for c in range(25):
        seg = perm[offset[c]:offset[c + 1]]
        assert np.all(np.diff(seg) > 0)
    # tiles partition [0, len(perm)) and never cross a cluster boundary
    cov = np.zeros(len(perm), dtype=int)
    for c, s, n in tiles:
        assert 1 <= n <= 128 and offset[c] <= s and s + n <= offset[c + 1]
        cov[s:s + n] += 1
    assert np.all(cov == 1)
    assert len(tiles) <= (4096 + 127) // 128 + 25


def test_segment_all_unbound():
    ta = np.full(64, -1, dtype=np.int32)
    perm, offset, tiles = segment_ref(ta, np.zeros(4, np.int32), 1)
    assert perm.size == 0 and offset.tolist() == [0, 0] and tiles.shape == (0, 3)
