"""The shared input generators: bf16 rounding pinned to torch's RNE cast, determinism, shapes."""
import numpy as np
import torch

from workloads import (activations, bf16_round, bf16_to_f64, cluster_map, decode_tokens,
                       direct_bank, prefill_tokens)


def test_bf16_round_matches_torch_on_fp32_inputs():
    g = np.random.default_rng(0)
    a = np.concatenate([g.standard_normal(100000) * 10.0 ** g.integers(-40, 38, 100000),
                        [0.0, -0.0, 1e-45, -3e-39, 3.3895314e38, 3.4e38, np.inf, -np.inf]])
    a32 = a.astype(np.float32)
    ref = torch.from_numpy(a32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    mine = bf16_round(a32.astype(np.float64))
    np.testing.assert_array_equal(mine, ref)


def test_bf16_ties_round_to_even_directly_from_fp64():
    # 1 + 2^-8 is a tie between 1 and 1 + 2^-7: even mantissa -> 1.0
    assert bf16_to_f64(bf16_round(1 + 2.0 ** -8)) == 1.0
    # just above the tie (not representable in fp32): must round up, no double rounding
    assert bf16_to_f64(bf16_round(1 + 2.0 ** -8 + 2.0 ** -40)) == 1 + 2.0 ** -7


def test_roundtrip_exact():
    b = bf16_round(activations(64, 64, 1))
    assert np.array_equal(bf16_round(bf16_to_f64(b)), b)


def test_generators_deterministic_and_shaped():
    b1 = direct_bank(64, 48, 10, 3, 4, 5)
    b2 = direct_bank(64, 48, 10, 3, 4, 5)
    for k in b1:
        np.testing.assert_array_equal(b1[k], b2[k])
    assert b1["in_basis"].shape == (3, 64, 4) and b1["out_basis"].shape == (3, 48, 4)
    np.testing.assert_allclose(np.einsum("cdr,cds->crs", b1["in_basis"], b1["in_basis"]),
                               np.broadcast_to(np.eye(4), (3, 4, 4)), atol=1e-12)
    assert not np.allclose(b1["sigma"], np.swapaxes(b1["sigma"], 1, 2))   # non-symmetric


def test_cluster_map_balanced():
    m = cluster_map(1000, 25, 0)
    assert np.bincount(m).tolist() == [40] * 25


def test_token_batches():
    d = decode_tokens(1024, 1000, 1, frac_none=0.1)
    assert d.min() >= -1 and d.max() < 1000 and (d == -1).any()
    p = prefill_tokens(16384, 1000, 1)
    runs = np.flatnonzero(np.diff(p)) + 1
    lens = np.diff(np.concatenate([[0], runs, [len(p)]]))
    assert lens[:-1].min() >= 128 and len(p) == 16384
