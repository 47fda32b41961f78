"""CUDA path (libcts.so through the C ABI) vs the fp64 oracle.  -m gpu."""
import numpy as np
import pytest
import torch

from oracle import apply_ref, jd_full, segment_ref
from workloads import (MISTRAL_MODULES, activations, bf16_round, bf16_to_f64, cluster_map,
                       decode_tokens, gen_loras, prefill_tokens)

from gpu_helpers import PARITY_TOL, bf16_ulp, dev_bf16, host_bits, quantized_bank, row_rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cts():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2407_00066_b200 as m
    return m


def make_bank(cts, banks_bits):
    return cts.Bank([dev_bf16(b["in_basis"]) for b in banks_bits],
                    [dev_bf16(b["out_basis"]) for b in banks_bits],
                    [dev_bf16(b["sigma"]) for b in banks_bits],
                    [torch.from_numpy(b["cluster_of"]).cuda() for b in banks_bits])


def run_apply(cts, plan, module, x_bits, y_bits, scale):
    x = dev_bf16(x_bits)
    y = dev_bf16(y_bits)
    plan.apply(module, x, y, scale)
    torch.cuda.synchronize()
    return host_bits(y)


def check_delta(ta, got_bits, f64, x_bits, scale, rows=None):
    dy, _ = apply_ref(bf16_to_f64(x_bits), ta, f64["cluster_of"], f64["in_basis"], f64["out_basis"],
                      f64["sigma"], scale)
    got = bf16_to_f64(got_bits)
    sel = np.arange(len(ta)) if rows is None else rows
    bound = sel[ta[sel] >= 0]
    err = row_rel_err(got[bound], dy[bound])
    assert err.size == 0 or err.max() <= PARITY_TOL, f"max per-row rel err {err.max():.3e}"
    unbound = sel[ta[sel] < 0]
    assert np.all(got_bits[unbound] == 0)
    return err


# ---------------------------------------------------------------- segmentation: bit-exact
@pytest.mark.parametrize("T,N,C,frac_none", [(1, 4, 1, 0.0), (32, 4, 1, 0.1), (257, 64, 1, 0.0),
                                             (1024, 1000, 25, 0.05), (999, 8192, 128, 0.0),
                                             (1000, 50, 1024, 0.2), (5, 3, 7, 0.0)])
def test_segment_bit_exact(cts, T, N, C, frac_none):
    bits, _ = quantized_bank(64, 64, N, C, 4, seed=T)
    maps = [cluster_map(N, C, s) for s in (1, 2)]
    banks = [dict(bits, cluster_of=m) for m in maps] + [dict(bits, cluster_of=maps[0])]
    bank = make_bank(cts, banks)
    plan = cts.Plan(bank, T + 5)
    ta = decode_tokens(T, N, seed=T + 1, frac_none=frac_none)
    plan.segment(torch.from_numpy(ta).cuda())
    for m in range(3):
        perm, offs, tiles = plan.readback(m)
        rp, ro, rt = segment_ref(ta, banks[m]["cluster_of"], C)
        assert np.array_equal(perm, rp) and np.array_equal(offs, ro) and np.array_equal(tiles, rt)
    assert plan.error() == (0, -1)


def test_segment_prefill_and_all_unbound(cts):
    bits, _ = quantized_bank(64, 64, 1000, 25, 16, seed=0)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, 16384)
    ta = prefill_tokens(16384, 1000, 5)
    plan.segment(torch.from_numpy(ta).cuda())
    perm, offs, tiles = plan.readback(0)
    rp, ro, rt = segment_ref(ta, bits["cluster_of"], 25)
    assert np.array_equal(perm, rp) and np.array_equal(offs, ro) and np.array_equal(tiles, rt)
    plan.segment(torch.full((100,), -1, dtype=torch.int32, device="cuda"))
    perm, offs, tiles = plan.readback(0)
    assert perm.size == 0 and offs.tolist() == [0] * 26 and tiles.shape[0] == 0


def test_invalid_adapter_poisons_plan(cts):
    bits, f64 = quantized_bank(64, 128, 10, 2, 4, seed=1)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, 64)
    ta = decode_tokens(64, 10, 2)
    ta[[9, 40]] = [10, -3]
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(64, 64, 3))
    y0 = bf16_round(activations(64, 128, 4))
    got = run_apply(cts, plan, 0, x, y0, 1.0)
    assert plan.error() == (3, 9)
    assert np.array_equal(got, y0)                 # untouched
    ta[[9, 40]] = 0                                # recovers on the next good batch
    plan.segment(torch.from_numpy(ta).cuda())
    torch.cuda.synchronize()
    assert plan.error() == (0, -1)


# ---------------------------------------------------------------- apply parity
def test_config1_tiny_jd_bank(cts):
    """Config 1: d=64, 4 LoRAs rank 2, JD-Full r=4, 1 cluster, 32 tokens."""
    Bs, As, _ = gen_loras("random", 64, 64, 4, 2, seed=11)
    res = jd_full(Bs, As, 4)
    bits = {"in_basis": bf16_round(res["V"][None]), "out_basis": bf16_round(res["U"][None]),
            "sigma": bf16_round(res["sigma"]), "cluster_of": np.zeros(4, np.int32)}
    f64 = {k: (bf16_to_f64(v) if k != "cluster_of" else v) for k, v in bits.items()}
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, 32)
    ta = decode_tokens(32, 4, 12, frac_none=0.1)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(32, 64, 13))
    got = run_apply(cts, plan, 0, x, np.zeros((32, 64), np.uint16), 1.0)
    check_delta(ta, got, f64, x, 1.0)


@pytest.mark.parametrize("r", [4, 16, 24, 32, 64])
@pytest.mark.parametrize("T", [1, 7, 130, 300])
def test_ranks_and_ragged_tiles(cts, r, T):
    """r padded to 16/32/64; tiles with len not a multiple of 4, several tiles per cluster."""
    bits, f64 = quantized_bank(192, 320, 20, 3, r, seed=r * 7 + T)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, 20, T + r, frac_none=0.1)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(T, 192, 1))
    got = run_apply(cts, plan, 0, x, np.zeros((T, 320), np.uint16), 0.75)
    check_delta(ta, got, f64, x, 0.75)


def test_config2_q_proj_r64(cts):
    """Config 2: q_proj 4096->4096, 64 LoRAs, JD r=64, 1 cluster, T=256 decode."""
    bits, f64 = quantized_bank(4096, 4096, 64, 1, 64, seed=2)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, 256)
    ta = decode_tokens(256, 64, 21)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(256, 4096, 22))
    got = run_apply(cts, plan, 0, x, np.zeros((256, 4096), np.uint16), 2.0)
    check_delta(ta, got, f64, x, 2.0)


@pytest.mark.parametrize("r,C,T", [(24, 6, 90), (24, 30, 500), (64, 6, 90), (64, 30, 500), (64, 2, 1000)])
def test_distributed_finisher(cts, r, C, T):
    """r_pad 32 / 64 with a K split (d_in 2048 = 32 K blocks, few slots): every CTA of a slot
    finishes 1/ks of its rows (shrink_sigma.cuh dist_finish).  Packed two-cluster slots, ragged
    lengths, unbound tokens, several tiles per cluster (C=2, T=1000); every row vs the oracle."""
    bits, f64 = quantized_bank(2048, 512, 40, C, r, seed=r * 100 + C)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, 40, T + C, frac_none=0.1)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(T, 2048, 3))
    for rep in range(2):                        # the slot counters reset themselves between launches
        got = run_apply(cts, plan, 0, x, np.zeros((T, 512), np.uint16), 1.5)
        check_delta(ta, got, f64, x, 1.5)


@pytest.mark.slow
def test_config2_jd_built_bank(cts):
    """Config 2 with the bank from the oracle's JD-Full of 64 trained-like rank-16 LoRAs."""
    Bs, As, _ = gen_loras("trained_like", 4096, 4096, 64, 16, seed=5, n_families=4)
    res = jd_full(Bs, As, 64, iters=3)
    bits = {"in_basis": bf16_round(res["V"][None]), "out_basis": bf16_round(res["U"][None]),
            "sigma": bf16_round(res["sigma"]), "cluster_of": np.zeros(64, np.int32)}
    f64 = {k: (bf16_to_f64(v) if k != "cluster_of" else v) for k, v in bits.items()}
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, 256)
    ta = decode_tokens(256, 64, 6)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(256, 4096, 7))
    got = run_apply(cts, plan, 0, x, np.zeros((256, 4096), np.uint16), 2.0)
    check_delta(ta, got, f64, x, 2.0)


def test_mistral_layer_decode_sampled(cts):
    """One Mistral-7B layer (q,k,v,o,gate,up,down) of config 3: N=1000, C=25, r=16, T=1024,
    per-module cluster maps; every row of every module."""
    N, C, r, T = 1000, 25, 16, 1024
    banks, f64s = [], []
    for m, (_, di, do) in enumerate(MISTRAL_MODULES):
        b, f = quantized_bank(di, do, N, C, r, seed=1000 + m, cluster_of=cluster_map(N, C, 50 + m))
        banks.append(b)
        f64s.append(f)
    bank = make_bank(cts, banks)
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, N, 1)
    plan.segment(torch.from_numpy(ta).cuda())
    for m, (_, di, do) in enumerate(MISTRAL_MODULES):
        x = bf16_round(activations(T, di, 2 + m))
        got = run_apply(cts, plan, m, x, np.zeros((T, do), np.uint16), 2.0)
        check_delta(ta, got, f64s[m], x, 2.0)


def test_prefill_sampled(cts):
    """Config 4 shape for one q module: T=16384 prefill (request runs, empty clusters)."""
    N, C, r, T = 1000, 25, 16, 16384
    bits, f64 = quantized_bank(4096, 4096, N, C, r, seed=44)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, T)
    ta = prefill_tokens(T, N, 45)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(T, 4096, 46))
    got = run_apply(cts, plan, 0, x, np.zeros((T, 4096), np.uint16), 2.0)
    rows = np.random.default_rng(1).choice(T, 512, replace=False)
    # oracle on the sampled rows only (row-local computation)
    dy, _ = apply_ref(bf16_to_f64(x[rows]), ta[rows], f64["cluster_of"], f64["in_basis"],
                      f64["out_basis"], f64["sigma"], 2.0)
    err = row_rel_err(bf16_to_f64(got[rows]), dy)
    assert err.max() <= PARITY_TOL


# ---------------------------------------------------------------- semantics
def test_residual_add_and_untouched_rows(cts):
    N, C, r, T = 30, 4, 16, 200
    bits, f64 = quantized_bank(256, 512, N, C, r, seed=9)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, N, 10, frac_none=0.25)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(T, 256, 11))
    yb = bf16_round(activations(T, 512, 12))
    got = run_apply(cts, plan, 0, x, yb, 1.0)
    assert np.array_equal(got[ta < 0], yb[ta < 0])                       # bit-identical
    dy, yref = apply_ref(bf16_to_f64(x), ta, f64["cluster_of"], f64["in_basis"], f64["out_basis"],
                         f64["sigma"], 1.0, y_base=bf16_to_f64(yb))
    g = bf16_to_f64(got)[ta >= 0]
    e = yref[ta >= 0]
    # y = bf16_rne(y_base + delta_y_fp32): one rounding of the exact sum (<= 1 ulp of the result)
    # plus the fp32 error of delta_y itself (t carried as bf16 hi+lo: ~2^-16 of the row's scale).
    # A mis-wired residual (wrong column chunk / row) would be off by ~|delta_y|, far above this.
    dscale = np.max(np.abs(dy[ta >= 0]), axis=1, keepdims=True)
    assert np.all(np.abs(g - e) <= bf16_ulp(e) + 1e-3 * dscale)


def test_sigma_zero_leaves_y(cts):
    N, C, r, T = 8, 2, 16, 64
    bits, _ = quantized_bank(128, 128, N, C, r, seed=3)
    bits["sigma"] = np.zeros_like(bits["sigma"])
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, N, 4)
    plan.segment(torch.from_numpy(ta).cuda())
    yb = bf16_round(activations(T, 128, 5))
    got = run_apply(cts, plan, 0, bf16_round(activations(T, 128, 6)), yb, 1.0)
    assert np.array_equal(bf16_to_f64(got), bf16_to_f64(yb))            # value-identical (+-0)


def test_deterministic_and_strided(cts):
    N, C, r, T = 100, 5, 16, 500
    bits, f64 = quantized_bank(512, 256, N, C, r, seed=8)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, N, 9)
    plan.segment(torch.from_numpy(ta).cuda())
    xfull = dev_bf16(bf16_round(activations(T, 640, 10)))
    x = xfull[:, 64:576]                                                  # ld_x = 640
    outs = []
    for _ in range(2):
        yfull = torch.zeros(T, 320, dtype=torch.bfloat16, device="cuda")
        plan.apply(0, x, yfull[:, :256], 1.0)                             # ld_y = 320
        torch.cuda.synchronize()
        outs.append(host_bits(yfull))
    assert np.array_equal(outs[0], outs[1])
    assert np.all(outs[0][:, 256:] == 0)
    check_delta(ta, outs[0][:, :256], f64, host_bits(x.contiguous()), 1.0)


def test_permutation_equivariance(cts):
    N, C, r, T = 40, 3, 16, 256
    bits, _ = quantized_bank(256, 256, N, C, r, seed=12)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, N, 13, frac_none=0.1)
    x = bf16_round(activations(T, 256, 14))
    plan.segment(torch.from_numpy(ta).cuda())
    a = run_apply(cts, plan, 0, x, np.zeros((T, 256), np.uint16), 1.0)
    p = np.random.default_rng(2).permutation(T)
    plan.segment(torch.from_numpy(np.ascontiguousarray(ta[p])).cuda())
    b = run_apply(cts, plan, 0, np.ascontiguousarray(x[p]), np.zeros((T, 256), np.uint16), 1.0)
    # same tokens in a different order: per-row results agree to rounding of the split-K order
    err = row_rel_err(bf16_to_f64(b), bf16_to_f64(a[p]))
    assert err.size == 0 or err.max() <= 2 * PARITY_TOL


def test_host_validation(cts):
    bits, _ = quantized_bank(64, 64, 4, 1, 4, seed=0)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, 8)
    plan.segment(torch.zeros(8, dtype=torch.int32, device="cuda"))
    x = torch.zeros(8, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(cts.CtsError):
        plan.apply(1, x, torch.zeros_like(x))                              # bad module
    with pytest.raises(cts.CtsError):
        plan.apply(0, x, x)                                                # aliasing
    with pytest.raises(cts.CtsError):                                     # ld_x * 2 % 16 != 0
        plan.apply(0, torch.zeros(8, 68, dtype=torch.bfloat16, device="cuda")[:, :64], torch.zeros_like(x))
    with pytest.raises(cts.CtsError):
        plan.segment(torch.zeros(9, dtype=torch.int32, device="cuda"))     # T > T_max
    assert bank.bytes > 0 and bank.params(0) == 1 * (64 + 64) * 4 + 4 * 16


def test_grouped_qkv_shared_x_and_mlp(cts):
    """cts_apply_group: q,k,v in one launch pair reading one x; gate,up in another; per-module maps."""
    N, C, r, T = 200, 6, 16, 777
    shapes = [(512, 512), (512, 128), (512, 128), (512, 1024), (512, 1024)]
    banks, f64s = [], []
    for m, (di, do) in enumerate(shapes):
        b, f = quantized_bank(di, do, N, C, r, seed=300 + m, cluster_of=cluster_map(N, C, 400 + m))
        banks.append(b)
        f64s.append(f)
    bank = make_bank(cts, banks)
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, N, 31, frac_none=0.05)
    plan.segment(torch.from_numpy(ta).cuda())
    xa = bf16_round(activations(T, 512, 32))
    xm = bf16_round(activations(T, 512, 33))
    x_attn, x_mlp = dev_bf16(xa), dev_bf16(xm)
    ys = [torch.zeros(T, do, dtype=torch.bfloat16, device="cuda") for (_, do) in shapes]
    plan.apply_group([0, 1, 2], [x_attn] * 3, ys[:3], 2.0)
    plan.apply_group([3, 4], [x_mlp] * 2, ys[3:], 2.0)
    torch.cuda.synchronize()
    for m in range(5):
        check_delta(ta, host_bits(ys[m]), f64s[m], xa if m < 3 else xm, 2.0)
    with pytest.raises(cts.CtsError):                                      # repeated module
        plan.apply_group([0, 0], [x_attn] * 2, ys[:2], 1.0)
    with pytest.raises(cts.CtsError):                                      # y aliases another y
        plan.apply_group([1, 2], [x_attn] * 2, [ys[1], ys[1]], 1.0)


def test_launch_count_and_split_path_agree(cts):
    """cts_launch_count: segment = 1 launch, apply_group = 1 (fused), shrink/expand = 1 each; the
    split path (shrink_group + expand_group) gives the same bits as the fused apply_group."""
    N, C, r, T = 64, 5, 16, 300
    shapes = [(512, 256), (512, 128)]
    banks = [quantized_bank(di, do, N, C, r, seed=700 + m, cluster_of=cluster_map(N, C, 710 + m))[0]
             for m, (di, do) in enumerate(shapes)]
    bank = make_bank(cts, banks)
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, N, 41, frac_none=0.05)
    x = dev_bf16(bf16_round(activations(T, 512, 42)))
    ya = [torch.zeros(T, do, dtype=torch.bfloat16, device="cuda") for (_, do) in shapes]
    yb = [torch.zeros(T, do, dtype=torch.bfloat16, device="cuda") for (_, do) in shapes]
    n0 = cts.cts_launch_count()
    plan.segment(torch.from_numpy(ta).cuda())
    n1 = cts.cts_launch_count()
    plan.apply_group([0, 1], [x, x], ya, 2.0)
    n2 = cts.cts_launch_count()
    plan.shrink_group([0, 1], [x, x], 2.0)
    plan.expand_group([0, 1], yb)
    n3 = cts.cts_launch_count()
    torch.cuda.synchronize()
    assert (n1 - n0, n2 - n1, n3 - n2) == (1, 1, 2)
    for a, b in zip(ya, yb):
        assert torch.equal(a, b)


@pytest.mark.parametrize("G,r,d_in", [(2, 16, 512), (4, 16, 512), (2, 64, 2048)])
def test_tensor_parallel_dsplit(cts, G, r, d_in):
    """TP d-split through the ABI, G shards simulated in one process: each shard's bank holds its
    d_in / d_out slices, cts_shrink_partial_group writes its fp32 partial, the partials are summed
    (the all-reduce), cts_expand_reduced_group adds each shard's slice of y.  The assembled y must
    meet the per-row 5e-3 bound against the unsharded fp64 oracle.  r = 64 with 1024 columns per
    shard splits K (the standalone shrink kernel: last-arriver finisher at r_pad 64)."""
    from paper_2407_00066_b200.tp import shard_bank, shard_cols
    N, C, T = 120, 5, 333
    shapes = [(d_in, 256), (d_in, 1024)]
    banks, f64s = [], []
    for m, (di, do) in enumerate(shapes):
        b, f = quantized_bank(di, do, N, C, r, seed=900 + m, cluster_of=cluster_map(N, C, 910 + m))
        banks.append(b)
        f64s.append(f)
    ins = [dev_bf16(b["in_basis"]) for b in banks]
    outs = [dev_bf16(b["out_basis"]) for b in banks]
    sig = [dev_bf16(b["sigma"]) for b in banks]
    cmaps = [torch.from_numpy(b["cluster_of"]).cuda() for b in banks]
    ta = decode_tokens(T, N, 51, frac_none=0.05)
    tok = torch.from_numpy(ta).cuda()
    xb = bf16_round(activations(T, d_in, 52))
    x = dev_bf16(xb)
    ys = [torch.zeros(T, do, dtype=torch.bfloat16, device="cuda") for (_, do) in shapes]
    shards = []
    for g in range(G):
        si, so = shard_bank(ins, outs, g, G)
        bank = cts.Bank(si, so, sig, cmaps)
        plan = cts.Plan(bank, T)
        plan.segment(tok)
        shards.append((bank, plan, plan.new_partials(2)))
    for g, (_, plan, parts) in enumerate(shards):
        xg = shard_cols(x, g, G)
        plan.shrink_partial_group([0, 1], [xg, xg], parts, 2.0)
    total = [sum(s[2][i] for s in shards) for i in range(2)]     # stands in for the all-reduce
    for g, (_, plan, _) in enumerate(shards):
        n0 = cts.cts_launch_count()
        plan.expand_reduced_group([0, 1], total, [shard_cols(y, g, G) for y in ys])
        assert cts.cts_launch_count() - n0 == 2
    torch.cuda.synchronize()
    for m in range(2):
        check_delta(ta, host_bits(ys[m]), f64s[m], xb, 2.0)


# ---------------------------------------------------------------- uncompressed multi-LoRA bank
@pytest.mark.parametrize("T,prefill", [(300, False), (700, True)])
def test_uncompressed_multi_lora_bank(cts, T, prefill):
    """the paper's baseline (N separate rank-16 LoRAs) through
    the same kernels -- every adapter its own cluster, in_basis = A_i^T, out_basis = B_i,
    Sigma_i = I -- must equal the plain LoRA update B_i (A_i x) (Sec. 3) of the oracle on
    the same bf16 factors."""
    from oracle import apply_lora_ref
    N, d_in, d_out, r = 150, 256, 384, 16
    Bs, As, _ = gen_loras("random", d_in, d_out, N, r, seed=5)
    Ab = [bf16_round(A / np.sqrt(d_in)) for A in As]
    Bb = [bf16_round(B / np.sqrt(r)) for B in Bs]
    bits = {"in_basis": np.stack([A.T for A in Ab]), "out_basis": np.stack(Bb),
            "sigma": bf16_round(np.broadcast_to(np.eye(r), (N, r, r)).copy()),
            "cluster_of": np.arange(N, dtype=np.int32)}
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, T)
    ta = prefill_tokens(T, N, 21) if prefill else decode_tokens(T, N, 21, frac_none=0.05)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(T, d_in, 22))
    got = bf16_to_f64(run_apply(cts, plan, 0, x, np.zeros((T, d_out), np.uint16), 2.0))
    ref = apply_lora_ref(bf16_to_f64(x), ta, [bf16_to_f64(b) for b in Bb], [bf16_to_f64(a) for a in Ab], 2.0)
    bound = ta >= 0
    err = row_rel_err(got[bound], ref[bound])
    assert err.max() <= PARITY_TOL, f"max per-row rel err {err.max():.3e}"
    assert np.all(got[~bound] == 0)
    plan.close()
    bank.close()


def test_diagonal_sigma_jd_diag(cts):
    """JD-Diag (Sigma_i diagonal) runs the same apply: the r x r matvec of App D
    reduces to an r-vector scale; checked against the oracle on a diagonal bank."""
    bits, f64 = quantized_bank(512, 256, 40, 4, 16, seed=77)
    d = bf16_round(np.stack([np.diag(np.diag(bf16_to_f64(s))) for s in bits["sigma"]]))
    bits["sigma"] = d
    f64["sigma"] = bf16_to_f64(d)
    bank = make_bank(cts, [bits])
    T = 257
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, 40, 31)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(T, 512, 32))
    got = run_apply(cts, plan, 0, x, np.zeros((T, 256), np.uint16), 1.5)
    check_delta(ta, got, f64, x, 1.5)
    plan.close()
    bank.close()


@pytest.mark.parametrize("r,T,prefill", [(16, 1024, False), (4, 300, False), (16, 3000, True), (24, 257, False),
                                         (64, 256, False), (32, 700, True)])
def test_diag_bank_kind(cts, r, T, prefill):
    """CTS_SIGMA_DIAG banks (JD-Diag, Eq. 3): Sigma_i stored as its r diagonal entries and
    applied as an r-vector scale (App D).  Every row of a grouped launch vs the fp64 oracle on
    diag(sigma_i); the same diagonals loaded as a FULL bank give bit-identical y (the full matvec only
    adds exact zeros); the split path, the TP partial path and App F's parameter count (r, not r^2)."""
    shapes = [(1024, 512), (1024, 256)]
    N, C = 300, 12
    banks, f64s, diags = [], [], []
    for m, (di, do) in enumerate(shapes):
        bits, f64 = quantized_bank(di, do, N, C, r, seed=1300 + m, cluster_of=cluster_map(N, C, 1310 + m))
        dg = bf16_round(np.stack([np.diag(bf16_to_f64(s_)) for s_ in bits["sigma"]]))      # [N][r]
        full = bf16_round(np.stack([np.diag(d_) for d_ in bf16_to_f64(dg)]))                  # [N][r][r]
        bits["sigma"] = full
        f64["sigma"] = bf16_to_f64(full)
        banks.append(bits)
        f64s.append(f64)
        diags.append(dg)
    bank_full = make_bank(cts, banks)
    bank_diag = cts.Bank([dev_bf16(b["in_basis"]) for b in banks], [dev_bf16(b["out_basis"]) for b in banks],
                         [dev_bf16(d_) for d_ in diags], [torch.from_numpy(b["cluster_of"]).cuda() for b in banks])
    assert bank_diag.sigma_diag and not bank_full.sigma_diag
    for m, (di, do) in enumerate(shapes):
        assert bank_diag.params(m) == C * (di + do) * r + N * (r + 1)
        assert bank_full.params(m) == C * (di + do) * r + N * (r * r + 1)
    assert bank_diag.bytes < bank_full.bytes
    ta = prefill_tokens(T, N, 1321) if prefill else decode_tokens(T, N, 1321, frac_none=0.05)
    xb = bf16_round(activations(T, 1024, 1322))
    x = dev_bf16(xb)
    outs = {}
    for name, bank in (("diag", bank_diag), ("full", bank_full)):
        plan = cts.Plan(bank, T)
        plan.segment(torch.from_numpy(ta).cuda())
        ys = [torch.zeros(T, do, dtype=torch.bfloat16, device="cuda") for (_, do) in shapes]
        plan.apply_group([0, 1], [x, x], ys, 1.5)
        ys2 = [torch.zeros_like(y) for y in ys]
        plan.shrink_group([0, 1], [x, x], 1.5)
        plan.expand_group([0, 1], ys2)
        parts = plan.new_partials(2)
        ys3 = [torch.zeros_like(y) for y in ys]
        plan.shrink_partial_group([0, 1], [x, x], parts, 1.5)
        plan.expand_reduced_group([0, 1], parts, ys3)
        torch.cuda.synchronize()
        outs[name] = [[host_bits(y) for y in v] for v in (ys, ys2, ys3)]
        plan.close()
    for m in range(2):
        check_delta(ta, outs["diag"][0][m], f64s[m], xb, 1.5)
        for v in range(3):
            assert np.array_equal(outs["diag"][v][m], outs["full"][v][m]), (m, v)
        assert np.array_equal(outs["diag"][1][m], outs["diag"][0][m])
    bank_full.close()
    bank_diag.close()


# ---------------------------------------------------------------- fused base + LoRA projection
@pytest.mark.parametrize("w_zero", [False, True])
@pytest.mark.parametrize("d_in,d_out,T,prefill,frac_none", [(512, 512, 300, False, 0.1), (256, 768, 700, True, 0.0),
                                                            (1024, 256, 130, False, 1.0), (256, 512, 5, False, 0.0)])
def test_fused_projection(cts, d_in, d_out, T, prefill, frac_none, w_zero):
    """cts_project: y = W0 x + scale U_c Sigma_i V_c^T x for EVERY token
    (unbound ones get W0 x) vs the fp64 oracle on the same bf16 bits; packed and whole slots,
    several 256-column blocks, all-unbound and tiny batches.  With W0 = 0 the output IS the LoRA
    term, so the per-row 5e-3 bound holds on Delta y alone (with W0 != 0 the row norm is dominated
    by W0 x and a wrong Delta y could hide inside the tolerance)."""
    from oracle import project_ref
    N, C = 40, 5
    bits, f64 = quantized_bank(d_in, d_out, N, C, 16, seed=d_in + T)
    g = np.random.default_rng(T)
    w_bits = bf16_round(g.standard_normal((d_out, d_in)) / np.sqrt(d_in))
    if w_zero:
        w_bits = np.zeros_like(w_bits)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, T)
    if frac_none >= 1.0:
        ta = np.full(T, -1, np.int32)
    else:
        ta = prefill_tokens(T, N, 41) if prefill else decode_tokens(T, N, 41, frac_none=frac_none)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(T, d_in, 42))
    y = torch.full((T, d_out), float("nan"), dtype=torch.bfloat16, device="cuda")
    plan.project(0, dev_bf16(x), dev_bf16(w_bits), y, 2.0)
    torch.cuda.synchronize()
    got = bf16_to_f64(host_bits(y))
    ref = project_ref(bf16_to_f64(x), bf16_to_f64(w_bits), ta, f64["cluster_of"], f64["in_basis"], f64["out_basis"],
                      f64["sigma"], 2.0)
    assert np.all(np.isfinite(got)), "some rows of y were not written"
    err = row_rel_err(got, ref)
    assert err.size == 0 or err.max() <= PARITY_TOL, f"max per-row rel err {err.max():.3e}"
    if w_zero:
        assert np.all(got[ta < 0] == 0), "unbound rows must be exactly W0 x = 0"
        assert err.size == np.count_nonzero(ta >= 0), "every bound row carries a nonzero Delta y"
    plan.close()
    bank.close()


def test_fused_projection_unsupported_rank(cts):
    bits, _ = quantized_bank(256, 256, 8, 2, 24, seed=1)          # r = 24 pads to 32: not supported
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, 16)
    plan.segment(torch.zeros(16, dtype=torch.int32, device="cuda"))
    x = torch.zeros(16, 256, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(256, 256, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(16, 256, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(cts.CtsError):
        plan.project(0, x, w, y, 1.0)
    plan.close()
    bank.close()


# ---------------------------------------------------------------- full-size, bench launch configuration
def _layer_bank(cts, N, C, r, seed0):
    banks, f64s = [], []
    for m, (_, di, do) in enumerate(MISTRAL_MODULES):
        b, f = quantized_bank(di, do, N, C, r, seed=seed0 + m, cluster_of=cluster_map(N, C, seed0 + 50 + m))
        banks.append(b)
        f64s.append(f)
    return make_bank(cts, banks), f64s


@pytest.mark.parametrize("N,C,T,prefill,sample", [(1000, 25, 1024, False, None), (8192, 128, 1024, False, None),
                                                  (1000, 25, 16384, True, 384)])
def test_layer_grouped_bench_configuration(cts, N, C, T, prefill, sample):
    """One Mistral-7B layer in the launch configuration bench.py times (configs 3, 5 and 4): one
    segment launch, then the fused grouped launches {q,k,v} (one x), {o}, {gate,up} (one x),
    {down}; every row (decode) or sampled rows (prefill) of every module vs the oracle."""
    r = 16
    bank, f64s = _layer_bank(cts, N, C, r, seed0=3000 + C)
    plan = cts.Plan(bank, T)
    ta = prefill_tokens(T, N, 7) if prefill else decode_tokens(T, N, 7)
    plan.segment(torch.from_numpy(ta).cuda())
    slots = {"attn": [0, 1, 2], "o": [3], "mlp": [4, 5], "down": [6]}
    rows = np.arange(T) if sample is None else np.sort(np.random.default_rng(8).choice(T, sample, replace=False))
    dys = {}
    for si, (slot, mods) in enumerate(slots.items()):
        di = MISTRAL_MODULES[mods[0]][1]
        x = bf16_round(activations(T, di, 10 + si))
        ybits = [bf16_round(activations(T, MISTRAL_MODULES[m][2], 20 + m)) for m in mods]
        ys = [dev_bf16(b) for b in ybits]
        plan.apply_group(mods, [dev_bf16(x)] * len(mods), ys, 2.0)
        torch.cuda.synchronize()
        for m, y, yb in zip(mods, ys, ybits):
            dy, yref = apply_ref(bf16_to_f64(x[rows]), ta[rows], f64s[m]["cluster_of"], f64s[m]["in_basis"],
                                 f64s[m]["out_basis"], f64s[m]["sigma"], 2.0, y_base=bf16_to_f64(yb)[rows])
            # y = bf16_rne(y_base + Delta y): within 1 bf16 ulp of the exact sum plus the fp32 error
            # of Delta y (1e-3 of the row's |Delta y|), the residual contract of DESIGN 5
            ygot = bf16_to_f64(host_bits(y))[rows]
            bound = np.abs(ygot - yref) <= bf16_ulp(yref) + 1e-3 * np.abs(dy).max(axis=1, keepdims=True)
            assert bound.all(), f"module {m}: {np.count_nonzero(~bound)} elements off"
            dys[m] = dy
        # the same launches with y_base = 0: y IS bf16(Delta y), so north_star's per-row 5e-3 bound
        # is checked on every row (decode) / every sampled row (prefill) of every module in the
        # timed launch configuration (with y_base ~ N(0,1) the residual contract above dominates)
        yz = [torch.zeros(T, MISTRAL_MODULES[m][2], dtype=torch.bfloat16, device="cuda") for m in mods]
        plan.apply_group(mods, [dev_bf16(x)] * len(mods), yz, 2.0)
        torch.cuda.synchronize()
        for m, y in zip(mods, yz):
            got = bf16_to_f64(host_bits(y))[rows]
            err = row_rel_err(got, dys[m])
            assert err.size == np.count_nonzero(ta[rows] >= 0)
            assert err.max() <= PARITY_TOL, f"module {m}: max per-row rel err {err.max():.3e}"
            assert np.all(got[ta[rows] < 0] == 0)
    plan.close()
    bank.close()


@pytest.mark.parametrize("w_zero", [False, True])
def test_fused_projection_full_size_sampled(cts, w_zero):
    """cts_project at config 4 size for q (4096 -> 4096, T=16384 prefill) and at decode size for
    down (14336 -> 4096, T=1024), sampled rows vs the oracle.  w_zero: W0 = 0, so the per-row
    bound is held by the LoRA term alone (the timed GEMM's K = 16 expand stage)."""
    from oracle import project_ref
    N, C, r = 1000, 25, 16
    for (di, do, T, prefill, seed) in ((4096, 4096, 16384, True, 61), (14336, 4096, 1024, False, 62)):
        bits, f64 = quantized_bank(di, do, N, C, r, seed=seed)
        bank = make_bank(cts, [bits])
        plan = cts.Plan(bank, T)
        ta = prefill_tokens(T, N, seed) if prefill else decode_tokens(T, N, seed, frac_none=0.05)
        plan.segment(torch.from_numpy(ta).cuda())
        x = bf16_round(activations(T, di, seed + 1))
        if w_zero:
            w = np.zeros((do, di), np.uint16)
        else:
            w = bf16_round(np.random.default_rng(seed).standard_normal((do, di)) / np.sqrt(di))
        y = torch.empty(T, do, dtype=torch.bfloat16, device="cuda")
        plan.project(0, dev_bf16(x), dev_bf16(w), y, 2.0)
        torch.cuda.synchronize()
        rows = np.sort(np.random.default_rng(seed).choice(T, 256, replace=False))
        ref = project_ref(bf16_to_f64(x[rows]), bf16_to_f64(w), ta[rows], f64["cluster_of"], f64["in_basis"],
                          f64["out_basis"], f64["sigma"], 2.0)
        got = bf16_to_f64(host_bits(y))[rows]
        err = row_rel_err(got, ref)
        assert err.max() <= PARITY_TOL, f"{di}->{do}: max per-row rel err {err.max():.3e}"
        if w_zero:
            assert np.all(got[ta[rows] < 0] == 0)
        plan.close()
        bank.close()


# ---------------------------------------------------------------- GPU compression (App A.2)
def _jd_problem(Bs, As, U0, V0):
    f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()  # noqa: E731
    n, r = len(Bs), U0.shape[1]
    return {"a_stack": f32(np.concatenate(As, axis=0)), "bt_stack": f32(np.concatenate([B.T for B in Bs], axis=0)),
            "U": f32(U0), "V": f32(V0), "sigma": torch.empty(n, r, r, device="cuda")}


@pytest.mark.parametrize("r,dims,iters,shapes", [
    (8, (96, 80), 6, None), (16, (256, 192), 8, None), (16, (4096, 4096), 4, None),
    (32, (512, 384), 5, ((6, 16), (5, 8))),          # tensor-core path at r = 32 (K = 40 < 2r: d-space)
    (32, (512, 384), 6, ((6, 16), (4, 16), (9, 8))),  # K-space iterations at r = 32 (every K >= 2r)
    (16, (1024, 4096), 12, ((40, 16), (21, 16))),   # K-space, K = 640 / 336 (partial 128-row Gram tiles)
    (16, (256, 192), 4, ((64, 16),)),                # K-space at its largest stack, K = 1024
    (32, (256, 192), 4, ((64, 16),)),                # the same at r = 32
    (16, (256, 192), 5, ((3, 6),)),                  # stacked K = 18 (not a multiple of 4): CUDA-core path
])
def test_gpu_jd_eigen_iteration(cts, r, dims, iters, shapes):
    """cts_jd_eigen_iteration vs the fp64 oracle of App A.2 on the
    same fp32 factors and the same initial bases: a batch of clusters with different sizes and
    LoRA ranks; U, V unique (QR with positive R diagonal) -> compared elementwise, Sigma per adapter."""
    from oracle import jd_eigen_iteration, orthogonalize
    d_in, d_out = dims
    g = np.random.default_rng(r + d_in)
    probs, refs = [], []
    if shapes is None:
        shapes = ((5, 16), (9, 8), (3, 16)) if d_in < 1000 else ((40, 16),)
    for k, (n, ri) in enumerate(shapes):
        Bs, As, _ = gen_loras("trained_like", d_in, d_out, n, ri, seed=100 * k + r, n_families=2)
        Bs = [B.astype(np.float32).astype(np.float64) for B in Bs]
        As = [A.astype(np.float32).astype(np.float64) for A in As]
        U0 = orthogonalize(g.standard_normal((d_out, r))).astype(np.float32).astype(np.float64)
        V0 = orthogonalize(g.standard_normal((d_in, r))).astype(np.float32).astype(np.float64)
        probs.append(_jd_problem(Bs, As, U0, V0))
        refs.append(jd_eigen_iteration(Bs, As, U0, V0, iters))
    ws = cts.cts_jd_eigen_iteration(probs, r, iters)
    torch.cuda.synchronize()
    del ws
    for q, ref in zip(probs, refs):
        U, V, S = (q[k].cpu().numpy().astype(np.float64) for k in ("U", "V", "sigma"))
        assert np.abs(U - ref["U"]).max() <= 2e-4, np.abs(U - ref["U"]).max()
        assert np.abs(V - ref["V"]).max() <= 2e-4, np.abs(V - ref["V"]).max()
        rel = np.linalg.norm(S - ref["sigma"], axis=(1, 2)) / np.linalg.norm(ref["sigma"], axis=(1, 2))
        assert rel.max() <= 1e-4, rel.max()
        assert np.allclose(U.T @ U, np.eye(r), atol=1e-5) and np.allclose(V.T @ V, np.eye(r), atol=1e-5)


def test_gpu_jd_more_problems_than_one_batch(cts):
    """cts_jd_eigen_iteration with 210 problems: more than one launch batch (kJdMaxBatch = 200), the
    stacked-space path in both batches (K = 48 >= 2r); a sample of problems from each batch vs the
    fp64 App A.2 oracle on the same factors and initial bases."""
    from oracle import jd_eigen_iteration, orthogonalize
    r, d_in, d_out, iters, n, ri = 16, 128, 96, 3, 3, 16
    g = np.random.default_rng(11)
    probs, refs = [], {}
    for k in range(210):
        Bs, As, _ = gen_loras("trained_like", d_in, d_out, n, ri, seed=1000 + k, n_families=2)
        Bs = [B.astype(np.float32).astype(np.float64) for B in Bs]
        As = [A.astype(np.float32).astype(np.float64) for A in As]
        U0 = orthogonalize(g.standard_normal((d_out, r))).astype(np.float32).astype(np.float64)
        V0 = orthogonalize(g.standard_normal((d_in, r))).astype(np.float32).astype(np.float64)
        probs.append(_jd_problem(Bs, As, U0, V0))
        if k in (0, 1, 99, 199, 200, 209):
            refs[k] = jd_eigen_iteration(Bs, As, U0, V0, iters)
    ws = cts.cts_jd_eigen_iteration(probs, r, iters)
    torch.cuda.synchronize()
    del ws
    for k, ref in refs.items():
        q = probs[k]
        U, V, S = (q[key].cpu().numpy().astype(np.float64) for key in ("U", "V", "sigma"))
        assert np.abs(U - ref["U"]).max() <= 2e-4, (k, np.abs(U - ref["U"]).max())
        assert np.abs(V - ref["V"]).max() <= 2e-4, (k, np.abs(V - ref["V"]).max())
        rel = np.linalg.norm(S - ref["sigma"], axis=(1, 2)) / np.linalg.norm(ref["sigma"], axis=(1, 2))
        assert rel.max() <= 1e-4, (k, rel.max())


# ---------------------------------------------------------------- edge cases
def test_empty_batch_then_normal_batch(cts):
    """T = 0: segment, grouped apply and projection are no-ops (y untouched); the same plan then
    serves a normal batch correctly."""
    bits, f64 = quantized_bank(256, 256, 20, 3, 16, seed=71)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, 64)
    plan.segment(torch.empty(0, dtype=torch.int32, device="cuda"))
    x = torch.zeros(0, 256, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(0, 256, dtype=torch.bfloat16, device="cuda")
    plan.apply_group([0], [x], [y], 1.0)
    plan.project(0, x, torch.zeros(256, 256, dtype=torch.bfloat16, device="cuda"), y, 1.0)
    torch.cuda.synchronize()
    assert plan.error() == (0, -1)
    ta = decode_tokens(64, 20, 72)
    plan.segment(torch.from_numpy(ta).cuda())
    xb = bf16_round(activations(64, 256, 73))
    got = run_apply(cts, plan, 0, xb, np.zeros((64, 256), np.uint16), 1.0)
    check_delta(ta, got, f64, xb, 1.0)
    plan.close()
    bank.close()


def test_all_tokens_one_adapter_prefill(cts):
    """Degenerate batch: all 16384 tokens bound to ONE adapter (one cluster holds every slot, the
    other clusters are empty); sampled rows vs the oracle."""
    N, C, T = 100, 10, 16384
    bits, f64 = quantized_bank(1024, 512, N, C, 16, seed=74)
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, T)
    ta = np.full(T, 37, np.int32)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(T, 1024, 75))
    got = run_apply(cts, plan, 0, x, np.zeros((T, 512), np.uint16), 2.0)
    check_delta(ta, got, f64, x, 2.0, rows=np.random.default_rng(2).choice(T, 300, replace=False))
    plan.close()
    bank.close()


def test_maximum_clusters_singletons(cts):
    """C = N = 1024 (the library's cluster limit, segment.cuh) with every token on a distinct
    adapter (1024 one-token tiles, packed two per slot): every row vs the oracle."""
    N = C = T = 1024
    bits, f64 = quantized_bank(256, 192, N, C, 16, seed=76, cluster_of=np.arange(N, dtype=np.int32))
    bank = make_bank(cts, [bits])
    plan = cts.Plan(bank, T)
    ta = np.random.default_rng(77).permutation(N).astype(np.int32)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(T, 256, 78))
    got = run_apply(cts, plan, 0, x, np.zeros((T, 192), np.uint16), 1.0)
    check_delta(ta, got, f64, x, 1.0)
    plan.close()
    bank.close()


# ---------------------------------------------------------------- cluster-affinity placement
def test_route_and_rows_move_exact(cts):
    """cts_route == a stable partition of the token indices by owning rank (unbound tokens to
    `self`), bit-exact; cts_rows_move gathers / scatters bf16 and int32 rows exactly."""
    g = np.random.default_rng(90)
    N, T, world, me = 300, 777, 4, 2
    owner = g.integers(0, world, N).astype(np.int32)
    ta = decode_tokens(T, N, 91, frac_none=0.1)
    perm, counts = cts.cts_route(torch.from_numpy(ta).cuda(), torch.from_numpy(owner).cuda(), world, me)
    dest = np.where(ta >= 0, owner[np.maximum(ta, 0)], me)
    assert np.array_equal(perm.cpu().numpy(), np.argsort(dest, kind="stable"))
    assert np.array_equal(counts.cpu().numpy(), np.bincount(dest, minlength=world))
    x = torch.randn(T, 96, device="cuda").to(torch.bfloat16)
    p = perm.long()
    out = torch.empty_like(x)
    cts.cts_rows_move(x, out, perm, scatter=False)
    assert torch.equal(out, x[p])
    back = torch.empty_like(x)
    cts.cts_rows_move(out, back, perm, scatter=True)
    assert torch.equal(back, x)
    ids = torch.from_numpy(ta).cuda()[:, None]
    ids_out = torch.empty_like(ids)
    cts.cts_rows_move(ids, ids_out, perm, scatter=False)
    assert torch.equal(ids_out[:, 0], ids[p, 0])


def test_cluster_affinity_single_rank(cts):
    """ClusterAffinityApply end to end on one GPU (world = 1, NCCL): route, pack, all-to-all,
    segment + grouped apply on the (whole) shard, return, scatter -- y vs the oracle."""
    import os

    import torch.distributed as dist
    from paper_2407_00066_b200.placement import ClusterAffinityApply, adapter_owner, shard_bank_by_cluster
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    own_pg = not dist.is_initialized()
    if own_pg:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    N, C, r, T = 200, 8, 16, 300
    cmap = cluster_map(N, C, 92)
    mods = [(512, 384), (512, 256)]
    bits, f64 = zip(*[quantized_bank(di, do, N, C, r, seed=93 + m, cluster_of=cmap) for m, (di, do) in enumerate(mods)])
    shards = [shard_bank_by_cluster(dev_bf16(b["in_basis"]), dev_bf16(b["out_basis"]),
                                    torch.from_numpy(b["cluster_of"]).cuda(), 0, 1) for b in bits]
    bank = cts.Bank([s[0] for s in shards], [s[1] for s in shards], [dev_bf16(b["sigma"]) for b in bits],
                    [s[2] for s in shards])
    ta = decode_tokens(T, N, 94, frac_none=0.1)
    aff = ClusterAffinityApply(bank, adapter_owner(torch.from_numpy(cmap).cuda(), 1), T, 1, 0)
    x = bf16_round(activations(T, 512, 95))
    ys = [dev_bf16(np.zeros((T, do), np.uint16)) for (_, do) in mods]
    aff.apply_group([0, 1], dev_bf16(x), ys, torch.from_numpy(ta).cuda(), 2.0)
    torch.cuda.synchronize()
    for m in range(2):
        check_delta(ta, host_bits(ys[m]), f64[m], x, 2.0)
    aff.plan.close()
    bank.close()
    if own_pg:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["singleton", "duplicates", "ill_conditioned", "kspace_duplicates",
                                  "kspace_ill_conditioned"])
def test_gpu_jd_rank_deficient_cluster(cts, case):
    """App A.2 on clusters whose stacked rank n*r_i is below r (a singleton or duplicated adapters)
    or nearly so (one adapter a 1e-4 perturbation of another): Cholesky-QR alone would return
    Inf/NaN; the kernel completes the basis deterministically (jd_eigen.cuh kJdCollapse).  U, V
    must come back finite and orthonormal, and since r covers the whole span, the compressed
    adapters must reconstruct B_i A_i (Prop. 1) up to fp32 rounding."""
    from oracle import orthogonalize
    r, d_in, d_out = 32, 384, 256
    g = np.random.default_rng(5)
    if case == "kspace_duplicates":
        # 8 copies of one rank-4 LoRA at r = 16: n*r_i = 32 >= 2r, so the stacked-space (Gram)
        # iterations run although the span (rank 4) is far below r
        r = 16
        B1, A1, _ = gen_loras("random", d_in, d_out, 1, 4, seed=6)
        Bs, As = [B1[0]] * 8, [A1[0]] * 8
    elif case == "kspace_ill_conditioned":
        # 4 rank-8 LoRAs at r = 16 (n*r_i = 32 = 2r: stacked-space iterations), the second and fourth
        # 1e-4 perturbations of the first and third: the Grams square that conditioning
        r = 16
        B1, A1, _ = gen_loras("random", d_in, d_out, 2, 8, seed=7)
        Bs = [B1[0], B1[0] + 1e-4 * g.standard_normal(B1[0].shape), B1[1], B1[1] + 1e-4 * g.standard_normal(B1[1].shape)]
        As = [A1[0], A1[0].copy(), A1[1], A1[1].copy()]
    elif case == "singleton":
        Bs, As, _ = gen_loras("random", d_in, d_out, 1, 16, seed=3)
    else:
        Bs, As, _ = gen_loras("random", d_in, d_out, 1, 16, seed=4)
        B2 = Bs[0] + (1e-4 * g.standard_normal(Bs[0].shape) if case == "ill_conditioned" else 0)
        Bs, As = [Bs[0], B2], [As[0], As[0].copy()]
    U0 = orthogonalize(g.standard_normal((d_out, r)))
    V0 = orthogonalize(g.standard_normal((d_in, r)))
    q = _jd_problem(Bs, As, U0, V0)
    ws = cts.cts_jd_eigen_iteration([q], r, 5)
    torch.cuda.synchronize()
    del ws
    U, V, S = (q[k].cpu().numpy().astype(np.float64) for k in ("U", "V", "sigma"))
    assert np.all(np.isfinite(U)) and np.all(np.isfinite(V)) and np.all(np.isfinite(S))
    assert np.allclose(U.T @ U, np.eye(r), atol=1e-4) and np.allclose(V.T @ V, np.eye(r), atol=1e-4)
    for i, (B, A) in enumerate(zip(Bs, As)):
        BA = B.astype(np.float32).astype(np.float64) @ A.astype(np.float32).astype(np.float64)
        rel = np.linalg.norm(U @ S[i] @ V.T - BA) / np.linalg.norm(BA)
        assert rel < (1e-3 if "ill_conditioned" in case else 2e-4), (case, i, rel)


@pytest.mark.parametrize("shapes,N,C,T,frac_none", [
    ([(1024, 1024), (1024, 256), (1024, 256)], 300, 12, 1024, 0.0),   # q,k,v-like group, decode
    ([(512, 320)], 40, 5, 257, 0.1),                                 # ragged last 256-column job
    ([(768, 512), (768, 512)], 500, 200, 333, 0.05),                 # many clusters, tiny pieces
    ([(256, 256)], 8, 3, 5, 0.0),                                    # a handful of rows
])
def test_grouped_decode_shapes(cts, shapes, N, C, T, frac_none):
    """Grouped fused launches at decode-like shapes (q,k,v-like group, a ragged last column block,
    many clusters with tiny slots, a handful of rows): every row of every module vs the fp64 oracle,
    unbound rows untouched, residual contract with a random y_base."""
    banks, f64s = [], []
    for m, (di, do) in enumerate(shapes):
        b, f = quantized_bank(di, do, N, C, 16, seed=500 + m, cluster_of=cluster_map(N, C, 510 + m))
        banks.append(b)
        f64s.append(f)
    bank = make_bank(cts, banks)
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, N, 521, frac_none=frac_none)
    plan.segment(torch.from_numpy(ta).cuda())
    x = bf16_round(activations(T, shapes[0][0], 522))
    ybits = [bf16_round(activations(T, do, 523 + m)) for m, (_, do) in enumerate(shapes)]
    ys = [dev_bf16(b) for b in ybits]
    yz = [torch.zeros(T, do, dtype=torch.bfloat16, device="cuda") for (_, do) in shapes]
    mods = list(range(len(shapes)))
    plan.apply_group(mods, [dev_bf16(x)] * len(mods), ys, 1.5)
    plan.apply_group(mods, [dev_bf16(x)] * len(mods), yz, 1.5)
    torch.cuda.synchronize()
    for m in mods:
        check_delta(ta, host_bits(yz[m]), f64s[m], x, 1.5)
        dy, yref = apply_ref(bf16_to_f64(x), ta, f64s[m]["cluster_of"], f64s[m]["in_basis"], f64s[m]["out_basis"],
                             f64s[m]["sigma"], 1.5, y_base=bf16_to_f64(ybits[m]))
        got = host_bits(ys[m])
        assert np.array_equal(got[ta < 0], ybits[m][ta < 0])
        g = bf16_to_f64(got)
        assert np.all(np.abs(g - yref) <= bf16_ulp(yref) + 1e-3 * np.abs(dy).max(axis=1, keepdims=True))
    plan.close()
    bank.close()


def test_two_streams_concurrent_applies(cts):
    """cts.h allows several plans / streams to apply the same bank concurrently: two plans on two
    streams, 40 grouped launches each, interleaved; both results vs the oracle (a deadlock would hang
    the test under its timeout)."""
    N, C, T = 400, 16, 512
    shapes = [(1024, 1024), (1024, 512)]
    banks, f64s = [], []
    for m, (di, do) in enumerate(shapes):
        b, f = quantized_bank(di, do, N, C, 16, seed=600 + m, cluster_of=cluster_map(N, C, 610 + m))
        banks.append(b)
        f64s.append(f)
    bank = make_bank(cts, banks)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    plans, tas, xs, ys = [], [], [], []
    for k in range(2):
        plan = cts.Plan(bank, T)
        ta = decode_tokens(T, N, 620 + k)
        with torch.cuda.stream(streams[k]):
            plan.segment(torch.from_numpy(ta).cuda())
        plans.append(plan)
        tas.append(ta)
        xs.append(bf16_round(activations(T, 1024, 630 + k)))
        ys.append([torch.zeros(T, do, dtype=torch.bfloat16, device="cuda") for (_, do) in shapes])
    torch.cuda.synchronize()
    xd = [dev_bf16(x) for x in xs]
    for rep in range(40):
        for k in range(2):
            with torch.cuda.stream(streams[k]):
                if rep == 39:
                    for y in ys[k]:
                        y.zero_()
                plans[k].apply_group([0, 1], [xd[k], xd[k]], ys[k], 1.0)
    torch.cuda.synchronize()
    for k in range(2):
        for m in range(2):
            check_delta(tas[k], host_bits(ys[k][m]), f64s[m], xs[k], 1.0)
    for pl in plans:
        pl.close()
    bank.close()


def test_bank_write_clusters_slot_pagein(cts):
    """cts_bank_write_clusters (slot page-in of a resident pool, the matched-memory baseline): load a
    bank, overwrite the bases of clusters {5, 1, 6} of module 1 with new ones on a side stream, then
    apply: every row vs the oracle on the UPDATED bank; module 0 and the untouched clusters keep
    their old bases (rows of those clusters compare against the old oracle bank)."""
    N, C, r, T = 64, 8, 16, 600
    shapes = [(512, 256), (512, 512)]
    old = [quantized_bank(di, do, N, C, r, seed=1500 + m, cluster_of=cluster_map(N, C, 1510 + m))
           for m, (di, do) in enumerate(shapes)]
    bank = make_bank(cts, [b for b, _ in old])
    new_bits, _ = quantized_bank(512, 512, 3, 3, r, seed=1520, cluster_of=np.arange(3, dtype=np.int32))
    targets = [5, 1, 6]
    s_ = torch.cuda.Stream()
    with torch.cuda.stream(s_):
        bank.write_clusters(1, targets, dev_bf16(new_bits["in_basis"]), dev_bf16(new_bits["out_basis"]), stream=s_)
    s_.synchronize()
    upd_bits = {k: old[1][0][k].copy() for k in ("in_basis", "out_basis", "sigma")}
    for q, c in enumerate(targets):
        upd_bits["in_basis"][c] = new_bits["in_basis"][q]
        upd_bits["out_basis"][c] = new_bits["out_basis"][q]
    upd = {k: bf16_to_f64(upd_bits[k]) for k in upd_bits}
    upd["cluster_of"] = old[1][1]["cluster_of"]
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, N, 1521, frac_none=0.05)
    plan.segment(torch.from_numpy(ta).cuda())
    xb = bf16_round(activations(T, 512, 1522))
    x = dev_bf16(xb)
    ys = [torch.zeros(T, do, dtype=torch.bfloat16, device="cuda") for (_, do) in shapes]
    plan.apply_group([0, 1], [x, x], ys, 2.0)
    torch.cuda.synchronize()
    check_delta(ta, host_bits(ys[0]), old[0][1], xb, 2.0)
    check_delta(ta, host_bits(ys[1]), upd, xb, 2.0)
    with pytest.raises(cts.CtsError):
        bank.write_clusters(1, [2, 2], dev_bf16(new_bits["in_basis"][:2]), dev_bf16(new_bits["out_basis"][:2]))
    with pytest.raises(cts.CtsError):
        bank.write_clusters(1, [C], dev_bf16(new_bits["in_basis"][:1]), dev_bf16(new_bits["out_basis"][:1]))
    plan.close()
    bank.close()


def test_exclusive_device_same_bits(cts):
    """cts_set_exclusive_device(1) (non-cooperative fused launches) computes exactly what the default
    cooperative launch computes: a Mistral-like grouped layer, both modes, bit-identical y."""
    shapes = [(1024, 1024), (1024, 256), (1024, 256)]
    N, C, T = 300, 12, 1024
    banks = [quantized_bank(di, do, N, C, 16, seed=1400 + m, cluster_of=cluster_map(N, C, 1410 + m))[0]
             for m, (di, do) in enumerate(shapes)]
    bank = make_bank(cts, banks)
    plan = cts.Plan(bank, T)
    plan.segment(torch.from_numpy(decode_tokens(T, N, 1421, frac_none=0.05)).cuda())
    x = dev_bf16(bf16_round(activations(T, 1024, 1422)))
    got = []
    try:
        for excl in (False, True):
            cts.cts_set_exclusive_device(excl)
            ys = [torch.zeros(T, do, dtype=torch.bfloat16, device="cuda") for (_, do) in shapes]
            plan.apply_group([0, 1, 2], [x, x, x], ys, 2.0)
            torch.cuda.synchronize()
            got.append([host_bits(y) for y in ys])
    finally:
        cts.cts_set_exclusive_device(False)
    for a, b in zip(*got):
        assert np.array_equal(a, b)
    plan.close()
    bank.close()


def test_apply_tp_nccl_inside_library_world1(cts):
    """cts_comm_create + cts_apply_tp: the TP d-split with the NCCL all-reduce issued
    by libcts.  One rank (the box has one GPU): shrink partial -> ncclAllReduce over a 1-rank
    communicator -> split + expand; every row vs the oracle, then the same sequence captured in a
    CUDA graph and replayed (NCCL is graph-capturable) gives identical bits."""
    N, C, T = 120, 5, 333
    shapes = [(1024, 512), (1024, 1024)]
    banks, f64s = [], []
    for m, (di, do) in enumerate(shapes):
        b, f = quantized_bank(di, do, N, C, 16, seed=940 + m, cluster_of=cluster_map(N, C, 950 + m))
        banks.append(b)
        f64s.append(f)
    bank = make_bank(cts, banks)
    plan = cts.Plan(bank, T)
    ta = decode_tokens(T, N, 961, frac_none=0.05)
    plan.segment(torch.from_numpy(ta).cuda())
    comm = cts.Comm(cts.cts_comm_unique_id(), 1, 0)
    xb = bf16_round(activations(T, 1024, 962))
    x = dev_bf16(xb)
    ys = [torch.zeros(T, do, dtype=torch.bfloat16, device="cuda") for (_, do) in shapes]
    plan.apply_tp([0, 1], [x, x], ys, comm, 2.0)
    torch.cuda.synchronize()
    for m in range(2):
        check_delta(ta, host_bits(ys[m]), f64s[m], xb, 2.0)
    first = [host_bits(y) for y in ys]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for y in ys:
            y.zero_()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            plan.apply_tp([0, 1], [x, x], ys, comm, 2.0)
        for y in ys:
            y.zero_()
        g.replay()
    torch.cuda.synchronize()
    for m in range(2):
        assert np.array_equal(host_bits(ys[m]), first[m])
    comm.close()
    plan.close()
    bank.close()
