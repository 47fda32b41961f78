"""Device-side (torch) generators for the full-size bench banks (configs 3-5: 224 modules,
2.2 GB at 1000 adapters) -- same recipe as gen.direct_bank, drawn on the GPU because the host
would need ~8 GB of fp64 to draw them.  Seeded torch generators; no method arithmetic."""
import torch


def direct_bank_torch(d_in: int, d_out: int, N: int, C: int, r: int, seed: int, device,
                      cluster_seed: int | None = None):
    """bf16 tensors in the C-ABI layout: in_basis [C][d_in][r] (paper V_c, orthonormal columns),
    out_basis [C][d_out][r] (paper U_c), sigma [N][r][r] = G a / ||G||_F with
    a = exp(U[ln 1/2, ln 2]), cluster_of [N] int32 = pi(i) mod C."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def ortho(rows):
        q, rr = torch.linalg.qr(torch.randn(C, rows, r, generator=g, device=device, dtype=torch.float32))
        s = torch.sign(torch.diagonal(rr, dim1=-2, dim2=-1))
        s[s == 0] = 1
        return (q * s[:, None, :]).to(torch.bfloat16).contiguous()

    in_basis = ortho(d_in)
    out_basis = ortho(d_out)
    G = torch.randn(N, r, r, generator=g, device=device, dtype=torch.float32)
    a = torch.exp(torch.empty(N, device=device).uniform_(-0.6931471805599453, 0.6931471805599453, generator=g))
    sigma = (G * (a / G.flatten(1).norm(dim=1))[:, None, None]).to(torch.bfloat16).contiguous()
    gc = torch.Generator()
    gc.manual_seed(seed + 7919 if cluster_seed is None else cluster_seed)
    cluster_of = (torch.randperm(N, generator=gc) % C).to(torch.int32).to(device)
    return {"in_basis": in_basis, "out_basis": out_basis, "sigma": sigma, "cluster_of": cluster_of}


def tokens_torch(T: int, N: int, seed: int, prefill: bool, device):
    """Decode: adapter uniform per token.  Prefill: requests of U{128..256} tokens, adapter uniform
    per request (same recipe as gen.decode_tokens / gen.prefill_tokens, torch RNG)."""
    g = torch.Generator()
    g.manual_seed(seed)
    if not prefill:
        return torch.randint(0, N, (T,), generator=g, dtype=torch.int32).to(device)
    out = torch.empty(T, dtype=torch.int32)
    pos = 0
    while pos < T:
        L = int(torch.randint(128, 257, (1,), generator=g))
        out[pos:pos + L] = int(torch.randint(0, N, (1,), generator=g))
        pos += L
    return out.to(device)


def lora_bank_torch(d_in: int, d_out: int, N: int, r: int, seed: int, device):
    """The UNCOMPRESSED multi-LoRA collection in the same bank layout (the paper's baseline:
    serving N separate rank-r LoRAs; Punica/vLLM multi-LoRA, App F):
    every adapter is its own cluster, in_basis[i] = A_i^T [d_in][r], out_basis[i] = B_i [d_out][r],
    sigma_i = I_r, cluster_of = identity, so the apply computes y += scale * B_i (A_i x).
    A_i ~ N(0, 1/d_in), B_i ~ N(0, 1/r) (trained-LoRA-like magnitudes); bf16."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    A_t = (torch.randn(N, d_in, r, generator=g, device=device) / d_in ** 0.5).to(torch.bfloat16)
    B = (torch.randn(N, d_out, r, generator=g, device=device) / r ** 0.5).to(torch.bfloat16)
    sigma = torch.eye(r, device=device, dtype=torch.bfloat16).expand(N, r, r).contiguous()
    cluster_of = torch.arange(N, dtype=torch.int32, device=device)
    return {"in_basis": A_t, "out_basis": B, "sigma": sigma, "cluster_of": cluster_of}


def planted_lora_clusters_torch(d_in: int, d_out: int, N: int, C: int, r_i: int, seed: int, device,
                                cluster_seed: int | None = None, families: int = 4, noise: float = 0.3):
    """Trained-like rank-r_i LoRAs B_i A_i for GPU compression, grouped by a given cluster assignment
    (cluster_of = pi(i) mod C, the direct_bank_torch recipe).  Inside a cluster the adapters come from
    `families` planted factor pairs plus Gaussian noise (App H: trained LoRAs share structure, random
    ones do not); A ~ N(0, 1/d_in), B ~ N(0, 1/r_i).  fp32.  Returns cluster_of [N] int32 and per
    cluster c: members (adapter ids, increasing), a_stack [n_c*r_i][d_in] = [A_i; ...] and bt_stack
    [n_c*r_i][d_out] = [B_i^T; ...] in member order -- the cts_jd_eigen_iteration layout."""
    gc = torch.Generator()
    gc.manual_seed(seed + 7919 if cluster_seed is None else cluster_seed)
    cluster_of = torch.randperm(N, generator=gc) % C
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    members, a_st, bt_st = [], [], []
    for c in range(C):
        mem = torch.nonzero(cluster_of == c).flatten()
        n = mem.numel()
        fam_a = torch.randn(families, r_i, d_in, generator=g, device=device) / d_in ** 0.5
        fam_b = torch.randn(families, d_out, r_i, generator=g, device=device) / r_i ** 0.5
        f = torch.arange(n, device=device) % families
        A = fam_a[f] + noise * torch.randn(n, r_i, d_in, generator=g, device=device) / d_in ** 0.5
        B = fam_b[f] + noise * torch.randn(n, d_out, r_i, generator=g, device=device) / r_i ** 0.5
        members.append(mem)
        a_st.append(A.reshape(n * r_i, d_in).contiguous())
        bt_st.append(B.transpose(1, 2).reshape(n * r_i, d_out).contiguous())
    return {"cluster_of": cluster_of.to(torch.int32).to(device), "members": members, "a_stack": a_st,
            "bt_stack": bt_st}


def orthonormal_torch(rows: int, r: int, g, device):
    """A random orthonormal [rows][r] fp32 basis (QR of a Gaussian, sign-fixed): JD's initial bases."""
    q, rr = torch.linalg.qr(torch.randn(rows, r, generator=g, device=device, dtype=torch.float32))
    s = torch.sign(torch.diagonal(rr))
    s[s == 0] = 1
    return (q * s[None, :]).contiguous()
