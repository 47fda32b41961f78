// shrink_sigma.cuh -- kernel 1 of the apply: shrink s_t = V_c^T x_t (tcgen05 grouped GEMM over
// cluster tiles) fused with the per-token Sigma_i matvec t_t = scale * Sigma_i s_t.
//
// Paper: App D broadcast product "V^T x" then "Sigma (V^T x)"; Punica BGMV #1/#2 of
// add_lora_slice_with_sigma with fp32 buffers.  Here both live in ONE kernel and
// the rank-r intermediate never round-trips through HBM as fp32.
//
// Work decomposition: one thread-block cluster of KS CTAs per 128-token tile of one cluster c.
// CTA q of the cluster owns the K-slice [q*K/KS, (q+1)*K/KS) of d_in (split-K), so decode-sized
// tiles (~41 tokens) still spread the x stream over >= 148 SMs.
//   warp 0      TMA producer: x rows gathered by token index (tile::gather4, 128B swizzle) and the
//               in_basis K-slab (tile), STAGES-deep mbarrier ring
//   warp 1      one elected lane issues tcgen05.mma (M=128 tokens, N=r_pad, K=16) into TMEM
//   warps 0-3   epilogue: tcgen05.ld (thread = token row) -> smem partials -> cluster barrier ->
//               CTA q reduces rows q, q+KS, ... over the KS partials through DSMEM in rank order
//               (deterministic) -> Sigma_i row gather (L2-resident, 16-byte loads) + r x r matvec
//               -> t split into bf16 hi + lo (t ~= hi + lo to ~2^-16 relative) for the expand.
// Rows past the tile's valid length up to a multiple of 4 duplicate the last valid token (so the
// expand's 4-row TMA scatter writes identical bytes for duplicates).
#pragma once
#include "sm100.cuh"
#include "segment.cuh"

namespace cts {

constexpr int kShrinkStages = 4;
constexpr int kBK = 64;                      // bf16 elements per K block = one 128-byte row
constexpr int kShrinkThreads = 128;

struct ShrinkArgs {
  const int4* tiles;                // this module's tile list
  const int32_t* n_tiles;           // -> count for this module's map
  const int32_t* perm;              // this module's permutation
  const int32_t* tok_adapter;       // plan copy of token -> adapter
  const __nv_bfloat16* sigma;       // [N][RP][RP], row = out index
  __nv_bfloat16* tbuf;              // [max_tiles*128][2*RP]  (hi | lo)
  int kblocks;                      // d_in / 64
  float scale;
};

template <int RP>
struct ShrinkSmem {
  static constexpr int kA = kTileM * 128;          // bytes per A stage
  static constexpr int kB = RP * 128;              // bytes per B stage
  static constexpr int kRed = kTileM * (RP + 1) * 4;
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + kShrinkStages * kA;
  static constexpr int kOffRed = kOffB + kShrinkStages * kB;
  static constexpr int kOffSred = kOffRed + kRed;
  static constexpr int kOffRows = kOffSred + kRed;
  static constexpr int kOffBar = kOffRows + kTileM * 4;
  static constexpr int kOffTmem = kOffBar + (2 * kShrinkStages + 1) * 8;
  static constexpr int kBytes = kOffTmem + 16 + 1024;  // + alignment slack
  static constexpr uint32_t kTmemCols = RP <= 32 ? 32 : 64;
};

template <int RP>
__global__ void __launch_bounds__(kShrinkThreads, 1)
    shrink_sigma_kernel(const __grid_constant__ CUtensorMap tm_x,
                        const __grid_constant__ CUtensorMap tm_in, ShrinkArgs a) {
  using L = ShrinkSmem<RP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem + L::kOffA;
  uint8_t* sB = smem + L::kOffB;
  float* red = reinterpret_cast<float*>(smem + L::kOffRed);
  float* sred = reinterpret_cast<float*>(smem + L::kOffSred);
  int* rows = reinterpret_cast<int*>(smem + L::kOffRows);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* empty = full + kShrinkStages;
  uint64_t* acc_bar = empty + kShrinkStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kOffTmem);

  const int tile_idx = blockIdx.y;
  if (tile_idx >= *a.n_tiles) return;              // uniform across the cluster
  const int4 tile = a.tiles[tile_idx];             // (c, start, len, -)
  const int c = tile.x, start = tile.y, len = tile.z;
  const int len4 = min(kTileM, (len + 3) & ~3);
  const int ngroups = len4 >> 2;
  const int ks = gridDim.x;
  const int q = static_cast<int>(cluster_ctarank());
  const int kb0 = q * a.kblocks / ks, kb1 = (q + 1) * a.kblocks / ks;
  const int nkb = kb1 - kb0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int j = threadIdx.x; j < kTileM; j += kShrinkThreads) rows[j] = a.perm[start + min(j, len - 1)];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kShrinkStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_bar, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_in);
  }
  if (warp == 2) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    const uint32_t stage_bytes = static_cast<uint32_t>(ngroups * 512 + L::kB);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kShrinkStages;
      const uint32_t ph = (i / kShrinkStages) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], stage_bytes);
      __syncwarp();
      const int k0 = (kb0 + i) * kBK;
      uint8_t* dstA = sA + s * L::kA;
      for (int g = lane; g < ngroups; g += 32)
        tma_gather4(dstA + g * 512, &tm_x, &full[s], k0, rows[4 * g], rows[4 * g + 1],
                    rows[4 * g + 2], rows[4 * g + 3]);
      if (lane == 0) tma_load_2d(sB + s * L::kB, &tm_in, &full[s], k0, c * RP);
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(kTileM, RP);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kShrinkStages;
        const uint32_t ph = (i / kShrinkStages) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sA + s * L::kA);
        const uint32_t b_base = smem_u32(sB + s * L::kB);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          umma_bf16(tmem, umma_desc_kmajor(a_base + k * 32, 128), umma_desc_kmajor(b_base + k * 32, 128),
                    idesc, (i | k) != 0);
        umma_commit(&empty[s]);
      }
      umma_commit(acc_bar);
    }
    __syncwarp();
  }

  // ---------------- epilogue 1: TMEM -> smem partial sums (thread = token row)
  mbar_wait(acc_bar, 0);
  tc_fence_after();
  {
    const int row = warp * 32 + lane;
#pragma unroll
    for (int col = 0; col < RP; col += 16) {
      float v[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + col, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) red[row * (RP + 1) + col + i] = v[i];
    }
  }
  tc_fence_before();
  cluster_sync();

  // ---------------- epilogue 2: deterministic split-K reduction through DSMEM
  const int my_rows = (len4 - q + ks - 1) / ks;     // rows q, q+ks, ... < len4
  const uint32_t red_base = smem_u32(red);
  for (int idx = threadIdx.x; idx < my_rows * RP; idx += kShrinkThreads) {
    const int row = q + (idx / RP) * ks, col = idx % RP;
    const uint32_t off = red_base + static_cast<uint32_t>((row * (RP + 1) + col) * 4);
    float sum = 0.f;
    for (int p = 0; p < ks; ++p) sum += ld_dsmem_f32(mapa_shared(off, p));
    sred[row * (RP + 1) + col] = sum;
  }
  __syncthreads();

  // ---------------- epilogue 3: t = scale * Sigma_i s  -> bf16 hi/lo
  for (int idx = threadIdx.x; idx < my_rows * RP; idx += kShrinkThreads) {
    const int row = q + (idx / RP) * ks, o = idx % RP;
    const int adapter = a.tok_adapter[rows[row]];
    const uint4* srow = reinterpret_cast<const uint4*>(a.sigma + (static_cast<size_t>(adapter) * RP + o) * RP);
    const float* sv = sred + row * (RP + 1);
    float t = 0.f;
#pragma unroll
    for (int v8 = 0; v8 < RP / 8; ++v8) {
      const uint4 w = __ldg(srow + v8);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        t = fmaf(f.x, sv[v8 * 8 + 2 * e], t);
        t = fmaf(f.y, sv[v8 * 8 + 2 * e + 1], t);
      }
    }
    t *= a.scale;
    const __nv_bfloat16 hi = __float2bfloat16_rn(t);
    const __nv_bfloat16 lo = __float2bfloat16_rn(t - __bfloat162float(hi));
    __nv_bfloat16* dst = a.tbuf + (static_cast<size_t>(tile_idx) * kTileM + row) * (2 * RP);
    dst[o] = hi;
    dst[RP + o] = lo;
  }

  cluster_sync();                                  // remote reads of `red` are done
  if (warp == 2) tmem_dealloc<L::kTmemCols>(tmem);
}

}  // namespace cts
