// shrink_sigma.cuh -- kernel 1 of the apply: shrink s_t = V_c^T x_t (tcgen05 grouped GEMM over
// cluster tiles) fused with the per-token Sigma_i matvec t_t = scale * Sigma_i s_t.
//
// Paper: App D broadcast product "V^T x" then "Sigma (V^T x)"; Punica BGMV #1/#2 of
// add_lora_slice_with_sigma with fp32 buffers.  Here both live in ONE kernel and the
// rank-r intermediate never round-trips through HBM as fp32.
//
// Persistent, grouped: one launch covers a group of modules (e.g. q,k,v which share x); the grid is
// one CTA per SM and every CTA walks a static round-robin list of work items
//     item = (module g, 128-token tile of one cluster, K-chunk kc of d_in)
// so the TMA ring keeps streaming across item boundaries (no per-tile launch/prologue latency).
//   warps 0-3   TMA producers: x rows gathered by token index (tile::gather4, 128B swizzle) and
//               the in_basis K-slab (tile) into a kStages-deep mbarrier ring shared by all items;
//               K blocks are dealt round-robin to the 4 warps because one warp's gather4 issue
//               rate caps at ~2 TB/s per GPU (measured, profiles/microbench), four reach the
//               tile-load rate
//   warp 4      one elected lane issues tcgen05.mma (M=128 tokens, N=r_pad, K=16) into one of
//               kAccSlots TMEM accumulators, commit -> acc_full[slot]
//   warps 5-8   epilogue, thread = token row (TMEM lane quarter w%4): tcgen05.ld the partial s;
//               split-K: the partial goes to an fp32 workspace, the LAST CTA to finish a tile
//               (per-tile arrival counter) sums the KS partials in kc order (deterministic),
//               gathers Sigma_i (L2-resident, 16-byte loads) and writes t = scale*Sigma_i s as a
//               bf16 hi + lo pair (t ~= hi + lo to ~2^-16 relative) for the expand.
// Rows of a tile past its length, up to a multiple of 4, duplicate the last valid token, so the
// expand's 4-row TMA scatter writes identical bytes for duplicates.
#pragma once
#include "sm100.cuh"
#include "segment.cuh"

namespace cts {

constexpr int kBK = 64;                 // bf16 elements per K block = one 128-byte swizzle row
constexpr int kMaxGroup = 16;           // modules per grouped launch
constexpr int kProducerWarps = 4;
constexpr int kMmaWarp = kProducerWarps;
constexpr int kEpiWarp0 = kProducerWarps + 1;
constexpr int kShrinkThreads = 32 * (kProducerWarps + 1 + 4);   // producers, MMA, 4 epilogue warps
constexpr int kShrinkAccSlots = 4;

struct alignas(64) ShrinkMod {
  CUtensorMap tm_x;                     // x [T][d_in], box {64, 1}, 128B swizzle (per call)
  const CUtensorMap* tm_in;             // in_basis [C*rp][d_in], box {64, rp} (bank, global mem)
  const int4* tiles;                    // (cluster, start, len, -)
  const int32_t* n_tiles;
  const int32_t* perm;
  const __nv_bfloat16* sigma;           // [N][rp][rp], row = out index
  __nv_bfloat16* tbuf;                  // [max_tiles*128][2*rp]  (hi | lo)
  float* ws;                            // [ks][max_tiles*128][rp] split-K partials
  int32_t* counters;                    // [max_tiles] arrivals per tile (self-resetting)
  int kblocks;                          // d_in / 64
  int ks;                               // K chunks per tile
  int ws_rows;                          // max_tiles * 128
  float scale;
};

struct ShrinkParams {
  ShrinkMod mod[kMaxGroup];
  const int32_t* tok_adapter;
  int n_mod;
};

template <int RP>
struct ShrinkCfg {
  static constexpr int kStages = 8;
  static constexpr int kA = kTileM * 128;           // bytes per A stage (x rows)
  static constexpr int kB = RP * 128;               // bytes per B stage (in_basis rows)
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + kStages * kA;
  static constexpr int kOffBar = kOffB + kStages * kB;
  static constexpr int kNumBars = 2 * kStages + 2 * kShrinkAccSlots;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kBytes = kOffMisc + 64 + 1024;
  static constexpr uint32_t kSlotCols = RP < 32 ? 32 : RP;
  static constexpr uint32_t kTmemCols = kSlotCols * kShrinkAccSlots;   // 128 or 256
};

// item -> (module g, local index j) through the per-module item prefix sums kept in smem
__device__ __forceinline__ int find_module(const int* prefix, int n_mod, int item) {
  int g = 0;
  while (g + 1 < n_mod && item >= prefix[g + 1]) ++g;
  return g;
}

template <int RP>
__global__ void __launch_bounds__(kShrinkThreads, 1) shrink_sigma_kernel(const __grid_constant__ ShrinkParams p) {
  using L = ShrinkCfg<RP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem + L::kOffA;
  uint8_t* sB = smem + L::kOffB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* empty = full + L::kStages;
  uint64_t* acc_full = empty + L::kStages;
  uint64_t* acc_empty = acc_full + kShrinkAccSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kOffMisc);
  int* s_last = reinterpret_cast<int*>(smem + L::kOffMisc + 16);
  __shared__ int prefix[kMaxGroup + 1];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    prefix[0] = 0;
    for (int g = 0; g < p.n_mod; ++g) prefix[g + 1] = prefix[g] + *p.mod[g].n_tiles * p.mod[g].ks;
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kShrinkAccSlots; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 4);       // one arrival per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = prefix[p.n_mod];

  if (warp < kProducerWarps) {
    // ------------------------------------------------------------ TMA producers (K blocks dealt round-robin)
    int li = 0;
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      const int g = find_module(prefix, p.n_mod, item);
      const ShrinkMod& m = p.mod[g];
      const int tile = (item - prefix[g]) / m.ks, kc = (item - prefix[g]) % m.ks;
      const int4 t4 = m.tiles[tile];
      const int len4 = min(kTileM, (t4.z + 3) & ~3);
      const int ngroups = len4 >> 2;
      const int kb0 = kc * m.kblocks / m.ks, kb1 = (kc + 1) * m.kblocks / m.ks;
      const uint32_t bytes = static_cast<uint32_t>(ngroups * 512 + L::kB);
      // token rows of this tile (4 per lane, clamped duplicates past len)
      int r4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) r4[q] = m.perm[t4.y + min(4 * lane + q, t4.z - 1)];
      for (int kb = kb0; kb < kb1; ++kb, ++li) {
        if (li % kProducerWarps != warp) continue;
        const int stage = li % L::kStages;
        const uint32_t phase = (li / L::kStages) & 1;
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&full[stage], bytes);
        __syncwarp();
        uint8_t* dA = sA + stage * L::kA;
        if (lane < ngroups) tma_gather4(dA + lane * 512, &m.tm_x, &full[stage], kb * kBK, r4[0], r4[1], r4[2], r4[3]);
        if (lane == 0) tma_load_2d(sB + stage * L::kB, m.tm_in, &full[stage], kb * kBK, t4.x * RP);
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(kTileM, RP);
    int stage = 0, slot = 0;
    uint32_t phase = 0, aphase = 0;
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      const int g = find_module(prefix, p.n_mod, item);
      const ShrinkMod& m = p.mod[g];
      const int kc = (item - prefix[g]) % m.ks;
      const int kb0 = kc * m.kblocks / m.ks, kb1 = (kc + 1) * m.kblocks / m.ks;
      mbar_wait(&acc_empty[slot], aphase ^ 1);
      tc_fence_after();
      const uint32_t acc = tmem + slot * L::kSlotCols;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_base = smem_u32(sA + stage * L::kA);
          const uint32_t b_base = smem_u32(sB + stage * L::kB);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16(acc, umma_desc_kmajor(a_base + k * 32, 128), umma_desc_kmajor(b_base + k * 32, 128), idesc,
                      (kb > kb0 || k > 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == L::kStages) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) umma_commit(&acc_full[slot]);
      __syncwarp();
      if (++slot == kShrinkAccSlots) { slot = 0; aphase ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 5..8)
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int ep_tid = threadIdx.x - 32 * kEpiWarp0;
    int slot = 0;
    uint32_t aphase = 0;
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      const int g = find_module(prefix, p.n_mod, item);
      const ShrinkMod& m = p.mod[g];
      const int tile = (item - prefix[g]) / m.ks, kc = (item - prefix[g]) % m.ks;
      const int4 t4 = m.tiles[tile];
      const int len4 = min(kTileM, (t4.z + 3) & ~3);
      mbar_wait(&acc_full[slot], aphase);
      tc_fence_after();
      float s[RP];
#pragma unroll
      for (int c = 0; c < RP; c += 16) tmem_ld16(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + slot * L::kSlotCols + c, s + c);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[slot]);
      if (++slot == kShrinkAccSlots) { slot = 0; aphase ^= 1; }

      bool finisher = true;
      if (m.ks > 1) {
        // split-K: publish this chunk's partial, the last arriving CTA reduces in kc order
        if (row < len4) {
          float4* dst = reinterpret_cast<float4*>(m.ws + (static_cast<size_t>(kc) * m.ws_rows + tile * kTileM + row) * RP);
#pragma unroll
          for (int c = 0; c < RP / 4; ++c) dst[c] = make_float4(s[4 * c], s[4 * c + 1], s[4 * c + 2], s[4 * c + 3]);
        }
        __threadfence();
        named_bar_sync(1, 128);
        if (ep_tid == 0) *s_last = (atomicAdd(&m.counters[tile], 1) == m.ks - 1);
        named_bar_sync(1, 128);
        finisher = *s_last != 0;
        if (finisher) {
          __threadfence();
          if (row < len4) {
#pragma unroll
            for (int c = 0; c < RP; ++c) s[c] = 0.f;
            for (int q = 0; q < m.ks; ++q) {
              const float4* src = reinterpret_cast<const float4*>(
                  m.ws + (static_cast<size_t>(q) * m.ws_rows + tile * kTileM + row) * RP);
#pragma unroll
              for (int c = 0; c < RP / 4; ++c) {
                const float4 v = __ldcg(src + c);
                s[4 * c] += v.x; s[4 * c + 1] += v.y; s[4 * c + 2] += v.z; s[4 * c + 3] += v.w;
              }
            }
          }
          if (ep_tid == 0) m.counters[tile] = 0;       // ready for the next launch
        }
      }
      if (finisher && row < len4) {
        // t = scale * Sigma_i s ; thread = token row
        const int adapter = p.tok_adapter[m.perm[t4.y + min(row, t4.z - 1)]];
        const uint4* srow = reinterpret_cast<const uint4*>(m.sigma + static_cast<size_t>(adapter) * RP * RP);
        __nv_bfloat16* dst = m.tbuf + (static_cast<size_t>(tile) * kTileM + row) * (2 * RP);
#pragma unroll 1
        for (int o0 = 0; o0 < RP; o0 += 8) {
          float t8[8];
#pragma unroll
          for (int oo = 0; oo < 8; ++oo) {
            const int o = o0 + oo;
            float acc = 0.f;
#pragma unroll
            for (int v8 = 0; v8 < RP / 8; ++v8) {
              const uint4 w = __ldg(srow + (o * RP) / 8 + v8);
              const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                acc = fmaf(f.x, s[v8 * 8 + 2 * e], acc);
                acc = fmaf(f.y, s[v8 * 8 + 2 * e + 1], acc);
              }
            }
            t8[oo] = acc * m.scale;
          }
          uint4 hi, lo;
          __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&hi);
          __nv_bfloat162* ll = reinterpret_cast<__nv_bfloat162*>(&lo);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(t8[2 * e], t8[2 * e + 1]);
            const float2 hf = __bfloat1622float2(h2);
            hh[e] = h2;
            ll[e] = __floats2bfloat162_rn(t8[2 * e] - hf.x, t8[2 * e + 1] - hf.y);
          }
          *reinterpret_cast<uint4*>(dst + o0) = hi;
          *reinterpret_cast<uint4*>(dst + RP + o0) = lo;
        }
      }
    }
  }
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc<L::kTmemCols>(tmem);
}

}  // namespace cts
