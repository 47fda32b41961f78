// expand.cuh -- kernel 2 of the apply: expand Delta y = U_c t (tcgen05, K = r) fused with the
// residual add into the base projection output y (in place).
//
// Paper: App D "U (Sigma V^T x) ... broadcasted"; Punica BGMV #3 "apply matrix B and
// update y" with `scale` -- here scale was already folded into t by kernel 1.
//
// One CTA per (128-token tile, BN-column block of d_out):
//   warp 0      TMA: t_hi / t_lo tile (A operand, K-major), out_basis block (B operand, K-major),
//               and the tile's y rows gathered by token index (tile::gather4, 64-column segments,
//               128B swizzle) -- the y read overlaps the MMA.
//   warp 1      one lane issues D = t_hi U^T + t_lo U^T (M=128 tokens, N=BN, K=16 per MMA).
//   warps 0-3   epilogue, thread = token row: tcgen05.ld 32 fp32 columns, add y_base from smem,
//               round to bf16 (RNE), write back in place; then 4-row TMA scatter to y.
#pragma once
#include "sm100.cuh"
#include "segment.cuh"

namespace cts {

constexpr int kExpandThreads = 128;
constexpr int kExpandMaxBN = 256;

struct ExpandArgs {
  const int4* tiles;
  const int32_t* n_tiles;
  const int32_t* perm;
  int bn;                            // columns per CTA: 64..256, multiple of 64
};

template <int RP>
struct ExpandSmem {
  static constexpr int kY = kTileM * 128;               // one 64-column segment of y rows
  static constexpr int kOffY = 0;
  static constexpr int kOffAhi = kOffY + (kExpandMaxBN / 64) * kY;
  static constexpr int kOffAlo = kOffAhi + kTileM * RP * 2;
  static constexpr int kOffB = kOffAlo + kTileM * RP * 2;
  static constexpr int kOffRows = kOffB + kExpandMaxBN * RP * 2;
  static constexpr int kOffBar = kOffRows + kTileM * 4;
  static constexpr int kOffTmem = kOffBar + 3 * 8;
  static constexpr int kBytes = kOffTmem + 16 + 1024;
  static constexpr uint32_t kTmemCols = 256;
};

template <int RP>
__global__ void __launch_bounds__(kExpandThreads, 1)
    expand_kernel(const __grid_constant__ CUtensorMap tm_t, const __grid_constant__ CUtensorMap tm_out,
                  const __grid_constant__ CUtensorMap tm_y, ExpandArgs a) {
  using L = ExpandSmem<RP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sY = smem + L::kOffY;
  uint8_t* sAhi = smem + L::kOffAhi;
  uint8_t* sAlo = smem + L::kOffAlo;
  uint8_t* sB = smem + L::kOffB;
  int* rows = reinterpret_cast<int*>(smem + L::kOffRows);
  uint64_t* bar_ab = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* bar_y = bar_ab + 1;
  uint64_t* bar_acc = bar_ab + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kOffTmem);

  const int tile_idx = blockIdx.y;
  if (tile_idx >= *a.n_tiles) return;
  const int4 tile = a.tiles[tile_idx];
  const int c = tile.x, start = tile.y, len = tile.z;
  const int len4 = min(kTileM, (len + 3) & ~3);
  const int ngroups = len4 >> 2;
  const int bn = a.bn;
  const int nseg = bn / 64;
  const int n0 = blockIdx.x * bn;
  const int d_out = gridDim.x * bn;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int j = threadIdx.x; j < kTileM; j += kExpandThreads) rows[j] = a.perm[start + min(j, len - 1)];
  if (threadIdx.x == 0) {
    mbar_init(bar_ab, 1);
    mbar_init(bar_y, 1);
    mbar_init(bar_acc, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm_t);
    tma_prefetch_desc(&tm_out);
    tma_prefetch_desc(&tm_y);
  }
  if (warp == 2) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(bar_ab, static_cast<uint32_t>(2 * kTileM * RP * 2 + bn * RP * 2));
      tma_load_2d(sAhi, &tm_t, bar_ab, 0, tile_idx * kTileM);
      tma_load_2d(sAlo, &tm_t, bar_ab, RP, tile_idx * kTileM);
      tma_load_2d(sB, &tm_out, bar_ab, 0, c * d_out + n0);
      mbar_arrive_expect_tx(bar_y, static_cast<uint32_t>(nseg * ngroups * 512));
    }
    __syncwarp();
    for (int g = lane; g < ngroups; g += 32)
      for (int s = 0; s < nseg; ++s)
        tma_gather4(sY + s * L::kY + g * 512, &tm_y, bar_y, n0 + s * 64, rows[4 * g], rows[4 * g + 1],
                    rows[4 * g + 2], rows[4 * g + 3]);
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(kTileM, static_cast<uint32_t>(bn));
      mbar_wait(bar_ab, 0);
      tc_fence_after();
      const uint32_t hi = smem_u32(sAhi), lo = smem_u32(sAlo), b = smem_u32(sB);
#pragma unroll
      for (int k = 0; k < RP / 16; ++k)
        umma_bf16(tmem, umma_desc_kmajor(hi + k * 32, RP * 2), umma_desc_kmajor(b + k * 32, RP * 2), idesc,
                  k != 0);
#pragma unroll
      for (int k = 0; k < RP / 16; ++k)
        umma_bf16(tmem, umma_desc_kmajor(lo + k * 32, RP * 2), umma_desc_kmajor(b + k * 32, RP * 2), idesc, 1);
      umma_commit(bar_acc);
    }
    __syncwarp();
  }

  // ---------------- epilogue: y = bf16(y_base + acc), in smem
  mbar_wait(bar_acc, 0);
  mbar_wait(bar_y, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  for (int j = 0; j < bn / 32; ++j) {
    float v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + j * 32, v);
    tmem_ld_wait();
    if (row < len4) {
      uint8_t* base = sY + (j >> 1) * L::kY + row * 128;
#pragma unroll
      for (int qd = 0; qd < 4; ++qd) {
        const int phys = (((j & 1) * 4 + qd) ^ (row & 7)) * 16;
        uint4 w = *reinterpret_cast<uint4*>(base + phys);
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
          h[e] = __floats2bfloat162_rn(f.x + v[qd * 8 + 2 * e], f.y + v[qd * 8 + 2 * e + 1]);
        }
        *reinterpret_cast<uint4*>(base + phys) = w;
      }
    }
  }
  tc_fence_before();
  fence_proxy_async_smem();
  __syncthreads();
  if (warp == 0) {
    for (int g = lane; g < ngroups; g += 32)
      for (int s = 0; s < nseg; ++s)
        tma_scatter4(&tm_y, sY + s * L::kY + g * 512, n0 + s * 64, rows[4 * g], rows[4 * g + 1],
                     rows[4 * g + 2], rows[4 * g + 3]);
    bulk_commit();
    bulk_wait_read0();
  }
  if (warp == 2) tmem_dealloc<L::kTmemCols>(tmem);
}

}  // namespace cts
