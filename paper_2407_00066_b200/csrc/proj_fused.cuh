// proj_fused.cuh -- SURVEY 8(f) NEXT 1: the fused base + compressed-LoRA projection
//     y_t = W0 x_t + scale * U_c Sigma_i V_c^T x_t
// for every token t of a cluster-sorted 128-row slot (paper: the LoRA'd projection (W0 + B_i A_i) x,
// Sec. 3, with B_i A_i ~ U_c Sigma_i V_c^T, Eq. 1 P:L124-126 / clustered Sec. 4.3
// P:L162-166; App D P:L971-982 evaluates the LoRA term right-to-left).
//
// One tcgen05 GEMM per (slot, 256-column block of d_out): the K loop accumulates x W0^T into a
// 128 x 256 fp32 TMEM accumulator; one more pipeline stage then carries the slot's t = scale Sigma_i
// V_c^T x (written by the shrink + Sigma kernel, bf16 hi + lo) and the out_basis blocks of the
// slot's (at most two) clusters, and four K=16 MMAs add t U_c^T into the SAME accumulator -- the
// LoRA expand costs 0.4% of the tile's MMA work and no extra pass over y.  For a packed slot
// (two <= 64-token tiles of clusters c0, c1 in the two 64-row halves) each half's t is loaded into
// its own A buffer with the other half's rows zero (TMA out-of-bounds fill), so
//     D += t_half0 U_c0^T + t_half1 U_c1^T
// applies the right basis to every row.  The epilogue rounds D to bf16 and stores the valid rows
// to y in token order (register-direct, thread = token row).
//
// A operand: the slot's token rows of x.  The TMA unit takes one instruction at a time, and 32
// tile::gather4 (4 rows each) per K block kept the MMA ~30% idle (ncu: tensor pipe 66% active,
// L2 at 51%), so runs of consecutive tokens -- at prefill a request is a contiguous run of 128-256
// tokens with one adapter -- are loaded as the largest aligned {64 x 128 | 32 | 8} box; only groups
// at run boundaries fall back to gather4.  (A slot-ordered copy of x, loaded as {64 x 128} tiles,
// measured no better: the copy costs an extra pass over x.)
// Persistent, one CTA per SM, 12 warps: 3 TMA producer warps (kProducerWarps) (x rows as above and W0 tiles
// {64 x 256} by 2-D TMA, 4-stage ring of 48 KB), 1 MMA warp (one elected
// lane, M=128 N=256 K=16), 8 epilogue warps (set s stores columns [128 s, 128 s + 128)).  Two TMEM
// accumulators (2 x 256 columns = all of TMEM) let the epilogue of tile i overlap the K loop of
// tile i+1.  Work items are laid over the REAL slot count (device-side, as in the apply kernels),
// followed by base-only tiles over the tokens without an adapter (no LoRA stage).
// r_pad = 16 only (the LoRA stage must fit one 48 KB stage).
#pragma once
#include "sm100.cuh"
#include "segment.cuh"
#include "shrink_sigma.cuh"

namespace cts {

constexpr int kProjBN = 256;
constexpr int kProjAccSlots = 2;

struct ProjParams {
  CUtensorMap tm_w;                      // W0 [d_out][d_in] (nn.Linear layout), box {64, 256}, 128B swizzle
  CUtensorMap tm_t3;                     // tbuf as [2*max_tiles halves][64 rows][2*rp], box {rp, 64, 1}, 32B swizzle
  const CUtensorMap* tm_out;             // out_basis [C*d_out][rp], box {rp, 64}, 32B swizzle (bank)
  const int4* tiles;                     // [slot][2]: (cluster, start, len, -) per 64-row half
  const int32_t* n_tiles;                // real slot count
  const int32_t* tile_rows;              // [slot*128 + row] token index
  const int32_t* unbound_rows;           // tokens with no adapter (segment kernel), padded to 128 rows
  const int32_t* n_unbound;              // their count: base-only tiles y = W0 x
  __nv_bfloat16* y;                      // y [T][ld_y] (written, not accumulated)
  int64_t ld_y;
  int kblocks;                           // d_in / 64
  int nblk;                              // d_out / 256
  int d_out;
  int meta_ready;
  int y32;                               // y base and row stride 32-byte aligned: 256-bit stores
  CUtensorMap tm_x4;                     // x [T][d_in], box {64, 1}, 128B swizzle (gather4)
  CUtensorMap tm_x8;                     // x [T][d_in], box {64, 8}, 128B swizzle (runs of 8 tokens)
  CUtensorMap tm_x32;                    // x [T][d_in], box {64, 32} (runs of 32 tokens)
  CUtensorMap tm_x128;                   // x [T][d_in], box {64, 128} (a slot that is one run)
};

struct ProjCfg {
  static constexpr int kA = kTileM * 128;                   // x rows, one 64-column K block (16 KB)
  static constexpr int kB = kProjBN * 128;                  // W0 tile {64 x 256} (32 KB)
  static constexpr int kStage = kA + kB;
  static constexpr int kStages = 4;
  static constexpr int kT = kTileM * 16 * 2;                // one t (hi or lo) buffer, 128 rows x 32 B
  static constexpr int kU = kProjBN * 16 * 2;               // one out_basis block, 256 rows x 32 B
  static_assert(4 * kT <= kA && 2 * kU <= kB, "LoRA stage must fit a K stage");
  static constexpr int kArena = kStages * kStage;
  static constexpr int kNumBars = 2 * kStages + 2 * kProjAccSlots;
  static constexpr int kOffBar = kArena;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kBytes = kOffMisc + 64 + 1024;
  static constexpr uint32_t kTmemCols = kProjBN * kProjAccSlots;   // 512
};

__global__ void __launch_bounds__(kApplyThreads, 1) proj_fused_kernel(const __grid_constant__ ProjParams p) {
  using L = ProjCfg;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* empty = full + L::kStages;
  uint64_t* acc_full = empty + L::kStages;
  uint64_t* acc_empty = acc_full + kProjAccSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kOffMisc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kProjAccSlots; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 4 * kEpiSets);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<L::kTmemCols>(tmem_slot);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&p.tm_x4);
    tma_prefetch_desc(&p.tm_x8);
    tma_prefetch_desc(&p.tm_x32);
    tma_prefetch_desc(&p.tm_x128);
    tma_prefetch_desc(&p.tm_w);
    tma_prefetch_desc(&p.tm_t3);
    tma_prefetch_desc(p.tm_out);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  int nt = 0, nu = 0;
  if (p.meta_ready) { nt = *p.n_tiles; nu = *p.n_unbound; }
  griddep_wait();
  if (threadIdx.x == 0) griddep_launch_dependents();
  if (!p.meta_ready) { nt = *p.n_tiles; nu = *p.n_unbound; }
  // items: (slot, 256-column block) for the nt cluster slots, nb fastest, then (unbound tile, block)
  const int bound_items = nt * p.nblk;
  const int total = bound_items + (nu + kTileM - 1) / kTileM * p.nblk;

  if (warp < kProducerWarps) {
    // ------------------------------------------------------------ TMA producers
    int li = 0;                                        // stage sequence over this CTA's items
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      const bool lora = item < bound_items;
      const int slot = (lora ? item : item - bound_items) / p.nblk, nb = item % p.nblk;
      int4 t0, t1;
      if (lora) {
        t0 = p.tiles[2 * slot];
        t1 = p.tiles[2 * slot + 1];
      } else {
        t0 = make_int4(0, 0, min(kTileM, nu - slot * kTileM), 0);
        t1 = make_int4(0, 0, 0, 0);
      }
      const int c1 = t1.z > 0 ? t1.x : t0.x;           // cluster of the second half (= c0 if unpacked)
      // lane l covers slot rows 4l..4l+3; lanes 2g, 2g+1 form 8-row group g, loaded as ONE {64 x 8}
      // box when its 8 tokens are consecutive, else as two gather4
      const int4 r4 = *reinterpret_cast<const int4*>((lora ? p.tile_rows : p.unbound_rows) + slot * kTileM + 4 * lane);
      const int l0 = (t0.z + 3) & ~3, l1 = (t1.z + 3) & ~3;
      const bool gvalid = t1.z > 0 ? (lane < 16 ? 4 * lane < l0 : 4 * (lane - 16) < l1) : 4 * lane < l0;
      // The fewest TMA instructions that load the slot's valid rows: the TMA unit issues them one at
      // a time, so 32 gather4 per K block starve the MMA; contiguous token runs use the largest
      // aligned box (128, 32 or 8 rows), the rest gather4.  Lane 4j's 4-row group starts row 4j.
      // run[j]: the 4 rows of group j are consecutive tokens continuing group j-1 (j > 0).
      const bool run4 = gvalid && r4.y == r4.x + 1 && r4.z == r4.x + 2 && r4.w == r4.x + 3;
      const int prev_w = __shfl_up_sync(0xffffffffu, r4.w, 1);
      const bool cont = run4 && (lane == 0 || prev_w + 1 == r4.x);     // continues the previous group
      const uint32_t mrun = __ballot_sync(0xffffffffu, run4), mcont = __ballot_sync(0xffffffffu, cont);
      // a box of 4b groups starting at group j is one run iff run4 for all and cont for j+1..j+b-1
      auto is_box = [&](int j, int b) {
        const uint32_t all = (b == 32 ? 0xffffffffu : ((1u << b) - 1u)) << j;
        const uint32_t inner = all & ~(1u << j);
        return (mrun & all) == all && (mcont & inner) == inner;
      };
      const bool box128 = is_box(0, 32);
      const bool box32 = !box128 && (lane & 7) == 0 && is_box(lane, 8);       // quarter lane/8
      const bool in32 = !box128 && is_box(lane & ~7, 8);                      // my quarter is one box
      const bool box8 = !box128 && !in32 && (lane & 1) == 0 && is_box(lane, 2);
      const bool in8 = box128 || in32 || is_box(lane & ~1, 2);
      const bool g4 = gvalid && !in8;                                          // gather4 fallback
      const uint32_t abytes = static_cast<uint32_t>(__popc(__ballot_sync(0xffffffffu, gvalid)) * 512);
      const int steps = p.kblocks + (lora ? 1 : 0);    // K blocks (+ the LoRA stage)
      for (int k = 0; k < steps; ++k, ++li) {
        if (li % kProducerWarps != warp) continue;
        const int stage = li % L::kStages;
        const uint32_t phase = (li / L::kStages) & 1;
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sA = smem + stage * L::kStage;
        uint8_t* sB = sA + L::kA;
        if (k < p.kblocks) {
          if (lane == 0) {
            mbar_arrive_expect_tx(&full[stage], abytes + static_cast<uint32_t>(L::kB));
            tma_load_2d(sB, &p.tm_w, &full[stage], k * kBK, nb * kProjBN);
          }
          __syncwarp();
          if (box128 && lane == 0) tma_load_2d(sA, &p.tm_x128, &full[stage], k * kBK, r4.x);
          if (box32) tma_load_2d(sA + lane * 512, &p.tm_x32, &full[stage], k * kBK, r4.x);
          if (box8) tma_load_2d(sA + lane * 512, &p.tm_x8, &full[stage], k * kBK, r4.x);
          if (g4) tma_gather4(sA + lane * 512, &p.tm_x4, &full[stage], k * kBK, r4.x, r4.y, r4.z, r4.w);
        } else if (lane == 0) {
          // LoRA stage: A = [hi0 | lo0 | hi1 | lo1], each 128 rows with the other half's rows zero
          // (out-of-bounds boxes fill zeros); B = [U_c0 block | U_c1 block]
          mbar_arrive_expect_tx(&full[stage], static_cast<uint32_t>(4 * L::kT + 2 * L::kU));
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int part = 0; part < 2; ++part) {      // 0 = hi columns [0, rp), 1 = lo columns [rp, 2 rp)
              uint8_t* dst = sA + (2 * h + part) * L::kT;
              // rows 0-63 of the buffer: half h's data if h == 0, zeros (rows -64..-1) if h == 1
              tma_load_3d(dst, &p.tm_t3, &full[stage], part * 16, h == 0 ? 0 : -64, 2 * slot + h);
              // rows 64-127: zeros (rows 64..127 of a 64-row half) if h == 0, half 1's data if h == 1
              tma_load_3d(dst + 64 * 32, &p.tm_t3, &full[stage], part * 16, h == 0 ? 64 : 0, 2 * slot + h);
            }
          }
#pragma unroll
          for (int s4 = 0; s4 < kProjBN / 64; ++s4) {
            tma_load_2d(sB + s4 * 64 * 32, p.tm_out, &full[stage], 0, t0.x * p.d_out + nb * kProjBN + s4 * 64);
            tma_load_2d(sB + L::kU + s4 * 64 * 32, p.tm_out, &full[stage], 0, c1 * p.d_out + nb * kProjBN + s4 * 64);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(kTileM, kProjBN);
    int stage = 0, slot = 0;
    uint32_t phase = 0, aphase = 0;
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      mbar_wait(&acc_empty[slot], aphase ^ 1);
      tc_fence_after();
      const uint32_t acc = tmem + slot * kProjBN;
      const int steps = p.kblocks + (item < bound_items ? 1 : 0);
      for (int k = 0; k < steps; ++k) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a = smem_u32(smem + stage * L::kStage), b = a + L::kA;
          if (k < p.kblocks) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma_bf16(acc, umma_desc_kmajor(a + kk * 32, 128), umma_desc_kmajor(b + kk * 32, 128), idesc,
                        (k > 0 || kk > 0) ? 1u : 0u);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)                 // hi0 U0, lo0 U0, hi1 U1, lo1 U1
              umma_bf16(acc, umma_desc_kmajor(a + q * L::kT, 32), umma_desc_kmajor(b + (q >> 1) * L::kU, 32), idesc,
                        1u);
          }
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == L::kStages) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) umma_commit(&acc_full[slot]);
      __syncwarp();
      if (++slot == kProjAccSlots) { slot = 0; aphase ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ epilogue: TMEM -> bf16 -> y
    const int ew = warp - kEpiWarp0, set = ew >> 2, quarter = warp & 3;
    const int row = quarter * 32 + lane;
    int slot = 0;
    uint32_t aphase = 0;
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      const bool lora = item < bound_items;
      const int s = (lora ? item : item - bound_items) / p.nblk, nb = item % p.nblk;
      bool valid;
      int tok = 0;
      if (lora) {
        const int4 t0 = p.tiles[2 * s], t1 = p.tiles[2 * s + 1];
        valid = t1.z > 0 ? (row < kTileM / 2 ? row < t0.z : row - kTileM / 2 < t1.z) : row < t0.z;
        if (valid) tok = p.tile_rows[s * kTileM + row];
      } else {
        valid = s * kTileM + row < nu;
        if (valid) tok = p.unbound_rows[s * kTileM + row];
      }
      mbar_wait(&acc_full[slot], aphase);
      tc_fence_after();
      __nv_bfloat16* yrow = p.y + static_cast<size_t>(tok) * p.ld_y + nb * kProjBN + set * 128;
#pragma unroll 1
      for (int c = 0; c < 128; c += 32) {
        float v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + slot * kProjBN + set * 128 + c, v);
        tmem_ld_wait();
        if (valid) {
          uint4 w[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w[q]);
#pragma unroll
            for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
          }
          if (p.y32) {                                   // 32-byte (full-sector) stores
            st_global_v8(yrow + c, w[0], w[1]);
            st_global_v8(yrow + c + 16, w[2], w[3]);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(yrow + c + 8 * q) = w[q];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[slot]);
      if (++slot == kProjAccSlots) { slot = 0; aphase ^= 1; }
    }
  }
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc<L::kTmemCols>(tmem);
}

}  // namespace cts
