// expand.cuh -- kernel 2 of the apply: expand Delta y = U_c t (tcgen05, K = r) fused with the
// residual add into the base projection output y (in place).
//
// Paper: App D "U (Sigma V^T x) ... broadcasted"; Punica BGMV #3 "apply matrix B and
// update y" with `scale` -- here scale was already folded into t by kernel 1.
//
// Persistent, grouped (same scheme as the shrink): one CTA per SM walks a static round-robin list
// of work items item = (module g, 128-row tile slot, BN-column block of d_out), laid out over the
// host-known tile bound (empty slots skipped); a slot holds one cluster's tile or two <=64-token
// tiles (one per 64-row half, two MMAs against the two clusters' out_basis blocks):
//   warps 0-3   TMA producers (items dealt round-robin, one warp's gather4 issue rate is not
//               enough): t_hi / t_lo tile (A operand, K-major), the out_basis block (B operand,
//               K-major) and the tile's y rows gathered by token index (tile::gather4, 64-column
//               segments, 128B swizzle) into a kStages-deep ring.  The producer also leaves the
//               item's token rows and tile descriptor in the stage.
//   warp 4      one lane issues D = t_hi U^T + t_lo U^T (M=128 tokens, N=BN, K=16 per MMA) into
//               one of kAccSlots TMEM accumulators.
//   warps 5-12  epilogue: two sets of 4 warps take alternate items; in a set each warp owns one
//               32-row quarter (its TMEM lanes).  Thread = token row: tcgen05.ld 64 fp32 columns at
//               a time, add y_base from smem, round to bf16 (RNE) in place; then the warp itself
//               TMA-scatters its 8 four-row groups to y and releases the stage as soon as the
//               scatter has read it (eager release; measured faster than deferring the release by
//               an item, and faster than coalesced STG row stores from smem).
#pragma once
#include "sm100.cuh"
#include "segment.cuh"
#include "shrink_sigma.cuh"

namespace cts {

constexpr int kExpandThreads = 32 * (kProducerWarps + 1 + 4 * kEpiSets);
constexpr int kBN = 128;                 // d_out columns per work item
constexpr int kExpandAccSlots = 2;       // 2 x (D0 | D1) x 128 fp32 columns = all of TMEM

struct alignas(64) ExpandMod {
  CUtensorMap tm_y;                      // y [T][d_out], box {64, 1}, 128B swizzle (per call)
  const CUtensorMap* tm_t;               // tbuf [max_tiles*128][2*rp], box {rp, 128} (plan, global mem)
  const CUtensorMap* tm_out;             // out_basis [C*d_out][rp], box {rp, 64} (bank, global mem)
  const int4* tiles;                     // [slot][2]: (cluster, start, len, -) per 64-row half
  const int32_t* n_tiles;                // real tile count of this module's map
  const int32_t* tile_rows;              // [tile*128 + row] token index
  __nv_bfloat16* y;                      // y base (register-direct store variant)
  int64_t ld_y;                          // elements
  int nblk;                              // ceil(d_out / kBN)
  int d_out;
};

struct ExpandParams {
  ExpandMod mod[kMaxGroup];
  int prefix[kMaxGroup + 1];             // item prefix over modules (tile bound * nblk each)
  int n_mod;
};

template <int RP>
struct ExpandCfg {
  static constexpr int kY = kTileM * 128;                    // one 64-column segment of y rows (16 KB)
  static constexpr int kSeg = kBN / 64;
  static constexpr int kA = kTileM * RP * 2;                 // t_hi (or t_lo) tile
  static constexpr int kB1 = kBN * RP * 2;                   // one out_basis block
  static constexpr int kB = 2 * kB1;                         // one block per slot half
  static constexpr int kMeta = kTileM * 4 + 32;              // token rows + 2 x int4 descriptors
  static constexpr int kStage = kSeg * kY + 2 * kA + kB;
  static constexpr int kStages = (200 * 1024) / (kStage + kMeta);   // 4 at rp=16, 3 at rp=32, 2 at rp=64
  static constexpr int kOffMeta = kStages * kStage;
  static constexpr int kOffBar = kOffMeta + kStages * kMeta;
  static constexpr int kNumBars = 2 * kStages + 2 * kExpandAccSlots;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kBytes = kOffMisc + 64 + 1024;
  static constexpr uint32_t kSlotCols = 2 * kBN;            // D0 | D1
  static constexpr uint32_t kTmemCols = kSlotCols * kExpandAccSlots;
};

// DIRECT = false: results go back into the stage and each warp TMA-scatters its rows, releasing the
// stage once the scatter has read it.  DIRECT = true: each thread stores its row's 16-byte chunks
// straight from registers (st.global) and the stage is released right after the y_base reads.
template <int RP, bool DIRECT>
__global__ void __launch_bounds__(kExpandThreads, 1) expand_kernel(const __grid_constant__ ExpandParams p) {
  using L = ExpandCfg<RP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* empty = full + L::kStages;
  uint64_t* acc_full = empty + L::kStages;
  uint64_t* acc_empty = acc_full + kExpandAccSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kOffMisc);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    CTS_STAMP(0);
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);            // one arrival per epilogue warp of the owning set
    }
    for (int s = 0; s < kExpandAccSlots; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = p.prefix[p.n_mod];
  griddep_wait();                         // t (previous kernel) and y are ready past this point
  griddep_launch_dependents();
  if (threadIdx.x == 0) CTS_STAMP(1);
  // real tile count of each module's map: lane g holds module g's (one load per warp); work items
  // over the tile bound with tile >= count are empty and skipped without touching memory
  const int nt_lane = lane < p.n_mod ? *p.mod[lane].n_tiles : 0;
  auto tile_count = [&](int g) { return __shfl_sync(0xffffffffu, nt_lane, g); };

  auto stage_y = [&](int s) { return smem + s * L::kStage; };
  auto stage_a = [&](int s) { return smem + s * L::kStage + L::kSeg * L::kY; };
  auto stage_b = [&](int s) { return smem + s * L::kStage + L::kSeg * L::kY + 2 * L::kA; };
  auto stage_rows = [&](int s) { return reinterpret_cast<int*>(smem + L::kOffMeta + s * L::kMeta); };
  auto stage_info = [&](int s) { return reinterpret_cast<int4*>(smem + L::kOffMeta + s * L::kMeta + kTileM * 4); };

  if (warp < kProducerWarps) {
    // ------------------------------------------------------------ TMA producers (items round-robin)
    int li = 0;                                   // index over this CTA's non-empty items
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      const int g = find_module(p.prefix, p.n_mod, item);
      const ExpandMod& m = p.mod[g];
      const int tile = (item - p.prefix[g]) / m.nblk, nb = (item - p.prefix[g]) % m.nblk;
      if (tile >= tile_count(g)) continue;
      const int my = li++;
      if (my % kProducerWarps != warp) continue;
      const int4 t0 = m.tiles[2 * tile], t1 = m.tiles[2 * tile + 1];
      const int4 r4 = *reinterpret_cast<const int4*>(m.tile_rows + tile * kTileM + 4 * lane);
      const int stage = my % L::kStages;
      const uint32_t phase = (my / L::kStages) & 1;
      const bool shared = t1.z > 0;
      const int l0 = (t0.z + 3) & ~3, l1 = (t1.z + 3) & ~3;
      const bool gvalid = shared ? (lane < 16 ? 4 * lane < l0 : 4 * (lane - 16) < l1) : 4 * lane < l0;
      const int ngroups = (l0 + l1) >> 2;
      mbar_wait(&empty[stage], phase ^ 1);
      *reinterpret_cast<int4*>(stage_rows(stage) + 4 * lane) = r4;
      if (lane == 0) {
        stage_info(stage)[0] = make_int4(g, t0.x, nb, t0.z);
        stage_info(stage)[1] = make_int4(t1.x, t1.z, 0, 0);
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[stage], static_cast<uint32_t>(2 * L::kA + (shared ? 2 : 1) * L::kB1 +
                                                                   L::kSeg * ngroups * 512));
        tma_load_2d(stage_a(stage), m.tm_t, &full[stage], 0, tile * kTileM);
        tma_load_2d(stage_a(stage) + L::kA, m.tm_t, &full[stage], RP, tile * kTileM);
#pragma unroll
        for (int s = 0; s < L::kSeg; ++s) {
          tma_load_2d(stage_b(stage) + s * 64 * RP * 2, m.tm_out, &full[stage], 0, t0.x * m.d_out + nb * kBN + s * 64);
          if (shared)
            tma_load_2d(stage_b(stage) + L::kB1 + s * 64 * RP * 2, m.tm_out, &full[stage], 0,
                        t1.x * m.d_out + nb * kBN + s * 64);
        }
      }
      __syncwarp();
      if (gvalid) {
#pragma unroll
        for (int s = 0; s < L::kSeg; ++s)
          tma_gather4(stage_y(stage) + s * L::kY + lane * 512, &m.tm_y, &full[stage], nb * kBN + s * 64, r4.x, r4.y,
                      r4.z, r4.w);
      }
      if (lane == 0 && my < 4) CTS_STAMP(10 + my);
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // N = 2 kBN: the two halves' out_basis blocks are contiguous in the B stage (256 rows), so one
    // MMA per K step gives D0 = t U_c0^T (cols [0,128)) and D1 = t U_c1^T (cols [128,256)); for an
    // unshared slot the second block is stale and D1 is never read.
    constexpr uint32_t idesc = umma_idesc_bf16(kTileM, 2 * kBN);
    int stage = 0, slot = 0;
    uint32_t phase = 0, aphase = 0;
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      const int g = find_module(p.prefix, p.n_mod, item);
      const ExpandMod& m = p.mod[g];
      if ((item - p.prefix[g]) / m.nblk >= tile_count(g)) continue;
      mbar_wait(&acc_empty[slot], aphase ^ 1);
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t acc = tmem + slot * L::kSlotCols;
        const uint32_t hi = smem_u32(stage_a(stage)), lo = hi + L::kA, b = smem_u32(stage_b(stage));
#pragma unroll
        for (int k = 0; k < RP / 16; ++k)
          umma_bf16(acc, umma_desc_kmajor(hi + k * 32, RP * 2), umma_desc_kmajor(b + k * 32, RP * 2), idesc, k != 0);
#pragma unroll
        for (int k = 0; k < RP / 16; ++k)
          umma_bf16(acc, umma_desc_kmajor(lo + k * 32, RP * 2), umma_desc_kmajor(b + k * 32, RP * 2), idesc, 1);
        umma_commit(&acc_full[slot]);
        if (item == static_cast<int>(blockIdx.x)) CTS_STAMP(14);
      }
      __syncwarp();
      if (++stage == L::kStages) { stage = 0; phase ^= 1; }
      if (++slot == kExpandAccSlots) { slot = 0; aphase ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ epilogue (2 sets x 4 warps)
    const int ew = warp - kEpiWarp0;           // 0..7
    const int set = ew >> 2;
    const int quarter = warp & 3;              // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    int li = 0;
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      const int g = find_module(p.prefix, p.n_mod, item);
      const ExpandMod& m = p.mod[g];
      if ((item - p.prefix[g]) / m.nblk >= tile_count(g)) continue;
      const int my = li++;
      if (my % kEpiSets != set) continue;
      const int stage = my % L::kStages, slot = my % kExpandAccSlots;
      const uint32_t phase = (my / L::kStages) & 1, aphase = (my / kExpandAccSlots) & 1;
      mbar_wait(&acc_full[slot], aphase);
      mbar_wait(&full[stage], phase);        // y rows + metadata landed (acquire for this thread)
      tc_fence_after();
      const int4 info = stage_info(stage)[0];   // (g, cluster0, nb, len0)
      const int4 info1 = stage_info(stage)[1];  // (cluster1, len1, -, -)
      const int sub = (info1.y > 0 && quarter >= 2) ? 1 : 0;   // which half's tile these rows hold
      const int sbase = sub * (kTileM / 2);                    // first slot row of that tile
      const int len4 = sbase + (((sub ? info1.y : info.w) + 3) & ~3);   // rows < len4 are live
      uint8_t* ys = stage_y(stage);
      const bool active = quarter * 32 < len4;  // warp-uniform: this quarter holds live rows
      if (active) {
#pragma unroll 1
        for (int j2 = 0; j2 < kBN / 64; ++j2) {
          float v[64];
          const uint32_t taddr =
              tmem + (static_cast<uint32_t>(quarter * 32) << 16) + slot * L::kSlotCols + sub * kBN + j2 * 64;
          tmem_ld32(taddr, v);
          tmem_ld32(taddr + 32, v + 32);
          tmem_ld_wait();
          // rows len..len4 duplicate the last token (identical bytes for the 4-row scatter);
          // the direct variant stores real rows only
          const bool live = DIRECT ? (row - sbase < (sub ? info1.y : info.w)) : (row < len4);
          if (live) {
            uint8_t* base = ys + j2 * L::kY + row * 128;   // 64 columns = one segment
            const ExpandMod& mo = p.mod[info.x];
            const int col0 = info.z * kBN + j2 * 64;
            __nv_bfloat16* yrow = DIRECT ? mo.y + static_cast<size_t>(stage_rows(stage)[row]) * mo.ld_y + col0 : nullptr;
#pragma unroll
            for (int qd = 0; qd < 8; ++qd) {
              const int phys = (qd ^ (row & 7)) * 16;
              uint4 w = *reinterpret_cast<uint4*>(base + phys);
              __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                h[e] = __floats2bfloat162_rn(f.x + v[qd * 8 + 2 * e], f.y + v[qd * 8 + 2 * e + 1]);
              }
              if (DIRECT) {
                if (col0 + qd * 8 < mo.d_out) *reinterpret_cast<uint4*>(yrow + qd * 8) = w;
              } else {
                *reinterpret_cast<uint4*>(base + phys) = w;
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[slot]);
      if (!DIRECT && active) {
        // this warp's 8 four-row groups: lane -> (group, segment); TMA scatter of the rows
        fence_proxy_async_smem();
        __syncwarp();
        const int grp = quarter * 8 + (lane & 7), seg = lane >> 3;
        if (grp * 4 < len4 && seg < L::kSeg) {
          const int4 r4 = *reinterpret_cast<const int4*>(stage_rows(stage) + 4 * grp);
          tma_scatter4(&p.mod[info.x].tm_y, ys + seg * L::kY + grp * 512, info.z * kBN + seg * 64, r4.x, r4.y, r4.z,
                       r4.w);
        }
        bulk_commit();
        bulk_wait_read<0>();                  // the scatter has read this warp's rows out of the stage
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (lane == 0 && quarter == 0 && my < 8) CTS_STAMP(2 + my);
    }
    bulk_wait0();                             // this warp's global writes complete before exit
  }
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc<L::kTmemCols>(tmem);
  if (threadIdx.x == 0) CTS_STAMP(15);
}

}  // namespace cts
