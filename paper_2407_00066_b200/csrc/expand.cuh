// expand.cuh -- kernel 2 of the apply: expand Delta y = U_c t (tcgen05, K = r) fused with the
// residual add into the base projection output y (in place).
//
// Paper: App D "U (Sigma V^T x) ... broadcasted"; Punica BGMV #3 "apply matrix B and
// update y" with `scale` -- here scale was already folded into t by kernel 1.
//
// Persistent, grouped (same scheme as the shrink): one CTA per SM walks a static round-robin list
// of work items item = (module g, 128-row tile slot, BN-column block of d_out), laid out over the
// host-known tile bound (empty slots skipped); a slot holds one cluster's tile or two <=64-token
// tiles (one per 64-row half; one N = 256 MMA covers both clusters' stacked out_basis blocks):
//   warps 0-2   TMA producers (items dealt round-robin, one warp's gather4 issue rate is not
//               enough): t_hi / t_lo tile (A operand, K-major), the out_basis blocks (B operand,
//               K-major) and the tile's y rows gathered by token index (tile::gather4, 64-column
//               segments, 128B swizzle) into a kStages-deep ring.  The producer also leaves the
//               item's token rows and slot descriptor in the stage.  In the fused kernel it first
//               waits for the slot's "t ready" flag.
//   warp 3      one lane issues D = t_hi U^T + t_lo U^T (M=128 tokens, N=256, K=16 per MMA) into
//               one of kAccSlots TMEM accumulators.
//   warps 4-11  epilogue: two sets of 4 warps take alternate items; in a set each warp owns one
//               32-row quarter (its TMEM lanes).  Thread = token row: tcgen05.ld 64 fp32 columns at
//               a time, add y_base from smem, round to bf16 (RNE), then (STORE mode)
//                 kStoreScatter:   write back into the stage; the warp TMA-scatters its 8 four-row
//                                  groups and releases the stage once the scatter has read it;
//                 kStoreDirect:    store the row's 32-byte pieces straight from registers and
//                                  release the stage right after the y_base reads.
#pragma once
#include "sm100.cuh"
#include "segment.cuh"
#include "shrink_sigma.cuh"

namespace cts {

constexpr int kExpandThreads = kApplyThreads;
#ifndef CTS_EXPAND_BN
#define CTS_EXPAND_BN 128
#endif
constexpr int kBN = CTS_EXPAND_BN;       // d_out columns per work item
constexpr int kExpandAccSlots = 512 / (2 * kBN);   // (D0 | D1) x kBN fp32 columns each: all of TMEM
constexpr int kStoreScatter = 0, kStoreDirect = 1;   // expand epilogue store paths
#ifndef CTS_Y_STORE_HINT
#define CTS_Y_STORE_HINT ""       // e.g. ".cs" (evict-first) -- tuning aid
#endif
#ifndef CTS_WEIGHTED_DEAL
#define CTS_WEIGHTED_DEAL 1       // fused: CTAs with an extra shrink item get fewer expand items
#endif
#ifndef CTS_DEAL_DIV
#define CTS_DEAL_DIV 2            // K = d_in / (ks * CTS_DEAL_DIV * kBN): x bytes of a shrink item / y bytes of an expand item
#endif
#ifndef CTS_EXPAND_BOXES
#define CTS_EXPAND_BOXES 1   // runs of consecutive tokens as box loads / stores (row_boxes)
#endif
// Epilogue work split.  kEpiSplit: BOTH epilogue sets work on every item, set s on 64-column
// segment s (the two warps of a TMEM lane quarter split the columns), so an item's accumulator
// and stage are released after half the epilogue latency.  Otherwise the sets alternate items.
#ifndef CTS_EPI_SPLIT
#define CTS_EPI_SPLIT (CTS_EXPAND_BN == 128)
#endif
constexpr bool kEpiSplit = CTS_EPI_SPLIT != 0;
constexpr int kEpiArrivals = kEpiSplit ? 4 * kEpiSets : 4;   // arrivals per item on acc_empty / empty

struct alignas(64) ExpandMod {
  CUtensorMap tm_y;                      // y [T][d_out], box {64, 1}, 128B swizzle (per call)
  CUtensorMap tm_y8;                     // y, box {64, 8}  (runs of consecutive tokens, row_boxes)
  CUtensorMap tm_y32;                    // y, box {64, 32}
  const CUtensorMap* tm_t;               // tbuf [max_tiles*128][2*rp], box {rp, 128} (plan, global mem)
  const CUtensorMap* tm_out;             // out_basis [C*d_out][rp], box {rp, 64} (bank, global mem)
  const int4* tiles;                     // [slot][2]: (cluster, start, len, -) per 64-row half
  const int32_t* n_tiles;                // real slot count of this module's map
  const int32_t* tile_rows;              // [slot*128 + row] token index
  const int32_t* ready;                  // [slot] "t ready" flags (fused kernel only; else null)
  __nv_bfloat16* y;                      // y base (register-direct stores)
  int y32;                               // y base and row stride 32-byte aligned: 256-bit stores
  int64_t ld_y;                          // elements
  int nblk;                              // ceil(d_out / kBN)
  int d_out;
};

struct ExpandParams {
  ExpandMod mod[kMaxGroup];
  int n_mod;
  int meta_ready;                        // 1: segment outputs are complete before griddep_wait
  int poll_first;                        // fused: 1 = wait for t before issuing the item's loads
  int early_items;                       // fused, poll_first = 0: only this CTA's first early_items items
                                         // issue their y / out_basis loads before their t is ready
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
  static constexpr int kArena = kOffMeta + kStages * kMeta;   // bytes of staged operands + metadata
  static constexpr int kNumBars = 2 * kStages + 2 * kExpandAccSlots;
  static constexpr uint32_t kSlotCols = 2 * kBN;            // D0 | D1
  static constexpr uint32_t kTmemCols = kSlotCols * kExpandAccSlots;
};

struct ExpandRing {
  uint8_t* arena;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* acc_full;
  uint64_t* acc_empty;
  uint32_t tmem;
};

template <int RP>
__device__ __forceinline__ ExpandRing expand_ring(uint8_t* arena, uint64_t* bars) {
  using L = ExpandCfg<RP>;
  ExpandRing R;
  R.arena = arena;
  R.full = bars;
  R.empty = bars + L::kStages;
  R.acc_full = R.empty + L::kStages;
  R.acc_empty = R.acc_full + kExpandAccSlots;
  R.tmem = 0;
  return R;
}

template <int RP>
__device__ __forceinline__ void expand_init_barriers(const ExpandRing& R) {   // one thread
  for (int s = 0; s < ExpandCfg<RP>::kStages; ++s) {
    mbar_init(&R.full[s], 1);
    mbar_init(&R.empty[s], kEpiArrivals);   // one arrival per epilogue warp working on the item
  }
  for (int s = 0; s < kExpandAccSlots; ++s) {
    mbar_init(&R.acc_full[s], 1);
    mbar_init(&R.acc_empty[s], kEpiArrivals);
  }
}

__device__ __forceinline__ ItemMap expand_map(const ExpandParams& p, int nt_lane, int lane) {
  return make_item_map(p.n_mod, nt_lane, lane < p.n_mod ? p.mod[lane].nblk : 0, lane);
}

// Weighted static deal (fused kernel).  When the shrink has more items than CTAs, CTAs
// b < r0 = shrink_items % grid run one more shrink item than the rest and would start (and end)
// their expand that much later.  Items [0, A) go round-robin to every CTA, the last nB = K * (grid -
// r0) only to CTAs b >= r0, K = expand items worth one shrink item.  r0 = 0: plain round-robin.
struct ExpandDeal {
  int A, r0, nB;
};

__device__ __forceinline__ ExpandDeal expand_deal(int S, int r0, int K) {
  ExpandDeal d{S, 0, 0};
  if (r0 > 0 && K > 0) {
    d.r0 = r0;
    d.nB = min(K * (static_cast<int>(gridDim.x) - r0), S);
    d.A = S - d.nB;
  }
  return d;
}

__device__ __forceinline__ int expand_deal_count(const ExpandDeal& d) {
  const int G = gridDim.x, b = blockIdx.x;
  int n = d.A > b ? (d.A - b + G - 1) / G : 0;
  if (d.nB > 0 && b >= d.r0) {
    const int GB = G - d.r0, bb = b - d.r0;
    n += d.nB > bb ? (d.nB - bb + GB - 1) / GB : 0;
  }
  return n;
}

__device__ __forceinline__ int expand_deal_count_a(const ExpandDeal& d) {     // round-robin part
  const int G = gridDim.x, b = blockIdx.x;
  return d.A > b ? (d.A - b + G - 1) / G : 0;
}

__device__ __forceinline__ int expand_deal_item(const ExpandDeal& d, int j, int nA) {   // this CTA's j-th item
  const int G = gridDim.x, b = blockIdx.x;
  return j < nA ? b + j * G : d.A + (b - d.r0) + (j - nA) * (G - d.r0);
}

template <int RP> __device__ __forceinline__ uint8_t* stage_y(const ExpandRing& R, int s) {
  return R.arena + s * ExpandCfg<RP>::kStage;
}
template <int RP> __device__ __forceinline__ uint8_t* stage_a(const ExpandRing& R, int s) {
  return R.arena + s * ExpandCfg<RP>::kStage + ExpandCfg<RP>::kSeg * ExpandCfg<RP>::kY;
}
template <int RP> __device__ __forceinline__ uint8_t* stage_b(const ExpandRing& R, int s) {
  return stage_a<RP>(R, s) + 2 * ExpandCfg<RP>::kA;
}
template <int RP> __device__ __forceinline__ int* stage_rows(const ExpandRing& R, int s) {
  return reinterpret_cast<int*>(R.arena + ExpandCfg<RP>::kOffMeta + s * ExpandCfg<RP>::kMeta);
}
template <int RP> __device__ __forceinline__ int4* stage_info(const ExpandRing& R, int s) {
  return reinterpret_cast<int4*>(R.arena + ExpandCfg<RP>::kOffMeta + s * ExpandCfg<RP>::kMeta + kTileM * 4);
}

// ------------------------------------------------------------------ TMA producers (warps 0..kProducerWarps-1)
template <int RP>
__device__ __forceinline__ void expand_produce(const ExpandParams& p, const ExpandRing& R, const ItemMap& M, int item,
                                               int my, int lane, int ready_target);

template <int RP>
__device__ void expand_producer(const ExpandParams& p, const ExpandRing& R, int nt_lane, int warp, int lane,
                                int ready_target = 1,       // fused: arrivals on a slot's "t ready" flag
                                int deal_r0 = 0, int deal_k = 0) {   // fused: weighted deal
  using L = ExpandCfg<RP>;
  const ItemMap M = expand_map(p, nt_lane, lane);
  const ExpandDeal D = expand_deal(M.total, deal_r0, deal_k);
  if (D.nB == 0) {                                // plain round-robin (decode: always)
    int li = 0;                                   // index over this CTA's items
    for (int item = blockIdx.x; item < M.total; item += gridDim.x) {
      const int my = li++;
      if (my % kProducerWarps != warp) continue;
      expand_produce<RP>(p, R, M, item, my, lane, ready_target);
    }
  } else {
    const int n_static = expand_deal_count(D), n_a = expand_deal_count_a(D);
    for (int j = warp; j < n_static; j += kProducerWarps)   // local item j -> producer warp j % 4
      expand_produce<RP>(p, R, M, expand_deal_item(D, j, n_a), j, lane, ready_target);
  }
}

// One work item's loads into ring stage my % kStages (one producer warp, all lanes).
template <int RP>
__device__ __forceinline__ void expand_produce(const ExpandParams& p, const ExpandRing& R, const ItemMap& M, int item,
                                               int my, int lane, int ready_target) {
  using L = ExpandCfg<RP>;
  {
    int local;
    const int g = map_item(M, p.n_mod, item, lane, &local);
    const ExpandMod& m = p.mod[g];
    const int tile = local / m.nblk, nb = local % m.nblk;
    const int4 t0 = m.tiles[2 * tile], t1 = m.tiles[2 * tile + 1];
    const int4 r4 = *reinterpret_cast<const int4*>(m.tile_rows + tile * kTileM + 4 * lane);
    const int stage = my % L::kStages;
    const uint32_t phase = (my / L::kStages) & 1;
    const bool shared = t1.z > 0;
    const int l0 = (t0.z + 3) & ~3, l1 = (t1.z + 3) & ~3;
    const bool gvalid = shared ? (lane < 16 ? 4 * lane < l0 : 4 * (lane - 16) < l1) : 4 * lane < l0;
    const int ngroups = (l0 + l1) >> 2;
    const bool early = !p.poll_first && my < p.early_items;
    const bool poll_late = m.ready != nullptr && early;
    if (m.ready != nullptr && !early) {
      if (lane == 0) {
        while (ld_acquire_gpu(m.ready + tile) < ready_target) nanosleep_ns(64);
        fence_proxy_async_global();
        if (my == 0) CTS_STAMP(8);
      }
      __syncwarp();
    }
    mbar_wait(&R.empty[stage], phase ^ 1);
    *reinterpret_cast<int4*>(stage_rows<RP>(R, stage) + 4 * lane) = r4;
    if (lane == 0) {
      stage_info<RP>(R, stage)[0] = make_int4(g, t0.x, nb, t0.z);
      stage_info<RP>(R, stage)[1] = make_int4(t1.x, t1.z, 0, 0);
    }
    __syncwarp();
    // out_basis blocks and y rows do not depend on the shrink: issue them first, so in the fused
    // kernel they stream in while this slot's t is still being reduced
    if (lane == 0) {
      mbar_arrive_expect_tx(&R.full[stage], static_cast<uint32_t>(2 * L::kA + (shared ? 2 : 1) * L::kB1 +
                                                                   L::kSeg * ngroups * 512));
#pragma unroll
      for (int s = 0; s < L::kSeg; ++s) {
        tma_load_2d(stage_b<RP>(R, stage) + s * 64 * RP * 2, m.tm_out, &R.full[stage], 0,
                    t0.x * m.d_out + nb * kBN + s * 64);
        if (shared)
          tma_load_2d(stage_b<RP>(R, stage) + L::kB1 + s * 64 * RP * 2, m.tm_out, &R.full[stage], 0,
                      t1.x * m.d_out + nb * kBN + s * 64);
      }
    }
    __syncwarp();
    {
      RowBoxes rb = row_boxes(r4, gvalid, lane);
      if (!CTS_EXPAND_BOXES) rb = RowBoxes{false, false, gvalid};
#pragma unroll
      for (int s = 0; s < L::kSeg; ++s) {
        uint8_t* dst = stage_y<RP>(R, stage) + s * L::kY + lane * 512;
        const int c0 = nb * kBN + s * 64;
        if (rb.box32) tma_load_2d(dst, &m.tm_y32, &R.full[stage], c0, r4.x);
        if (rb.box8) tma_load_2d(dst, &m.tm_y8, &R.full[stage], c0, r4.x);
        if (rb.g4) tma_gather4(dst, &m.tm_y, &R.full[stage], c0, r4.x, r4.y, r4.z, r4.w);
      }
    }
    if (lane == 0) {
      if (poll_late) {                            // fused kernel: t of this slot published?
        while (ld_acquire_gpu(m.ready + tile) < ready_target) nanosleep_ns(64);
        fence_proxy_async_global();
        if (my == 0) CTS_STAMP(8);                // first expand item's t available
      }
      tma_load_2d(stage_a<RP>(R, stage), m.tm_t, &R.full[stage], 0, tile * kTileM);
      tma_load_2d(stage_a<RP>(R, stage) + L::kA, m.tm_t, &R.full[stage], RP, tile * kTileM);
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ MMA issuer (warp 4)
template <int RP>
__device__ void expand_mma(const ExpandParams& p, const ExpandRing& R, int nt_lane, int lane, int deal_r0 = 0,
                           int deal_k = 0) {
  using L = ExpandCfg<RP>;
  // N = 2 kBN: the two halves' out_basis blocks are contiguous in the B stage (256 rows), so one
  // MMA per K step gives D0 = t U_c0^T (cols [0,128)) and D1 = t U_c1^T (cols [128,256)); for an
  // unshared slot the second block is stale and D1 is never read.
  constexpr uint32_t idesc = umma_idesc_bf16(kTileM, 2 * kBN);
  const ItemMap M = expand_map(p, nt_lane, lane);
  const int n_items = expand_deal_count(expand_deal(M.total, deal_r0, deal_k));
  int stage = 0, slot = 0;
  uint32_t phase = 0, aphase = 0;
  for (int li = 0; li < n_items; ++li) {
    mbar_wait(&R.acc_empty[slot], aphase ^ 1);
    if (lane == 0 && li >= 1 && li <= 3) CTS_STAMP(27 + 4 * (li - 1));   // MMA: accumulator free
    mbar_wait(&R.full[stage], phase);
    if (lane == 0 && li >= 1 && li <= 3) CTS_STAMP(36 + (li - 1));       // MMA: operands (t) landed
    tc_fence_after();
    if (lane == 0) {
      const uint32_t acc = R.tmem + slot * L::kSlotCols;
      const uint32_t hi = smem_u32(stage_a<RP>(R, stage)), lo = hi + L::kA, b = smem_u32(stage_b<RP>(R, stage));
#pragma unroll
      for (int k = 0; k < RP / 16; ++k)
        umma_bf16(acc, umma_desc_kmajor(hi + k * 32, RP * 2), umma_desc_kmajor(b + k * 32, RP * 2), idesc, k != 0);
#pragma unroll
      for (int k = 0; k < RP / 16; ++k)
        umma_bf16(acc, umma_desc_kmajor(lo + k * 32, RP * 2), umma_desc_kmajor(b + k * 32, RP * 2), idesc, 1);
      umma_commit(&R.acc_full[slot]);
    }
    __syncwarp();
    if (++stage == L::kStages) { stage = 0; phase ^= 1; }
    if (++slot == kExpandAccSlots) { slot = 0; aphase ^= 1; }
  }
}

// ------------------------------------------------------------------ epilogue (warps kEpiWarp0 .. kEpiWarp0+7)
template <int RP, int STORE>
__device__ void expand_epilogue(const ExpandParams& p, const ExpandRing& R, int nt_lane, int warp, int lane,
                                int deal_r0 = 0, int deal_k = 0) {
  using L = ExpandCfg<RP>;
  const ItemMap M = expand_map(p, nt_lane, lane);
  const int ew = warp - kEpiWarp0;               // 0..7
  const int set = ew >> 2;
  const int quarter = warp & 3;                  // TMEM lane quarter this warp may access
  const int row = quarter * 32 + lane;
  const int n_items = expand_deal_count(expand_deal(M.total, deal_r0, deal_k));
  for (int my = 0; my < n_items; ++my) {
    if (!kEpiSplit && my % kEpiSets != set) continue;
    static_assert(!kEpiSplit || kEpiSets == kBN / 64, "split epilogue: one 64-column segment per set");
    const int seg0 = kEpiSplit ? set : 0, seg1 = kEpiSplit ? set + 1 : kBN / 64;   // this warp's segments
    const int stage = my % L::kStages, slot = my % kExpandAccSlots;
    const uint32_t phase = (my / L::kStages) & 1, aphase = (my / kExpandAccSlots) & 1;
    mbar_wait(&R.acc_full[slot], aphase);
    if (warp == kEpiWarp0 && lane == 0 && my >= 1 && my <= 3) CTS_STAMP(24 + 4 * (my - 1));   // acc ready
    mbar_wait(&R.full[stage], phase);            // y rows + metadata landed (acquire for this thread)
    tc_fence_after();
    const int4 info = stage_info<RP>(R, stage)[0];    // (g, cluster0, nb, len0)
    const int4 info1 = stage_info<RP>(R, stage)[1];   // (cluster1, len1, -, -)
    const int sub = (info1.y > 0 && quarter >= 2) ? 1 : 0;   // which half's tile these rows hold
    const int sbase = sub * (kTileM / 2);                    // first slot row of that tile
    const int slen = sub ? info1.y : info.w;
    const int len4 = sbase + ((slen + 3) & ~3);              // rows < len4 are live
    uint8_t* ys = stage_y<RP>(R, stage);
    const bool active = quarter * 32 < len4;     // warp-uniform: this quarter holds live rows
    if (active) {
#pragma unroll 1
      for (int j2 = seg0; j2 < seg1; ++j2) {
        float v[64];
        const uint32_t taddr =
            R.tmem + (static_cast<uint32_t>(quarter * 32) << 16) + slot * L::kSlotCols + sub * kBN + j2 * 64;
        tmem_ld32(taddr, v);
        tmem_ld32(taddr + 32, v + 32);
        tmem_ld_wait();
        if (warp == kEpiWarp0 && lane == 0 && my >= 1 && my <= 3) CTS_STAMP(25 + 4 * (my - 1));   // TMEM read
        // rows len..len4 duplicate the last token (identical bytes for the 4-row scatter); the
        // direct variant stores real rows only
        constexpr bool DIRECT = STORE == kStoreDirect;
        const bool live = DIRECT ? (row - sbase < slen) : (row < len4);
        if (live) {
          uint8_t* base = ys + j2 * L::kY + row * 128;   // 64 columns = one segment
          const ExpandMod& mo = p.mod[info.x];
          const int col0 = info.z * kBN + j2 * 64;
          __nv_bfloat16* yrow =
              DIRECT ? mo.y + static_cast<size_t>(stage_rows<RP>(R, stage)[row]) * mo.ld_y + col0 : nullptr;
#pragma unroll
          for (int qd = 0; qd < 8; qd += 2) {
            uint4 w[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int phys = ((qd + u) ^ (row & 7)) * 16;
              w[u] = *reinterpret_cast<uint4*>(base + phys);
              __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w[u]);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                h[e] = __floats2bfloat162_rn(f.x + v[(qd + u) * 8 + 2 * e], f.y + v[(qd + u) * 8 + 2 * e + 1]);
              }
              if (!DIRECT) *reinterpret_cast<uint4*>(base + phys) = w[u];
            }
            if (DIRECT && col0 + qd * 8 < mo.d_out) {
              if (mo.y32) {
                // one 32-byte (full-sector) store for the two 16-byte chunks (256-bit LSU path, sm_100)
                asm volatile("st.global" CTS_Y_STORE_HINT ".v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(yrow + qd * 8),
                             "r"(w[0].x), "r"(w[0].y), "r"(w[0].z), "r"(w[0].w), "r"(w[1].x), "r"(w[1].y), "r"(w[1].z),
                             "r"(w[1].w)
                             : "memory");
              } else {
                *reinterpret_cast<uint4*>(yrow + qd * 8) = w[0];
                *reinterpret_cast<uint4*>(yrow + qd * 8 + 8) = w[1];
              }
            }
          }
        }
      }
    }
    if (warp == kEpiWarp0 && lane == 0 && my >= 1 && my <= 3) CTS_STAMP(26 + 4 * (my - 1));     // stores issued
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&R.acc_empty[slot]);
    if (STORE == kStoreScatter && active) {
      // this warp's 8 four-row groups: lane -> (group, segment); TMA scatter of the rows
      fence_proxy_async_smem();
      __syncwarp();
      // lane l plans 4-row group l of the slot (row_boxes), then this warp stores its quarter's
      // 8 groups (lane -> (group, segment)) as 32-row / 8-row boxes or scatter4
      const int4 rl = *reinterpret_cast<const int4*>(stage_rows<RP>(R, stage) + 4 * lane);
      RowBoxes rb = row_boxes(rl, 4 * lane < len4 && (lane >> 3) == quarter, lane);
      if (!CTS_EXPAND_BOXES) rb = RowBoxes{false, false, 4 * lane < len4 && (lane >> 3) == quarter};
      const uint32_t m32 = __ballot_sync(0xffffffffu, rb.box32), m8 = __ballot_sync(0xffffffffu, rb.box8);
      const uint32_t mg4 = __ballot_sync(0xffffffffu, rb.g4);
      const int grp = quarter * 8 + (lane & 7), seg = seg0 + (lane >> 3);
      if (seg < seg1) {
        const int4 r4 = *reinterpret_cast<const int4*>(stage_rows<RP>(R, stage) + 4 * grp);
        const CUtensorMap* tm = nullptr;
        if (m32 >> grp & 1) tm = &p.mod[info.x].tm_y32;
        else if (m8 >> grp & 1) tm = &p.mod[info.x].tm_y8;
        if (tm) tma_store_2d(tm, ys + seg * L::kY + grp * 512, info.z * kBN + seg * 64, r4.x);
        else if (mg4 >> grp & 1)
          tma_scatter4(&p.mod[info.x].tm_y, ys + seg * L::kY + grp * 512, info.z * kBN + seg * 64, r4.x, r4.y, r4.z,
                       r4.w);
      }
      bulk_commit();
      bulk_wait_read<0>();                      // the scatter has read this warp's rows out of the stage
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&R.empty[stage]);
    if (warp == kEpiWarp0 && lane == 0 && my < 4) CTS_STAMP(20 + my);   // trace: item my's epilogue done
  }
  if (STORE == kStoreScatter) bulk_wait0();     // this warp's global writes complete before exit
}

// ------------------------------------------------------------------ TP: reduced fp32 t -> hi | lo
// After the caller's all-reduce of the per-rank partials (cts_expand_reduced_group): gather each
// slot row's token from the token-ordered fp32 t and split it into the bf16 hi + lo pair the
// expand MMA consumes (same split as the shrink epilogue).
struct SplitArgs {
  const float* part[kMaxGroup];          // [T][rp] token order
  __nv_bfloat16* tbuf[kMaxGroup];        // [slot*128 + row][2*rp]
  const int32_t* n_tiles[kMaxGroup];
  const int32_t* tile_rows[kMaxGroup];
  int n_mod, rp;
};

__global__ void __launch_bounds__(256) t_split_kernel(const __grid_constant__ SplitArgs a) {
  griddep_wait();
  if (threadIdx.x == 0) griddep_launch_dependents();
  for (int g = 0; g < a.n_mod; ++g) {
    const size_t n = static_cast<size_t>(*a.n_tiles[g]) * kTileM * a.rp;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
      const size_t row = i / a.rp;
      const int c = static_cast<int>(i % a.rp);
      const float v = a.part[g][static_cast<size_t>(a.tile_rows[g][row]) * a.rp + c];
      const __nv_bfloat16 hi = __float2bfloat16_rn(v);
      a.tbuf[g][row * 2 * a.rp + c] = hi;
      a.tbuf[g][row * 2 * a.rp + a.rp + c] = __float2bfloat16_rn(v - __bfloat162float(hi));
    }
  }
}

// ------------------------------------------------------------------ standalone kernel
template <int RP>
struct ExpandKernelSmem {
  using L = ExpandCfg<RP>;
  static constexpr int kOffBar = L::kArena;
  static constexpr int kOffMisc = kOffBar + L::kNumBars * 8;
  static constexpr int kBytes = kOffMisc + 64 + 1024;
};

template <int RP, int STORE>
__global__ void __launch_bounds__(kApplyThreads, 1) expand_kernel(const __grid_constant__ ExpandParams p) {
  using S = ExpandKernelSmem<RP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::kOffMisc);
  ExpandRing R = expand_ring<RP>(smem, reinterpret_cast<uint64_t*>(smem + S::kOffBar));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    expand_init_barriers<RP>(R);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<ExpandCfg<RP>::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  R.tmem = *tmem_slot;
  int nt_lane = 0;
  if (p.meta_ready) nt_lane = lane < p.n_mod ? *p.mod[lane].n_tiles : 0;
  griddep_wait();                         // t (previous kernel) and y are ready past this point
  if (threadIdx.x == 0) griddep_launch_dependents();
  if (!p.meta_ready) nt_lane = lane < p.n_mod ? *p.mod[lane].n_tiles : 0;

  if (warp < kProducerWarps) expand_producer<RP>(p, R, nt_lane, warp, lane);
  else if (warp == kMmaWarp) expand_mma<RP>(p, R, nt_lane, lane);
  else expand_epilogue<RP, STORE>(p, R, nt_lane, warp, lane);

  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc<ExpandCfg<RP>::kTmemCols>(R.tmem);
}

}  // namespace cts
