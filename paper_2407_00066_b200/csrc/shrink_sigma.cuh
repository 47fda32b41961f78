// shrink_sigma.cuh -- kernel 1 of the apply: shrink s_t = V_c^T x_t (tcgen05 grouped GEMM over
// cluster tiles) fused with the per-token Sigma_i matvec t_t = scale * Sigma_i s_t.
//
// Paper: App D broadcast product "V^T x" then "Sigma (V^T x)"; Punica BGMV #1/#2 of
// add_lora_slice_with_sigma with fp32 buffers.  Here both live in ONE kernel and the
// rank-r intermediate never round-trips through HBM as fp32.
//
// Persistent, grouped: one launch covers a group of modules (e.g. q,k,v which share x); the grid is
// one CTA per SM and every CTA walks a static round-robin list of work items
//     item = (module g, 128-row tile slot, K-chunk kc of d_in)
// where a slot holds one cluster's tile or two <=64-token tiles of two clusters (one per half; one
// N = 2 r_pad MMA per K step against both clusters' stacked basis slabs; segment.cuh "packing")
// laid out over the host-known tile BOUND (tile slots past the real count are empty and skipped), so
// no CTA waits on a device-side count before issuing its first load; the TMA ring keeps streaming
// across item boundaries.
//   warps 0-2   TMA producers (kProducerWarps): x rows gathered by token index (tile::gather4, 128B swizzle) and
//               the in_basis K-slab (tile) into a kStages-deep mbarrier ring shared by all items;
//               K blocks are dealt round-robin to the 4 warps because one warp's gather4 issue
//               rate caps at ~2 TB/s per GPU (measured, profiles/microbench), four reach the
//               tile-load rate.  Token rows come from the segment kernel's per-slot row list.
//   warp 3      one elected lane issues tcgen05.mma (M=128 tokens, N=2 r_pad, K=16) into one of
//               kAccSlots TMEM accumulators, commit -> acc_full[slot]
//   warps 4-11  epilogue, two sets of 4 warps on alternate items, thread = token row (TMEM lane
//               quarter w%4): tcgen05.ld the partial s;
//               split-K: the partial goes to an fp32 workspace, the LAST CTA to finish a tile
//               (acq_rel per-tile arrival counter) sums the KS partials in kc order (deterministic),
//               gathers Sigma_i (L2-resident, 16-byte loads) and writes t = scale*Sigma_i s as a
//               bf16 hi + lo pair (t ~= hi + lo to ~2^-16 relative) for the expand; in the fused
//               kernel it then publishes the slot's "t ready" flag.
// Rows of a tile past its length, up to a multiple of 4, duplicate the last valid token.
// The roles are device functions so apply_fused.cuh can run them as the first phase of one launch.
#pragma once
#include "sm100.cuh"
#include "segment.cuh"

namespace cts {

#ifdef CTS_TRACE
__device__ unsigned long long g_cts_trace[kTraceCtas][kTraceSlots];
#define CTS_STAMP(slot) do { if (blockIdx.x < kTraceCtas) g_cts_trace[blockIdx.x][slot] = globaltimer(); } while (0)
#else
#define CTS_STAMP(slot) do {} while (0)
#endif

constexpr int kBK = 64;                 // bf16 elements per K block = one 128-byte swizzle row
constexpr int kMaxGroup = 16;           // modules per grouped launch
#ifndef CTS_PRODUCER_WARPS
// TMA producer warps.  3, not 4: with 1 MMA warp and 8 epilogue warps the CTA has 12 warps, 3 per
// SM sub-partition, whose 16K-register files then allow 168 registers per thread instead of 128
// (13 warps put 4 on one sub-partition) -- the r_pad 32/64 instantiations stop spilling.  Measured
// (profiles/r02/s3/producer_warps3_ab.txt): cfg3 decode 25.70 vs 25.82 us per launch, cfg5 60.4 vs
// 61.7, q_proj (r_pad 64) 18.5 vs 20.0, prefill unchanged.
#define CTS_PRODUCER_WARPS 3
#endif
constexpr int kProducerWarps = CTS_PRODUCER_WARPS;
constexpr int kMmaWarp = kProducerWarps;
constexpr int kEpiWarp0 = kProducerWarps + 1;
constexpr int kEpiSets = 2;             // epilogue warp-sets working on alternate items
constexpr int kApplyThreads = 32 * (kProducerWarps + 1 + 4 * kEpiSets);   // producers, MMA, epilogue
constexpr int kShrinkThreads = kApplyThreads;
constexpr int kShrinkAccSlots = 4;
#ifndef CTS_DIST_FINISH
#define CTS_DIST_FINISH 1     // r_pad >= 32: every CTA of a split slot finishes 1/ks of its rows
#endif
#ifndef CTS_DIST_MIN_RP
#define CTS_DIST_MIN_RP 32    // smallest r_pad that uses distributed finishing
#endif
#ifndef CTS_SHRINK_STAGES
#define CTS_SHRINK_STAGES 8   // x / in_basis ring depth cap (the fused kernel shares its arena with the expand)
#endif
#ifndef CTS_KCHUNK_NUM
#define CTS_KCHUNK_NUM 48   // finisher: partials fetched per L2 round trip = CTS_KCHUNK_NUM / r_pad
#endif

struct alignas(64) ShrinkMod {
  CUtensorMap tm_x;                     // x [T][d_in], box {64, 1}, 128B swizzle (per call)
  CUtensorMap tm_x8;                    // x, box {64, 8}  (runs of consecutive tokens, row_boxes)
  CUtensorMap tm_x32;                   // x, box {64, 32}
  const CUtensorMap* tm_in;             // in_basis [C*rp][d_in], box {64, rp} (bank, global mem)
  const int4* tiles;                    // [slot][2]: (cluster, start, len, -) per 64-row half
  const int32_t* n_tiles;               // real slot count of this module's map
  const int32_t* tile_rows;             // [slot*128 + row] token index
  const int32_t* tile_adapters;         // [slot*128 + row] adapter id
  const __nv_bfloat16* sigma;           // [N][rp][rp], row = out index; sigma_diag: [N][rp]
  __nv_bfloat16* tbuf;                  // [max_tiles*128][2*rp]  (hi | lo)
  float* tpart;                         // TP partial mode: fp32 t in TOKEN order [T][rp] instead of tbuf
  float* ws;                            // [(slot*ks + kc)*128 + row][rp] split-K partials
  int32_t* counters;                    // [max_tiles] arrivals per slot (self-resetting)
  int32_t* ready;                       // [max_tiles] "t ready" flags (fused kernel only; else null)
  int kblocks;                          // d_in / 64
  float scale;
};

struct ShrinkParams {
  ShrinkMod mod[kMaxGroup];
  int n_mod;
  int tiles_bound;                      // host-known slot bound per module (flag clearing)
  int ks_max;                           // K chunks per slot: cap (>= 4 K blocks each, workspace fit)
  int target_items;                     // wanted items per SM (K chunks sized on the device)
  int meta_ready;                       // 1: segment outputs are complete before griddep_wait
  int sigma_diag;                       // bank of kind CTS_SIGMA_DIAG (JD-Diag): t = scale * sigma_i .* s
};

template <int RP>
struct ShrinkCfg {
  static constexpr int kA = kTileM * 128;           // bytes per A stage (x rows)
  static constexpr int kB1 = RP * 128;              // one in_basis K-slab (rp rows x 64 cols)
  static constexpr int kB = 2 * kB1;                // bytes per B stage: one slab per slot half
  static constexpr int kStages = (200 * 1024) / (kA + kB) < CTS_SHRINK_STAGES ? (200 * 1024) / (kA + kB) : CTS_SHRINK_STAGES;
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + kStages * kA;
  static constexpr int kArena = kOffB + kStages * kB;          // bytes of staged operands
  static constexpr int kNumBars = 2 * kStages + 2 * kShrinkAccSlots;
  static constexpr uint32_t kSlotCols = 2 * RP < 32 ? 32 : 2 * RP;   // D0 | D1 (one per slot half)
  // r_pad = 16: each epilogue set stages its row's Sigma_i (16 x 16 bf16 = 128 TMEM columns) in
  // TMEM while the MMA runs, so the finisher's Sigma matvec reads TMEM instead of doing two
  // dependent global round trips on the split-K critical path
  static constexpr bool kSigmaTmem = RP == 16;
  static constexpr uint32_t kSigmaCol0 = kSlotCols * kShrinkAccSlots;
  static constexpr uint32_t kSigmaCols = kSigmaTmem ? RP * RP / 2 : 0;  // per set
  static constexpr uint32_t kUsedCols = kSigmaCol0 + kEpiSets * kSigmaCols;
  static constexpr uint32_t kTmemCols = kUsedCols <= 128 ? 128 : (kUsedCols <= 256 ? 256 : 512);
};

// ------------------------------------------------------------------ device-side work map
// Work items are laid over the REAL slot counts the segment kernel produced (lane g of every warp
// holds module g's count, nt_lane), so no item is empty and the K split is sized from the real
// slot total: ks = floor(target_items * grid / slots), capped by the host.  Every role of every CTA
// derives the identical map from the same counts.
struct ItemMap {
  int pre;                              // lane g < n_mod: first item of module g
  int total;                            // items in the launch
  int per;                              // items per slot of this lane's module (ks or nblk)
};

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ ItemMap make_item_map(int n_mod, int nt_lane, int per_lane, int lane) {
  ItemMap M;
  const int cnt = lane < n_mod ? nt_lane * per_lane : 0;
  int inc = cnt;                                           // inclusive scan over lanes
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  M.pre = inc - cnt;
  M.total = __shfl_sync(0xffffffffu, inc, 31);
  M.per = per_lane;
  return M;
}

// K chunks per slot for the shrink, from the real slot total of the group
__device__ __forceinline__ int shrink_ks(const ShrinkParams& p, int nt_lane, int lane) {
  const int slots = warp_sum(lane < p.n_mod ? nt_lane : 0);
  if (slots == 0) return 1;
  // floor, not ceil: items <= target * grid, so no CTA takes a second shrink item whose slot's
  // split-K exchange (and every expand item waiting on it) would then finish a whole item later
  const int want = (p.target_items * static_cast<int>(gridDim.x)) / slots;
  return max(1, min(want, p.ks_max));
}

// The shrink's work map of a launch: K chunks per slot and the item map (per warp, lane g holding
// module g's values).  Computed once per warp -- before griddep_wait when the segment outputs are
// already complete -- so the parameter and shuffle latency stays off the critical path.
struct ShrinkWork {
  int ks;
  ItemMap M;
};

// Distributed finishing (r_pad >= 32).  The r x r Sigma_i matvec of a 128-row slot reads 128
// different Sigma_i (8 KB each at r_pad = 64) with one L1 wavefront per lane and 32-byte load: ~40
// us for the one last-arriving CTA (profiles/r01/decode_tuning/trace_fused_q*.txt).  Instead every
// CTA of the slot waits until all ks partials are published and finishes rows [kc*128/ks, ...),
// so the Sigma traffic spreads over ks SMs; the slot's "t ready" flag then counts ks arrivals.
// Needs every CTA to hold at most one shrink item (all chunks of a slot in flight at once: the
// floor K split guarantees it when items <= grid) and all CTAs co-resident -- so only the fused
// kernel (ready flags set), which already relies on co-residency, uses it; the standalone shrink
// kernel (CTS_FUSED=0, TP partials) keeps the wait-free last-arriver finisher.
template <int RP>
__device__ __forceinline__ bool shrink_dist_finish(const ShrinkParams& p, const ShrinkWork& W) {
  return CTS_DIST_FINISH && RP >= CTS_DIST_MIN_RP && !p.sigma_diag && p.mod[0].ready != nullptr && W.ks > 1 &&
         W.M.total <= static_cast<int>(gridDim.x);
}

// item -> (module g, index within the module); warp-uniform item, all lanes participate
__device__ __forceinline__ int map_item(const ItemMap& M, int n_mod, int item, int lane, int* local) {
  const unsigned b = __ballot_sync(0xffffffffu, lane < n_mod && M.pre <= item);
  const int g = 31 - __clz(b);
  *local = item - __shfl_sync(0xffffffffu, M.pre, g);
  return g;
}

// Shared-memory handles of the shrink pipeline (operand ring in `arena`, barriers elsewhere).
struct ShrinkRing {
  uint8_t* sA;
  uint8_t* sB;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* acc_full;
  uint64_t* acc_empty;
  int* s_last;                          // [kEpiSets]
  uint32_t tmem;
};

template <int RP>
__device__ __forceinline__ ShrinkRing shrink_ring(uint8_t* arena, uint64_t* bars, int* s_last) {
  using L = ShrinkCfg<RP>;
  ShrinkRing R;
  R.sA = arena + L::kOffA;
  R.sB = arena + L::kOffB;
  R.full = bars;
  R.empty = bars + L::kStages;
  R.acc_full = R.empty + L::kStages;
  R.acc_empty = R.acc_full + kShrinkAccSlots;
  R.s_last = s_last;
  R.tmem = 0;
  return R;
}

template <int RP>
__device__ __forceinline__ void shrink_init_barriers(const ShrinkRing& R) {   // one thread
  for (int s = 0; s < ShrinkCfg<RP>::kStages; ++s) {
    mbar_init(&R.full[s], 1);
    mbar_init(&R.empty[s], 1);
  }
  for (int s = 0; s < kShrinkAccSlots; ++s) {
    mbar_init(&R.acc_full[s], 1);
    mbar_init(&R.acc_empty[s], 4);      // one arrival per epilogue warp of the owning set
  }
}

// ------------------------------------------------------------------ TMA producers (warps 0..kProducerWarps-1)
// Tile metadata of a CTA's first non-empty item, loaded before griddep_wait when the segment
// outputs are already complete (meta_ready), so the first gathers issue right after the wait
// instead of after two dependent global loads.
struct ShrinkFirst {
  int item = -1;
  int4 t0, t1, r4;
};

__device__ __forceinline__ ShrinkWork shrink_work(const ShrinkParams& p, int nt_lane, int lane) {
  ShrinkWork w;
  w.ks = shrink_ks(p, nt_lane, lane);
  w.M = make_item_map(p.n_mod, nt_lane, w.ks, lane);
  return w;
}

__device__ __forceinline__ ShrinkFirst shrink_first_meta(const ShrinkParams& p, const ShrinkWork& W, int lane) {
  ShrinkFirst f;
  const int ks = W.ks;
  const ItemMap& M = W.M;
  const int item = blockIdx.x;
  if (item < M.total) {
    int local;
    const int g = map_item(M, p.n_mod, item, lane, &local);
    const ShrinkMod& m = p.mod[g];
    const int tile = local / ks;
    f.item = item;
    f.t0 = m.tiles[2 * tile];
    f.t1 = m.tiles[2 * tile + 1];
    f.r4 = *reinterpret_cast<const int4*>(m.tile_rows + tile * kTileM + 4 * lane);
  }
  return f;
}

template <int RP>
__device__ void shrink_producer(const ShrinkParams& p, const ShrinkRing& R, const ShrinkWork& W, int warp, int lane,
                                const ShrinkFirst& first = ShrinkFirst()) {
  using L = ShrinkCfg<RP>;
  const int ks = W.ks;
  const ItemMap& M = W.M;
  int li = 0;                                     // K-block sequence index over this CTA's items
  for (int item = blockIdx.x; item < M.total; item += gridDim.x) {
    int local;
    const int g = map_item(M, p.n_mod, item, lane, &local);
    const ShrinkMod& m = p.mod[g];
    const int tile = local / ks, kc = local % ks;
    const bool pre = item == first.item;
    const int4 t0 = pre ? first.t0 : m.tiles[2 * tile], t1 = pre ? first.t1 : m.tiles[2 * tile + 1];
    const int4 r4 = pre ? first.r4 : *reinterpret_cast<const int4*>(m.tile_rows + tile * kTileM + 4 * lane);
    const bool shared = t1.z > 0;                 // two <=64-token tiles, one per half
    const int l0 = (t0.z + 3) & ~3, l1 = (t1.z + 3) & ~3;
    const bool gvalid = shared ? (lane < 16 ? 4 * lane < l0 : 4 * (lane - 16) < l1) : 4 * lane < l0;
    const int ngroups = (l0 + l1) >> 2;
    const RowBoxes rb = row_boxes(r4, gvalid, lane);
    const int kb0 = kc * m.kblocks / ks, kb1 = (kc + 1) * m.kblocks / ks;
    const uint32_t bbytes = static_cast<uint32_t>((shared ? 2 : 1) * L::kB1);
    const uint32_t bytes = static_cast<uint32_t>(ngroups * 512) + bbytes;
    for (int kb = kb0; kb < kb1; ++kb, ++li) {
      if (li % kProducerWarps != warp) continue;
      const int stage = li % L::kStages;
      const uint32_t phase = (li / L::kStages) & 1;
      if (li == 0 && lane == 0) CTS_STAMP(16);          // first item mapped
      mbar_wait(&R.empty[stage], phase ^ 1);
      if (lane == 0) mbar_arrive_expect_tx(&R.full[stage], bytes);
      if (li == 0 && lane == 0) CTS_STAMP(17);          // expect_tx armed
      __syncwarp();
      uint8_t* dA = R.sA + stage * L::kA;
      if (rb.box32) tma_load_2d(dA + lane * 512, &m.tm_x32, &R.full[stage], kb * kBK, r4.x);
      if (rb.box8) tma_load_2d(dA + lane * 512, &m.tm_x8, &R.full[stage], kb * kBK, r4.x);
      if (rb.g4) tma_gather4(dA + lane * 512, &m.tm_x, &R.full[stage], kb * kBK, r4.x, r4.y, r4.z, r4.w);
      if (li == 0 && lane == 0) CTS_STAMP(18);          // first x gathers issued
      if (lane == 0) {
        tma_load_2d(R.sB + stage * L::kB, m.tm_in, &R.full[stage], kb * kBK, t0.x * RP);
        if (shared) tma_load_2d(R.sB + stage * L::kB + L::kB1, m.tm_in, &R.full[stage], kb * kBK, t1.x * RP);
      }
      if (li == 0 && lane == 0) CTS_STAMP(2);
    }
  }
}

// ------------------------------------------------------------------ MMA issuer (warp 4)
// Returns once every MMA is issued (the fused kernel then waits for its tmem_free barrier before
// reusing the TMEM columns).
template <int RP>
__device__ void shrink_mma(const ShrinkParams& p, const ShrinkRing& R, const ShrinkWork& W, int lane) {
  using L = ShrinkCfg<RP>;
  // N = 2 r_pad: the two halves' basis slabs are contiguous in the B stage, so ONE MMA per K step
  // yields D0 = A B0^T (cols [0, rp)) and D1 = A B1^T (cols [rp, 2rp)); for an unshared slot the
  // second slab is stale and D1 is never read.  (A second MMA per K step measurably slowed the
  // single issuing thread.)
  constexpr uint32_t idesc = umma_idesc_bf16(kTileM, 2 * RP);
  const int ks = W.ks;
  const ItemMap& M = W.M;
  int stage = 0, slot = 0;
  uint32_t phase = 0, aphase = 0;
  for (int item = blockIdx.x; item < M.total; item += gridDim.x) {
    int local;
    const int g = map_item(M, p.n_mod, item, lane, &local);
    const ShrinkMod& m = p.mod[g];
    const int kc = local % ks;
    const int kb0 = kc * m.kblocks / ks, kb1 = (kc + 1) * m.kblocks / ks;
    mbar_wait(&R.acc_empty[slot], aphase ^ 1);
    tc_fence_after();
    const uint32_t acc = R.tmem + slot * L::kSlotCols;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&R.full[stage], phase);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a_base = smem_u32(R.sA + stage * L::kA);
        const uint32_t b_base = smem_u32(R.sB + stage * L::kB);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          umma_bf16(acc, umma_desc_kmajor(a_base + k * 32, 128), umma_desc_kmajor(b_base + k * 32, 128), idesc,
                    (kb > kb0 || k > 0) ? 1u : 0u);
        umma_commit(&R.empty[stage]);
      }
      __syncwarp();
      if (++stage == L::kStages) { stage = 0; phase ^= 1; }
    }
    if (lane == 0) umma_commit(&R.acc_full[slot]);
    __syncwarp();
    if (++slot == kShrinkAccSlots) { slot = 0; aphase ^= 1; }
  }
}

// Distributed finishing of rows [kc*rpc, (kc+1)*rpc) of a slot (shrink_dist_finish), by the 128
// threads of one epilogue set: kTpr = r_pad/4 threads per row, 128/kTpr rows per pass.  Thread
// `sub` of a row sums the ks partials of its kCols = 4 columns of s (kc order, as the single finisher),
// forms partial dot products Sigma_i[o][cols] . s[cols] for every output o (the 16 threads of a
// row read each Sigma_i row as one contiguous line), then a recursive-halving reduce-scatter
// over the kTpr threads leaves it kCols consecutive outputs of t.
template <int RP>
__device__ __forceinline__ void dist_finish(const ShrinkMod& m, int tile, int kc, int ks, int rpc, int set_tid,
                                            int4 t0, int4 t1) {
  constexpr int kCols = 4, kTpr = RP / kCols;                     // 4 / 8 / 16 threads per row
  static_assert(kTpr >= 4 && kTpr <= 16, "dist_finish: r_pad 16, 32 or 64");
  const int sub = set_tid & (kTpr - 1);
  const int r_end = min((kc + 1) * rpc, kTileM);
  const float* const wtile = m.ws + static_cast<size_t>(tile) * ks * kTileM * RP;
  for (int r0 = kc * rpc; r0 < r_end; r0 += kTileM / kTpr) {     // set-uniform trip count
    const int row = r0 + set_tid / kTpr;
    const int half = (t1.z > 0 && row >= kTileM / 2) ? 1 : 0;
    const int slen4 = ((half ? t1.z : t0.z) + 3) & ~3;
    const bool rvalid = row < r_end && row - half * (kTileM / 2) < slen4;
    float sc[kCols];
#pragma unroll
    for (int c = 0; c < kCols; ++c) sc[c] = 0.f;
    if (rvalid) {
      const float* src = wtile + static_cast<size_t>(row) * RP + sub * kCols;
      constexpr int kB = 8;                                        // partials per L2 round trip
      for (int q0 = 0; q0 < ks; q0 += kB) {
        float buf[kB][kCols];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
          if (q0 + j < ks) {
            const float* a = src + static_cast<size_t>(q0 + j) * kTileM * RP;
            if constexpr (kCols == 4) {
              const float4 f = __ldcg(reinterpret_cast<const float4*>(a));
              buf[j][0] = f.x; buf[j][1] = f.y; buf[j][2] = f.z; buf[j][3] = f.w;
            } else {
              const float2 f = __ldcg(reinterpret_cast<const float2*>(a));
              buf[j][0] = f.x; buf[j][1] = f.y;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) {
          if (q0 + j >= ks) break;
#pragma unroll
          for (int c = 0; c < kCols; ++c) sc[c] += buf[j][c];
        }
      }
    }
    const int adapter = rvalid ? m.tile_adapters[tile * kTileM + row] : 0;
    const __nv_bfloat16* sg = m.sigma + static_cast<size_t>(adapter) * RP * RP + sub * kCols;
    float v[RP];
    constexpr int kOB = 16;                                        // Sigma rows per L2 round trip
#pragma unroll
    for (int o0 = 0; o0 < RP; o0 += kOB) {
      uint32_t w[kOB][kCols / 2];
#pragma unroll
      for (int j = 0; j < kOB; ++j) {
        if constexpr (kCols == 4) {
          const uint2 q = rvalid ? __ldg(reinterpret_cast<const uint2*>(sg + (o0 + j) * RP)) : make_uint2(0, 0);
          w[j][0] = q.x; w[j][1] = q.y;
        } else {
          w[j][0] = rvalid ? __ldg(reinterpret_cast<const unsigned int*>(sg + (o0 + j) * RP)) : 0u;
        }
      }
#pragma unroll
      for (int j = 0; j < kOB; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int e = 0; e < kCols / 2; ++e) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j][e]));
          acc = fmaf(f.x, sc[2 * e], acc);
          acc = fmaf(f.y, sc[2 * e + 1], acc);
        }
        v[o0 + j] = acc;
      }
    }
    int base = 0;                                                  // first output this thread keeps
#pragma unroll
    for (int mk = kTpr / 2, n = RP / 2; mk >= 1; mk >>= 1, n >>= 1) {
      const bool up = (sub & mk) != 0;
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const float keep = up ? v[n + i] : v[i];
        const float give = up ? v[i] : v[n + i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, give, mk);
      }
      if (up) base += n;
    }
    if (rvalid) {
      if (m.tpart != nullptr) {
        float* dp = m.tpart + static_cast<size_t>(m.tile_rows[tile * kTileM + row]) * RP + base;
#pragma unroll
        for (int i = 0; i < kCols; ++i) dp[i] = v[i] * m.scale;
      } else {
        __nv_bfloat16* dst = m.tbuf + (static_cast<size_t>(tile) * kTileM + row) * (2 * RP) + base;
        uint32_t hi[kCols / 2], lo[kCols / 2];
#pragma unroll
        for (int e = 0; e < kCols / 2; ++e) {
          const float a = v[2 * e] * m.scale, b = v[2 * e + 1] * m.scale;
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
          const float2 hf = __bfloat1622float2(h2);
          const __nv_bfloat162 l2 = __floats2bfloat162_rn(a - hf.x, b - hf.y);
          hi[e] = *reinterpret_cast<const uint32_t*>(&h2);
          lo[e] = *reinterpret_cast<const uint32_t*>(&l2);
        }
        if constexpr (kCols == 4) {
          *reinterpret_cast<uint2*>(dst) = make_uint2(hi[0], hi[1]);
          *reinterpret_cast<uint2*>(dst + RP) = make_uint2(lo[0], lo[1]);
        } else {
          *reinterpret_cast<uint32_t*>(dst) = hi[0];
          *reinterpret_cast<uint32_t*>(dst + RP) = lo[0];
        }
      }
    }
  }
}

// Eight finished entries t[o0 .. o0+8) of a row (fp32, scale applied) out: TP partial mode -> fp32
// in token order; else the bf16 hi + lo pair the expand MMA consumes (t ~= hi + lo to ~2^-16).
template <int RP>
__device__ __forceinline__ void store_t8(const ShrinkMod& m, int tile, int row, int o0, const float* t8) {
  if (m.tpart != nullptr) {
    float4* dp = reinterpret_cast<float4*>(m.tpart + static_cast<size_t>(m.tile_rows[tile * kTileM + row]) * RP + o0);
    dp[0] = make_float4(t8[0], t8[1], t8[2], t8[3]);
    dp[1] = make_float4(t8[4], t8[5], t8[6], t8[7]);
    return;
  }
  __nv_bfloat16* dst = m.tbuf + (static_cast<size_t>(tile) * kTileM + row) * (2 * RP) + o0;
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
  *reinterpret_cast<uint4*>(dst) = hi;
  *reinterpret_cast<uint4*>(dst + RP) = lo;
}

// ------------------------------------------------------------------ epilogue (warps kEpiWarp0 .. kEpiWarp0+7)
// DIAG: the bank is of kind CTS_SIGMA_DIAG (a separate instantiation, so the diagonal path adds no
// register pressure to the full-Sigma path).
template <int RP, bool DIAG>
__device__ void shrink_epilogue(const ShrinkParams& p, const ShrinkRing& R, const ShrinkWork& W, int warp, int lane) {
  using L = ShrinkCfg<RP>;
  const int ks = W.ks;
  const ItemMap& M = W.M;
  const int ew = warp - kEpiWarp0;              // 0..7
  const int set = ew >> 2;
  const int quarter = warp & 3;                  // TMEM lane quarter this warp may access
  const int row = quarter * 32 + lane;
  const int set_tid = (ew & 3) * 32 + lane;      // 0..127 within the set
  const bool dist = shrink_dist_finish<RP>(p, W);   // launch-uniform
  constexpr bool diag = DIAG;
  const int rpc = (kTileM + ks - 1) / ks;        // dist: rows finished per CTA of a slot
  int li = 0;                                    // index over this CTA's items
  for (int item = blockIdx.x; item < M.total; item += gridDim.x) {
    int local;
    const int g = map_item(M, p.n_mod, item, lane, &local);
    const ShrinkMod& m = p.mod[g];
    const int tile = local / ks, kc = local % ks;
    const bool my_rows = !dist || (row >= kc * rpc && row < (kc + 1) * rpc);
    const bool mine = (li % kEpiSets) == set;
    const int slot = li % kShrinkAccSlots;
    const uint32_t aphase = (li / kShrinkAccSlots) & 1;
    ++li;
    if (!mine) continue;
    const int4 t0 = m.tiles[2 * tile], t1 = m.tiles[2 * tile + 1];
    const int sub = (t1.z > 0 && quarter >= 2) ? 1 : 0;   // which half's tile this warp's rows hold
    const int slen4 = ((sub ? t1.z : t0.z) + 3) & ~3;
    const bool rvalid = row - sub * (kTileM / 2) < slen4;
    const int adapter = rvalid ? m.tile_adapters[tile * kTileM + row] : 0;
    const uint32_t tsig = R.tmem + (static_cast<uint32_t>(quarter * 32) << 16) + L::kSigmaCol0 + set * L::kSigmaCols;
    if (diag) {                                    // warm L2 with this row's sigma_i (RP bf16)
      if (rvalid) prefetch_l2(m.sigma + static_cast<size_t>(adapter) * RP);
    } else if (L::kSigmaTmem && !dist) {
      // this row's Sigma_i -> TMEM lane `row`, 64 columns (8 rows of Sigma_i) per global round trip
      const uint4* sg = reinterpret_cast<const uint4*>(m.sigma + static_cast<size_t>(adapter) * RP * RP);
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        uint32_t w[64];
#pragma unroll
        for (int v = 0; v < 16; v += 2) {              // 32-byte loads
          uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0;
          if (rvalid) ld_global_nc_v8(sg + 16 * h + v, q0, q1);
          w[4 * v] = q0.x; w[4 * v + 1] = q0.y; w[4 * v + 2] = q0.z; w[4 * v + 3] = q0.w;
          w[4 * v + 4] = q1.x; w[4 * v + 5] = q1.y; w[4 * v + 6] = q1.z; w[4 * v + 7] = q1.w;
        }
        tmem_st32(tsig + 64 * h, w);
        tmem_st32(tsig + 64 * h + 32, w + 32);
      }
      tmem_st_wait();
    } else if (rvalid && my_rows) {               // warm L2 with this row's Sigma_i while the MMA runs
      const uint8_t* sp = reinterpret_cast<const uint8_t*>(m.sigma + static_cast<size_t>(adapter) * RP * RP);
#pragma unroll
      for (int off = 0; off < RP * RP * 2; off += 128) prefetch_l2(sp + off);
    }
    mbar_wait(&R.acc_full[slot], aphase);
    tc_fence_after();
    if (li <= 2 && set_tid == 0) CTS_STAMP(19);        // first accumulator ready
    float s[RP];
#pragma unroll
    for (int c = 0; c < RP; c += 16)
      tmem_ld16(R.tmem + (static_cast<uint32_t>(quarter * 32) << 16) + slot * L::kSlotCols + sub * RP + c, s + c);
    tmem_ld_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&R.acc_empty[slot]);

    bool finisher = true;                          // this thread's row is finished here
    if (ks > 1) {
      // split-K: publish this chunk's partial; the LAST arriving CTA (acq_rel counter) sums the
      // ks partials in kc order, so the result does not depend on scheduling.
      // Workspace row = (slot*ks + kc)*128 + row.
      float* const wbase = m.ws + (static_cast<size_t>(tile) * ks * kTileM + row) * RP;   // + kc*128*RP
      if (rvalid) {
        float4* dst = reinterpret_cast<float4*>(wbase + static_cast<size_t>(kc) * kTileM * RP);
#pragma unroll
        for (int c = 0; c < RP / 4; c += 2)            // 32-byte stores (full sectors)
          st_global_v8(dst + c, make_uint4(__float_as_uint(s[4 * c]), __float_as_uint(s[4 * c + 1]),
                                           __float_as_uint(s[4 * c + 2]), __float_as_uint(s[4 * c + 3])),
                       make_uint4(__float_as_uint(s[4 * c + 4]), __float_as_uint(s[4 * c + 5]),
                                  __float_as_uint(s[4 * c + 6]), __float_as_uint(s[4 * c + 7])));
      }
      named_bar_sync(1 + set, 128);
      if (dist) {
        if (set_tid == 0) {
          atom_add_acq_rel_gpu(&m.counters[tile], 1);
          while (ld_acquire_gpu(&m.counters[tile]) < ks) nanosleep_ns(32);
          // second arrival: the last CTA past the wait resets the counter for the next launch
          if (atom_add_acq_rel_gpu(&m.counters[tile], 1) == 2 * ks - 1) m.counters[tile] = 0;
        }
        named_bar_sync(1 + set, 128);
        dist_finish<RP>(m, tile, kc, ks, rpc, set_tid, t0, t1);
        finisher = false;                          // rows done above; every CTA publishes below
      } else {
        if (set_tid == 0) R.s_last[set] = (atom_add_acq_rel_gpu(&m.counters[tile], 1) == ks - 1);
        named_bar_sync(1 + set, 128);
        finisher = R.s_last[set] != 0;
      }
      if (set_tid == 0 && finisher) CTS_STAMP(12);         // last arrival known
      if (finisher) {
        if (rvalid) {
          // sum in kc order (deterministic), this CTA's own chunk included (it is in L2 from the
          // store above); kChunk partials are fetched at a time, all their loads in flight
          // together: ceil(ks/kChunk) L2 round trips instead of ks
          constexpr int kChunk = CTS_KCHUNK_NUM / RP > 1 ? CTS_KCHUNK_NUM / RP : 1;
#pragma unroll
          for (int c = 0; c < RP; ++c) s[c] = 0.f;
          for (int q0 = 0; q0 < ks; q0 += kChunk) {
            float4 buf[kChunk][RP / 4];
#pragma unroll
            for (int j = 0; j < kChunk; ++j) {
              if (q0 + j < ks) {
                const float4* src = reinterpret_cast<const float4*>(wbase + static_cast<size_t>(q0 + j) * kTileM * RP);
#pragma unroll
                for (int c = 0; c < RP / 4; c += 2) {
                  uint4 a, b;
                  ld_global_cg_v8(src + c, a, b);
                  buf[j][c] = make_float4(__uint_as_float(a.x), __uint_as_float(a.y), __uint_as_float(a.z),
                                          __uint_as_float(a.w));
                  buf[j][c + 1] = make_float4(__uint_as_float(b.x), __uint_as_float(b.y), __uint_as_float(b.z),
                                              __uint_as_float(b.w));
                }
              }
            }
#pragma unroll
            for (int j = 0; j < kChunk; ++j) {
              if (q0 + j >= ks) break;
#pragma unroll
              for (int c = 0; c < RP / 4; ++c) {
                s[4 * c] += buf[j][c].x; s[4 * c + 1] += buf[j][c].y;
                s[4 * c + 2] += buf[j][c].z; s[4 * c + 3] += buf[j][c].w;
              }
            }
          }
        }
        if (set_tid == 0 && !dist) m.counters[tile] = 0;   // ready for the next launch
        if (set_tid == 0) CTS_STAMP(13);                // partials summed
      }
    }
    if (diag && finisher && rvalid) {
      // JD-Diag (Eq. 3): t = scale * sigma_i .* s -- no r x r matvec (App D)
      const uint4* sg = reinterpret_cast<const uint4*>(m.sigma + static_cast<size_t>(adapter) * RP);
#pragma unroll
      for (int v = 0; v < RP / 8; ++v) {
        const uint4 q = __ldg(sg + v);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
        float t8[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
          t8[2 * e] = f.x * s[8 * v + 2 * e] * m.scale;
          t8[2 * e + 1] = f.y * s[8 * v + 2 * e + 1] * m.scale;
        }
        store_t8<RP>(m, tile, row, 8 * v, t8);
      }
    }
    if (L::kSigmaTmem && !diag && finisher) {
      // t = scale * Sigma_i s from the TMEM-staged Sigma_i (warp-collective loads: whole warps)
      float t[RP];
#pragma unroll 1
      for (int h = 0; h < 4; ++h) {             // (t is indexed by h: a 64-byte local array)
        float w[32];
        tmem_ld32(tsig + 32 * h, w);
        tmem_ld_wait();
#pragma unroll
        for (int oo = 0; oo < 4; ++oo) {               // Sigma rows 4h .. 4h+3, 16 bf16 each
          float acc = 0.f;
#pragma unroll
          for (int e = 0; e < RP / 2; ++e) {
            const uint32_t u = __float_as_uint(w[oo * (RP / 2) + e]);
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
            acc = fmaf(f.x, s[2 * e], acc);
            acc = fmaf(f.y, s[2 * e + 1], acc);
          }
          t[4 * h + oo] = acc * m.scale;
        }
      }
      if (rvalid) {
        if (m.tpart != nullptr) {
          const int tok = m.tile_rows[tile * kTileM + row];
          float4* dp = reinterpret_cast<float4*>(m.tpart + static_cast<size_t>(tok) * RP);
#pragma unroll
          for (int c = 0; c < RP / 4; ++c) dp[c] = make_float4(t[4 * c], t[4 * c + 1], t[4 * c + 2], t[4 * c + 3]);
        } else {
          __nv_bfloat16* dst = m.tbuf + (static_cast<size_t>(tile) * kTileM + row) * (2 * RP);
          uint4 hi[RP / 8], lo[RP / 8];
#pragma unroll
          for (int o0 = 0; o0 < RP; o0 += 8) {
            __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&hi[o0 / 8]);
            __nv_bfloat162* ll = reinterpret_cast<__nv_bfloat162*>(&lo[o0 / 8]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const __nv_bfloat162 h2 = __floats2bfloat162_rn(t[o0 + 2 * e], t[o0 + 2 * e + 1]);
              const float2 hf = __bfloat1622float2(h2);
              hh[e] = h2;
              ll[e] = __floats2bfloat162_rn(t[o0 + 2 * e] - hf.x, t[o0 + 2 * e + 1] - hf.y);
            }
          }
#pragma unroll
          for (int q = 0; q < RP / 8; q += 2) {           // 32-byte stores: hi | lo rows of 2*RP bf16
            st_global_v8(dst + 8 * q, hi[q], hi[q + 1]);
            st_global_v8(dst + RP + 8 * q, lo[q], lo[q + 1]);
          }
        }
      }
    }
    if (!L::kSigmaTmem && !diag && finisher && rvalid) {
      // t = scale * Sigma_i s ; thread = token row
      const uint4* srow = reinterpret_cast<const uint4*>(m.sigma + static_cast<size_t>(adapter) * RP * RP);
      const int tok = m.tpart != nullptr ? m.tile_rows[tile * kTileM + row] : 0;
      __nv_bfloat16* dst = m.tbuf + (static_cast<size_t>(tile) * kTileM + row) * (2 * RP);
#pragma unroll 1
      for (int o0 = 0; o0 < RP; o0 += 8) {
        float t8[8];
#pragma unroll
        for (int oo = 0; oo < 8; ++oo) {
          const int o = o0 + oo;
          float acc = 0.f;
          // 32-byte loads: every lane reads a different Sigma_i (one L1 wavefront per lane and
          // load), so the access width sets the wavefront count
#pragma unroll
          for (int v8 = 0; v8 < RP / 8; v8 += 2) {
            uint4 w[2];
            ld_global_nc_v8(srow + (o * RP) / 8 + v8, w[0], w[1]);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[hh]);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                acc = fmaf(f.x, s[(v8 + hh) * 8 + 2 * e], acc);
                acc = fmaf(f.y, s[(v8 + hh) * 8 + 2 * e + 1], acc);
              }
            }
          }
          t8[oo] = acc * m.scale;
        }
        if (m.tpart != nullptr) {                   // TP: this rank's fp32 partial, summed over ranks later
          // rows past a tile's length repeat its last token with identical values: benign rewrites
          float4* dp = reinterpret_cast<float4*>(m.tpart + static_cast<size_t>(tok) * RP + o0);
          dp[0] = make_float4(t8[0], t8[1], t8[2], t8[3]);
          dp[1] = make_float4(t8[4], t8[5], t8[6], t8[7]);
          continue;
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
    if ((finisher || dist) && m.ready != nullptr) {   // set-uniform (dist: every CTA of the slot)
      // fused kernel: make the slot's t visible to other CTAs' TMA (async proxy), then publish
      if (set_tid == 0) CTS_STAMP(14);                  // t stored
      fence_proxy_async_global();
      named_bar_sync(1 + set, 128);
      if (set_tid == 0) {
        if (dist) red_release_add_gpu(&m.ready[tile], 1);   // the expand waits for ks arrivals
        else st_release_gpu(&m.ready[tile], 1);
      }
      if (set_tid == 0) CTS_STAMP(15);                  // flag published
    }
  }
}

// ------------------------------------------------------------------ standalone kernel
template <int RP>
struct ShrinkKernelSmem {
  using L = ShrinkCfg<RP>;
  static constexpr int kOffBar = L::kArena;
  static constexpr int kOffMisc = kOffBar + L::kNumBars * 8;
  static constexpr int kBytes = kOffMisc + 64 + 1024;
};

template <int RP, bool DIAG>
__global__ void __launch_bounds__(kApplyThreads, 1) shrink_sigma_kernel(const __grid_constant__ ShrinkParams p) {
  using S = ShrinkKernelSmem<RP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::kOffMisc);
  ShrinkRing R = shrink_ring<RP>(smem, reinterpret_cast<uint64_t*>(smem + S::kOffBar),
                                 reinterpret_cast<int*>(smem + S::kOffMisc + 16));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    CTS_STAMP(0);
    shrink_init_barriers<RP>(R);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<ShrinkCfg<RP>::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  R.tmem = *tmem_slot;
  // the prologue above overlaps the previous kernel's tail under PDL.  Segment outputs may be read
  // before griddep_wait once another kernel separates this one from cts_segment (meta_ready): the
  // predecessor only triggers its dependents after its own griddep_wait.
  int nt_lane = 0;
  ShrinkWork W;
  ShrinkFirst first;
  if (p.meta_ready) {
    nt_lane = lane < p.n_mod ? *p.mod[lane].n_tiles : 0;
    W = shrink_work(p, nt_lane, lane);
    if (warp < kProducerWarps) first = shrink_first_meta(p, W, lane);
  }
  griddep_wait();
  if (threadIdx.x == 0) griddep_launch_dependents();
  if (!p.meta_ready) {
    nt_lane = lane < p.n_mod ? *p.mod[lane].n_tiles : 0;
    W = shrink_work(p, nt_lane, lane);
  }
  if (threadIdx.x == 0) CTS_STAMP(1);

  if (warp < kProducerWarps) shrink_producer<RP>(p, R, W, warp, lane, first);
  else if (warp == kMmaWarp) shrink_mma<RP>(p, R, W, lane);
  else shrink_epilogue<RP, DIAG>(p, R, W, warp, lane);

  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc<ShrinkCfg<RP>::kTmemCols>(R.tmem);
  if (threadIdx.x == 0) CTS_STAMP(11);
}

}  // namespace cts
