// apply_fused.cuh -- the whole apply of a module group in ONE persistent launch: phase 1 runs the
// shrink + Sigma roles (shrink_sigma.cuh) over all shrink work items, phase 2 the expand + residual
// roles (expand.cuh) over all expand work items.
//
// Why: at decode each grouped launch moves only a few MB, so a separate expand launch pays its own
// launch latency, prologue (barrier init, TMEM alloc) and tile-metadata round trips, and cannot
// start any item before the last shrink CTA has finished its split-K reduction.  Here an expand
// item waits only for ITS slot: the split-K finisher publishes a per-slot "t ready" flag
// (st.release after fence.proxy.async, so the TMA reads of other CTAs see the bf16 t rows) and the
// expand producer polls it (ld.acquire) before loading t.  Progress is guaranteed because the grid
// is at most one CTA per SM (all CTAs co-resident), every role of a CTA finishes its shrink work
// before it takes expand work, and no shrink step ever waits on an expand step.
//
// Shared memory: the two phases reuse one operand arena and keep separate mbarrier sets; TMEM is
// allocated once (512 columns) and reused.  The phase change is per role (see below), not a CTA
// barrier, so a CTA's expand loads overlap its own split-K finisher work.  The ready flags are
// cleared by the last CTA to exit (per-plan exit counter), so the next launch starts from zero even
// when replayed from a CUDA graph.
#pragma once
#include "expand.cuh"
#include "shrink_sigma.cuh"

namespace cts {

struct FusedParams {
  ShrinkParams s;
  ExpandParams e;
  int32_t* exit_count;                   // per plan; self-resetting
};

template <int RP>
struct FusedSmem {
  static constexpr int kArena = ShrinkCfg<RP>::kArena > ExpandCfg<RP>::kArena ? ShrinkCfg<RP>::kArena
                                                                                : ExpandCfg<RP>::kArena;
  static constexpr int kOffBarS = kArena;
  static constexpr int kOffBarE = kOffBarS + ShrinkCfg<RP>::kNumBars * 8;
  static constexpr int kOffBarF = kOffBarE + ExpandCfg<RP>::kNumBars * 8;   // "shrink operands consumed"
  static constexpr int kOffBarT = kOffBarF + 8;                                // "shrink TMEM released"
  static constexpr int kOffMisc = kOffBarT + 8;
  static constexpr int kBytes = kOffMisc + 64 + 1024;
  static constexpr uint32_t kTmemCols = 512;
  static_assert(ShrinkCfg<RP>::kTmemCols <= kTmemCols && ExpandCfg<RP>::kTmemCols <= kTmemCols, "TMEM");
};

template <int RP, int STORE, bool DIAG>
__global__ void __launch_bounds__(kApplyThreads, 1) apply_fused_kernel(const __grid_constant__ FusedParams p) {
  using S = FusedSmem<RP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::kOffMisc);
  int* s_last_exit = reinterpret_cast<int*>(smem + S::kOffMisc + 32);
  ShrinkRing RS = shrink_ring<RP>(smem, reinterpret_cast<uint64_t*>(smem + S::kOffBarS),
                                  reinterpret_cast<int*>(smem + S::kOffMisc + 16));
  ExpandRing RE = expand_ring<RP>(smem, reinterpret_cast<uint64_t*>(smem + S::kOffBarE));
  uint64_t* arena_free = reinterpret_cast<uint64_t*>(smem + S::kOffBarF);
  uint64_t* tmem_free = reinterpret_cast<uint64_t*>(smem + S::kOffBarT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    CTS_STAMP(0);
    shrink_init_barriers<RP>(RS);
    expand_init_barriers<RP>(RE);
    mbar_init(arena_free, 1);
    mbar_init(tmem_free, 4 * kEpiSets);       // every epilogue warp, after its last shrink TMEM access
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<S::kTmemCols>(tmem_slot);
  if (warp == 0 && lane < p.s.n_mod) {   // descriptors never depend on the previous kernel
    tma_prefetch_desc(&p.s.mod[lane].tm_x);
    tma_prefetch_desc(p.s.mod[lane].tm_in);
    tma_prefetch_desc(&p.e.mod[lane].tm_y);
    tma_prefetch_desc(p.e.mod[lane].tm_t);
    tma_prefetch_desc(p.e.mod[lane].tm_out);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  RS.tmem = RE.tmem = *tmem_slot;
  // shrink and expand items cover the same modules, so one per-module slot count serves both
  int nt_lane = 0;
  ShrinkWork W;
  ShrinkFirst first;
  if (p.s.meta_ready) {
    nt_lane = lane < p.s.n_mod ? *p.s.mod[lane].n_tiles : 0;
    W = shrink_work(p.s, nt_lane, lane);
    if (warp < kProducerWarps) first = shrink_first_meta(p.s, W, lane);
  }
  griddep_wait();
  if (threadIdx.x == 0) griddep_launch_dependents();
  if (!p.s.meta_ready) {
    nt_lane = lane < p.s.n_mod ? *p.s.mod[lane].n_tiles : 0;
    W = shrink_work(p.s, nt_lane, lane);
  }
  if (threadIdx.x == 0) CTS_STAMP(1);

  // ---------------------------------------------------------------- phase 1 -> phase 2, per role
  // No CTA-wide barrier between the phases: each role moves on as soon as what it reuses is free.
  //   producers: the operand arena, once the shrink MMAs have consumed every stage (arena_free,
  //              committed by the MMA warp after its last MMA);
  //   MMA warp:  the TMEM columns, once every epilogue warp is done with its shrink TMEM (the
//              accumulators and the staged Sigma_i, tmem_free);
  //   epilogue:  nothing -- it takes expand items after its own split-K / Sigma work, so expand
  //              loads and MMAs of this CTA overlap its shrink finisher chain.
  // weighted expand deal: r0 = CTAs holding one more shrink item than the rest, K = expand items
  // (128 x kBN y read + written) worth one shrink item (128 rows x its K chunk of x)
  const int deal_r0 = (CTS_WEIGHTED_DEAL && W.M.total > static_cast<int>(gridDim.x))
                          ? W.M.total % static_cast<int>(gridDim.x) : 0;
  const int deal_k = p.s.mod[0].kblocks * kBK / (W.ks * CTS_DEAL_DIV * kBN);
  if (warp < kProducerWarps) {
    shrink_producer<RP>(p.s, RS, W, warp, lane, first);
    if (threadIdx.x == 0) CTS_STAMP(3);               // producers done issuing
    mbar_wait(arena_free, 0);
    if (threadIdx.x == 0) CTS_STAMP(7);
    expand_producer<RP>(p.e, RE, nt_lane, warp, lane, shrink_dist_finish<RP>(p.s, W) ? W.ks : 1, deal_r0,
                        deal_k);
  } else if (warp == kMmaWarp) {
    shrink_mma<RP>(p.s, RS, W, lane);
    if (lane == 0) { umma_commit(arena_free); CTS_STAMP(4); }
    __syncwarp();
    mbar_wait(tmem_free, 0);                  // shrink accumulators and staged Sigma all read
    tc_fence_after();
    expand_mma<RP>(p.e, RE, nt_lane, lane, deal_r0, deal_k);
  } else {
    shrink_epilogue<RP, DIAG>(p.s, RS, W, warp, lane);
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(tmem_free);
    if (threadIdx.x == 32 * kEpiWarp0) CTS_STAMP(5);        // epilogue set 0 done
    if (threadIdx.x == 32 * (kEpiWarp0 + 4)) CTS_STAMP(6);  // epilogue set 1 done
    expand_epilogue<RP, STORE>(p.e, RE, nt_lane, warp, lane, deal_r0, deal_k);
  }

  // ---------------------------------------------------------------- exit: last CTA clears flags
  if (threadIdx.x == 0) CTS_STAMP(9);
  if (threadIdx.x == 32 * kEpiWarp0) CTS_STAMP(10);
  __syncthreads();
  if (threadIdx.x == 0) CTS_STAMP(11);
  if (threadIdx.x == 0) *s_last_exit = atomicAdd(p.exit_count, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (*s_last_exit) {
    for (int g = 0; g < p.s.n_mod; ++g)
      for (int i = threadIdx.x; i < p.s.tiles_bound; i += blockDim.x) p.s.mod[g].ready[i] = 0;
    if (threadIdx.x == 0) {
      *p.exit_count = 0;
    }
  }
  if (warp == kMmaWarp) tmem_dealloc<S::kTmemCols>(RS.tmem);
}

}  // namespace cts
