// apply_local.cuh -- the decode-regime apply of a module group in ONE persistent launch with NO
// inter-CTA exchange (round 2).
//
// Paper: App D evaluates the compressed update right to left, V^T x, then Sigma_i (.), then U (.)
// (P:L976-980); Punica's add_lora_slice_with_sigma runs the same three products as three launches
// (App F.4).  Here every CTA owns whole PIECES = (module g, cluster c, a range of c's
// cluster-sorted tokens, <= 64 rows) and runs the full chain for them on chip:
//     s    = V_c^T x            tcgen05, M = 128 token rows, N = r_pad, K = d_in (A = x rows)
//     t    = scale Sigma_i s    epilogue set A, thread = token row, Sigma_i staged in TMEM
//     dy^T = U_c t^T            tcgen05, M = 128 OUTPUT COLUMNS, N = tokens, K = r_pad (A = the
//                               out_basis block, B = t hi / lo): transposed, so all 128 TMEM lanes
//                               hold useful outputs even when a piece has 8 rows
//     y    = bf16(y + dy)       epilogue set B, thread = output column, y rows staged by TMA
// The split-K design of apply_fused.cuh spreads a slot's K over ~3-11 CTAs and pays a chain of
// global round trips (partials, last-arriver reduction, t publication, flag polling) on every
// launch -- ~6 us of a 20-25 us decode launch (profiles/r02/).  Here nothing crosses CTAs: the
// price is that a cluster's bases are read once per piece (from L2 after the first), which at
// decode (~7-28 rows per CTA) is the cheaper side.  All waits are CTA-local, so the kernel makes
// progress with any number of co-resident CTAs (no co-residency assumption).
//
// Work map (device side, identical in every role): per module the cluster-sorted bound tokens of
// cluster c (segment kernel: offsets, perm, sorted adapters) are cut into k_c = max(round(n_c/u_g),
// ceil(n_c/lcap)) near-equal pieces, u_g = the host's rows-per-CTA target for module g (weighted by
// its bytes per row, d_in + 2 d_out, so every CTA gets ~ the same bytes); pieces are numbered in
// (module, cluster) order and dealt round-robin to the CTAs.
//
// Warps (16): 0-3 x rows (tile::gather4, 512 B / op: one warp issues ~14 GB/s, profiles/r02
// tma_rate.txt) + in_basis (one 3-D box of kLocKB K blocks); 4-6 y rows (gather4 of 256-column
// rows, 2 KB / op) + out_basis blocks; 7 MMA; 8-11 set A (t); 12-15 set B (y).
#pragma once
#include "sm100.cuh"
#include "segment.cuh"
#include "shrink_sigma.cuh"

namespace cts {

#ifdef CTS_TRACE
// per-job timeline of CTA kJobTraceCta: [event][job] globaltimer stamps (debug builds only)
constexpr int kJobTraceCta = 5, kJobTraceN = 128;
__device__ unsigned long long g_cts_jobtrace[8][kJobTraceN];
#define CTS_JOB_STAMP(ev, j) do { if (blockIdx.x == kJobTraceCta && (j) < kJobTraceN) g_cts_jobtrace[ev][j] = globaltimer(); } while (0)
#else
#define CTS_JOB_STAMP(ev, j) do {} while (0)
#endif

#ifndef CTS_LOC_NO_YMATH
#define CTS_LOC_NO_YMATH 0     // timing knob: skip the y epilogue arithmetic
#endif
#ifndef CTS_LOC_NO_SCATTER
#define CTS_LOC_NO_SCATTER 0   // timing knob: skip the y scatter
#endif
#ifndef CTS_LOC_SFRAC
#define CTS_LOC_SFRAC 45       // percent of the ring budget given to the shrink ring
#endif

constexpr int kLocXWarps = 4;
constexpr int kLocYWarps = 3;
constexpr int kLocMmaWarp = kLocXWarps + kLocYWarps;
constexpr int kLocAWarp0 = kLocMmaWarp + 1;
constexpr int kLocBWarp0 = kLocAWarp0 + 4;
constexpr int kLocThreads = 32 * (kLocBWarp0 + 4);
constexpr int kLocKB = 4;          // 64-column K blocks per shrink stage (one 3-D in_basis box)
constexpr int kLocBN = 256;        // output columns per expand job (two M = 128 MMAs)
constexpr int kLocMaxRows = 64;    // piece row cap (decode regime; larger batches use apply_fused)
constexpr int kLocTable = 2048;    // work-map entries n_mod * (C + 1) held in shared memory
constexpr int kLocRP = 16;         // r_pad served by this kernel (Sigma_i staged in 128 TMEM columns)
constexpr int kLocSigCol = 2 * kLocRP;            // TMEM: [0, 2 rp) shrink accumulators
constexpr int kLocE0 = kLocSigCol + kLocRP * kLocRP / 2;   // then Sigma_i, then expand accumulators

struct alignas(64) LocMod {
  CUtensorMap tm_x;                // x [T][d_in] bf16, box {64, 1}, 128B swizzle (gather4 rows)
  CUtensorMap tm_y;                // y [T][d_out] bf16, box {256, 1}, no swizzle (gather4 rows)
  const CUtensorMap* tm_in3;       // bank: in_basis viewed {64, C*rp, d_in/64}, box {64, rp, kLocKB}
  const CUtensorMap* tm_out;       // bank: out_basis [C*d_out][rp], box {rp, 256}, 32B swizzle
  const int32_t* offsets;          // plan: [C+1] cluster offsets of the module's map
  const int32_t* perm;             // plan: sorted position -> token
  const int32_t* sadapter;         // plan: sorted position -> adapter
  const __nv_bfloat16* sigma;      // bank: [N][rp][rp], row = out index
  __nv_bfloat16* y;
  int64_t ld_y;
  int d_in, d_out, unit_rows;
  float scale;
};

struct LocParams {
  LocMod mod[kMaxGroup];
  int n_mod, C;
  int lcap;                        // piece row cap (multiple of 8, <= kLocMaxRows)
  int npad;                        // roundup16(lcap): TMEM columns per expand half-accumulator
  int s_stages, e_stages, n_acc;
  int meta_ready;                  // 1: segment outputs complete before griddep_wait
};

// ------------------------------------------------------------------ shared-memory layout
struct LocLayout {
  int tab, sring, tt, ering, tok, bars, total;
  int a_bytes, s_bytes, e_bytes, t_bytes;
};

__host__ __device__ inline LocLayout loc_layout(int n_mod, int C, int lcap, int npad, int s_stages, int e_stages,
                                                int n_acc) {
  auto up = [](int v, int a) { return (v + a - 1) / a * a; };
  LocLayout L;
  L.a_bytes = up(lcap, 8) / 8 * 1024;                  // rows of one K block, 8-row 1 KB atoms
  L.s_bytes = kLocKB * (L.a_bytes + kLocRP * 128);     // x rows + in_basis slabs of kLocKB K blocks
  L.e_bytes = kLocBN * kLocRP * 2 + lcap * kLocBN * 2; // out_basis block + y rows
  L.t_bytes = npad * kLocRP * 2;                       // one t tile (hi or lo)
  L.tab = 0;
  L.sring = up(2 * (n_mod * (C + 1) + 1) * 4, 1024);
  L.tt = L.sring + s_stages * L.s_bytes;
  L.ering = L.tt + up(4 * L.t_bytes, 1024);
  L.tok = L.ering + e_stages * L.e_bytes;
  L.bars = up(L.tok + 4 * kLocMaxRows * 4, 64);
  L.total = L.bars + (2 * s_stages + 2 * e_stages + 8 + 2 * n_acc) * 8 + 64 + 1024;   // + base alignment
  return L;
}

struct LocBars {
  uint64_t *full_s, *empty_s, *full_e, *empty_e, *acc_s_full, *acc_s_empty, *t_full, *t_empty, *acc_full, *acc_empty;
  int* total;
};

__device__ __forceinline__ LocBars loc_bars(uint8_t* smem, const LocLayout& L, const LocParams& p) {
  LocBars B;
  uint64_t* b = reinterpret_cast<uint64_t*>(smem + L.bars);
  B.full_s = b; b += p.s_stages;
  B.empty_s = b; b += p.s_stages;
  B.full_e = b; b += p.e_stages;
  B.empty_e = b; b += p.e_stages;
  B.acc_s_full = b; b += 2;
  B.acc_s_empty = b; b += 2;
  B.t_full = b; b += 2;
  B.t_empty = b; b += 2;
  B.acc_full = b; b += p.n_acc;
  B.acc_empty = b; b += p.n_acc;
  B.total = reinterpret_cast<int*>(b);
  return B;
}

// ------------------------------------------------------------------ work map
struct Piece {
  int g, c, lo, L;
};

// Block-wide exclusive scan for any blockDim that is a multiple of 32 (<= 1024); warp_sums[33].
__device__ __forceinline__ int loc_block_scan(int v, int* warp_sums, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int s = lane < nw ? warp_sums[lane] : 0;
    int si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += n;
    }
    warp_sums[lane] = si - s;
    if (lane == 31) warp_sums[32] = si;
  }
  __syncthreads();
  const int res = warp_sums[warp] + incl - v;
  total = warp_sums[32];
  __syncthreads();
  return res;
}

// off[g*(C+1) + c] = cluster offsets of module g; pre[f] (f = g*C + c) = first piece index of
// (g, c) in the launch, pre[n_mod*C] = total.  All threads of the CTA.
__device__ void loc_build_map(const LocParams& p, int* off, int* pre, int* total, int* warp_sums) {
  const int C = p.C, n_off = p.n_mod * (C + 1), n = p.n_mod * C;
  for (int i = threadIdx.x; i < n_off; i += blockDim.x) off[i] = p.mod[i / (C + 1)].offsets[i % (C + 1)];
  __syncthreads();
  int carry = 0;
  for (int f0 = 0; f0 < n; f0 += blockDim.x) {
    const int f = f0 + threadIdx.x;
    int k = 0;
    if (f < n) {
      const int g = f / C, c = f % C;
      const int cnt = off[g * (C + 1) + c + 1] - off[g * (C + 1) + c];
      if (cnt > 0) {
        const int u = p.mod[g].unit_rows;
        k = max(max(1, (cnt + u / 2) / u), (cnt + p.lcap - 1) / p.lcap);
      }
    }
    int tot;
    const int ex = loc_block_scan(k, warp_sums, tot);
    if (f < n) pre[f] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    pre[n] = carry;
    *total = carry;
  }
  __syncthreads();
}

__device__ __forceinline__ Piece loc_piece(const LocParams& p, const int* off, const int* pre, int u) {
  const int C = p.C;
  int lo = 0, hi = p.n_mod * C;                     // pre[lo] <= u < pre[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] <= u) lo = mid;
    else hi = mid;
  }
  const int g = lo / C, c = lo % C;
  const int k = pre[lo + 1] - pre[lo], sub = u - pre[lo];
  const int base = off[g * (C + 1) + c], cnt = off[g * (C + 1) + c + 1] - base;
  const int r0 = base + sub * cnt / k, r1 = base + (sub + 1) * cnt / k;
  return Piece{g, c, r0, r1 - r0};
}

// tokens of this lane's 4-row group of a piece (rows past L repeat the last row)
__device__ __forceinline__ int4 loc_rows4(const int32_t* perm, const Piece& P, int lane) {
  const int b = 4 * lane;
  int4 r;
  r.x = perm[P.lo + min(b, P.L - 1)];
  r.y = perm[P.lo + min(b + 1, P.L - 1)];
  r.z = perm[P.lo + min(b + 2, P.L - 1)];
  r.w = perm[P.lo + min(b + 3, P.L - 1)];
  return r;
}

// ------------------------------------------------------------------ the kernel
__global__ void __launch_bounds__(kLocThreads, 1) apply_local_kernel(const __grid_constant__ LocParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const LocLayout L = loc_layout(p.n_mod, p.C, p.lcap, p.npad, p.s_stages, p.e_stages, p.n_acc);
  const LocBars B = loc_bars(smem, L, p);
  int* off = reinterpret_cast<int*>(smem + L.tab);
  int* pre = off + p.n_mod * (p.C + 1);
  __shared__ int warp_sums[33];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.s_stages, E = p.e_stages, NA = p.n_acc;
  if (threadIdx.x == 0) {
    CTS_STAMP(0);
    for (int i = 0; i < S; ++i) { mbar_init(&B.full_s[i], 1); mbar_init(&B.empty_s[i], 1); }
    // an expand stage is free once the MMA consumed its out_basis block (commit) AND the four set-B
    // warps read its y rows
    for (int i = 0; i < E; ++i) { mbar_init(&B.full_e[i], 1); mbar_init(&B.empty_e[i], 5); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.acc_s_full[i], 1);
      mbar_init(&B.acc_s_empty[i], 4);
      mbar_init(&B.t_full[i], 1);
      mbar_init(&B.t_empty[i], 1);
    }
    for (int i = 0; i < NA; ++i) { mbar_init(&B.acc_full[i], 1); mbar_init(&B.acc_empty[i], 4); }
    fence_barrier_init();
  }
  if (warp == kLocMmaWarp) tmem_alloc<512>(&tmem_slot);
  if (warp == 0 && lane < p.n_mod) {                 // descriptors never depend on the previous kernel
    tma_prefetch_desc(&p.mod[lane].tm_x);
    tma_prefetch_desc(&p.mod[lane].tm_y);
    tma_prefetch_desc(p.mod[lane].tm_in3);
    tma_prefetch_desc(p.mod[lane].tm_out);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (p.meta_ready) loc_build_map(p, off, pre, B.total, warp_sums);
  griddep_wait();
  if (threadIdx.x == 0) griddep_launch_dependents();
  if (!p.meta_ready) loc_build_map(p, off, pre, B.total, warp_sums);
  const int total = *B.total;
  const int G = gridDim.x;
  if (threadIdx.x == 0) CTS_STAMP(1);

  if (warp < kLocXWarps) {
    // ---------------------------------------------------------------- x rows + in_basis
    // every stage's kLocKB K blocks are issued by the kLocXWarps warps in parallel (warp w: K block w)
    // -- one warp issuing a whole stage's gathers (~70 cycles each) took ~0.9 us per stage
    static_assert(kLocKB == kLocXWarps, "one K block of every shrink stage per x producer warp");
    int js = 0;
    for (int u = blockIdx.x; u < total; u += G) {
      const Piece P = loc_piece(p, off, pre, u);
      const LocMod& m = p.mod[P.g];
      const int nst = m.d_in / (64 * kLocKB);
      const int ngroups = (P.L + 3) >> 2;
      const uint32_t bytes = static_cast<uint32_t>(kLocKB * (ngroups * 512 + kLocRP * 128));
      const int4 r4 = 4 * lane < P.L ? loc_rows4(m.perm, P, lane) : make_int4(0, 0, 0, 0);
      for (int st = 0; st < nst; ++st, ++js) {
        const int stage = js % S;
        // every warp passes every stage: none can run two rounds ahead of the MMA (a round's full
        // barrier needs all warps' bytes), so the parity wait cannot alias
        mbar_wait(&B.empty_s[stage], ((js / S) & 1) ^ 1);
        uint8_t* sA = smem + L.sring + stage * L.s_bytes;
        uint8_t* sB = sA + kLocKB * L.a_bytes;
        if (warp == 0 && lane == 0) {
          if (js == 0) CTS_STAMP(2);
          CTS_JOB_STAMP(1, js);
          mbar_arrive_expect_tx(&B.full_s[stage], bytes);
          tma_load_3d(sB, m.tm_in3, &B.full_s[stage], 0, P.c * kLocRP, st * kLocKB);
        }
        if (4 * lane < P.L)
          tma_gather4(sA + warp * L.a_bytes + lane * 512, &m.tm_x, &B.full_s[stage], (st * kLocKB + warp) * 64, r4.x,
                      r4.y, r4.z, r4.w);
        __syncwarp();
      }
    }
    if (threadIdx.x == 0) CTS_STAMP(3);
  } else if (warp < kLocMmaWarp) {
    // ---------------------------------------------------------------- y rows + out_basis blocks
    const int yw = warp - kLocXWarps;
    int je = 0;
    for (int u = blockIdx.x; u < total; u += G) {
      const Piece P = loc_piece(p, off, pre, u);
      const LocMod& m = p.mod[P.g];
      const int nj = (m.d_out + kLocBN - 1) / kLocBN;
      const int ngroups = (P.L + 3) >> 2;
      const uint32_t bytes = static_cast<uint32_t>(kLocBN * kLocRP * 2 + ngroups * 4 * kLocBN * 2);
      const int4 r4 = 4 * lane < P.L ? loc_rows4(m.perm, P, lane) : make_int4(0, 0, 0, 0);
      for (int j = 0; j < nj; ++j, ++je) {
        if ((je % E) % kLocYWarps != yw) continue;   // stage -> warp fixed (see above)
        const int stage = je % E;
        mbar_wait(&B.empty_e[stage], ((je / E) & 1) ^ 1);
        if (lane == 0) CTS_JOB_STAMP(0, je);
        uint8_t* sO = smem + L.ering + stage * L.e_bytes;
        uint8_t* sY = sO + kLocBN * kLocRP * 2;
        if (lane == 0) {
          if (je == 0) CTS_STAMP(6);
          mbar_arrive_expect_tx(&B.full_e[stage], bytes);
          tma_load_2d(sO, m.tm_out, &B.full_e[stage], 0, P.c * m.d_out + j * kLocBN);
        }
        __syncwarp();
        if (4 * lane < P.L)
          tma_gather4(sY + lane * 4 * kLocBN * 2, &m.tm_y, &B.full_e[stage], j * kLocBN, r4.x, r4.y, r4.z, r4.w);
      }
    }
    if (threadIdx.x == 32 * kLocXWarps) CTS_STAMP(12);
  } else if (warp == kLocMmaWarp) {
    // ---------------------------------------------------------------- MMA issue: S(0) S(1) E(0) S(2) E(1) ...
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, kLocRP);
    int js = 0, je = 0, pc = 0;
    Piece prev{0, 0, 0, 0};
    bool have_prev = false;
    for (int u = blockIdx.x;; u += G) {
      const bool have = u < total;
      Piece P{0, 0, 0, 0};
      if (have) {
        P = loc_piece(p, off, pre, u);
        const LocMod& m = p.mod[P.g];
        const int buf = pc & 1;
        mbar_wait(&B.acc_s_empty[buf], ((pc >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * kLocRP;
        const int nst = m.d_in / (64 * kLocKB);
        for (int st = 0; st < nst; ++st, ++js) {
          const int stage = js % S;
          mbar_wait(&B.full_s[stage], (js / S) & 1);
          tc_fence_after();
          if (lane == 0) {
            CTS_JOB_STAMP(7, js);
            const uint32_t a0 = smem_u32(smem + L.sring + stage * L.s_bytes);
            const uint32_t b0 = a0 + kLocKB * L.a_bytes;
#pragma unroll
            for (int kk = 0; kk < kLocKB; ++kk)
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k)
                umma_bf16(acc, umma_desc_kmajor(a0 + kk * L.a_bytes + k * 32, 128),
                          umma_desc_kmajor(b0 + kk * kLocRP * 128 + k * 32, 128), idesc_s,
                          (st | kk | k) != 0 ? 1u : 0u);
            umma_commit(&B.empty_s[stage]);
          }
          __syncwarp();
        }
        if (lane == 0) {
          umma_commit(&B.acc_s_full[buf]);
          if (pc == 0) CTS_STAMP(4);
        }
        __syncwarp();
      }
      if (have_prev) {
        const LocMod& m = p.mod[prev.g];
        const int pbuf = (pc - 1) & 1;
        mbar_wait(&B.t_full[pbuf], ((pc - 1) >> 1) & 1);
        tc_fence_after();
        if (pc == 1 && lane == 0) CTS_STAMP(7);
        const int npad = max(16, (prev.L + 15) & ~15);
        const uint32_t idesc_e = umma_idesc_bf16(128, npad);
        const uint32_t thi = smem_u32(smem + L.tt + pbuf * 2 * L.t_bytes), tlo = thi + L.t_bytes;
        const int nj = (m.d_out + kLocBN - 1) / kLocBN;
        for (int j = 0; j < nj; ++j, ++je) {
          const int slot = je % NA, stage = je % E;
          mbar_wait(&B.acc_empty[slot], ((je / NA) & 1) ^ 1);
          if (lane == 0) CTS_JOB_STAMP(2, je);
          mbar_wait(&B.full_e[stage], (je / E) & 1);
          tc_fence_after();
          if (lane == 0) {
            CTS_JOB_STAMP(3, je);
            const uint32_t acc = tmem + kLocE0 + slot * 2 * p.npad;
            const uint32_t ob = smem_u32(smem + L.ering + stage * L.e_bytes);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t a = ob + h * 128 * kLocRP * 2;
#pragma unroll
              for (int k = 0; k < kLocRP / 16; ++k)
                umma_bf16(acc + h * p.npad, umma_desc_kmajor(a + k * 32, kLocRP * 2),
                          umma_desc_kmajor(thi + k * 32, kLocRP * 2), idesc_e, k != 0);
#pragma unroll
              for (int k = 0; k < kLocRP / 16; ++k)
                umma_bf16(acc + h * p.npad, umma_desc_kmajor(a + k * 32, kLocRP * 2),
                          umma_desc_kmajor(tlo + k * 32, kLocRP * 2), idesc_e, 1u);
            }
            umma_commit(&B.empty_e[stage]);
            umma_commit(&B.acc_full[slot]);
          }
          __syncwarp();
        }
        if (lane == 0) umma_commit(&B.t_empty[pbuf]);
        __syncwarp();
      }
      if (!have) break;
      prev = P;
      have_prev = true;
      ++pc;
    }
  } else if (warp < kLocBWarp0) {
    // ---------------------------------------------------------------- set A: t = scale Sigma_i s
    const int q = warp & 3;                          // TMEM lane quarter of this warp
    const int row = 32 * q + lane;
    int pc = 0;
    for (int u = blockIdx.x; u < total; u += G, ++pc) {
      const Piece P = loc_piece(p, off, pre, u);
      const LocMod& m = p.mod[P.g];
      const int buf = pc & 1;
      const bool active = 32 * q < P.L;              // warp-uniform
      const bool valid = row < P.L;
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * q) << 16);
      if (active) {                                  // this row's Sigma_i -> TMEM (128 columns)
        const int adapter = valid ? m.sadapter[P.lo + row] : 0;
        const uint4* sg = reinterpret_cast<const uint4*>(m.sigma + static_cast<size_t>(adapter) * kLocRP * kLocRP);
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          uint32_t w[64];
#pragma unroll
          for (int v = 0; v < 16; v += 2) {
            uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0;
            if (valid) ld_global_nc_v8(sg + 16 * h + v, q0, q1);
            w[4 * v] = q0.x; w[4 * v + 1] = q0.y; w[4 * v + 2] = q0.z; w[4 * v + 3] = q0.w;
            w[4 * v + 4] = q1.x; w[4 * v + 5] = q1.y; w[4 * v + 6] = q1.z; w[4 * v + 7] = q1.w;
          }
          tmem_st32(lane_base + kLocSigCol + 64 * h, w);
          tmem_st32(lane_base + kLocSigCol + 64 * h + 32, w + 32);
        }
        tmem_st_wait();
      }
      mbar_wait(&B.acc_s_full[buf], (pc >> 1) & 1);
      tc_fence_after();
      float s[kLocRP];
      if (active) {
        tmem_ld16(lane_base + buf * kLocRP, s);
        tmem_ld_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&B.acc_s_empty[buf]);
      mbar_wait(&B.t_empty[buf], ((pc >> 1) & 1) ^ 1);
      if (active) {
        float t[kLocRP];
#pragma unroll 1
        for (int h = 0; h < 4; ++h) {                // Sigma rows 4h .. 4h+3 (16 bf16 each)
          float w[32];
          tmem_ld32(lane_base + kLocSigCol + 32 * h, w);
          tmem_ld_wait();
#pragma unroll
          for (int oo = 0; oo < 4; ++oo) {
            float acc = 0.f;
#pragma unroll
            for (int e = 0; e < kLocRP / 2; ++e) {
              const uint32_t uu = __float_as_uint(w[oo * (kLocRP / 2) + e]);
              const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uu));
              acc = fmaf(f.x, s[2 * e], acc);
              acc = fmaf(f.y, s[2 * e + 1], acc);
            }
            t[4 * h + oo] = acc * m.scale;
          }
        }
        if (valid) {
          // t = hi + lo (two bf16, ~2^-16 relative), rows of 32 bytes in the 32B-swizzled K-major
          // layout the UMMA descriptor expects: 16-byte chunk c of row r at 32 r + 16 (c ^ (r>>2 & 1))
          uint8_t* thi = smem + L.tt + buf * 2 * L.t_bytes;
          uint8_t* tlo = thi + L.t_bytes;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint4 hi, lo;
            __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&hi);
            __nv_bfloat162* ll = reinterpret_cast<__nv_bfloat162*>(&lo);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a = t[8 * c + 2 * e], b = t[8 * c + 2 * e + 1];
              const __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
              const float2 hf = __bfloat1622float2(h2);
              hh[e] = h2;
              ll[e] = __floats2bfloat162_rn(a - hf.x, b - hf.y);
            }
            const int phys = 32 * row + 16 * (c ^ ((row >> 2) & 1));
            *reinterpret_cast<uint4*>(thi + phys) = hi;
            *reinterpret_cast<uint4*>(tlo + phys) = lo;
          }
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (warp == kLocAWarp0 && lane == 0) {
        mbar_arrive(&B.t_full[buf]);
        if (pc == 0) CTS_STAMP(5);
      }
    }
  } else {
    // ---------------------------------------------------------------- set B: y = bf16(y + dy)
    const int q = warp & 3;
    int* tok = reinterpret_cast<int*>(smem + L.tok) + (warp - kLocBWarp0) * kLocMaxRows;
    int je = 0;
    for (int u = blockIdx.x; u < total; u += G) {
      const Piece P = loc_piece(p, off, pre, u);
      const LocMod& m = p.mod[P.g];
      for (int j = lane; j < P.L; j += 32) tok[j] = m.perm[P.lo + j];
      __syncwarp();
      const int nj = (m.d_out + kLocBN - 1) / kLocBN;
      for (int jb = 0; jb < nj; ++jb, ++je) {
        const int slot = je % NA, stage = je % E;
        mbar_wait(&B.acc_full[slot], (je / NA) & 1);
        if (lane == 0 && q == 0) CTS_JOB_STAMP(4, je);
        mbar_wait(&B.full_e[stage], (je / E) & 1);
        tc_fence_after();
        if (lane == 0 && q == 0) CTS_JOB_STAMP(5, je);
        // y_new = bf16(y_base + dy) written back into the staged rows (thread = column: conflict-free
        // 2-byte smem accesses), then moved out by TMA scatter4 (4 rows x 512 B per op): 2-byte
        // per-lane global stores capped set B at ~1.3 us per 256-column job (profiles/r02 trace).
        // Rows L .. 4*ngroups-1 repeat row L-1 (the gather duplicated its token), so a scatter4 group
        // writes identical bytes for its duplicate rows.
        __nv_bfloat16* yrow = reinterpret_cast<__nv_bfloat16*>(smem + L.ering + stage * L.e_bytes + kLocBN * kLocRP * 2);
        const int ngroups = (P.L + 3) >> 2;
#pragma unroll 1
        for (int h = 0; h < (CTS_LOC_NO_YMATH ? 0 : 2); ++h) {
          const int col_in = h * 128 + 32 * q + lane;
          const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * q) << 16) + kLocE0 + slot * 2 * p.npad + h * p.npad;
#pragma unroll 1
          for (int j0 = 0; j0 < 4 * ngroups; j0 += 16) {
            float v[16];
            tmem_ld16(taddr + j0, v);
            __nv_bfloat16 yb[16];
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) yb[jj] = ld_shared_bf16(yrow + min(j0 + jj, P.L - 1) * kLocBN + col_in);
            tmem_ld_wait();
            __nv_bfloat16 o_last = __float2bfloat16_rn(0.f);
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const int j = j0 + jj;
              if (j < 4 * ngroups) {
                // duplicate rows (j >= L) repeat row L-1, which comes earlier in this same chunk
                const __nv_bfloat16 o = j < P.L ? __float2bfloat16_rn(__bfloat162float(yb[jj]) + v[jj]) : o_last;
                o_last = o;
                st_shared_bf16(yrow + j * kLocBN + col_in, o);
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&B.acc_empty[slot]);          // accumulator read: MMA may reuse it
        fence_proxy_async_smem();
        named_bar_sync(2, 128);                                 // all four warps' columns written
        if (!CTS_LOC_NO_SCATTER && lane < ngroups && (lane & 3) == q) {   // warp q scatters groups g = q mod 4
          const int4 r4 = make_int4(tok[min(4 * lane, P.L - 1)], tok[min(4 * lane + 1, P.L - 1)],
                                    tok[min(4 * lane + 2, P.L - 1)], tok[min(4 * lane + 3, P.L - 1)]);
          tma_scatter4(&m.tm_y, yrow + 4 * lane * kLocBN, jb * kLocBN, r4.x, r4.y, r4.z, r4.w);
        }
        bulk_commit();
        bulk_wait_read<0>();                                    // this warp's scatters have read the stage
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&B.empty_e[stage]);
          if (je == 0 && warp == kLocBWarp0) CTS_STAMP(8);
          if (q == 0) CTS_JOB_STAMP(6, je);
        }
      }
    }
    bulk_wait0();                                               // global writes complete before exit
    if (threadIdx.x == 32 * kLocBWarp0) CTS_STAMP(10);
  }
  __syncthreads();
  if (threadIdx.x == 0) CTS_STAMP(11);
  if (warp == kLocMmaWarp) tmem_dealloc<512>(tmem);
}

}  // namespace cts
