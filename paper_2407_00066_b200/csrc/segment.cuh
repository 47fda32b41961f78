// segment.cuh -- token segmentation by cluster, one CTA per distinct map.
//
// For a module whose adapter->cluster map is cmap:  tc[t] = cmap[token_adapter[t]] (or -1),
// perm = bound tokens stably sorted by (cluster, token index), offsets = exclusive prefix sum of
// per-cluster counts, tiles = (cluster, start, len <= 128).  Grouping tokens that share weights
// is SGMV's idea; grouping by cluster makes App D's broadcast products real GEMMs.
//
// Algorithm (deterministic, no atomics on the data path):
//   A. warp w owns the contiguous token range [w*seg, (w+1)*seg); per 32-token chunk,
//      __match_any_sync groups lanes with equal keys; the group's highest lane adds the group
//      size (popc) to the warp-private histogram hist[w][c].
//   B. per cluster c, exclusive scan over warps (cluster-major, warp-minor) plus a block scan over
//      clusters of the totals gives every (warp, cluster) its first output slot.
//   C. each warp re-walks its range: a token's slot = base[w][key] + popc(peers & lanes_below).
// Stable by construction: warps own increasing token ranges, chunks are walked in order, and the
// within-chunk rank counts lower lanes (= lower token indices) only.
//   D. tiles: each cluster's group is cut into 128-token tiles in order; the GEMM kernels see SLOTS
//      of 128 rows: a whole tile (full, or a remainder of 65..127 tokens) or two remainders of
//      <= 64 tokens, one per 64-row half ("packing": at decode ~41 tokens per cluster, so a 128-row
//      MMA tile is otherwise 2/3 empty).  Halves are paired in cluster order.  Every logical tile is
//      still one contiguous perm range (c, start, len), as in oracle.segment_ref.
#pragma once
#include <cstdint>
#include "sm100.cuh"

namespace cts {

constexpr int kTileM = 128;          // token rows per GEMM tile (tcgen05 M)
constexpr int kSegThreads = 1024;
constexpr int kSegWarps = kSegThreads / 32;

struct SegArgs {
  const int32_t* token_adapter;  // [T] caller buffer
  int32_t* tok_adapter_copy;     // [T_max] plan copy (for the Sigma lookup)
  const int32_t* maps;           // [n_maps][N]
  int32_t* perm;                 // [n_maps][T_max]
  int32_t* offsets;              // [n_maps][C+1]
  int4* tiles;                   // [n_maps][max_tiles][2] slots: (c, start, len, 0) per 64-row half;
                                 //   second half len = 0 for a whole tile; both 0 past n_tiles
  int32_t* n_tiles;              // [n_maps] number of slots
  int32_t* tile_rows;            // [n_maps][max_tiles*128] token of each tile row (dup of last past len)
  int32_t* tile_adapters;        // [n_maps][max_tiles*128] adapter of that token
  int32_t* err;                  // [2] code, first bad token
  int32_t* unbound_rows;         // [T_max + 128] tokens with id -1 in order, padded to a multiple of 128
  int32_t* n_unbound;            // [1] (0 if the batch is invalid)
  int n_maps;                    // CTAs 0..n_maps-1 segment one map each; CTA n_maps lists unbound tokens
  int T, T_max, N, C, max_tiles;
  int pack;                      // 1: pair <=64-token remainders into shared slots
};

__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_sums, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int s = warp_sums[lane];
    int si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int n = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += n;
    }
    warp_sums[lane] = si - s;       // exclusive per-warp base
    if (lane == 31) warp_sums[32] = si;
  }
  __syncthreads();
  const int res = warp_sums[warp] + incl - v;
  total = warp_sums[32];
  __syncthreads();
  return res;
}

// CTA n_maps: the stable list of UNBOUND tokens (id -1), for the fused projection (proj_fused.cuh),
// which must still compute y = W0 x for them.  Chunks of 1024 tokens, block scan per chunk; the
// list is padded with its last token to a multiple of 128 rows.
__device__ void unbound_list(const SegArgs& a, int* warp_sums) {
  __shared__ int s_bad_u;
  if (threadIdx.x == 0) s_bad_u = 0;
  __syncthreads();
  int base = 0;
  for (int t0 = 0; t0 < a.T; t0 += kSegThreads) {
    const int t = t0 + threadIdx.x;
    const int id = t < a.T ? a.token_adapter[t] : 0;
    if (t < a.T && (id < -1 || id >= a.N)) s_bad_u = 1;
    const int f = (t < a.T && id == -1) ? 1 : 0;
    int total;
    const int pos = block_exclusive_scan(f, warp_sums, total);
    if (f) a.unbound_rows[base + pos] = t;
    base += total;
  }
  __syncthreads();
  const int n = s_bad_u ? 0 : base;
  const int padded = (n + kTileM - 1) / kTileM * kTileM;
  for (int i = n + threadIdx.x; i < padded; i += kSegThreads) a.unbound_rows[i] = a.unbound_rows[n - 1];
  if (threadIdx.x == 0) *a.n_unbound = n;
}

__global__ void __launch_bounds__(kSegThreads, 1) segment_kernel(SegArgs a) {
  extern __shared__ int seg_smem[];
  int* hist = seg_smem;                            // [kSegWarps][C]
  int* cnt = hist + kSegWarps * a.C;               // [C]
  int* tile_base = cnt + a.C;                      // [C] first whole slot of the cluster
  int* half_base = tile_base + a.C;                // [C] index of the cluster's half remainder
  __shared__ int warp_sums[33];
  __shared__ int s_bad;

  const int map_id = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int* cmap = a.maps + static_cast<size_t>(map_id) * a.N;
  int32_t* perm = a.perm + static_cast<size_t>(map_id) * a.T_max;
  int32_t* offsets = a.offsets + static_cast<size_t>(map_id) * (a.C + 1);
  int4* tiles = a.tiles + static_cast<size_t>(map_id) * a.max_tiles * 2;

  griddep_wait();                                   // previous step's applies still read the plan
  griddep_launch_dependents();
  if (map_id == a.n_maps) {
    unbound_list(a, warp_sums);
    return;
  }
  if (threadIdx.x == 0) s_bad = 0x7fffffff;
  for (int i = threadIdx.x; i < kSegWarps * a.C; i += kSegThreads) hist[i] = 0;
  __syncthreads();

  // Validation (+ plan copy of the ids, done once by CTA 0).
  for (int t = threadIdx.x; t < a.T; t += kSegThreads) {
    const int id = a.token_adapter[t];
    if (id < -1 || id >= a.N) atomicMin(&s_bad, t);
    if (map_id == 0) a.tok_adapter_copy[t] = id;
  }
  __syncthreads();
  if (s_bad != 0x7fffffff) {                       // poison: no tiles / no bound rows for any module
    for (int i = threadIdx.x; i < 2 * a.max_tiles; i += kSegThreads) tiles[i] = make_int4(0, 0, 0, 0);
    for (int i = threadIdx.x; i <= a.C; i += kSegThreads) offsets[i] = 0;
    if (threadIdx.x == 0) {
      a.n_tiles[map_id] = 0;
      if (map_id == 0) {
        a.err[0] = 3;  // CTS_ERR_INDEX_OUT_OF_RANGE
        a.err[1] = s_bad;
      }
    }
    return;
  }
  if (map_id == 0 && threadIdx.x == 0) {
    a.err[0] = 0;
    a.err[1] = -1;
  }

  // A. per-warp histograms over contiguous token ranges.
  const int seg = ((a.T + kSegWarps - 1) / kSegWarps + 31) & ~31;
  const int t_lo = warp * seg, t_hi = min(a.T, t_lo + seg);
  int* my_hist = hist + warp * a.C;
  for (int t0 = t_lo; t0 < t_hi; t0 += 32) {
    const int t = t0 + lane;
    int key = -1;
    if (t < t_hi) {
      const int id = a.token_adapter[t];
      key = id >= 0 ? cmap[id] : -1;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (key >= 0 && lane == 31 - __clz(peers)) my_hist[key] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();

  // B. (cluster-major, warp-minor) exclusive scan.
  for (int c0 = 0; c0 < a.C; c0 += kSegThreads) {
    const int c = c0 + threadIdx.x;
    int run = 0;
    if (c < a.C) {
      for (int w = 0; w < kSegWarps; ++w) {
        const int h = hist[w * a.C + c];
        hist[w * a.C + c] = run;
        run += h;
      }
      cnt[c] = run;
    }
  }
  __syncthreads();
  int carry = 0, tcarry = 0, hcarry = 0;
  for (int c0 = 0; c0 < a.C; c0 += kSegThreads) {
    const int c = c0 + threadIdx.x;
    const int v = c < a.C ? cnt[c] : 0;
    const int rem = v % kTileM;
    const int lim = a.pack ? kTileM / 2 : 0;
    const int whole = v / kTileM + (rem > lim ? 1 : 0);           // slots owned outright
    const int half = (rem > 0 && rem <= lim) ? 1 : 0;             // a remainder that shares a slot
    int tot, wtot, htot;
    const int ex = block_exclusive_scan(v, warp_sums, tot);
    const int wex = block_exclusive_scan(whole, warp_sums, wtot);
    const int hex = block_exclusive_scan(half, warp_sums, htot);
    if (c < a.C) {
      offsets[c] = carry + ex;
      tile_base[c] = tcarry + wex;
      half_base[c] = half ? hcarry + hex : -1;
      cnt[c] = v;
    }
    carry += tot;
    tcarry += wtot;
    hcarry += htot;
  }
  const int n_whole = tcarry, n_half = hcarry;
  const int n_slots = n_whole + (n_half + 1) / 2;
  if (threadIdx.x == 0) {
    offsets[a.C] = carry;
    a.n_tiles[map_id] = n_slots;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kSegWarps * a.C; i += kSegThreads) hist[i] += offsets[i % a.C];
  __syncthreads();

  // C. stable scatter.
  for (int t0 = t_lo; t0 < t_hi; t0 += 32) {
    const int t = t0 + lane;
    int key = -1;
    if (t < t_hi) {
      const int id = a.token_adapter[t];
      key = id >= 0 ? cmap[id] : -1;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (key >= 0) {
      const int rank = __popc(peers & ((1u << lane) - 1u));
      perm[my_hist[key] + rank] = t;
    }
    __syncwarp();
    if (key >= 0 && lane == 31 - __clz(peers)) my_hist[key] += __popc(peers);
    __syncwarp();
  }

  // D. slots (empty descriptors past n_slots: kernels map work statically over the bound).
  for (int c = threadIdx.x; c < a.C; c += kSegThreads) {
    const int n = cnt[c], off = offsets[c], full = n / kTileM, rem = n % kTileM;
    int slot = tile_base[c];
    for (int j = 0; j < full; ++j, ++slot) {
      tiles[2 * slot] = make_int4(c, off + j * kTileM, kTileM, 0);
      tiles[2 * slot + 1] = make_int4(0, 0, 0, 0);
    }
    if (rem > (a.pack ? kTileM / 2 : 0)) {
      tiles[2 * slot] = make_int4(c, off + full * kTileM, rem, 0);
      tiles[2 * slot + 1] = make_int4(0, 0, 0, 0);
    } else if (rem > 0) {
      const int k = half_base[c];
      const int hs = n_whole + k / 2;
      tiles[2 * hs + (k & 1)] = make_int4(c, off + full * kTileM, rem, 0);
      if ((k & 1) == 0 && k == n_half - 1) tiles[2 * hs + 1] = make_int4(0, 0, 0, 0);
    }
  }
  for (int i = 2 * n_slots + threadIdx.x; i < 2 * a.max_tiles; i += kSegThreads) tiles[i] = make_int4(0, 0, 0, 0);
  __syncthreads();                                 // perm and slots complete (block scope)

  // E. per-slot row lists: token and adapter of every slot row (rows 64..127 belong to the second
  //    half when the slot is shared; rows past a tile's length repeat its last token), so the GEMM
  //    kernels fetch a slot's rows with one dependent load.
  int32_t* trows = a.tile_rows + static_cast<size_t>(map_id) * a.max_tiles * kTileM;
  int32_t* tads = a.tile_adapters + static_cast<size_t>(map_id) * a.max_tiles * kTileM;
  for (int i = threadIdx.x; i < n_slots * kTileM; i += kSegThreads) {
    const int slot = i / kTileM, r = i % kTileM;
    const int4 s1 = tiles[2 * slot + 1];
    const bool second = s1.z > 0 && r >= kTileM / 2;
    const int4 tl = second ? s1 : tiles[2 * slot];
    const int local = second ? r - kTileM / 2 : r;
    const int tok = perm[tl.y + min(local, tl.z - 1)];
    trows[i] = tok;
    tads[i] = a.token_adapter[tok];
  }
}

}  // namespace cts

namespace cts {

// ------------------------------------------------------------------ cluster-affinity routing
// SURVEY 8(f) NEXT 4 ("clustering offers opportunities for efficient scheduling"): tokens
// go to the rank that owns their cluster.  route_kernel: one 1024-thread CTA; dest[t] =
// owner[adapter[t]] (unbound tokens stay on `self`); perm = token indices stably partitioned by
// destination rank, counts[r] = tokens for rank r.  Per destination a block scan per 1024-token
// chunk (world <= 64): deterministic, no atomics.
struct RouteArgs {
  const int32_t* token_adapter;  // [T]
  const int32_t* owner;          // [N] adapter -> rank
  int32_t* perm;                 // [T]
  int32_t* counts;               // [world]
  int T, N, world, self;
};

__global__ void __launch_bounds__(kSegThreads, 1) route_kernel(RouteArgs a) {
  __shared__ int warp_sums[33];
  int base = 0;
  for (int r = 0; r < a.world; ++r) {
    const int start = base;
    for (int t0 = 0; t0 < a.T; t0 += kSegThreads) {
      const int t = t0 + threadIdx.x;
      int dst = -1;
      if (t < a.T) {
        const int id = a.token_adapter[t];
        dst = (id >= 0 && id < a.N) ? a.owner[id] : a.self;
        if (dst < 0 || dst >= a.world) dst = a.self;   // an out-of-range owner keeps the token local
      }
      const int f = dst == r ? 1 : 0;
      int total;
      const int pos = block_exclusive_scan(f, warp_sums, total);
      if (f) a.perm[base + pos] = t;
      base += total;
    }
    if (threadIdx.x == 0) a.counts[r] = base - start;
  }
}

// dst[k] = src[idx[k]] (gather) or dst[idx[k]] = src[k] (scatter) for rows of row_bytes bytes:
// 16-byte chunks when rows and strides are 16-byte multiples (bf16 activations), else 4-byte
// chunks (int32 token ids)
struct RowsArgs {
  const uint8_t* src;
  uint8_t* dst;
  const int32_t* idx;
  int64_t ld_src, ld_dst;        // bytes
  int n, row_bytes, scatter;
};

template <typename V>
__global__ void __launch_bounds__(256) rows_move_kernel(RowsArgs a) {
  const int chunks = a.row_bytes / static_cast<int>(sizeof(V));
  const int64_t total = static_cast<int64_t>(a.n) * chunks;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i / chunks), c = static_cast<int>(i % chunks);
    const int64_t sr = a.scatter ? k : a.idx[k], dr = a.scatter ? a.idx[k] : k;
    *reinterpret_cast<V*>(a.dst + dr * a.ld_dst + c * sizeof(V)) =
        *reinterpret_cast<const V*>(a.src + sr * a.ld_src + c * sizeof(V));
  }
}

}  // namespace cts
