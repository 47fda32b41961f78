// cts.cu -- host side of libcts.so: bank relayout, plans, segmentation and grouped apply launches.
// See include/cts.h for the contract of every entry point.
#include <cuda.h>
#include <cuda_runtime.h>

#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/cts.h"
#include "apply_fused.cuh"
#include "expand.cuh"
#include "proj_fused.cuh"
#include "jd_eigen.cuh"
#include "jd_tc.cuh"
#include "jd_gram.cuh"
#include "segment.cuh"
#include "shrink_sigma.cuh"

using namespace cts;

namespace {

// ------------------------------------------------------------------ driver entry point (TMA maps)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

CUtensorMapSwizzle swizzle_for(int row_bytes) {
  switch (row_bytes) {
    case 32: return CU_TENSOR_MAP_SWIZZLE_32B;
    case 64: return CU_TENSOR_MAP_SWIZZLE_64B;
    default: return CU_TENSOR_MAP_SWIZZLE_128B;
  }
}

// 2-D bf16 tensor map: `inner` contiguous elements per row, `outer` rows, `row_stride` bytes.
bool make_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride,
               uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 2-D map (GPU compression, jd_tc.cuh): rows of `inner` floats, 128B swizzle
bool make_tmap_f32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                   uint32_t box_outer) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D tiled map (used for the fused projection's masked t halves: out-of-bounds boxes fill zeros)
bool make_tmap3(CUtensorMap* m, const void* ptr, const uint64_t dims_in[3], const uint64_t strides_in[2],
                const uint32_t box_in[3], CUtensorMapSwizzle sw) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {dims_in[0], dims_in[1], dims_in[2]};
  cuuint64_t strides[2] = {strides_in[0], strides_in[1]};
  cuuint32_t box[3] = {box_in[0], box_in[1], box_in[2]};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int pad_rank(int r) { return r <= 16 ? 16 : (r <= 32 ? 32 : 64); }

int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      (void)cudaGetLastError();
      v = 148;
    }
    return v;
  }();
  return n;
}

// ------------------------------------------------------------------ relayout kernels
// in_basis [C][d_in][r] (paper V_c, row-major) -> [C][rp][d_in], zero rows for k >= r.
__global__ void relayout_in_kernel(const __nv_bfloat16* src, __nv_bfloat16* dst, int C, int d_in, int r, int rp) {
  const size_t n = static_cast<size_t>(C) * rp * d_in;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i % d_in);
    const int k = static_cast<int>((i / d_in) % rp);
    const int c = static_cast<int>(i / (size_t(d_in) * rp));
    dst[i] = k < r ? src[(size_t(c) * d_in + j) * r + k] : __float2bfloat16_rn(0.f);
  }
}
// out_basis rows [rows][r] -> [rows][rp]
__global__ void relayout_pad_kernel(const __nv_bfloat16* src, __nv_bfloat16* dst, size_t rows, int r, int rp) {
  const size_t n = rows * rp;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % rp);
    dst[i] = k < r ? src[(i / rp) * r + k] : __float2bfloat16_rn(0.f);
  }
}
// cts_bank_write_clusters: n clusters' bases, sources [n][d][r], into the bank slices of clusters
// cl.c[q] ([C][rp][d_in] for in_basis, [C][d_out][rp] for out_basis)
constexpr int kMaxWriteClusters = 64;
struct ClusterList {
  int32_t c[kMaxWriteClusters];
};
__global__ void write_in_kernel(const __nv_bfloat16* src, __nv_bfloat16* dst, ClusterList cl, int n, int d_in, int r,
                                int rp) {
  const size_t per = size_t(rp) * d_in;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n * per; i += size_t(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(i / per);
    const int k = static_cast<int>((i % per) / d_in), j = static_cast<int>(i % d_in);
    dst[size_t(cl.c[q]) * per + size_t(k) * d_in + j] =
        k < r ? src[(size_t(q) * d_in + j) * r + k] : __float2bfloat16_rn(0.f);
  }
}
__global__ void write_out_kernel(const __nv_bfloat16* src, __nv_bfloat16* dst, ClusterList cl, int n, int d_out, int r,
                                 int rp) {
  const size_t per = size_t(d_out) * rp;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n * per; i += size_t(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(i / per);
    const int row = static_cast<int>((i % per) / rp), k = static_cast<int>(i % rp);
    dst[size_t(cl.c[q]) * per + size_t(row) * rp + k] =
        k < r ? src[(size_t(q) * d_out + row) * r + k] : __float2bfloat16_rn(0.f);
  }
}
// Sigma [N][r][r] -> [N][rp][rp]
__global__ void relayout_sigma_kernel(const __nv_bfloat16* src, __nv_bfloat16* dst, int N, int r, int rp) {
  const size_t n = static_cast<size_t>(N) * rp * rp;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % rp);
    const int o = static_cast<int>((i / rp) % rp);
    const int a = static_cast<int>(i / (size_t(rp) * rp));
    dst[i] = (k < r && o < r) ? src[(size_t(a) * r + o) * r + k] : __float2bfloat16_rn(0.f);
  }
}

struct Module {
  int d_in, d_out, map_id;
  __nv_bfloat16* in_t;    // [C][rp][d_in]
  __nv_bfloat16* out;     // [C][d_out][rp]
  __nv_bfloat16* sigma;   // [N][rp][rp], or [N][rp] (diagonal kind)
};

}  // namespace

struct cts_bank_s {
  int n_modules, N, C, r, rp;
  int sigma_diag;         // CTS_SIGMA_DIAG: Sigma_i stored as its diagonal (JD-Diag, Eq. 3)
  std::vector<Module> mods;
  int n_maps;
  int32_t* maps;          // [n_maps][N]
  CUtensorMap* d_tm_in;   // [n_modules] device copies (TMA descriptors in global memory)
  CUtensorMap* d_tm_out;  // [n_modules]
  void* arena;
  size_t bytes;
};

struct cts_plan_s {
  cts_bank_t bank;
  int T_max, max_tiles;
  int T;                  // tokens of the last segmented batch (host view)
  void* arena;
  int32_t* tok_adapter;   // [T_max]
  int32_t* perm;          // [n_maps][T_max]
  int32_t* offsets;       // [n_maps][C+1]
  int4* tiles;            // [n_maps][max_tiles]
  int32_t* n_tiles;       // [n_maps]
  int32_t* tile_rows;     // [n_maps][max_tiles*128]
  int32_t* tile_adapters; // [n_maps][max_tiles*128]
  int32_t* err;           // [2]
  int32_t* unbound_rows;  // [T_max + 128] tokens with id -1 (fused projection)
  int32_t* n_unbound;     // [1]
  __nv_bfloat16* tbuf;    // [n_modules][max_tiles*128][2*rp]  rank-r intermediate (t hi | t lo)
  CUtensorMap* d_tm_t;    // [n_modules] device copies
  float* ws;              // [kMaxGroup][ws_cap rows][rp]  split-K partials
  size_t ws_cap_rows;
  int32_t* counters;      // [kMaxGroup][max_tiles]
  int32_t* ready;         // [kMaxGroup][max_tiles] per-slot "t ready" flags (fused kernel)
  int32_t* exit_count;    // fused kernel: CTAs exited (last one clears the flags)
  float* tp_parts;        // [kMaxGroup][T_max][rp] fp32 TP partials (cts_apply_tp)
  int launches_since_segment;  // host view, for meta_ready (see next_meta_ready)
};

namespace {

#define CTS_CUDA(call)                                  \
  do {                                                  \
    if ((call) != cudaSuccess) {                        \
      (void)cudaGetLastError();                         \
      return CTS_ERR_CUDA;                              \
    }                                                   \
  } while (0)

template <typename T>
bool aligned16(const T* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

constexpr int kTargetItemsPerSMMax = 4;   // sizes the split-K workspace

// Run-time tuning aids, read once from the environment.  Every default is the measured best (the
// A/B behind each is logged in DESIGN.md section 8 and profiles/); none changes results, only how
// the work is split, issued or launched.
//   CTS_ITEMS_PER_SM  shrink work items per SM per launch (K split target), 1..4        default 1
//   CTS_KS_MAX        cap on K chunks per slot, 1..16                                   default 16
//   CTS_EXPAND_STORE  expand store path: 0 TMA scatter, 1 register-direct  default by tokens/cluster
//   CTS_POLL_FIRST    fused: poll t-ready before issuing an item's y / out_basis loads   default idem
//   CTS_EARLY_ITEMS   fused: items whose loads may be issued before their t is ready    default 4
//   CTS_PACK          segment: pack two <=64-token clusters per 128-row slot (0 = off)  default 1
//   CTS_FUSED         0: shrink and expand as two launches (no inter-CTA waits)         default 1
//   CTS_JD_KSPACE     0: GPU compression iterates in the d-space only (no K-space Grams) default 1
//   CTS_JD_KS_RECOMPUTE  K-space Cholesky-QR2: 1 = second pass recomputes G C, 0 = reuses Y R1^-1  default 0
//                     (the last iteration is always the d-space Cholesky-QR2, so the result is orthonormal)
struct Tuning {
  int items_per_sm = 1, ks_max = 16, expand_store = -1, poll_first = -1, early_items = 4, pack = 1;
  bool fused = true;
  bool jd_kspace = true;
  bool jd_ks_recompute = false;
};

const Tuning& tuning() {
  static const Tuning t = [] {
    Tuning v;
    auto env = [](const char* name, int dflt) {
      const char* e = std::getenv(name);
      return e ? std::atoi(e) : dflt;
    };
    v.items_per_sm = std::max(1, std::min(kTargetItemsPerSMMax, env("CTS_ITEMS_PER_SM", v.items_per_sm)));
    v.ks_max = std::max(1, std::min(16, env("CTS_KS_MAX", v.ks_max)));
    v.expand_store = env("CTS_EXPAND_STORE", v.expand_store);
    v.poll_first = env("CTS_POLL_FIRST", v.poll_first);
    v.early_items = env("CTS_EARLY_ITEMS", v.early_items);
    v.pack = env("CTS_PACK", v.pack);
    v.fused = env("CTS_FUSED", 1) != 0;
    v.jd_kspace = env("CTS_JD_KSPACE", 1) != 0;
    v.jd_ks_recompute = env("CTS_JD_KS_RECOMPUTE", 0) != 0;
    return v;
  }();
  return t;
}

int target_items_per_sm() { return tuning().items_per_sm; }

template <typename Kern>
cudaError_t set_smem(Kern kernel, int bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// expand store path (expand.cuh STORE modes): register-direct stores when tiles are small
// (latency-bound decode: the stage is freed right after the y_base reads), TMA scatter when tiles
// are full (bandwidth-bound prefill).  Measured on B200 (expand us per launch, decode / prefill):
// scatter 21.4 / 150.7, direct 19.4 / 179.1 (row copies out of the stage, 23.7 / 160.9, were
// removed: the extra shared-memory round trip cost more than the fewer store wavefronts saved).
int expand_store_mode(int T, int C) {
  const int v = tuning().expand_store;
  if (v == 0 || v == 1) return v;
  return T < 96 * C ? kStoreDirect : kStoreScatter;   // mean tokens per cluster < 96
}

// fused kernel, expand producer: poll the slot's t-ready flag before (1) or after (0) issuing the
// item's out_basis / y loads.
int poll_first_default(int T, int C) {
  const int v = tuning().poll_first;
  if (v >= 0) return v != 0;
  return T < 96 * C ? 0 : 1;
}

// fused kernel, expand producer: how many of a CTA's expand items may load y / out_basis before
// their t is ready (the rest poll first, so their loads do not queue ahead of the split-K
// exchange's round trips).
int early_items_default() { return tuning().early_items; }

// cts_apply[_group] runs the fused single-launch kernel unless CTS_FUSED=0.
bool use_fused() { return tuning().fused; }

// The fused kernel launches cooperatively unless the caller declared exclusive use of the device
// (cts_set_exclusive_device): a cooperative launch cannot start before every CTA fits, so it loses
// the PDL overlap of its prologue with the previous kernel's tail (measured ~1.3 us per launch).
std::atomic<int> g_exclusive{0};
bool use_cooperative() { return g_exclusive.load(std::memory_order_relaxed) == 0; }

// Launch with programmatic stream serialization (PDL): the kernel may start while the previous
// kernel in the stream drains; every kernel calls griddep_wait() before touching dependent data.
std::atomic<uint64_t> g_launches{0};          // kernels this library enqueued (cts_launch_count)

// cooperative = 1: the launch is cooperative, i.e. the runtime only starts it when every CTA can be
// resident at once -- the fused kernel's inter-CTA waits (expand producers polling t-ready flags
// published by other CTAs) rely on that, also when other streams run kernels concurrently.
template <typename Kern, typename... Args>
cudaError_t launch_pdl_ex(Kern kernel, int grid, int block, size_t smem, cudaStream_t stream, bool cooperative,
                          Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(block, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cooperative ? 2 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
  if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
  return e;
}

template <typename Kern, typename... Args>
cudaError_t launch_pdl(Kern kernel, int grid, int block, size_t smem, cudaStream_t stream, Args... args) {
  return launch_pdl_ex(kernel, grid, block, smem, stream, false, args...);
}

__nv_bfloat16* module_tbuf(cts_plan_t p, int module) {
  return p->tbuf + size_t(module) * p->max_tiles * kTileM * 2 * p->bank->rp;
}

// K chunks per slot: the DEVICE sizes them from the real slot count (shrink_ks: ~target items per
// SM over the slots the segment kernel produced); the host only caps them: each chunk >= 4 K
// blocks, <= 16 chunks.  The workspace holds (target * SMs + slots) * 128 rows per module, which
// bounds slots * ks for any slot count.
int ks_cap(int min_kblocks) { return std::max(1, std::min(tuning().ks_max, min_kblocks / 4)); }

// Segment outputs may be read before griddep_wait by every kernel but the first after cts_segment:
// each kernel triggers its dependents only after its own griddep_wait, so when launch k starts,
// launch k-2 (at the latest cts_segment) has completed.
int next_meta_ready(cts_plan_t p) { return p->launches_since_segment++ > 0 ? 1 : 0; }

cts_status_t fill_shrink(cts_plan_t p, int n, const int32_t* modules, const void* const* xs, const int64_t* ld_x,
                         float scale, bool fused, ShrinkParams& prm, int& items, float* const* parts = nullptr) {
  const cts_bank_t b = p->bank;
  const int T = p->T;
  const int tiles_bound = cts_plan_max_tiles(p, T);
  int min_kb = 1 << 30;
  for (int i = 0; i < n; ++i) min_kb = std::min(min_kb, b->mods[modules[i]].d_in / kBK);
  const int ks_max = ks_cap(min_kb);
  std::memset(&prm, 0, sizeof(prm));
  prm.n_mod = n;
  prm.tiles_bound = tiles_bound;
  prm.ks_max = ks_max;
  prm.target_items = target_items_per_sm();
  prm.sigma_diag = b->sigma_diag;
  for (int i = 0; i < n; ++i) {
    const Module& m = b->mods[modules[i]];
    ShrinkMod& sm = prm.mod[i];
    if (!make_tmap(&sm.tm_x, xs[i], m.d_in, T, ld_x[i] * 2, 64, 1, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap(&sm.tm_x8, xs[i], m.d_in, T, ld_x[i] * 2, 64, 8, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap(&sm.tm_x32, xs[i], m.d_in, T, ld_x[i] * 2, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B))
      return CTS_ERR_CUDA;
    sm.tm_in = b->d_tm_in + modules[i];
    const size_t mid = m.map_id;
    sm.tiles = p->tiles + mid * p->max_tiles * 2;
    sm.n_tiles = p->n_tiles + mid;
    sm.tile_rows = p->tile_rows + mid * p->max_tiles * kTileM;
    sm.tile_adapters = p->tile_adapters + mid * p->max_tiles * kTileM;
    sm.sigma = m.sigma;
    sm.tbuf = module_tbuf(p, modules[i]);
    sm.tpart = parts ? parts[i] : nullptr;
    sm.ws = p->ws + size_t(i) * p->ws_cap_rows * b->rp;
    sm.counters = p->counters + size_t(i) * p->max_tiles;
    sm.ready = fused ? p->ready + size_t(i) * p->max_tiles : nullptr;
    sm.kblocks = m.d_in / kBK;
    sm.scale = scale;
  }
  items = tiles_bound * n * ks_max;                // upper bound (grid sizing)
  return CTS_OK;
}

cts_status_t fill_expand(cts_plan_t p, int n, const int32_t* modules, void* const* ys, const int64_t* ld_y,
                         bool fused, ExpandParams& prm, int& items) {
  const cts_bank_t b = p->bank;
  const int T = p->T;
  const int tiles_bound = cts_plan_max_tiles(p, T);
  std::memset(&prm, 0, sizeof(prm));
  prm.n_mod = n;
  items = 0;
  for (int i = 0; i < n; ++i) {
    const Module& m = b->mods[modules[i]];
    ExpandMod& em = prm.mod[i];
    if (!make_tmap(&em.tm_y, ys[i], m.d_out, T, ld_y[i] * 2, 64, 1, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap(&em.tm_y8, ys[i], m.d_out, T, ld_y[i] * 2, 64, 8, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap(&em.tm_y32, ys[i], m.d_out, T, ld_y[i] * 2, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B))
      return CTS_ERR_CUDA;
    em.tm_t = p->d_tm_t + modules[i];
    em.tm_out = b->d_tm_out + modules[i];
    const size_t mid = m.map_id;
    em.tiles = p->tiles + mid * p->max_tiles * 2;
    em.n_tiles = p->n_tiles + mid;
    em.tile_rows = p->tile_rows + mid * p->max_tiles * kTileM;
    em.ready = fused ? p->ready + size_t(i) * p->max_tiles : nullptr;
    em.y = static_cast<__nv_bfloat16*>(ys[i]);
    em.y32 = (reinterpret_cast<uintptr_t>(ys[i]) % 32 == 0 && (ld_y[i] * 2) % 32 == 0 && m.d_out % 16 == 0) ? 1 : 0;
    em.ld_y = ld_y[i];
    em.nblk = (m.d_out + kBN - 1) / kBN;
    em.d_out = m.d_out;
    items += tiles_bound * em.nblk;               // upper bound (grid sizing)
  }
  return CTS_OK;
}

template <int RP>
cts_status_t launch_shrink(cts_plan_t p, int n, const int32_t* modules, const void* const* xs, const int64_t* ld_x,
                           float scale, cudaStream_t stream, float* const* parts = nullptr) {
  static const cudaError_t attr = set_smem(shrink_sigma_kernel<RP, false>, ShrinkKernelSmem<RP>::kBytes);
  static const cudaError_t attr_d = set_smem(shrink_sigma_kernel<RP, true>, ShrinkKernelSmem<RP>::kBytes);
  CTS_CUDA(attr);
  CTS_CUDA(attr_d);
  ShrinkParams prm;
  int items = 0;
  cts_status_t st = fill_shrink(p, n, modules, xs, ld_x, scale, false, prm, items, parts);
  if (st != CTS_OK) return st;
  prm.meta_ready = next_meta_ready(p);
  CTS_CUDA(launch_pdl(prm.sigma_diag ? shrink_sigma_kernel<RP, true> : shrink_sigma_kernel<RP, false>,
                      std::min(sm_count(), items), kApplyThreads,
                      ShrinkKernelSmem<RP>::kBytes, stream, prm));
  return CTS_OK;
}

template <int RP, int STORE>
cts_status_t launch_expand(cts_plan_t p, int n, const int32_t* modules, void* const* ys, const int64_t* ld_y,
                           cudaStream_t stream) {
  static const cudaError_t attr = set_smem(expand_kernel<RP, STORE>, ExpandKernelSmem<RP>::kBytes);
  CTS_CUDA(attr);
  ExpandParams prm;
  int items = 0;
  cts_status_t st = fill_expand(p, n, modules, ys, ld_y, false, prm, items);
  if (st != CTS_OK) return st;
  prm.meta_ready = next_meta_ready(p);
  CTS_CUDA(launch_pdl(expand_kernel<RP, STORE>, std::min(sm_count(), items), kApplyThreads,
                      ExpandKernelSmem<RP>::kBytes, stream, prm));
  return CTS_OK;
}

template <int RP, int STORE>
cts_status_t launch_fused(cts_plan_t p, int n, const int32_t* modules, const void* const* xs, const int64_t* ld_x,
                          void* const* ys, const int64_t* ld_y, float scale, cudaStream_t stream) {
  static const cudaError_t attr = set_smem(apply_fused_kernel<RP, STORE, false>, FusedSmem<RP>::kBytes);
  static const cudaError_t attr_d = set_smem(apply_fused_kernel<RP, STORE, true>, FusedSmem<RP>::kBytes);
  CTS_CUDA(attr);
  CTS_CUDA(attr_d);
  FusedParams prm;
  int items_s = 0, items_e = 0;
  cts_status_t st = fill_shrink(p, n, modules, xs, ld_x, scale, true, prm.s, items_s);
  if (st != CTS_OK) return st;
  if ((st = fill_expand(p, n, modules, ys, ld_y, true, prm.e, items_e)) != CTS_OK) return st;
  prm.s.meta_ready = prm.e.meta_ready = next_meta_ready(p);
  prm.e.poll_first = poll_first_default(p->T, p->bank->C);
  prm.e.early_items = early_items_default();
  prm.exit_count = p->exit_count;
  CTS_CUDA(launch_pdl_ex(prm.s.sigma_diag ? apply_fused_kernel<RP, STORE, true> : apply_fused_kernel<RP, STORE, false>,
                         std::min(sm_count(), std::max(items_s, items_e)),
                         kApplyThreads, FusedSmem<RP>::kBytes, stream, use_cooperative(), prm));
  return CTS_OK;
}

cts_status_t check_group(cts_plan_t p, int32_t n, const int32_t* modules, const void* const* ptrs, const int64_t* lds,
                         bool is_x) {
  if (!p || n < 1 || !modules || !ptrs || !lds) return CTS_ERR_INVALID_ARGUMENT;
  if (n > kMaxGroup) return CTS_ERR_SHAPE;
  for (int i = 0; i < n; ++i) {
    if (modules[i] < 0 || modules[i] >= p->bank->n_modules) return CTS_ERR_SHAPE;
    for (int j = 0; j < i; ++j)
      if (modules[j] == modules[i]) return CTS_ERR_INVALID_ARGUMENT;
    if (!ptrs[i] && p->T > 0) return CTS_ERR_INVALID_ARGUMENT;   // an empty batch may pass null tensors
    const Module& m = p->bank->mods[modules[i]];
    const int64_t need = is_x ? m.d_in : m.d_out;
    if (lds[i] < need || (lds[i] * 2) % 16 || !aligned16(ptrs[i])) return CTS_ERR_SHAPE;
  }
  return CTS_OK;
}

cts_status_t do_shrink(cts_plan_t p, int n, const int32_t* mods, const void* const* xs, const int64_t* ld, float scale,
                       cudaStream_t s, float* const* parts = nullptr) {
  switch (p->bank->rp) {
    case 16: return launch_shrink<16>(p, n, mods, xs, ld, scale, s, parts);
    case 32: return launch_shrink<32>(p, n, mods, xs, ld, scale, s, parts);
    default: return launch_shrink<64>(p, n, mods, xs, ld, scale, s, parts);
  }
}

cts_status_t do_split(cts_plan_t p, int n, const int32_t* mods, const float* const* parts, cudaStream_t s) {
  SplitArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_mod = n;
  a.rp = p->bank->rp;
  for (int i = 0; i < n; ++i) {
    a.part[i] = parts[i];
    a.tbuf[i] = module_tbuf(p, mods[i]);
    const size_t mid = p->bank->mods[mods[i]].map_id;
    a.n_tiles[i] = p->n_tiles + mid;
    a.tile_rows[i] = p->tile_rows + mid * p->max_tiles * kTileM;
  }
  (void)next_meta_ready(p);   // one more launch separating the plan's segment from later kernels
  CTS_CUDA(launch_pdl(t_split_kernel, sm_count(), 256, 0, s, a));
  return CTS_OK;
}

bool check_parts(cts_plan_t p, int n, const void* const* parts) {
  if (!parts) return false;
  for (int i = 0; i < n; ++i)
    if (!parts[i] || !aligned16(parts[i])) return false;
  (void)p;
  return true;
}

// template dispatch over (r_pad, store mode)
template <template <int, int> class F, typename... A>
cts_status_t dispatch_rp_store(int rp, int store, A... a) {
  switch (rp * 4 + store) {
    case 16 * 4 + kStoreScatter: return F<16, kStoreScatter>::run(a...);
    case 16 * 4 + kStoreDirect: return F<16, kStoreDirect>::run(a...);
    case 32 * 4 + kStoreScatter: return F<32, kStoreScatter>::run(a...);
    case 32 * 4 + kStoreDirect: return F<32, kStoreDirect>::run(a...);
    case 64 * 4 + kStoreScatter: return F<64, kStoreScatter>::run(a...);
    default: return F<64, kStoreDirect>::run(a...);
  }
}
template <int RP, int STORE>
struct ExpandLaunch {
  static cts_status_t run(cts_plan_t p, int n, const int32_t* mods, void* const* ys, const int64_t* ld, cudaStream_t s) {
    return launch_expand<RP, STORE>(p, n, mods, ys, ld, s);
  }
};
template <int RP, int STORE>
struct FusedLaunch {
  static cts_status_t run(cts_plan_t p, int n, const int32_t* mods, const void* const* xs, const int64_t* ldx,
                          void* const* ys, const int64_t* ldy, float scale, cudaStream_t s) {
    return launch_fused<RP, STORE>(p, n, mods, xs, ldx, ys, ldy, scale, s);
  }
};

cts_status_t do_expand(cts_plan_t p, int n, const int32_t* mods, void* const* ys, const int64_t* ld, cudaStream_t s) {
  return dispatch_rp_store<ExpandLaunch>(p->bank->rp, expand_store_mode(p->T, p->bank->C), p, n, mods, ys, ld, s);
}

cts_status_t do_fused(cts_plan_t p, int n, const int32_t* mods, const void* const* xs, const int64_t* ldx,
                      void* const* ys, const int64_t* ldy, float scale, cudaStream_t s) {
  return dispatch_rp_store<FusedLaunch>(p->bank->rp, expand_store_mode(p->T, p->bank->C), p, n, mods, xs, ldx, ys,
                                        ldy, scale, s);
}

// fused base + LoRA projection (proj_fused.cuh): shrink + Sigma into the plan's t, then one GEMM
cts_status_t launch_project(cts_plan_t p, int32_t module, const void* x, int64_t ld_x, const void* w0, int64_t ld_w,
                            void* y, int64_t ld_y, float scale, cudaStream_t stream) {
  const cts_bank_t b = p->bank;
  const Module& m = b->mods[module];
  cts_status_t st = launch_shrink<16>(p, 1, &module, &x, &ld_x, scale, stream);
  if (st != CTS_OK) return st;
  static const cudaError_t attr = set_smem(proj_fused_kernel, ProjCfg::kBytes);
  CTS_CUDA(attr);
  ProjParams prm;
  std::memset(&prm, 0, sizeof(prm));
  if (!make_tmap(&prm.tm_x4, x, m.d_in, p->T, ld_x * 2, 64, 1, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_tmap(&prm.tm_x8, x, m.d_in, p->T, ld_x * 2, 64, 8, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_tmap(&prm.tm_x32, x, m.d_in, p->T, ld_x * 2, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_tmap(&prm.tm_x128, x, m.d_in, p->T, ld_x * 2, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_tmap(&prm.tm_w, w0, m.d_in, m.d_out, ld_w * 2, 64, kProjBN, CU_TENSOR_MAP_SWIZZLE_128B))
    return CTS_ERR_CUDA;
  {
    const uint64_t dims[3] = {uint64_t(2 * b->rp), 64, uint64_t(2 * p->max_tiles)};
    const uint64_t strides[2] = {uint64_t(4 * b->rp), uint64_t(64 * 4 * b->rp)};
    const uint32_t box[3] = {uint32_t(b->rp), 64, 1};
    if (!make_tmap3(&prm.tm_t3, module_tbuf(p, module), dims, strides, box, CU_TENSOR_MAP_SWIZZLE_32B))
      return CTS_ERR_CUDA;
  }
  prm.tm_out = b->d_tm_out + module;
  const size_t mid = m.map_id;
  prm.tiles = p->tiles + mid * p->max_tiles * 2;
  prm.n_tiles = p->n_tiles + mid;
  prm.tile_rows = p->tile_rows + mid * p->max_tiles * kTileM;
  prm.unbound_rows = p->unbound_rows;
  prm.n_unbound = p->n_unbound;
  prm.y = static_cast<__nv_bfloat16*>(y);
  prm.ld_y = ld_y;
  prm.y32 = (reinterpret_cast<uintptr_t>(y) % 32 == 0 && (ld_y * 2) % 32 == 0) ? 1 : 0;
  prm.kblocks = m.d_in / kBK;
  prm.nblk = m.d_out / kProjBN;
  prm.d_out = m.d_out;
  prm.meta_ready = next_meta_ready(p);
  const int items = (p->max_tiles + (p->T + kTileM - 1) / kTileM) * prm.nblk;
  CTS_CUDA(launch_pdl(proj_fused_kernel, std::min(sm_count(), std::max(items, 1)), kApplyThreads, ProjCfg::kBytes,
                      stream, prm));
  return CTS_OK;
}

// ------------------------------------------------------------------ GPU compression (App A.2)
// Tensor-core path (jd_tc.cuh) for r_pad >= 16 when every stacked K = n r_i is a multiple of 4
// (16-byte TMA row strides); otherwise the CUDA-core kernels of jd_eigen.cuh.
bool jd_tc_ok(const cts_jd_problem_t& q, int r) {
  return r >= 16 && (q.n * q.r_i) % 4 == 0 && reinterpret_cast<uintptr_t>(q.a_stack) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(q.bt_stack) % 16 == 0;
}

// K-space path (jd_gram.cuh): tensor-core shapes, 2r <= K <= kJdGramMaxK, r = 16 or 32
bool jd_gram_ok(const cts_jd_problem_t& q, int r) {
  const int K = q.n * q.r_i;
  return jd_tc_ok(q, r) && (r == 16 || r == 32) && K >= 2 * r && K <= kJdGramMaxK;
}

size_t jd_problem_floats(const cts_jd_problem_t& q, int r) {
  const size_t K = size_t(q.n) * q.r_i;
  const size_t gb = (size_t(q.d_in) + 255) / 256 + (size_t(q.d_out) + 255) / 256;
  const size_t dmax = size_t(std::max(q.d_in, q.d_out));
  const size_t part = std::max((dmax + kJdSeg - 1) / kJdSeg * K, (K + kJdKSeg - 1) / kJdKSeg * dmax) * r;
  size_t f = 4 * K * r + size_t(q.d_in + q.d_out) * r + gb * r * r + part + 64;   // + Gram, segment partials
  if (jd_tc_ok(q, r))   // A^T, Bt^T, V^T, U^T, W^T, Z^T (K-major operands of the tensor-core GEMMs)
    f += K * size_t(q.d_in + q.d_out) + size_t(r) * (q.d_in + q.d_out + 2 * K) + 64;
  if (jd_gram_ok(q, r)) f += 2 * K * K + 2 * K * size_t(r) + 64;   // G_A, G_B, Y_A, Y_B
  return f;
}

// One batch's tensor-core tables (maps, jobs, tile lists, transpose jobs) in one device block.
// Groups 0-3: the thin GEMMs; K-space path only: group 4 the Grams G_A = A A^T, G_B = Bt Bt^T,
// group 5 the per-iteration products Y_A = G_A Z, Y_B = G_B W (X = G, Y = Z^T / W^T).
struct JdTcTables {
  std::vector<uint8_t> host;
  void* dev = nullptr;
  size_t maps_bytes = 0;                 // the tensor maps sit at offset 0 of the device block
  size_t off_jobs[6] = {}, off_tiles[6] = {}, off_tr[3] = {};
  int n_tiles[6] = {}, n_tr[3] = {};
};

template <int R>
cts_status_t jd_tc_prepare(const JdBatch& jb, float* const* tc_base, bool gram, JdTcTables& T, cudaStream_t stream) {
  const int n = jb.count;
  // per problem: maps 0..7 = X: A, Bt, A^T, Bt^T; Y: V^T, U^T, W^T, Z^T
  std::vector<CUtensorMap> maps(size_t(n) * 10);
  std::vector<int4> tiles[6];
  std::vector<JdTransposeJob> tr[3];
  for (int i = 0; i < n; ++i) {
    const JdProblem& p = jb.pr[i];
    const int K = p.n * p.ri;
    float* at = tc_base[i];
    float* btt = at + size_t(K) * p.d_in;
    float* vt = btt + size_t(K) * p.d_out;
    float* ut = vt + size_t(R) * p.d_in;
    float* wt = ut + size_t(R) * p.d_out;
    float* zt = wt + size_t(R) * K;
    const int rowsP = (K + 127) / 128, rowsU = (p.d_out + 127) / 128, rowsV = (p.d_in + 127) / 128;
    for (int t = 0; t < rowsP; ++t) tiles[0].push_back(make_int4(i, t * 128, 0, 0));   // P = A V
    for (int t = 0; t < rowsP; ++t) tiles[1].push_back(make_int4(i, t * 128, 0, 0));   // Q = Bt U
    for (int t = 0; t < rowsU; ++t) tiles[2].push_back(make_int4(i, t * 128, 0, 0));   // U0 = Bt^T W
    for (int t = 0; t < rowsV; ++t) tiles[3].push_back(make_int4(i, t * 128, 0, 0));   // V0 = A^T Z
    if (gram)                                                                          // G_A, G_B tiles
      for (int side = 0; side < 2; ++side)
        for (int a = 0; a < rowsP; ++a)
          for (int c = a; c < rowsP; ++c)   // G symmetric: upper tiles, each off-diagonal one mirrored
            tiles[4].push_back(make_int4(2 * i + side, a * 128, c * 128, c > a ? 1 : 0));
    if (gram)                                                                          // G_A Z, G_B W tiles
      for (int side = 0; side < 2; ++side)
        for (int t = 0; t < rowsP; ++t) tiles[5].push_back(make_int4(2 * i + side, t * 128, 0, 0));
    tr[0].push_back({p.a, at, K, p.d_in});
    tr[0].push_back({p.bt, btt, K, p.d_out});
    tr[1].push_back({p.V, vt, p.d_in, R});
    tr[1].push_back({p.U, ut, p.d_out, R});
    tr[2].push_back({p.W, wt, K, R});
    tr[2].push_back({p.Z, zt, K, R});
  }
  auto al = [](size_t v) { return (v + 127) / 128 * 128; };
  size_t off = al(maps.size() * sizeof(CUtensorMap));
  for (int g = 0; g < 6; ++g) { T.off_jobs[g] = off; off = al(off + size_t(g >= 4 ? 2 * n : n) * sizeof(JdTcJob)); }
  for (int g = 0; g < 6; ++g) {
    T.off_tiles[g] = off;
    T.n_tiles[g] = int(tiles[g].size());
    off = al(off + tiles[g].size() * sizeof(int4));
  }
  for (int g = 0; g < 3; ++g) {
    if (tr[g].size() > size_t(kJdMaxTranspose)) return CTS_ERR_SHAPE;
    T.off_tr[g] = off;
    T.n_tr[g] = int(tr[g].size());
    off = al(off + sizeof(JdTransposeBatch));
  }
  T.host.assign(off, 0);
  if (cudaMallocAsync(&T.dev, off, stream) != cudaSuccess) { (void)cudaGetLastError(); return CTS_ERR_OUT_OF_MEMORY; }
  const CUtensorMap* dmaps = static_cast<const CUtensorMap*>(T.dev);
  for (int i = 0; i < n; ++i) {
    const JdProblem& p = jb.pr[i];
    const int K = p.n * p.ri;
    const CUtensorMap* m = dmaps + size_t(i) * 10;
    const JdTcJob jobs[4] = {{m + 0, m + 4, p.P, K, p.d_in, R, R}, {m + 1, m + 5, p.Q, K, p.d_out, R, R},
                             {m + 3, m + 6, p.U0, p.d_out, K, R, R}, {m + 2, m + 7, p.V0, p.d_in, K, R, R}};
    for (int g = 0; g < 4; ++g) std::memcpy(T.host.data() + T.off_jobs[g] + i * sizeof(JdTcJob), &jobs[g], sizeof(JdTcJob));
    if (gram) {   // X = Y = the stack (box {32, 128} serves both operands)
      const JdTcJob gj[2] = {{m + 0, m + 0, p.Ga, K, p.d_in, K, K}, {m + 1, m + 1, p.Gb, K, p.d_out, K, K}};
      std::memcpy(T.host.data() + T.off_jobs[4] + 2 * i * sizeof(JdTcJob), gj, sizeof(gj));
      const JdTcJob yj[2] = {{m + 8, m + 7, p.Ya, K, K, R, R}, {m + 9, m + 6, p.Yb, K, K, R, R}};
      std::memcpy(T.host.data() + T.off_jobs[5] + 2 * i * sizeof(JdTcJob), yj, sizeof(yj));
    }
  }
  for (int g = 0; g < 6; ++g) std::memcpy(T.host.data() + T.off_tiles[g], tiles[g].data(), tiles[g].size() * sizeof(int4));
  for (int g = 0; g < 3; ++g) std::memcpy(T.host.data() + T.off_tr[g], tr[g].data(), tr[g].size() * sizeof(JdTransposeJob));
  // jobs, tile lists and transpose batches now; the tensor maps (host encoding, ~1 us each) follow in
  // jd_tc_prepare_maps while the first transposes already run on the GPU
  T.maps_bytes = maps.size() * sizeof(CUtensorMap);
  if (cudaMemcpyAsync(static_cast<uint8_t*>(T.dev) + T.off_jobs[0], T.host.data() + T.off_jobs[0], off - T.off_jobs[0],
                      cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return CTS_ERR_CUDA;
  return CTS_OK;
}

// Phase 2 of the tables: encode every problem's tensor maps (0..7 = X: A, Bt, A^T, Bt^T; Y: V^T,
// U^T, W^T, Z^T; 8, 9 = the Grams) and copy them to the front of the device block.
template <int R>
cts_status_t jd_tc_prepare_maps(const JdBatch& jb, float* const* tc_base, bool gram, JdTcTables& T,
                                cudaStream_t stream) {
  const int n = jb.count;
  CUtensorMap* maps = reinterpret_cast<CUtensorMap*>(T.host.data());
  for (int i = 0; i < n; ++i) {
    const JdProblem& p = jb.pr[i];
    const int K = p.n * p.ri;
    float* at = tc_base[i];
    float* btt = at + size_t(K) * p.d_in;
    float* vt = btt + size_t(K) * p.d_out;
    float* ut = vt + size_t(R) * p.d_in;
    float* wt = ut + size_t(R) * p.d_out;
    float* zt = wt + size_t(R) * K;
    CUtensorMap* m = maps + size_t(i) * 10;
    if (!make_tmap_f32(&m[0], p.a, p.d_in, K, 32, 128) || !make_tmap_f32(&m[1], p.bt, p.d_out, K, 32, 128) ||
        !make_tmap_f32(&m[2], at, K, p.d_in, 32, 128) || !make_tmap_f32(&m[3], btt, K, p.d_out, 32, 128) ||
        !make_tmap_f32(&m[4], vt, p.d_in, R, 32, R) || !make_tmap_f32(&m[5], ut, p.d_out, R, 32, R) ||
        !make_tmap_f32(&m[6], wt, K, R, 32, R) || !make_tmap_f32(&m[7], zt, K, R, 32, R))
      return CTS_ERR_CUDA;
    if (gram && (!make_tmap_f32(&m[8], p.Ga, K, K, 32, 128) || !make_tmap_f32(&m[9], p.Gb, K, K, 32, 128)))
      return CTS_ERR_CUDA;
  }
  if (cudaMemcpyAsync(T.dev, T.host.data(), T.maps_bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return CTS_ERR_CUDA;
  return CTS_OK;
}

template <int R>
cts_status_t jd_run(const cts_jd_problem_t* problems, int32_t count, int32_t iters, float* ws,
                           cudaStream_t stream) {
  static const cudaError_t attr = cudaFuncSetAttribute(jd_small<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       96 * 1024);
  CTS_CUDA(attr);
  for (int b0 = 0; b0 < count; b0 += kJdMaxBatch) {
    std::unique_ptr<JdBatch> jbp(new (std::nothrow) JdBatch());   // 30 KB: not on the host stack
    if (!jbp) return CTS_ERR_OUT_OF_MEMORY;
    JdBatch& jb = *jbp;
    jb.count = std::min(kJdMaxBatch, count - b0);
    int kmax = 1, dmax = 1, nmax = 1, rimax = 1;
    bool tc = true, gram = true;
    float* tc_base[kJdMaxBatch];
    for (int i = 0; i < jb.count; ++i) {
      const cts_jd_problem_t& q = problems[b0 + i];
      JdProblem& p = jb.pr[i];
      const size_t K = size_t(q.n) * q.r_i;
      p.a = q.a_stack; p.bt = q.bt_stack; p.U = q.U; p.V = q.V; p.sigma = q.sigma;
      p.n = q.n; p.ri = q.r_i; p.d_in = q.d_in; p.d_out = q.d_out;
      float* w = ws;
      p.P = w; w += K * R;
      p.Q = w; w += K * R;
      p.W = w; w += K * R;
      p.Z = w; w += K * R;
      p.U0 = w; w += size_t(q.d_out) * R;
      p.V0 = w; w += size_t(q.d_in) * R;
      p.Gu = w; w += (size_t(q.d_out) + 255) / 256 * R * R;
      p.Gv = w; w += (size_t(q.d_in) + 255) / 256 * R * R;
      p.part = w;
      w += std::max((size_t(std::max(q.d_in, q.d_out)) + kJdSeg - 1) / kJdSeg * K,
                    (K + kJdKSeg - 1) / kJdKSeg * size_t(std::max(q.d_in, q.d_out))) * R;
      tc_base[i] = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(w) + 255) & ~uintptr_t(255));
      p.Ga = p.Gb = p.Ya = p.Yb = nullptr;
      if (jd_gram_ok(q, R)) {
        float* g0 = tc_base[i] + K * size_t(q.d_in + q.d_out) + size_t(R) * (q.d_in + q.d_out + 2 * K);
        p.Ga = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(g0) + 255) & ~uintptr_t(255));
        p.Gb = p.Ga + K * K;
        p.Ya = p.Gb + K * K;
        p.Yb = p.Ya + K * R;
      }
      tc = tc && jd_tc_ok(q, R);
      gram = gram && jd_gram_ok(q, R);
      ws += jd_problem_floats(q, R);
      kmax = std::max<int>(kmax, int(K));
      dmax = std::max({dmax, q.d_in, q.d_out});
      nmax = std::max(nmax, q.n);
      rimax = std::max(rimax, q.r_i);
    }
    const dim3 g_rows((kmax + kJdRowsPerBlock - 1) / kJdRowsPerBlock, (dmax + kJdSeg - 1) / kJdSeg, jb.count);
    const dim3 g_cols((dmax + 256 * JdColsPer<R>::v - 1) / (256 * JdColsPer<R>::v), (kmax + kJdKSeg - 1) / kJdKSeg,
                      jb.count);
    const dim3 g_red(std::max(1, kmax * R / 1024), jb.count), g_cred(std::max(1, dmax * R / 1024), jb.count);
    const dim3 g_small(nmax, jb.count), g_gram((dmax + kJdGramRows - 1) / kJdGramRows, jb.count, 2);
    const dim3 g_one(1, jb.count, 2), g_ew(std::max(1, (dmax + 255) / 256), jb.count, 2);
    const size_t small_smem = (2 * size_t(rimax) * R + R * R) * 4;
    if (small_smem > 96 * 1024) return CTS_ERR_SHAPE;
    if constexpr (R >= 16) {
      if (tc) {                          // tensor-core thin GEMMs (jd_tc.cuh); same orthogonalization
        JdTcTables T;
        gram = gram && iters >= 2 && tuning().jd_kspace;
        cts_status_t st = jd_tc_prepare<R>(jb, tc_base, gram, T, stream);
        if (st != CTS_OK) return st;
        static const cudaError_t attr_tc = set_smem(jd_tc_gemm<R>, JdTcCfg<R>::kBytes);
        CTS_CUDA(attr_tc);
        uint8_t* dv = static_cast<uint8_t*>(T.dev);
        auto gemm = [&](int g) {
          JdTcParams prm;
          prm.jobs = reinterpret_cast<const JdTcJob*>(dv + T.off_jobs[g]);
          prm.tiles = reinterpret_cast<const int4*>(dv + T.off_tiles[g]);
          prm.n_tiles = T.n_tiles[g];
          jd_tc_gemm<R><<<std::min(sm_count(), std::max(1, T.n_tiles[g])), 320, JdTcCfg<R>::kBytes, stream>>>(prm);
        };
        auto transpose = [&](int g) {
          jd_transpose<<<dim3(g == 0 ? 256 : 16, 1, std::min(T.n_tr[g], 65535)), 256, 0, stream>>>(
              reinterpret_cast<const JdTransposeBatch*>(dv + T.off_tr[g]), T.n_tr[g]);
        };
        transpose(0);                     // A^T, Bt^T (once)
        transpose(1);                     // V^T, U^T of the initial bases
        if ((st = jd_tc_prepare_maps<R>(jb, tc_base, gram, T, stream)) != CTS_OK) return st;
        int it0 = 0;
        if constexpr (R == 16 || R == 32) {
          if (gram) {                     // iterations 0 .. iters-2 in the K-space (jd_gram.cuh)
            static const cudaError_t attr_g = set_smem(jd_tc_gemm<128>, JdTcCfg<128>::kBytes);
            CTS_CUDA(attr_g);
            gemm(0);
            gemm(1);
            JdTcParams gp;
            gp.jobs = reinterpret_cast<const JdTcJob*>(dv + T.off_jobs[4]);
            gp.tiles = reinterpret_cast<const int4*>(dv + T.off_tiles[4]);
            gp.n_tiles = T.n_tiles[4];
            jd_tc_gemm<128><<<std::min(sm_count(), std::max(1, T.n_tiles[4])), 320, JdTcCfg<128>::kBytes, stream>>>(gp);
            const dim3 g_go(2, jb.count);
            for (; it0 < iters - 1; ++it0) {
              jd_small<R><<<g_small, 256, small_smem, stream>>>(jb);
              for (int pass = 0; pass < 2; ++pass) {
                if (pass == 0 || tuning().jd_ks_recompute) {   // pass 2: G C recomputed, or Y R1^-1 reused
                  transpose(2);              // C^T (W^T, Z^T), then Y = G C on the tensor cores
                  gemm(5);
                  g_launches.fetch_add(2, std::memory_order_relaxed);
                }
                jd_gorth<R><<<g_go, 256, 0, stream>>>(jb, pass);
              }
              g_launches.fetch_add(3, std::memory_order_relaxed);
            }
            g_launches.fetch_add(3, std::memory_order_relaxed);
          }
        }
        for (int it = it0; it < iters; ++it) {
          if (it > it0 || it0 == 0) {     // (the K-space iterations leave P, Q of the current iterate)
            gemm(0);                      // P = A V
            gemm(1);                      // Q = Bt U
          } else {
            g_launches.fetch_sub(2, std::memory_order_relaxed);
          }
          jd_small<R><<<g_small, 256, small_smem, stream>>>(jb);
          transpose(2);                   // W^T, Z^T
          gemm(2);                        // U0 = Bt^T W
          gemm(3);                        // V0 = A^T Z
          for (int pass = 0; pass < 2; ++pass) {
            jd_gram<R><<<g_gram, 256, 0, stream>>>(jb, pass);
            jd_chol<R><<<g_one, 32, 0, stream>>>(jb, pass);
            jd_apply<R><<<g_ew, 256, 0, stream>>>(jb, pass);
          }
          transpose(1);                   // V^T, U^T of the new bases
          g_launches.fetch_add(13, std::memory_order_relaxed);
        }
        gemm(0);
        gemm(1);
        jd_sigma<R><<<g_small, 256, 0, stream>>>(jb);
        g_launches.fetch_add(5, std::memory_order_relaxed);
        CTS_CUDA(cudaGetLastError());
        if (cudaFreeAsync(T.dev, stream) != cudaSuccess) return CTS_ERR_CUDA;
        continue;
      }
    }
    for (int it = 0; it < iters; ++it) {
      jd_rows_times<R><<<g_rows, 256, 0, stream>>>(jb, 0);
      jd_rows_reduce<R><<<g_red, 256, 0, stream>>>(jb, 0);
      jd_rows_times<R><<<g_rows, 256, 0, stream>>>(jb, 1);
      jd_rows_reduce<R><<<g_red, 256, 0, stream>>>(jb, 1);
      jd_small<R><<<g_small, 256, small_smem, stream>>>(jb);
      jd_cols_times<R><<<g_cols, 256, 0, stream>>>(jb, 0);
      jd_cols_reduce<R><<<g_cred, 256, 0, stream>>>(jb, 0);
      jd_cols_times<R><<<g_cols, 256, 0, stream>>>(jb, 1);
      jd_cols_reduce<R><<<g_cred, 256, 0, stream>>>(jb, 1);
      for (int pass = 0; pass < 2; ++pass) {
        jd_gram<R><<<g_gram, 256, 0, stream>>>(jb, pass);
        jd_chol<R><<<g_one, 32, 0, stream>>>(jb, pass);
        jd_apply<R><<<g_ew, 256, 0, stream>>>(jb, pass);
      }
      g_launches.fetch_add(15, std::memory_order_relaxed);
    }
    jd_rows_times<R><<<g_rows, 256, 0, stream>>>(jb, 0);
    jd_rows_reduce<R><<<g_red, 256, 0, stream>>>(jb, 0);
    jd_rows_times<R><<<g_rows, 256, 0, stream>>>(jb, 1);
    jd_rows_reduce<R><<<g_red, 256, 0, stream>>>(jb, 1);
    jd_sigma<R><<<g_small, 256, 0, stream>>>(jb);
    g_launches.fetch_add(5, std::memory_order_relaxed);
    CTS_CUDA(cudaGetLastError());
  }
  return CTS_OK;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const uint8_t* x = static_cast<const uint8_t*>(a);
  const uint8_t* y = static_cast<const uint8_t*>(b);
  return x < y + nb && y < x + na;
}

// ------------------------------------------------------------------ NCCL (loaded at run time)
// Only the handful of entry points cts_apply_tp needs; ABI types restated from nccl.h (stable since
// NCCL 2.0): ncclUniqueId is 128 opaque bytes, ncclFloat32 = 7, ncclSum = 0, ncclSuccess = 0.
struct NcclId { char internal[128]; };
using ncclComm_p = void*;
struct NcclApi {
  int (*get_unique_id)(NcclId*) = nullptr;
  int (*comm_init_rank)(ncclComm_p*, int, NcclId, int) = nullptr;
  int (*comm_destroy)(ncclComm_p) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_p, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<int (*)(NcclId*)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<int (*)(ncclComm_p*, int, NcclId, int)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<int (*)(ncclComm_p)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, ncclComm_p, cudaStream_t)>(
        dlsym(h, "ncclAllReduce"));
    api.group_start = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupEnd"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.group_start &&
             api.group_end;
  });
  return api;
}

}  // namespace

struct cts_comm_s {
  ncclComm_p comm;
  int nranks, rank;
};

extern "C" {

const char* cts_status_string(cts_status_t s) {
  switch (s) {
    case CTS_OK: return "ok";
    case CTS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case CTS_ERR_SHAPE: return "shape or alignment violation";
    case CTS_ERR_INDEX_OUT_OF_RANGE: return "index out of range";
    case CTS_ERR_UNSUPPORTED: return "unsupported device or configuration";
    case CTS_ERR_OUT_OF_MEMORY: return "out of device memory";
    case CTS_ERR_CUDA: return "CUDA error";
    case CTS_ERR_NCCL: return "NCCL unavailable or failed";
  }
  return "unknown status";
}

uint64_t cts_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

cts_status_t cts_set_exclusive_device(int32_t exclusive) {
  if (exclusive != 0 && exclusive != 1) return CTS_ERR_INVALID_ARGUMENT;
  g_exclusive.store(exclusive, std::memory_order_relaxed);
  return CTS_OK;
}

cts_status_t cts_bank_load(const cts_bank_desc_t* d, cudaStream_t stream, cts_bank_t* out) {
  if (!out) return CTS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (!d || !d->d_in || !d->d_out || !d->in_basis || !d->out_basis || !d->sigma || !d->cluster_of)
    return CTS_ERR_INVALID_ARGUMENT;
  if (d->n_modules < 1 || d->n_adapters < 1 || d->n_clusters < 1 || d->rank < 1) return CTS_ERR_SHAPE;
  if (d->rank > 64 || d->n_clusters > 1024) return CTS_ERR_UNSUPPORTED;
  if (d->sigma_kind != CTS_SIGMA_FULL && d->sigma_kind != CTS_SIGMA_DIAG) return CTS_ERR_INVALID_ARGUMENT;
  const bool diag = d->sigma_kind == CTS_SIGMA_DIAG;
  int dev = 0, major = 0;
  CTS_CUDA(cudaGetDevice(&dev));
  CTS_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) return CTS_ERR_UNSUPPORTED;
  if (!encode_fn()) return CTS_ERR_CUDA;
  const int M = d->n_modules, N = d->n_adapters, C = d->n_clusters, r = d->rank, rp = pad_rank(r);
  for (int m = 0; m < M; ++m) {
    if (d->d_in[m] <= 0 || d->d_out[m] <= 0 || d->d_in[m] % 64 || d->d_out[m] % 64) return CTS_ERR_SHAPE;
    if (!d->in_basis[m] || !d->out_basis[m] || !d->sigma[m] || !d->cluster_of[m]) return CTS_ERR_INVALID_ARGUMENT;
  }
  // cluster maps: bring to host, validate, dedupe
  std::vector<std::vector<int32_t>> uniq;
  std::vector<int> map_id(M);
  std::vector<int32_t> tmp(N);
  for (int m = 0; m < M; ++m) {
    if (d->sources_on_device) {   // ordered after the caller's pending writes on `stream`
      CTS_CUDA(cudaMemcpyAsync(tmp.data(), d->cluster_of[m], N * sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
      CTS_CUDA(cudaStreamSynchronize(stream));
    }
    else
      std::memcpy(tmp.data(), d->cluster_of[m], N * sizeof(int32_t));
    for (int i = 0; i < N; ++i)
      if (tmp[i] < 0 || tmp[i] >= C) return CTS_ERR_INDEX_OUT_OF_RANGE;
    int found = -1;
    for (size_t u = 0; u < uniq.size(); ++u)
      if (std::memcmp(uniq[u].data(), tmp.data(), N * sizeof(int32_t)) == 0) { found = int(u); break; }
    if (found < 0) { found = int(uniq.size()); uniq.push_back(tmp); }
    map_id[m] = found;
  }
  // arena layout
  std::vector<size_t> off_in(M), off_out(M), off_sig(M);
  size_t total = 0, stage = 0;
  for (int m = 0; m < M; ++m) {
    const size_t n_in = size_t(C) * rp * d->d_in[m], n_out = size_t(C) * d->d_out[m] * rp, n_sig = size_t(N) * rp * (diag ? 1 : rp);
    off_in[m] = total;  total = align_up(total + n_in * 2, 1024);
    off_out[m] = total; total = align_up(total + n_out * 2, 1024);
    off_sig[m] = total; total = align_up(total + n_sig * 2, 1024);
    stage = std::max(stage, std::max(size_t(C) * d->d_in[m] * r, std::max(size_t(C) * d->d_out[m] * r, size_t(N) * r * (diag ? 1 : r))) * 2);
  }
  const size_t off_maps = total;
  total = align_up(total + uniq.size() * N * sizeof(int32_t), 1024);
  const size_t off_tm = total;
  total = align_up(total + 2 * size_t(M) * sizeof(CUtensorMap), 1024);

  auto* b = new (std::nothrow) cts_bank_s();
  if (!b) return CTS_ERR_OUT_OF_MEMORY;
  b->n_modules = M; b->N = N; b->C = C; b->r = r; b->rp = rp;
  b->sigma_diag = diag ? 1 : 0;
  b->n_maps = int(uniq.size());
  b->bytes = total;
  if (cudaMalloc(&b->arena, total) != cudaSuccess) { (void)cudaGetLastError(); delete b; return CTS_ERR_OUT_OF_MEMORY; }
  void* staging = nullptr;
  if (!d->sources_on_device && cudaMalloc(&staging, stage) != cudaSuccess) {
    (void)cudaGetLastError(); cudaFree(b->arena); delete b; return CTS_ERR_OUT_OF_MEMORY;
  }
  auto fail = [&](cts_status_t s) { (void)cudaGetLastError(); if (staging) cudaFree(staging); cudaFree(b->arena); delete b; return s; };
  uint8_t* base = static_cast<uint8_t*>(b->arena);
  b->maps = reinterpret_cast<int32_t*>(base + off_maps);
  b->d_tm_in = reinterpret_cast<CUtensorMap*>(base + off_tm);
  b->d_tm_out = b->d_tm_in + M;
  for (size_t u = 0; u < uniq.size(); ++u)
    if (cudaMemcpyAsync(b->maps + u * N, uniq[u].data(), N * 4, cudaMemcpyHostToDevice, stream) != cudaSuccess) return fail(CTS_ERR_CUDA);
  std::vector<CUtensorMap> h_tm(2 * size_t(M));
  b->mods.resize(M);
  for (int m = 0; m < M; ++m) {
    Module& mod = b->mods[m];
    mod.d_in = d->d_in[m]; mod.d_out = d->d_out[m]; mod.map_id = map_id[m];
    mod.in_t = reinterpret_cast<__nv_bfloat16*>(base + off_in[m]);
    mod.out = reinterpret_cast<__nv_bfloat16*>(base + off_out[m]);
    mod.sigma = reinterpret_cast<__nv_bfloat16*>(base + off_sig[m]);
    const void* srcs[3] = {d->in_basis[m], d->out_basis[m], d->sigma[m]};
    const size_t nbytes[3] = {size_t(C) * mod.d_in * r * 2, size_t(C) * mod.d_out * r * 2, size_t(N) * r * (diag ? 1 : r) * 2};
    for (int k = 0; k < 3; ++k) {
      const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(srcs[k]);
      if (!d->sources_on_device) {
        if (cudaMemcpyAsync(staging, srcs[k], nbytes[k], cudaMemcpyHostToDevice, stream) != cudaSuccess) return fail(CTS_ERR_CUDA);
        src = static_cast<const __nv_bfloat16*>(staging);
      }
      if (k == 0) relayout_in_kernel<<<1184, 256, 0, stream>>>(src, mod.in_t, C, mod.d_in, r, rp);
      if (k == 1) relayout_pad_kernel<<<1184, 256, 0, stream>>>(src, mod.out, size_t(C) * mod.d_out, r, rp);
      if (k == 2 && diag) relayout_pad_kernel<<<1184, 256, 0, stream>>>(src, mod.sigma, size_t(N), r, rp);
      if (k == 2 && !diag) relayout_sigma_kernel<<<1184, 256, 0, stream>>>(src, mod.sigma, N, r, rp);
      if (cudaGetLastError() != cudaSuccess) return fail(CTS_ERR_CUDA);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      if (!d->sources_on_device && cudaStreamSynchronize(stream) != cudaSuccess) return fail(CTS_ERR_CUDA);
    }
    if (!make_tmap(&h_tm[m], mod.in_t, mod.d_in, uint64_t(C) * rp, uint64_t(mod.d_in) * 2, 64, rp,
                   CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap(&h_tm[M + m], mod.out, rp, uint64_t(C) * mod.d_out, uint64_t(rp) * 2, rp, 64, swizzle_for(rp * 2)))
      return fail(CTS_ERR_CUDA);
  }
  if (cudaMemcpyAsync(b->d_tm_in, h_tm.data(), h_tm.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return fail(CTS_ERR_CUDA);
  if (cudaStreamSynchronize(stream) != cudaSuccess) return fail(CTS_ERR_CUDA);
  if (staging) cudaFree(staging);
  *out = b;
  return CTS_OK;
}

cts_status_t cts_bank_bytes(cts_bank_t b, size_t* bytes) {
  if (!b || !bytes) return CTS_ERR_INVALID_ARGUMENT;
  *bytes = b->bytes;
  return CTS_OK;
}

cts_status_t cts_bank_params(cts_bank_t b, int32_t module, int64_t* params) {
  if (!b || !params) return CTS_ERR_INVALID_ARGUMENT;
  if (module < 0 || module >= b->n_modules) return CTS_ERR_SHAPE;
  const Module& m = b->mods[module];
  const int64_t sig = b->sigma_diag ? int64_t(b->r) : int64_t(b->r) * b->r;   // JD-Diag: r numbers (Eq. 3)
  *params = int64_t(b->C) * (m.d_in + m.d_out) * b->r + int64_t(b->N) * (sig + (b->C > 1 ? 1 : 0));
  return CTS_OK;
}

cts_status_t cts_bank_write_clusters(cts_bank_t b, int32_t module, int32_t n, const int32_t* clusters,
                                     const void* in_basis, const void* out_basis, cudaStream_t stream) {
  if (!b || !clusters || (n > 0 && (!in_basis || !out_basis))) return CTS_ERR_INVALID_ARGUMENT;
  if (module < 0 || module >= b->n_modules || n < 0 || n > kMaxWriteClusters) return CTS_ERR_SHAPE;
  ClusterList cl;
  for (int q = 0; q < n; ++q) {
    if (clusters[q] < 0 || clusters[q] >= b->C) return CTS_ERR_INDEX_OUT_OF_RANGE;
    for (int p = 0; p < q; ++p)
      if (clusters[p] == clusters[q]) return CTS_ERR_INVALID_ARGUMENT;
    cl.c[q] = clusters[q];
  }
  if (n == 0) return CTS_OK;
  const Module& m = b->mods[module];
  write_in_kernel<<<1184, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(in_basis), m.in_t, cl, n, m.d_in, b->r,
                                            b->rp);
  write_out_kernel<<<1184, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(out_basis), m.out, cl, n, m.d_out,
                                             b->r, b->rp);
  CTS_CUDA(cudaGetLastError());
  g_launches.fetch_add(2, std::memory_order_relaxed);
  return CTS_OK;
}

cts_status_t cts_bank_free(cts_bank_t b) {
  if (!b) return CTS_ERR_INVALID_ARGUMENT;
  cudaFree(b->arena);
  delete b;
  return CTS_OK;
}

int32_t cts_plan_max_tiles(cts_plan_t p, int32_t T) {
  if (!p || T <= 0) return 0;
  return (T + kTileM - 1) / kTileM + std::min(p->bank->C, T);
}

cts_status_t cts_plan_create(cts_bank_t b, int32_t T_max, cts_plan_t* out) {
  if (!out) return CTS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (!b || T_max < 1) return CTS_ERR_INVALID_ARGUMENT;
  auto* p = new (std::nothrow) cts_plan_s();
  if (!p) return CTS_ERR_OUT_OF_MEMORY;
  p->bank = b;
  p->T_max = T_max;
  p->T = 0;
  p->launches_since_segment = 0;
  p->max_tiles = cts_plan_max_tiles(p, T_max);
  // split-K workspace rows per group slot: ks * tiles_bound * 128 <= (target items + tiles) * 128
  p->ws_cap_rows = size_t(kTargetItemsPerSMMax * sm_count() + p->max_tiles) * kTileM;
  const size_t nm = b->n_maps;
  size_t off = 0;
  const size_t o_tok = off; off = align_up(off + size_t(T_max) * 4, 256);
  const size_t o_perm = off; off = align_up(off + nm * T_max * 4, 256);
  const size_t o_offs = off; off = align_up(off + nm * (b->C + 1) * 4, 256);
  const size_t o_tiles = off; off = align_up(off + nm * p->max_tiles * 32, 256);
  const size_t o_nt = off; off = align_up(off + nm * 4, 256);
  const size_t o_trows = off; off = align_up(off + nm * p->max_tiles * kTileM * 4, 256);
  const size_t o_tads = off; off = align_up(off + nm * p->max_tiles * kTileM * 4, 256);
  const size_t o_err = off; off = align_up(off + 16, 256);
  const size_t o_unb = off; off = align_up(off + (size_t(T_max) + kTileM + 4) * 4, 256);
  const size_t o_cnt = off; off = align_up(off + size_t(kMaxGroup) * p->max_tiles * 4, 1024);
  const size_t o_rdy = off; off = align_up(off + size_t(kMaxGroup) * p->max_tiles * 4 + 16, 1024);
  const size_t o_tm = off; off = align_up(off + size_t(b->n_modules) * sizeof(CUtensorMap), 1024);
  const size_t o_ws = off; off = align_up(off + size_t(kMaxGroup) * p->ws_cap_rows * b->rp * 4, 1024);
  const size_t o_t = off; off = align_up(off + size_t(b->n_modules) * p->max_tiles * kTileM * 2 * b->rp * 2, 1024);
  const size_t o_tp = off; off = align_up(off + size_t(kMaxGroup) * T_max * b->rp * 4, 1024);
  if (cudaMalloc(&p->arena, off) != cudaSuccess) { (void)cudaGetLastError(); delete p; return CTS_ERR_OUT_OF_MEMORY; }
  uint8_t* base = static_cast<uint8_t*>(p->arena);
  p->tok_adapter = reinterpret_cast<int32_t*>(base + o_tok);
  p->perm = reinterpret_cast<int32_t*>(base + o_perm);
  p->offsets = reinterpret_cast<int32_t*>(base + o_offs);
  p->tiles = reinterpret_cast<int4*>(base + o_tiles);
  p->n_tiles = reinterpret_cast<int32_t*>(base + o_nt);
  p->tile_rows = reinterpret_cast<int32_t*>(base + o_trows);
  p->tile_adapters = reinterpret_cast<int32_t*>(base + o_tads);
  p->err = reinterpret_cast<int32_t*>(base + o_err);
  p->n_unbound = reinterpret_cast<int32_t*>(base + o_unb);
  p->unbound_rows = p->n_unbound + 4;
  p->counters = reinterpret_cast<int32_t*>(base + o_cnt);
  p->ready = reinterpret_cast<int32_t*>(base + o_rdy);
  p->exit_count = p->ready + size_t(kMaxGroup) * p->max_tiles;
  p->d_tm_t = reinterpret_cast<CUtensorMap*>(base + o_tm);
  p->ws = reinterpret_cast<float*>(base + o_ws);
  p->tbuf = reinterpret_cast<__nv_bfloat16*>(base + o_t);
  p->tp_parts = reinterpret_cast<float*>(base + o_tp);
  const int32_t init_err[2] = {0, -1};
  bool ok = cudaMemset(p->n_tiles, 0, nm * 4) == cudaSuccess && cudaMemset(p->n_unbound, 0, 16) == cudaSuccess &&
            cudaMemset(p->tiles, 0, nm * p->max_tiles * 32) == cudaSuccess &&
            cudaMemset(p->counters, 0, size_t(kMaxGroup) * p->max_tiles * 4) == cudaSuccess &&
            cudaMemset(p->ready, 0, size_t(kMaxGroup) * p->max_tiles * 4 + 16) == cudaSuccess &&
            cudaMemcpy(p->err, init_err, 8, cudaMemcpyHostToDevice) == cudaSuccess;
  std::vector<CUtensorMap> h_tm(b->n_modules);
  for (int m = 0; ok && m < b->n_modules; ++m)
    ok = make_tmap(&h_tm[m], module_tbuf(p, m), 2 * b->rp, uint64_t(p->max_tiles) * kTileM, uint64_t(4 * b->rp),
                   b->rp, kTileM, swizzle_for(2 * b->rp));
  ok = ok && cudaMemcpy(p->d_tm_t, h_tm.data(), h_tm.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) {
    (void)cudaGetLastError();
    cudaFree(p->arena);
    delete p;
    return CTS_ERR_CUDA;
  }
  *out = p;
  return CTS_OK;
}

cts_status_t cts_plan_free(cts_plan_t p) {
  if (!p) return CTS_ERR_INVALID_ARGUMENT;
  cudaFree(p->arena);
  delete p;
  return CTS_OK;
}

cts_status_t cts_segment(cts_plan_t p, const int32_t* token_adapter, int32_t T, cudaStream_t stream) {
  if (!p || T < 0 || (T > 0 && !token_adapter)) return CTS_ERR_INVALID_ARGUMENT;
  if (T > p->T_max) return CTS_ERR_SHAPE;
  const cts_bank_t b = p->bank;
  SegArgs a;
  a.token_adapter = token_adapter;
  a.tok_adapter_copy = p->tok_adapter;
  a.maps = b->maps;
  a.perm = p->perm;
  a.offsets = p->offsets;
  a.tiles = p->tiles;
  a.n_tiles = p->n_tiles;
  a.tile_rows = p->tile_rows;
  a.tile_adapters = p->tile_adapters;
  a.err = p->err;
  a.unbound_rows = p->unbound_rows;
  a.n_unbound = p->n_unbound;
  a.n_maps = b->n_maps;
  a.T = T;
  a.T_max = p->T_max;
  a.N = b->N;
  a.C = b->C;
  a.max_tiles = p->max_tiles;
  a.pack = tuning().pack;
  static const cudaError_t seg_attr = cudaFuncSetAttribute(
      segment_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (kSegWarps + 3) * 1024 * 4);
  CTS_CUDA(seg_attr);
  CTS_CUDA(launch_pdl(segment_kernel, b->n_maps + 1, kSegThreads, size_t(kSegWarps + 3) * b->C * 4, stream, a));
  p->T = T;
  p->launches_since_segment = 0;
  return CTS_OK;
}

cts_status_t cts_segment_readback(cts_plan_t p, int32_t module, int32_t* perm, int32_t* offsets, int32_t* tiles,
                                  int32_t* n_tiles, cudaStream_t stream) {
  if (!p) return CTS_ERR_INVALID_ARGUMENT;
  const cts_bank_t b = p->bank;
  if (module < 0 || module >= b->n_modules) return CTS_ERR_SHAPE;
  const size_t mid = b->mods[module].map_id;
  CTS_CUDA(cudaStreamSynchronize(stream));
  if (perm && p->T > 0)
    CTS_CUDA(cudaMemcpy(perm, p->perm + mid * p->T_max, size_t(p->T) * 4, cudaMemcpyDeviceToHost));
  if (offsets)
    CTS_CUDA(cudaMemcpy(offsets, p->offsets + mid * (b->C + 1), size_t(b->C + 1) * 4, cudaMemcpyDeviceToHost));
  int32_t ns = 0;
  CTS_CUDA(cudaMemcpy(&ns, p->n_tiles + mid, 4, cudaMemcpyDeviceToHost));
  // slots -> the logical tile list (every tile is one perm range; sorted by start = cluster order)
  std::vector<int4> slots(size_t(ns) * 2);
  if (ns > 0)
    CTS_CUDA(cudaMemcpy(slots.data(), p->tiles + mid * p->max_tiles * 2, size_t(ns) * 32, cudaMemcpyDeviceToHost));
  std::vector<int4> logical;
  for (const int4& t : slots)
    if (t.z > 0) logical.push_back(t);
  std::sort(logical.begin(), logical.end(), [](const int4& a, const int4& b) { return a.y < b.y; });
  if (n_tiles) *n_tiles = static_cast<int32_t>(logical.size());
  if (tiles) {
    for (size_t i = 0; i < logical.size(); ++i) {
      tiles[3 * i] = logical[i].x;
      tiles[3 * i + 1] = logical[i].y;
      tiles[3 * i + 2] = logical[i].z;
    }
  }
  return CTS_OK;
}

cts_status_t cts_shrink_group(cts_plan_t p, int32_t n, const int32_t* modules, const void* const* xs,
                              const int64_t* ld_x, float scale, cudaStream_t stream) {
  cts_status_t st = check_group(p, n, modules, xs, ld_x, true);
  if (st != CTS_OK) return st;
  if (p->T == 0) return CTS_OK;
  return do_shrink(p, n, modules, xs, ld_x, scale, stream);
}

cts_status_t cts_expand_group(cts_plan_t p, int32_t n, const int32_t* modules, void* const* ys, const int64_t* ld_y,
                              cudaStream_t stream) {
  cts_status_t st = check_group(p, n, modules, ys, ld_y, false);
  if (st != CTS_OK) return st;
  if (p->T == 0) return CTS_OK;
  return do_expand(p, n, modules, ys, ld_y, stream);
}

cts_status_t cts_apply_group(cts_plan_t p, int32_t n, const int32_t* modules, const void* const* xs,
                             const int64_t* ld_x, void* const* ys, const int64_t* ld_y, float scale,
                             cudaStream_t stream) {
  cts_status_t st = check_group(p, n, modules, xs, ld_x, true);
  if (st != CTS_OK) return st;
  if ((st = check_group(p, n, modules, ys, ld_y, false)) != CTS_OK) return st;
  const int T = p->T;
  if (T == 0) return CTS_OK;
  // no y may overlap any x or another y of the group (x's may be shared: q, k, v read one x)
  for (int i = 0; i < n; ++i) {
    const Module& mi = p->bank->mods[modules[i]];
    const size_t yb = size_t(T - 1) * ld_y[i] * 2 + mi.d_out * 2;
    for (int j = 0; j < n; ++j) {
      const Module& mj = p->bank->mods[modules[j]];
      const size_t xb = size_t(T - 1) * ld_x[j] * 2 + mj.d_in * 2;
      if (overlaps(ys[i], yb, xs[j], xb)) return CTS_ERR_INVALID_ARGUMENT;
      if (j != i && overlaps(ys[i], yb, ys[j], size_t(T - 1) * ld_y[j] * 2 + mj.d_out * 2))
        return CTS_ERR_INVALID_ARGUMENT;
    }
  }
  if (use_fused()) return do_fused(p, n, modules, xs, ld_x, ys, ld_y, scale, stream);
  if ((st = do_shrink(p, n, modules, xs, ld_x, scale, stream)) != CTS_OK) return st;
  return do_expand(p, n, modules, ys, ld_y, stream);
}

cts_status_t cts_plan_partial_elems(cts_plan_t p, int64_t* elems) {
  if (!p || !elems) return CTS_ERR_INVALID_ARGUMENT;
  *elems = int64_t(p->T_max) * p->bank->rp;
  return CTS_OK;
}

cts_status_t cts_shrink_partial_group(cts_plan_t p, int32_t n, const int32_t* modules, const void* const* xs,
                                      const int64_t* ld_x, float scale, float* const* parts, cudaStream_t stream) {
  cts_status_t st = check_group(p, n, modules, xs, ld_x, true);
  if (st != CTS_OK) return st;
  if (!check_parts(p, n, reinterpret_cast<const void* const*>(parts))) return CTS_ERR_INVALID_ARGUMENT;
  if (p->T == 0) return CTS_OK;
  return do_shrink(p, n, modules, xs, ld_x, scale, stream, parts);
}

cts_status_t cts_expand_reduced_group(cts_plan_t p, int32_t n, const int32_t* modules, const float* const* parts,
                                      void* const* ys, const int64_t* ld_y, cudaStream_t stream) {
  cts_status_t st = check_group(p, n, modules, ys, ld_y, false);
  if (st != CTS_OK) return st;
  if (!check_parts(p, n, reinterpret_cast<const void* const*>(parts))) return CTS_ERR_INVALID_ARGUMENT;
  if (p->T == 0) return CTS_OK;
  if ((st = do_split(p, n, modules, parts, stream)) != CTS_OK) return st;
  return do_expand(p, n, modules, ys, ld_y, stream);
}

cts_status_t cts_comm_unique_id(void* id_out) {
  if (!id_out) return CTS_ERR_INVALID_ARGUMENT;
  const NcclApi& api = nccl();
  if (!api.ok) return CTS_ERR_NCCL;
  NcclId id;
  if (api.get_unique_id(&id) != 0) return CTS_ERR_NCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return CTS_OK;
}

cts_status_t cts_comm_create(const void* nccl_unique_id, int32_t nranks, int32_t rank, cts_comm_t* out) {
  if (!out) return CTS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (!nccl_unique_id || nranks < 1 || rank < 0 || rank >= nranks) return CTS_ERR_INVALID_ARGUMENT;
  const NcclApi& api = nccl();
  if (!api.ok) return CTS_ERR_NCCL;
  NcclId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  auto* c = new (std::nothrow) cts_comm_s();
  if (!c) return CTS_ERR_OUT_OF_MEMORY;
  c->nranks = nranks;
  c->rank = rank;
  if (api.comm_init_rank(&c->comm, nranks, id, rank) != 0) {
    delete c;
    return CTS_ERR_NCCL;
  }
  *out = c;
  return CTS_OK;
}

cts_status_t cts_comm_free(cts_comm_t c) {
  if (!c) return CTS_ERR_INVALID_ARGUMENT;
  const NcclApi& api = nccl();
  const int rc = api.ok ? api.comm_destroy(c->comm) : 1;
  delete c;
  return rc == 0 ? CTS_OK : CTS_ERR_NCCL;
}

cts_status_t cts_apply_tp(cts_plan_t p, int32_t n, const int32_t* modules, const void* const* xs, const int64_t* ld_x,
                          void* const* ys, const int64_t* ld_y, float scale, cts_comm_t comm, cudaStream_t stream) {
  if (!comm) return CTS_ERR_INVALID_ARGUMENT;
  cts_status_t st = check_group(p, n, modules, xs, ld_x, true);
  if (st != CTS_OK) return st;
  if ((st = check_group(p, n, modules, ys, ld_y, false)) != CTS_OK) return st;
  if (p->T == 0) return CTS_OK;
  const NcclApi& api = nccl();
  if (!api.ok) return CTS_ERR_NCCL;
  const int rp = p->bank->rp;
  float* parts[kMaxGroup];
  for (int i = 0; i < n; ++i) parts[i] = p->tp_parts + size_t(i) * p->T_max * rp;
  if ((st = do_shrink(p, n, modules, xs, ld_x, scale, stream, parts)) != CTS_OK) return st;
  if (api.group_start() != 0) return CTS_ERR_NCCL;
  for (int i = 0; i < n; ++i)
    if (api.all_reduce(parts[i], parts[i], size_t(p->T) * rp, /*ncclFloat32*/ 7, /*ncclSum*/ 0, comm->comm, stream) != 0) {
      api.group_end();
      return CTS_ERR_NCCL;
    }
  if (api.group_end() != 0) return CTS_ERR_NCCL;
  if ((st = do_split(p, n, modules, parts, stream)) != CTS_OK) return st;
  return do_expand(p, n, modules, ys, ld_y, stream);
}

cts_status_t cts_shrink(cts_plan_t p, int32_t module, const void* x, int64_t ld_x, float scale, cudaStream_t stream) {
  return cts_shrink_group(p, 1, &module, &x, &ld_x, scale, stream);
}

cts_status_t cts_expand(cts_plan_t p, int32_t module, void* y, int64_t ld_y, cudaStream_t stream) {
  return cts_expand_group(p, 1, &module, &y, &ld_y, stream);
}

cts_status_t cts_apply(cts_plan_t p, int32_t module, const void* x, int64_t ld_x, void* y, int64_t ld_y, float scale,
                       cudaStream_t stream) {
  return cts_apply_group(p, 1, &module, &x, &ld_x, &y, &ld_y, scale, stream);
}

cts_status_t cts_project(cts_plan_t p, int32_t module, const void* x, int64_t ld_x, const void* w0, int64_t ld_w,
                         void* y, int64_t ld_y, float scale, cudaStream_t stream) {
  if (!p || !w0 || (p->T > 0 && (!x || !y))) return CTS_ERR_INVALID_ARGUMENT;
  const cts_bank_t b = p->bank;
  if (module < 0 || module >= b->n_modules) return CTS_ERR_SHAPE;
  if (b->rp != 16) return CTS_ERR_UNSUPPORTED;
  const Module& m = b->mods[module];
  if (m.d_out % kProjBN || m.d_in % kBK) return CTS_ERR_UNSUPPORTED;
  if (ld_x < m.d_in || ld_w < m.d_in || ld_y < m.d_out || (ld_x * 2) % 16 || (ld_w * 2) % 16 || (ld_y * 2) % 16 ||
      !aligned16(x) || !aligned16(w0) || !aligned16(y))
    return CTS_ERR_SHAPE;
  const size_t nx = size_t(p->T) * ld_x * 2, nw = size_t(m.d_out) * ld_w * 2, ny = size_t(p->T) * ld_y * 2;
  if (p->T > 0 && (overlaps(y, ny, x, nx) || overlaps(y, ny, w0, nw))) return CTS_ERR_INVALID_ARGUMENT;
  if (p->T == 0) return CTS_OK;
  return launch_project(p, module, x, ld_x, w0, ld_w, y, ld_y, scale, stream);
}

cts_status_t cts_jd_workspace_bytes(const cts_jd_problem_t* problems, int32_t count, int32_t r, size_t* bytes) {
  if (!problems || count < 0 || !bytes) return CTS_ERR_INVALID_ARGUMENT;
  size_t f = 0;
  for (int i = 0; i < count; ++i) f += jd_problem_floats(problems[i], r);
  *bytes = f * 4;
  return CTS_OK;
}

cts_status_t cts_jd_eigen_iteration(const cts_jd_problem_t* problems, int32_t count, int32_t r, int32_t iters,
                                    void* workspace, size_t ws_bytes, cudaStream_t stream) {
  if (!problems || count < 0 || iters < 0 || (count > 0 && !workspace)) return CTS_ERR_INVALID_ARGUMENT;
  if (r != 8 && r != 16 && r != 32 && r != 64) return CTS_ERR_UNSUPPORTED;
  size_t need = 0;
  cts_status_t st = cts_jd_workspace_bytes(problems, count, r, &need);
  if (st != CTS_OK) return st;
  if (ws_bytes < need || !aligned16(workspace)) return CTS_ERR_SHAPE;
  for (int i = 0; i < count; ++i) {
    const cts_jd_problem_t& q = problems[i];
    if (!q.a_stack || !q.bt_stack || !q.U || !q.V || !q.sigma) return CTS_ERR_INVALID_ARGUMENT;
    if (q.n < 1 || q.r_i < 1 || q.d_in < r || q.d_out < r || q.d_in % 4 || q.d_out % 4) return CTS_ERR_SHAPE;
    if (!aligned16(q.a_stack) || !aligned16(q.bt_stack) || !aligned16(q.U) || !aligned16(q.V)) return CTS_ERR_SHAPE;
  }
  float* ws = static_cast<float*>(workspace);
  switch (r) {
    case 8: return jd_run<8>(problems, count, iters, ws, stream);
    case 16: return jd_run<16>(problems, count, iters, ws, stream);
    case 32: return jd_run<32>(problems, count, iters, ws, stream);
    default: return jd_run<64>(problems, count, iters, ws, stream);
  }
}

cts_status_t cts_route(const int32_t* token_adapter, int32_t T, const int32_t* owner, int32_t N, int32_t world,
                       int32_t self, int32_t* perm, int32_t* counts, cudaStream_t stream) {
  if (T < 0 || N < 1 || world < 1 || world > 64 || self < 0 || self >= world || !owner || !counts ||
      (T > 0 && (!token_adapter || !perm)))
    return CTS_ERR_INVALID_ARGUMENT;
  RouteArgs a{token_adapter, owner, perm, counts, T, N, world, self};
  route_kernel<<<1, kSegThreads, 0, stream>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  CTS_CUDA(cudaGetLastError());
  return CTS_OK;
}

cts_status_t cts_rows_move(const void* src, int64_t ld_src, void* dst, int64_t ld_dst, const int32_t* idx, int32_t n,
                           int32_t row_bytes, int32_t scatter, cudaStream_t stream) {
  if (n < 0 || row_bytes < 4 || (n > 0 && (!src || !dst || !idx))) return CTS_ERR_INVALID_ARGUMENT;
  if (row_bytes % 4 || ld_src < row_bytes || ld_dst < row_bytes || ld_src % 4 || ld_dst % 4 ||
      reinterpret_cast<uintptr_t>(src) % 4 || reinterpret_cast<uintptr_t>(dst) % 4)
    return CTS_ERR_SHAPE;
  if (n == 0) return CTS_OK;
  RowsArgs a{static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), idx, ld_src, ld_dst, n, row_bytes,
             scatter ? 1 : 0};
  const bool v16 = row_bytes % 16 == 0 && ld_src % 16 == 0 && ld_dst % 16 == 0 && aligned16(src) && aligned16(dst);
  const int64_t chunks = int64_t(n) * (row_bytes / (v16 ? 16 : 4));
  const int grid = static_cast<int>(std::min<int64_t>(8 * sm_count(), (chunks + 255) / 256));
  if (v16) rows_move_kernel<uint4><<<grid, 256, 0, stream>>>(a);
  else rows_move_kernel<uint32_t><<<grid, 256, 0, stream>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  CTS_CUDA(cudaGetLastError());
  return CTS_OK;
}

#ifdef CTS_TRACE
// debug-only (not part of cts.h): copy the per-CTA timeline of the last traced launch
int cts_debug_trace(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_cts_trace, std::min<size_t>(n, sizeof(g_cts_trace) / 8) * 8) == cudaSuccess ? 0 : 1;
}
#endif

cts_status_t cts_plan_error(cts_plan_t p, int32_t* code, int32_t* first_bad_token) {
  if (!p || !code || !first_bad_token) return CTS_ERR_INVALID_ARGUMENT;
  int32_t e[2];
  CTS_CUDA(cudaMemcpy(e, p->err, 8, cudaMemcpyDeviceToHost));
  *code = e[0];
  *first_bad_token = e[1];
  return CTS_OK;
}

}  // extern "C"
