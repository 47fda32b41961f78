// Microbenchmark: how fast can one persistent CTA per SM stream token rows with TMA?
// Modes: 0 = tile box {64 cols, 128 rows}, 1 = gather4 of 4 consecutive rows, 2 = gather4 of
// randomly permuted rows (the shrink's access pattern), 3 = plain LDG.128 by 256 threads.
// Stage = 128 rows x (64*KB) cols; KB boxes per stage.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_gather_bench tma_gather_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include "../../paper_2407_00066_b200/csrc/sm100.cuh"

using namespace cts;

constexpr int ROWS = 131072, COLS = 4096;   // 1 GiB of bf16: steady state dominates

template <int KB, int STAGES>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm_tile,
                                                        const __grid_constant__ CUtensorMap tm_g, const int* perm,
                                                        int mode, int n_items, unsigned long long* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStage = 128 * 128 * KB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStage);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int kblocks_per_tile = COLS / (64 * KB);
  if (warp == 0) {
    int stage = 0; uint32_t phase = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int tile = item / kblocks_per_tile, kb = item % kblocks_per_tile;
      int r4[4];
      for (int q = 0; q < 4; ++q) r4[q] = (mode == 2) ? perm[tile * 128 + 4 * lane + q] : tile * 128 + 4 * lane + q;
      mbar_wait(&empty[stage], phase ^ 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[stage], kStage);
      __syncwarp();
      uint8_t* dst = smem + stage * kStage;
      for (int b = 0; b < KB; ++b) {
        const int col = (kb * KB + b) * 64;
        if (mode == 0) {
          if (lane == 0) tma_load_2d(dst + b * 16384, &tm_tile, &full[stage], col, tile * 128);
        } else {
          tma_gather4(dst + b * 16384 + lane * 512, &tm_g, &full[stage], col, r4[0], r4[1], r4[2], r4[3]);
        }
      }
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  } else {
    int stage = 0; uint32_t phase = 0;
    unsigned long long acc = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      mbar_wait(&full[stage], phase);
      acc += smem[stage * kStage + lane * 64];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    if (lane == 0) atomicAdd(sink, acc);
  }
}


template <int KB, int STAGES, int P>
__global__ void __launch_bounds__(32 * (P + 1), 1) mp_kernel(const __grid_constant__ CUtensorMap tm_g, const int* perm,
                                                             int mode, int n_items, unsigned long long* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStage = 128 * 128 * KB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStage);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int kblocks_per_tile = COLS / (64 * KB);
  if (warp < P) {
    // producer warp `warp` handles every P-th local item
    int li = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++li) {
      if (li % P != warp) continue;
      const int stage = li % STAGES;
      const uint32_t phase = (li / STAGES) & 1;
      const int tile = item / kblocks_per_tile, kb = item % kblocks_per_tile;
      int r4[4];
      for (int q = 0; q < 4; ++q) r4[q] = (mode == 2) ? perm[tile * 128 + 4 * lane + q] : tile * 128 + 4 * lane + q;
      mbar_wait(&empty[stage], phase ^ 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[stage], kStage);
      __syncwarp();
      uint8_t* dst = smem + stage * kStage;
      for (int b = 0; b < KB; ++b)
        tma_gather4(dst + b * 16384 + lane * 512, &tm_g, &full[stage], (kb * KB + b) * 64, r4[0], r4[1], r4[2], r4[3]);
    }
  } else {
    int stage = 0; uint32_t phase = 0;
    unsigned long long acc = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      mbar_wait(&full[stage], phase);
      acc += smem[stage * kStage + lane * 64];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    if (lane == 0) atomicAdd(sink, acc);
  }
}

__global__ void ldg_kernel(const uint4* x, const int* perm, int mode, unsigned long long* sink) {
  // each CTA streams whole 128-row bands with 16-byte loads, rows permuted in mode 5
  unsigned long long acc = 0;
  const int vec_per_row = COLS * 2 / 16;
  for (int tile = blockIdx.x; tile < ROWS / 128; tile += gridDim.x) {
    for (int i = threadIdx.x; i < 128 * vec_per_row; i += blockDim.x) {
      const int r = i / vec_per_row, c = i % vec_per_row;
      const int row = mode == 5 ? perm[tile * 128 + r] : tile * 128 + r;
      uint4 v = __ldg(x + size_t(row) * vec_per_row + c);
      acc += v.x ^ v.w;
    }
  }
  if (acc == 0x12345) atomicAdd(sink, acc);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<EncodeFn>(fnp);
  __nv_bfloat16* x;
  cudaMalloc(&x, size_t(ROWS) * COLS * 2);
  cudaMemset(x, 1, size_t(ROWS) * COLS * 2);
  std::vector<int> h(ROWS);
  for (int i = 0; i < ROWS; ++i) h[i] = i;
  std::mt19937 rng(1);
  std::shuffle(h.begin(), h.end(), rng);
  int* perm;
  cudaMalloc(&perm, ROWS * 4);
  cudaMemcpy(perm, h.data(), ROWS * 4, cudaMemcpyHostToDevice);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  CUtensorMap tm_tile, tm_g;
  cuuint64_t dims[2] = {COLS, ROWS}, strides[1] = {COLS * 2};
  cuuint32_t box_t[2] = {64, 128}, box_g[2] = {64, 1}, es[2] = {1, 1};
  enc(&tm_tile, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box_t, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tm_g, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box_g, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  // flush buffer
  void* flush;
  cudaMalloc(&flush, 256ull << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto kern, int kb, int stages, int mode, int grid) {
    const int smem = stages * 128 * 128 * kb + 2 * stages * 8 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int items = (ROWS / 128) * (COLS / (64 * kb));
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemset(flush, it, 256ull << 20);
      cudaEventRecord(a);
      kern<<<grid, 64, smem>>>(tm_tile, tm_g, perm, mode, items, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = std::min(best, ms);
    }
    const double gbs = double(ROWS) * COLS * 2 / (best * 1e-3) / 1e9;
    printf("mode=%d (%s) KB=%d stages=%d grid=%d: %.1f us  %.0f GB/s  err=%s\n", mode,
           mode == 0 ? "tile" : (mode == 1 ? "gather4-contig" : "gather4-perm"), kb, stages, grid, best * 1e3, gbs,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(stream_kernel<1, 8>, 1, 8, 0, 148);
  run(stream_kernel<2, 6>, 2, 6, 0, 148);
  run(stream_kernel<1, 8>, 1, 8, 2, 148);
  for (int mode : std::vector<int>{}) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemset(flush, it, 256ull << 20);
      cudaEventRecord(a);
      ldg_kernel<<<148 * 4, 512>>>(reinterpret_cast<const uint4*>(x), perm, mode, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = std::min(best, ms);
    }
    printf("mode=%d (ldg %s): %.1f us %.0f GB/s\n", mode, mode == 4 ? "contig" : "perm", best * 1e3,
           double(ROWS) * COLS * 2 / (best * 1e-3) / 1e9);
  }

  auto runmp = [&](auto kern, int kb, int stages, int P, int mode, int grid) {
    const int smem = stages * 128 * 128 * kb + 2 * stages * 8 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int items = (ROWS / 128) * (COLS / (64 * kb));
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemset(flush, it, 256ull << 20);
      cudaEventRecord(a);
      kern<<<grid, 32 * (P + 1), smem>>>(tm_g, perm, mode, items, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = std::min(best, ms);
    }
    printf("MP mode=%d KB=%d stages=%d P=%d grid=%d: %.1f us  %.0f GB/s  err=%s\n", mode, kb, stages, P, grid, best * 1e3,
           double(ROWS) * COLS * 2 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int mode = 1; mode < 3; ++mode) {
    runmp(mp_kernel<1, 8, 4>, 1, 8, 4, mode, 148);
    runmp(mp_kernel<1, 12, 8>, 1, 12, 8, mode, 148);
    runmp(mp_kernel<1, 6, 4>, 1, 6, 4, mode, 296);
    runmp(mp_kernel<1, 6, 8>, 1, 6, 8, mode, 296);
  }
  return 0;
}
