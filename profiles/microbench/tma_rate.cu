// Microbenchmark (round 2): per-SM TMA row-gather throughput on B200, to size the decode redesign.
// One CTA per SM, W producer warps each lane issuing tile::gather4 (4 random rows x box width) into a
// ring of stages, one consumer warp releasing stages.  Source either L2-resident (32 MB) or
// DRAM-sized (2 GB).  Reports GB/s per SM and for the whole GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_rate tma_rate.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include "../../paper_2407_00066_b200/csrc/sm100.cuh"

using namespace cts;

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void __launch_bounds__(32 * 13, 1) gather_kernel(const __grid_constant__ CUtensorMap tm, const int* rows,
                                                          int n_rows_src, int W, int box_bytes, int stages,
                                                          int jobs_per_cta, int tile_mode, const __nv_bfloat16* gsrc, unsigned long long* sink, int pat) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = 128 * box_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], tile_mode == 2 ? 32 : 1); mbar_init(&empty[s], 1); }
    // tile_mode 3: one warp produces a whole stage with plain 32-byte loads (full count 1)
    fence_barrier_init();
  }
  __syncthreads();
  if (warp < W) {
    for (int j = warp; j < jobs_per_cta; j += W) {
      const int stage = j % stages;
      const uint32_t phase = (j / stages) & 1;
      mbar_wait(&empty[stage], phase ^ 1);
      if (tile_mode < 2 && lane == 0) mbar_arrive_expect_tx(&full[stage], stage_bytes);
      __syncwarp();
      uint8_t* dst = smem + stage * stage_bytes;
      // pat 1 (the decode shrink's order): the same 128 rows for 21 consecutive column blocks
      const int jj = pat ? j / 21 : j;
      const int base = ((blockIdx.x * 7919 + jj * 131) % (n_rows_src / 128)) * 128;
      // DRAM-sized source: also walk the column blocks, so the touched footprint is the whole
      // source (round-2 session 3 fix: with column 0 only, a "DRAM" run touched 32-64 MB = L2)
      const int ncb = 4096 / (box_bytes / 2);
      const int col = n_rows_src <= 4096 ? 0
                      : (pat ? ((j % 21) + 21 * (jj % 3)) % ncb : (blockIdx.x * 7 + j * 13) % ncb) * (box_bytes / 2);
      if (tile_mode == 3) {
        // plain loads into registers: 4 lanes per 128-byte row segment (ld.global.v8, 32 B each),
        // 8 rows per instruction, 8 instructions in flight, then 16-byte stores at the 128B-swizzled
        // offsets; one arrival per stage
        const int sub = lane & 3, r8 = lane >> 2;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          uint4 v[8][2];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int rr = h * 64 + u * 8 + r8;
            const int row = rows[base + rr];
            const uint8_t* src = reinterpret_cast<const uint8_t*>(gsrc) + (static_cast<size_t>(row) * 4096 + col) * 2 + sub * 32;
            ld_global_nc_v8(src, v[u][0], v[u][1]);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int rr = h * 64 + u * 8 + r8;
            *reinterpret_cast<uint4*>(dst + rr * 128 + (((2 * sub) ^ (rr & 7)) * 16)) = v[u][0];
            *reinterpret_cast<uint4*>(dst + rr * 128 + (((2 * sub + 1) ^ (rr & 7)) * 16)) = v[u][1];
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[stage]);
      } else if (tile_mode == 2) {
        // cp.async (LDGSTS) 16-byte pieces of the same 128 random rows x box_bytes, each placed at
        // its 128B-swizzled offset (as an MMA A tile would need); completion via the mbarrier
        const int chunks_per_row = box_bytes / 16;
        for (int i = lane; i < 128 * chunks_per_row; i += 32) {
          const int rr = i / chunks_per_row, ch = i % chunks_per_row;
          const int row = rows[base + rr];
          const uint8_t* src = reinterpret_cast<const uint8_t*>(gsrc) + (static_cast<size_t>(row) * 4096 + col) * 2 + ch * 16;
          const int off = rr * box_bytes + ((ch ^ (rr & 7)) * 16);
          cp_async16(dst + off, src);
        }
        cp_async_mbar_arrive(&full[stage]);
      } else if (tile_mode) {
        if (lane == 0) tma_load_2d(dst, &tm, &full[stage], col, base);
      } else {
        const int4 r = *reinterpret_cast<const int4*>(rows + base + 4 * lane);
        tma_gather4(dst + lane * 4 * box_bytes, &tm, &full[stage], col, r.x, r.y, r.z, r.w);
      }
    }
  } else if (warp == W) {
    unsigned long long acc = 0;
    for (int j = 0; j < jobs_per_cta; ++j) {
      const int stage = j % stages;
      mbar_wait(&full[stage], (j / stages) & 1);
      acc += smem[stage * stage_bytes + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
    }
    if (lane == 0) atomicAdd(sink, acc);
  }
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<EncodeTiledFn>(p);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int COLS = 4096;
  const int pat = getenv("PAT") ? atoi(getenv("PAT")) : 0;
  for (long long src_rows : {4096LL, 262144LL}) {          // 32 MB (L2) / 2 GB (DRAM)
    __nv_bfloat16* x = nullptr;
    cudaMalloc(&x, src_rows * COLS * 2);
    cudaMemset(x, 1, src_rows * COLS * 2);
    std::vector<int> h(src_rows);
    for (long long i = 0; i < src_rows; ++i) h[i] = int(i);
    std::mt19937 g(1);
    std::shuffle(h.begin(), h.end(), g);
    int* rows = nullptr;
    cudaMalloc(&rows, src_rows * 4);
    cudaMemcpy(rows, h.data(), src_rows * 4, cudaMemcpyHostToDevice);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    struct Mode { const char* name; int box; CUtensorMapSwizzle sw; int tile; };
    Mode modes[] = {{"gather4 64col SW128 (512B/op)", 64, CU_TENSOR_MAP_SWIZZLE_128B, 0},
                    {"gather4 128col noswz (1KB/op)", 128, CU_TENSOR_MAP_SWIZZLE_NONE, 0},
                    {"gather4 256col noswz (2KB/op)", 256, CU_TENSOR_MAP_SWIZZLE_NONE, 0},
                    {"tile 64colx128row SW128 (16KB/op)", 64, CU_TENSOR_MAP_SWIZZLE_128B, 1},
                    {"cp.async 16B x 128 rows x 128B", 64, CU_TENSOR_MAP_SWIZZLE_128B, 2},
                    {"cp.async 16B x 128 rows x 256B", 128, CU_TENSOR_MAP_SWIZZLE_NONE, 2},
                    {"ldg 32B x 4 lanes per 128B row", 64, CU_TENSOR_MAP_SWIZZLE_128B, 3}};
    for (const Mode& m : modes) {
      CUtensorMap tm;
      cuuint64_t dims[2] = {cuuint64_t(COLS), cuuint64_t(src_rows)};
      cuuint64_t strides[1] = {cuuint64_t(COLS) * 2};
      cuuint32_t box[2] = {cuuint32_t(m.box), cuuint32_t(m.tile == 1 ? 128 : 1)};
      cuuint32_t es[2] = {1, 1};
      CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, m.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", m.name, int(r)); continue; }
      const int box_bytes = m.box * 2;
      const int stage_bytes = 128 * box_bytes;
      const int stages = std::max(2, (200 * 1024) / stage_bytes);
      const int smem = stages * stage_bytes + 1024 + 2 * stages * 8 + 64;
      cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      for (int W : {1, 2, 3, 4, 6, 8, 12}) {
        if (m.tile != 3 && W > 8) continue;
        if (m.tile == 3 ? W + 2 > stages : 2 * W > stages) continue;
        const long long total_bytes = (src_rows == 4096 ? 4LL : 8LL) << 30;
        const int jobs = int(total_bytes / stage_bytes / sms);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        gather_kernel<<<sms, 32 * (W + 1), smem>>>(tm, rows, int(src_rows), W, box_bytes, stages, 4, m.tile, x, sink, pat);
        cudaEventRecord(a);
        gather_kernel<<<sms, 32 * (W + 1), smem>>>(tm, rows, int(src_rows), W, box_bytes, stages, jobs, m.tile, x, sink, pat);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = double(jobs) * stage_bytes * sms;
        printf("pat%d %-36s src=%s W=%d stages=%d: %8.1f GB/s total, %6.1f GB/s per SM  (%s)\n", pat, m.name,
               src_rows == 4096 ? "L2  " : "DRAM", W, stages, bytes / ms / 1e6, bytes / ms / 1e6 / sms,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
    cudaFree(x); cudaFree(rows); cudaFree(sink);
  }
  return 0;
}
