// jd_tc.cuh -- the four thin GEMMs of the App A.2 eigenvalue iteration (jd_eigen.cuh) on the
// 5th-generation tensor cores, fp32-accurate by the 3xTF32 split.
//
// Why tensor cores: per iteration one layer moves ~10.5 GB of fp32 LoRA factors through 84 GFLOP
// (8 FLOP/B), above the fp32 CUDA-core ridge (~36 TFLOP/s / 6.5 TB/s = 5.5 FLOP/B on B200: FFMA
// issues at one per 2 cycles per SMSP), so the CUDA-core kernels are compute-bound.  tcgen05
// kind::tf32 runs ~1.1 PFLOP/s dense; three MMAs per product keep fp32 accuracy:
//     x = hi + lo,  hi = x with the low 13 mantissa bits cleared (exactly a tf32 value),
//     lo = x - hi (exact in fp32, then read as tf32: relative error 2^-11 of lo, ~2^-21 of x),
//     X Y^T ~= X_hi Y_hi^T + X_hi Y_lo^T + X_lo Y_hi^T      (fp32 accumulation in TMEM)
// (the dropped X_lo Y_lo^T term is ~2^-22 relative).  The Y_hi and Y_lo tiles are adjacent in shared
// memory, so ONE MMA of N = 2R gives [X_hi Y_hi^T | X_hi Y_lo^T] and a second (N = R) adds X_lo Y_hi^T
// into the first half: X_hi is read once per K step, and the epilogue adds the two halves.
//
// Every GEMM is written D[M][R] = X[M][Kd] * Y[R][Kd]^T with BOTH operands K-major (row-major in
// memory, the reduction index contiguous), so the cts_jd driver keeps transposed copies where the
// paper's product reduces over a row index: P = A V -> (X = A, Y = V^T); Q = Bt U -> (Bt, U^T);
// U0 = Bt^T W -> (Bt^T, W^T); V0 = A^T Z -> (A^T, Z^T).  A^T and Bt^T are formed once per call.
//
// Persistent kernel over a flat tile list ((job, 128-row tile) entries), 10 warps:
//   warp 0       TMA producer (one lane): X tile {32 fp32, 128 rows} and Y tile {32, R}, 128B swizzle
//   warps 1-4    split: lo = x - hi into a second buffer (hi = the MMA's own tf32 read of x), fence.proxy.async
//   warp 5       MMA issuer: per 32-wide K block 4 k-steps x 2 tcgen05.mma.kind::tf32 (M=128, N=2R and R)
//   warps 6-9    epilogue: tcgen05.ld the 2R accumulator columns (thread = row), add halves, store D rows
// Two TMEM accumulators so a tile's epilogue overlaps the next tile's MMAs.  Deterministic.
#pragma once
#include <cstdint>
#include "sm100.cuh"

namespace cts {

struct JdTcJob {
  const CUtensorMap* tm_x;     // X [M][Kd] fp32, box {32, 128}, 128B swizzle
  const CUtensorMap* tm_y;     // Y [N][Kd] fp32, box {32, R}, 128B swizzle
  float* D;                    // [M][ldD]
  int M, Kd;
  int N, ldD;                  // rows of Y (columns of D); thin GEMMs: N = ldD = R
};

struct JdTcParams {
  const JdTcJob* jobs;
  const int4* tiles;           // (job, first row of X, first row of Y = first column of D, mirror)
  int n_tiles;
};

// One ring; a stage holds X (hi after the split, in place), its X_lo, Y_hi and Y_lo (Y_lo follows
// Y_hi: one N = 2R operand).  (A separate 3-slot X_lo ring under a 7-stage TMA ring measured slower:
// 41 vs 36 ms per layer -- the split then waits on MMA completions.)
template <int R>
struct JdTcCfg {
  static constexpr int kX = 128 * 128;                 // X tile: 128 rows x 128 B
  static constexpr int kY = R * 128;                   // Y tile: R rows x 128 B
  static constexpr int kStage = 2 * kX + 2 * kY;       // X, X_lo, Y_hi, Y_lo
  static constexpr int kStages = (200 * 1024) / kStage < 6 ? (200 * 1024) / kStage : 6;
  static constexpr int kNumBars = 3 * kStages + 4;
  static constexpr int kOffBar = kStages * kStage;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kBytes = kOffMisc + 64 + 1024;
  static constexpr uint32_t kTmemCols = 4 * R < 32 ? 32 : 4 * R;   // two accumulators of 2R columns
};

// Instruction descriptor, kind::tf32: A, B tf32, D f32, both K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_tf32(uint32_t M, uint32_t N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ float4 tf32_hi(float4 v) {
  return make_float4(__uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u),
                     __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u),
                     __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u),
                     __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
}

// The tensor core reads an fp32 value as tf32 by ignoring its 13 low mantissa bits (the reason
// cvt.rna.tf32.f32 exists), i.e. it already sees X_hi; writing X_hi back is only needed if that
// changed.  Default 0: measured 4% faster, App A.2 parity unchanged (test_gpu_jd_eigen_iteration).
#ifndef CTS_JD_HI_INPLACE
#define CTS_JD_HI_INPLACE 0
#endif

template <int R>
__global__ void __launch_bounds__(320, 1) jd_tc_gemm(const __grid_constant__ JdTcParams p) {
  using L = JdTcCfg<R>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* split = full + L::kStages;
  uint64_t* empty = split + L::kStages;
  uint64_t* acc_full = empty + L::kStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kOffMisc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto stage_x = [&](int s) { return smem + s * L::kStage; };
  auto stage_xlo = [&](int s) { return smem + s * L::kStage + L::kX; };
  auto stage_y = [&](int s) { return smem + s * L::kStage + 2 * L::kX; };
  auto stage_ylo = [&](int s) { return smem + s * L::kStage + 2 * L::kX + L::kY; };

  if (warp == 0) {                                          // ---------------- TMA producer
    int it = 0;
    for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
      const int4 tl = p.tiles[t];
      const JdTcJob& j = p.jobs[tl.x];
      const int nkb = (j.Kd + 31) / 32;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % L::kStages;
        const uint32_t ph = (it / L::kStages) & 1;
        if (lane == 0) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], L::kX + L::kY);
          tma_load_2d(stage_x(s), j.tm_x, &full[s], kb * 32, tl.y);
          tma_load_2d(stage_y(s), j.tm_y, &full[s], kb * 32, tl.z);
        }
        __syncwarp();
      }
    }
  } else if (warp <= 4) {                                   // ---------------- hi / lo split
    const int tid = threadIdx.x - 32;                       // 0..127
    int it = 0;
    for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
      const JdTcJob& j = p.jobs[p.tiles[t].x];
      const int nkb = (j.Kd + 31) / 32;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % L::kStages;
        const uint32_t ph = (it / L::kStages) & 1;
        mbar_wait(&full[s], ph);
        float4* x = reinterpret_cast<float4*>(stage_x(s));
        float4* xl = reinterpret_cast<float4*>(stage_xlo(s));
#pragma unroll 4
        for (int i = tid; i < L::kX / 16; i += 128) {
          const float4 v = x[i], h = tf32_hi(v);
          if (CTS_JD_HI_INPLACE) x[i] = h;                  // else the MMA's own tf32 read of x
          xl[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
        float4* y = reinterpret_cast<float4*>(stage_y(s));
        float4* yl = reinterpret_cast<float4*>(stage_ylo(s));
        for (int i = tid; i < L::kY / 16; i += 128) {
          const float4 v = y[i], h = tf32_hi(v);
          if (CTS_JD_HI_INPLACE) y[i] = h;                  // else the MMA's own tf32 read of y
          yl[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
        fence_proxy_async_smem();                           // generic writes -> tensor-core reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&split[s]);
      }
    }
  } else if (warp == 5) {                                   // ---------------- MMA issuer
    constexpr uint32_t idesc2 = umma_idesc_tf32(128, 2 * R), idesc = umma_idesc_tf32(128, R);
    int it = 0, tile_i = 0;
    for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++tile_i) {
      const JdTcJob& j = p.jobs[p.tiles[t].x];
      const int nkb = (j.Kd + 31) / 32;
      const int slot = tile_i & 1;
      mbar_wait(&acc_empty[slot], ((tile_i >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t acc = tmem + slot * 2 * R;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % L::kStages;
        const uint32_t ph = (it / L::kStages) & 1;
        mbar_wait(&split[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t xh = smem_u32(stage_x(s)), xl = smem_u32(stage_xlo(s));
          const uint32_t yh = smem_u32(stage_y(s)), yl = smem_u32(stage_ylo(s));
#pragma unroll
          for (int k = 0; k < 4; ++k) {                     // K = 8 tf32 (32 bytes) per MMA
            const uint32_t first = (kb == 0 && k == 0) ? 0u : 1u;
            (void)yl;                                       // Y_lo rows follow Y_hi: one N = 2R operand
            umma_tf32(acc, umma_desc_kmajor(xh + k * 32, 128), umma_desc_kmajor(yh + k * 32, 128), idesc2, first);
            umma_tf32(acc, umma_desc_kmajor(xl + k * 32, 128), umma_desc_kmajor(yh + k * 32, 128), idesc, 1);
          }
          umma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) umma_commit(&acc_full[slot]);
      __syncwarp();
    }
  } else {                                                  // ---------------- epilogue (warps 6-9)
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    int tile_i = 0;
    for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++tile_i) {
      const int4 tl = p.tiles[t];
      const JdTcJob& j = p.jobs[tl.x];
      const int slot = tile_i & 1;
      mbar_wait(&acc_full[slot], (tile_i >> 1) & 1);
      tc_fence_after();
      const uint32_t ta = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + slot * 2 * R;
      const int m = tl.y + row;
      const int ncols = min(R, j.N - tl.z);                 // Gram tiles: the last column block is partial
      float* drow = j.D + static_cast<size_t>(m) * j.ldD + tl.z;
      constexpr int kC = R < 32 ? R : 32;                   // accumulator columns per TMEM load
#pragma unroll 1
      for (int c0 = 0; c0 < R; c0 += kC) {
        float v[kC], w[kC];
#pragma unroll
        for (int c = 0; c < kC; c += 16) {
          tmem_ld16(ta + c0 + c, v + c);
          tmem_ld16(ta + R + c0 + c, w + c);
        }
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < kC; ++c) v[c] += w[c];          // X_hi Y_hi + X_lo Y_hi  +  X_hi Y_lo
        if (m < j.M) {
          if (c0 + kC <= ncols && (j.ldD & 3) == 0) {
            float4* dst = reinterpret_cast<float4*>(drow + c0);
#pragma unroll
            for (int c = 0; c < kC / 4; ++c) dst[c] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          } else {
#pragma unroll
            for (int c = 0; c < kC; ++c)
              if (c0 + c < ncols) drow[c0 + c] = v[c];
          }
          if (tl.w) {                                       // symmetric Gram: the mirrored tile too
#pragma unroll
            for (int c = 0; c < kC; ++c)                    // lanes = consecutive m: coalesced
              if (c0 + c < ncols) j.D[static_cast<size_t>(tl.z + c0 + c) * j.ldD + m] = v[c];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[slot]);
    }
  }
  __syncthreads();
  if (warp == 5) tmem_dealloc<L::kTmemCols>(tmem);
}

// Batched transposes for the K-major operands: out[c][r] = in[r][c] of a rows x cols fp32 matrix
// (32 x 32 tiles through shared memory; blockIdx.z = matrix).
struct JdTransposeJob {
  const float* in;
  float* out;
  int rows, cols;
};
constexpr int kJdMaxTranspose = 512;
struct JdTransposeBatch {
  JdTransposeJob j[kJdMaxTranspose];
};

__global__ void __launch_bounds__(256) jd_transpose(const JdTransposeBatch* __restrict__ b, int count) {
  // 64 x 64 tiles: 16-byte global loads along input rows, 16-byte global stores along output rows,
  // the turn through a padded shared tile (conflict-free scalar accesses)
  __shared__ float tile[64][65];
  const int tq = threadIdx.x & 15, tr = threadIdx.x >> 4;        // 16 float4 columns x 16 rows
  for (int z = blockIdx.z; z < count; z += gridDim.z) {
    const JdTransposeJob jb = b->j[z];
    const int tiles_c = (jb.cols + 63) / 64, tiles_r = (jb.rows + 63) / 64;
    const bool vec = (jb.cols % 4 == 0) && (jb.rows % 4 == 0);
    for (int t = blockIdx.x; t < tiles_r * tiles_c; t += gridDim.x) {
      const int r0 = (t / tiles_c) * 64, c0 = (t % tiles_c) * 64;
      for (int k = tr; k < 64; k += 16) {
        const int r = r0 + k, c = c0 + 4 * tq;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < jb.rows) {
          const float* src = jb.in + static_cast<size_t>(r) * jb.cols + c;
          if (vec && c + 3 < jb.cols) v = *reinterpret_cast<const float4*>(src);
          else {
            if (c < jb.cols) v.x = src[0];
            if (c + 1 < jb.cols) v.y = src[1];
            if (c + 2 < jb.cols) v.z = src[2];
            if (c + 3 < jb.cols) v.w = src[3];
          }
        }
        tile[k][4 * tq] = v.x; tile[k][4 * tq + 1] = v.y; tile[k][4 * tq + 2] = v.z; tile[k][4 * tq + 3] = v.w;
      }
      __syncthreads();
      for (int k = tr; k < 64; k += 16) {
        const int oc = c0 + k, orow = r0 + 4 * tq;                 // output row oc, columns orow..+3
        if (oc < jb.cols) {
          const float4 v = make_float4(tile[4 * tq][k], tile[4 * tq + 1][k], tile[4 * tq + 2][k], tile[4 * tq + 3][k]);
          float* dst = jb.out + static_cast<size_t>(oc) * jb.rows + orow;
          if (vec && orow + 3 < jb.rows) *reinterpret_cast<float4*>(dst) = v;
          else {
            if (orow < jb.rows) dst[0] = v.x;
            if (orow + 1 < jb.rows) dst[1] = v.y;
            if (orow + 2 < jb.rows) dst[2] = v.z;
            if (orow + 3 < jb.rows) dst[3] = v.w;
          }
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace cts
