// jd_gram.cuh -- the App A.2 eigenvalue iteration (jd_eigen.cuh) carried in the stacked-factor
// ("Gram") space, so a call streams the fp32 LoRA factors a fixed number of times instead of four
// times per iteration.
//
// The paper's iteration with the factors stacked, A = [A_1; ..; A_n] (K x d_in),
// Bt = [B_1^T; ..; B_n^T] (K x d_out), K = n r_i:
//     P = A V, Q = Bt U;  W_i = P_i (P_i^T Q_i), Z_i = Q_i (Q_i^T P_i)        (jd_small)
//     U' = orthogonalize(Bt^T W),  V' = orthogonalize(A^T Z)
// orthogonalize = the Q of a QR with a positive R diagonal = X R^-1 with R^T R = X^T X (Cholesky).
// For X = A^T Z:  X^T X = Z^T (A A^T) Z,  so with G_A = A A^T (K x K) and R from chol(Z^T G_A Z):
//     V' = A^T C_V,  C_V = Z R^-1,  and the next  P' = A V' = G_A C_V.
// The same holds for U' with G_B = Bt Bt^T and C_U = W R_U^-1, Q' = G_B C_U.  So after ONE pass
// that forms G_A and G_B on the tensor cores (jd_tc_gemm<128>, 3xTF32), every further iteration is
// K x K x r work: Y = G C as a thin tensor-core GEMM (jd_tc_gemm<R>, X = G, Y = C^T from the batched
// transpose), then the r x r orthogonalization below; only the last iteration returns to the
// d-space (explicit U0 = Bt^T W, V0 = A^T Z, Cholesky-QR2 with the collapse completion, then P, Q and
// Sigma) -- the same iterates in exact arithmetic, a different rounding.  As in the d-space path the
// orthogonalization is applied twice (Cholesky-QR2); the second pass reuses Y R1^-1 for G C of the
// updated C (CTS_JD_KS_RECOMPUTE=1 forms it again), with the r x r Gram and its Cholesky in fp64.
//
// Used when every problem of a batch has 2r <= K <= kJdGramMaxK (cts.cu jd_gram_ok).  A span below r
// (duplicated or low-rank adapters) makes Cholesky pivots collapse; the standard-basis completion of
// the d-space path cannot be expressed in the K-space, so there the collapsed directions are dropped
// and the last, explicit iteration completes the basis (test_gpu_jd_rank_deficient_cluster
// [kspace_duplicates]: reconstruction of every B_i A_i).  Above kJdGramMaxK the K x K Grams outgrow
// their purpose.
#pragma once
#include <cstdint>
#include "jd_eigen.cuh"

namespace cts {

constexpr int kJdGramMaxK = 1024;

// One Cholesky-QR pass in the K-space for side s (blockIdx.x), problem blockIdx.y:
//     M = C^T Y (= X^T X of the implicit X = A^T C), M = L L^T (fp64), Rinv = (L^T)^-1,
//     C <- C Rinv,  Y <- Y Rinv  (written to P / Q on the last pass: P = G_A C_V = A V').
// A pivot below kJdCollapse of its diagonal (a collapsed direction: the cluster's stacked span is
// below r, e.g. duplicated adapters) drops that column (zero in C and Y); the final d-space
// Cholesky-QR2 completes the basis with standard basis vectors as in the d-space path.
template <int R>
__global__ void __launch_bounds__(256, 2) jd_gorth(const __grid_constant__ JdBatch b, int last) {
  const JdProblem& p = b.pr[blockIdx.y];
  const int K = p.n * p.ri;
  const int side = blockIdx.x;
  float* C = side == 0 ? p.Z : p.W;
  const float* Y = side == 0 ? p.Ya : p.Yb;
  float* Yout = last ? (side == 0 ? p.P : p.Q) : (side == 0 ? p.Ya : p.Yb);
  constexpr int kE = R * R / 256;                  // M entries per thread (1 at R = 16, 4 at R = 32)
  constexpr int kCh = 64;                          // rows of C / Y staged per chunk
  constexpr int kV = kCh * R / 4 / 256;            // float4 of C (and of Y) per thread per chunk
  __shared__ float4 Cs[kCh * R / 4], Ys[kCh * R / 4];
  __shared__ double M[R][R + 1];
  __shared__ double dg[R];
  __shared__ bool drop[R];
  __shared__ float Ri[R][R];
  // M = C^T Y: fp32 products, fp64 accumulation, over staged 64-row chunks; the next chunk is
  // loaded into registers while the current one is reduced
  float4 cr[kV], yr[kV];
  auto load = [&](int k0) {
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      const int e = threadIdx.x + 256 * j;
      const bool in = k0 + e / (R / 4) < K;
      cr[j] = in ? reinterpret_cast<const float4*>(C + static_cast<size_t>(k0) * R)[e] : make_float4(0.f, 0.f, 0.f, 0.f);
      yr[j] = in ? reinterpret_cast<const float4*>(Y + static_cast<size_t>(k0) * R)[e] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  double acc[kE];
#pragma unroll
  for (int q = 0; q < kE; ++q) acc[q] = 0.0;
  load(0);
  for (int k0 = 0; k0 < K; k0 += kCh) {
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      Cs[threadIdx.x + 256 * j] = cr[j];
      Ys[threadIdx.x + 256 * j] = yr[j];
    }
    __syncthreads();
    if (k0 + kCh < K) load(k0 + kCh);
    const float* cs = reinterpret_cast<const float*>(Cs);
    const float* ys = reinterpret_cast<const float*>(Ys);
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      const int e = threadIdx.x + 256 * q, a = e / R, c = e % R;
      double s0 = 0.0, s1 = 0.0;                   // two chains (rows are zero-filled past K)
#pragma unroll 8
      for (int k = 0; k < kCh; k += 2) {
        s0 += static_cast<double>(cs[k * R + a] * ys[k * R + c]);
        s1 += static_cast<double>(cs[(k + 1) * R + a] * ys[(k + 1) * R + c]);
      }
      acc[q] += s0 + s1;
    }
  }
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    const int e = threadIdx.x + 256 * q;
    M[e / R][e % R] = acc[q];
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int j = lane; j < R; j += 32) dg[j] = M[j][j];
    __syncwarp();
    // symmetrize (M = C^T G C is symmetric in exact arithmetic), then L L^T = M in place (lower)
    for (int e = lane; e < R * R; e += 32) {
      const int a = e / R, c = e % R;
      if (a > c) M[a][c] = 0.5 * (M[a][c] + M[c][a]);
    }
    __syncwarp();
    for (int j = 0; j < R; ++j) {
      if (lane == 0) {
        double s = M[j][j];
        for (int k = 0; k < j; ++k) s -= M[j][k] * M[j][k];
        // a collapsed direction (already in the span of the earlier columns): DROPPED -- its column
        // of C and Y becomes zero below, so no amplified residual enters the next iterate; the span
        // is unchanged and the last (d-space) iteration completes the basis as the oracle does
        drop[j] = !(s > static_cast<double>(kJdCollapse) * dg[j]);
        M[j][j] = drop[j] ? 1.0 : sqrt(s);
      }
      __syncwarp();
      for (int i = j + 1 + lane; i < R; i += 32) {
        double t = M[i][j];
        for (int k = 0; k < j; ++k) t -= M[i][k] * M[j][k];
        M[i][j] = drop[j] ? 0.0 : t / M[j][j];
      }
      __syncwarp();
    }
    // Rinv = (L^T)^-1 (upper): lane c solves L^T x = e_c, back substitution in place in column c
    for (int c = lane; c < R; c += 32) {
#pragma unroll 1
      for (int i = R - 1; i >= 0; --i) {
        double t = i == c ? 1.0 : 0.0;
        for (int k = i + 1; k <= c; ++k) t -= M[k][i] * static_cast<double>(Ri[k][c]);
        Ri[i][c] = i <= c ? static_cast<float>(t / M[i][i]) : 0.f;
      }
    }
    __syncwarp();
    for (int e = lane; e < R * R; e += 32)          // dropped directions: zero row and column
      if (drop[e / R] || drop[e % R]) Ri[e / R][e % R] = 0.f;
  }
  __syncthreads();
  // C <- C Rinv, Y <- Y Rinv: thread = row, one matrix at a time (fewer live registers)
  for (int mat = 0; mat < 2; ++mat) {
    float* src = mat == 0 ? C : const_cast<float*>(Y);
    float* dst = mat == 0 ? C : Yout;
    for (int k = threadIdx.x; k < K; k += 256) {
      float x[R];
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4) {
        const float4 v = reinterpret_cast<const float4*>(src + static_cast<size_t>(k) * R)[c4];
        x[4 * c4] = v.x; x[4 * c4 + 1] = v.y; x[4 * c4 + 2] = v.z; x[4 * c4 + 3] = v.w;
      }
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4) {
        float o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = 4 * c4 + u;
          float s = 0.f;
#pragma unroll
          for (int a = 0; a <= c; ++a) s = fmaf(x[a], Ri[a][c], s);
          o[u] = s;
        }
        reinterpret_cast<float4*>(dst + static_cast<size_t>(k) * R)[c4] = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
  }
}

}  // namespace cts
