// jd_eigen.cuh -- SURVEY 8(f) NEXT 3: GPU compression.  The joint diagonalization of a cluster's
// LoRAs by the paper's GPU-oriented "Additional Eigenvalue Iteration Algorithm" (App A.2,
// P:L528-562), batched over clusters / modules:
//     P_i = A_i V,  Q_i = B_i^T U                                    (r_i x r each)
//     U0  = sum_i B_i (P_i (P_i^T Q_i)),   V0 = sum_i A_i^T (Q_i (Q_i^T P_i))
//     U <- orthogonalize(U0),  V <- orthogonalize(V0)                 (both from the k-th iterates)
// and finally Sigma_i = U^T B_i A_i V = Q_i^T P_i (Eq. sigmastar).  The paper's
// parenthesization is kept: nothing d x d is ever formed.  With the factors stacked --
// A_stack = [A_1; ..; A_n] (n r_i x d_in), Bt_stack = [B_1^T; ..; B_n^T] (n r_i x d_out) -- the four
// sums are four thin GEMMs (P = A_stack V, Q = Bt_stack U, U0 = Bt_stack^T W, V0 = A_stack^T Z) and
// W_i = P_i S_i, Z_i = Q_i S_i^T with S_i = P_i^T Q_i are per-adapter r x r products.
// orthogonalize = Cholesky-QR applied twice (Q = X R^-1 with R^T R = X^T X, diag(R) > 0: the
// reduced QR with a positive R diagonal, the oracle's convention).  fp32 (an offline step).
//
// All kernels take a batch of independent problems (blockIdx.z / blockIdx.y = problem), so one
// launch covers every cluster of a module (or several modules) and fills the SMs.
#pragma once
#include <cstdint>
#include "sm100.cuh"

namespace cts {

constexpr int kJdMaxBatch = 200;   // problems per launch (kernel parameter space: 200 x 160 B)

struct JdProblem {
  const float* a;        // A_stack [n*r_i][d_in]
  const float* bt;       // Bt_stack [n*r_i][d_out]
  float* U;              // [d_out][R] in/out
  float* V;              // [d_in][R] in/out
  float* sigma;          // [n][R][R] out (row = out index)
  float* P;              // workspace [n*r_i][R]
  float* Q;              // [n*r_i][R]
  float* W;              // [n*r_i][R]
  float* Z;              // [n*r_i][R]
  float* U0;             // [d_out][R]
  float* V0;             // [d_in][R]
  float* part;           // partials: [ceil(d/1024)][n*r_i][R] of P / Q, [ceil(n*r_i/128)][d][R] of U0 / V0
  float* Gu;             // [ceil(d_out/256)][R][R] partial Gram matrices; slot 0 then holds R^-1
  float* Gv;             // [ceil(d_in/256)][R][R]
  float* Ga;             // K-space path (jd_gram.cuh): G_A = A_stack A_stack^T [K][K]
  float* Gb;             // G_B = Bt_stack Bt_stack^T [K][K]
  float* Ya;             // [K][R] G_A C_V
  float* Yb;             // [K][R] G_B C_U
  int n, ri, d_in, d_out;
};

struct JdBatch {
  JdProblem pr[kJdMaxBatch];
  int count;
};

// out[K][R] = X[K][d] * Y[d][R], split over d: block (256 rows, d segment of kJdSeg) writes a partial
// [seg][K][R] to the workspace (jd_rows_reduce sums the segments in order -- deterministic).
// Thread = one row of X, all R outputs: its row streams in as 16-byte loads (the 128-byte lines of
// a warp's 32 rows are re-used from L1 over 8 consecutive loads), Y is staged in shared memory in
// chunks of kJdYChunk rows and read as warp-broadcast 16-byte loads -- 4R FMAs per R/4 + 1 loads,
// so the kernel streams X at close to HBM speed instead of being bound by shared-memory traffic.
constexpr int kJdSeg = 1024;
constexpr int kJdRowsPerBlock = 256;

template <int R>
__global__ void __launch_bounds__(256, R <= 16 ? 4 : (R <= 32 ? 2 : 1)) jd_rows_times(const __grid_constant__ JdBatch b, int which) {
  constexpr int kChunk = 4096 / R;                   // 16 KB of Y per stage
  const JdProblem& p = b.pr[blockIdx.z];
  const float* X = which == 0 ? p.a : p.bt;          // 0: P = A V, 1: Q = Bt U
  const float* Y = which == 0 ? p.V : p.U;
  const int d = which == 0 ? p.d_in : p.d_out;
  const int K = p.n * p.ri;
  const int row0 = blockIdx.x * kJdRowsPerBlock, d_lo = blockIdx.y * kJdSeg;
  if (row0 >= K || d_lo >= d) return;
  const int d_hi = min(d, d_lo + kJdSeg);
  float* part = p.part + (static_cast<size_t>(blockIdx.y) * K) * R;
  __shared__ float4 ys[kChunk * R / 4];              // [chunk row][R / 4]
  const int row = row0 + threadIdx.x;
  const bool live = row < K;
  const float* xr = X + static_cast<size_t>(live ? row : 0) * d;
  float acc[R];
#pragma unroll
  for (int c = 0; c < R; ++c) acc[c] = 0.f;
  for (int d0 = d_lo; d0 < d_hi; d0 += kChunk) {
    const int n = min(kChunk, d_hi - d0);
    __syncthreads();
    for (int i = threadIdx.x; i < kChunk * R / 4; i += 256)
      ys[i] = i < n * R / 4 ? reinterpret_cast<const float4*>(Y + static_cast<size_t>(d0) * R)[i]
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    if (live) {
#pragma unroll 2
      for (int k = 0; k < n; k += 4) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + d0 + k));
        const float xk[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
          for (int c4 = 0; c4 < R / 4; ++c4) {
            const float4 yv = ys[(k + u) * (R / 4) + c4];
            acc[4 * c4] = fmaf(xk[u], yv.x, acc[4 * c4]);
            acc[4 * c4 + 1] = fmaf(xk[u], yv.y, acc[4 * c4 + 1]);
            acc[4 * c4 + 2] = fmaf(xk[u], yv.z, acc[4 * c4 + 2]);
            acc[4 * c4 + 3] = fmaf(xk[u], yv.w, acc[4 * c4 + 3]);
          }
        }
      }
    }
  }
  if (live) {
    float4* dst = reinterpret_cast<float4*>(part + static_cast<size_t>(row) * R);
#pragma unroll
    for (int c4 = 0; c4 < R / 4; ++c4) dst[c4] = make_float4(acc[4 * c4], acc[4 * c4 + 1], acc[4 * c4 + 2], acc[4 * c4 + 3]);
  }
}

// out = sum over d segments of the partials, in segment order
template <int R>
__global__ void __launch_bounds__(256) jd_rows_reduce(const __grid_constant__ JdBatch b, int which) {
  const JdProblem& p = b.pr[blockIdx.y];
  float* out = which == 0 ? p.P : p.Q;
  const int d = which == 0 ? p.d_in : p.d_out;
  const int K = p.n * p.ri;
  const int S = (d + kJdSeg - 1) / kJdSeg;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K * R; i += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int g = 0; g < S; ++g) s += p.part[static_cast<size_t>(g) * K * R + i];
    out[i] = s;
  }
}

// per adapter i: S = P_i^T Q_i (R x R), W_i = P_i S, Z_i = Q_i S^T  (blockIdx.x = adapter)
template <int R>
__global__ void __launch_bounds__(256) jd_small(const __grid_constant__ JdBatch b) {
  const JdProblem& p = b.pr[blockIdx.y];
  const int i = blockIdx.x;
  if (i >= p.n) return;
  extern __shared__ float sm[];
  float* Ps = sm;                      // [ri][R]
  float* Qs = Ps + p.ri * R;           // [ri][R]
  float* S = Qs + p.ri * R;            // [R][R]
  const size_t base = static_cast<size_t>(i) * p.ri * R;
  for (int e = threadIdx.x; e < p.ri * R; e += blockDim.x) {
    Ps[e] = p.P[base + e];
    Qs[e] = p.Q[base + e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int a = e / R, c = e % R;
    float s = 0.f;
    for (int j = 0; j < p.ri; ++j) s = fmaf(Ps[j * R + a], Qs[j * R + c], s);
    S[e] = s;                          // S[a][c] = (P_i^T Q_i)[a][c]
  }
  __syncthreads();
  for (int e = threadIdx.x; e < p.ri * R; e += blockDim.x) {
    const int j = e / R, c = e % R;
    float w = 0.f, z = 0.f;
    for (int a = 0; a < R; ++a) {
      w = fmaf(Ps[j * R + a], S[a * R + c], w);   // (P_i S)[j][c]
      z = fmaf(Qs[j * R + a], S[c * R + a], z);   // (Q_i S^T)[j][c]
    }
    p.W[base + e] = w;
    p.Z[base + e] = z;
  }
}

// out[d][R] = X[K][d]^T * M[K][R], split over K: block (256 * kJdColsPer(R) columns of d, K segment
// of kJdKSeg rows) writes a partial [kseg][d][R] (jd_cols_reduce sums the segments in order).
// Thread = kJdColsPer consecutive columns of d, all R outputs: X rows stream in as coalesced
// 16/8-byte loads, M is staged in shared memory and read as warp-broadcast 16-byte loads.
constexpr int kJdKSeg = 320;

template <int R>
struct JdColsPer {
  static constexpr int v = R <= 16 ? 4 : (R <= 32 ? 2 : 1);
};

template <int R>
__global__ void __launch_bounds__(256, R <= 32 ? 2 : 1) jd_cols_times(const __grid_constant__ JdBatch b, int which) {
  constexpr int CP = JdColsPer<R>::v;
  const JdProblem& p = b.pr[blockIdx.z];
  const float* X = which == 0 ? p.bt : p.a;           // 0: U0 = Bt^T W, 1: V0 = A^T Z
  const float* Mt = which == 0 ? p.W : p.Z;
  const int d = which == 0 ? p.d_out : p.d_in;
  const int K = p.n * p.ri;
  const int col0 = (blockIdx.x * 256 + threadIdx.x) * CP, k_lo = blockIdx.y * kJdKSeg;
  if (blockIdx.x * 256 * CP >= d || k_lo >= K) return;
  const int k_hi = min(K, k_lo + kJdKSeg);
  float* part = p.part + static_cast<size_t>(blockIdx.y) * d * R;
  constexpr int kMs = 64;                             // M rows staged per pass
  __shared__ float4 ms[kMs * R / 4];
  const bool live = col0 < d;                         // d is a multiple of 64 (and of CP)
  float acc[CP][R];
#pragma unroll
  for (int j = 0; j < CP; ++j)
#pragma unroll
    for (int c = 0; c < R; ++c) acc[j][c] = 0.f;
  for (int k0 = k_lo; k0 < k_hi; k0 += kMs) {
    const int n = min(kMs, k_hi - k0);
    __syncthreads();
    for (int i = threadIdx.x; i < kMs * R / 4; i += 256)
      ms[i] = i < n * R / 4 ? reinterpret_cast<const float4*>(Mt + static_cast<size_t>(k0) * R)[i]
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    if (live) {
#pragma unroll 2
      for (int k = 0; k < n; ++k) {
        float xv[CP];
        const float* xp = X + static_cast<size_t>(k0 + k) * d + col0;
        if constexpr (CP == 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(xp));
          xv[0] = v.x; xv[1] = v.y; xv[2] = v.z; xv[3] = v.w;
        } else if constexpr (CP == 2) {
          const float2 v = __ldg(reinterpret_cast<const float2*>(xp));
          xv[0] = v.x; xv[1] = v.y;
        } else {
          xv[0] = __ldg(xp);
        }
#pragma unroll
        for (int c4 = 0; c4 < R / 4; ++c4) {
          const float4 mv = ms[k * (R / 4) + c4];
#pragma unroll
          for (int j = 0; j < CP; ++j) {
            acc[j][4 * c4] = fmaf(xv[j], mv.x, acc[j][4 * c4]);
            acc[j][4 * c4 + 1] = fmaf(xv[j], mv.y, acc[j][4 * c4 + 1]);
            acc[j][4 * c4 + 2] = fmaf(xv[j], mv.z, acc[j][4 * c4 + 2]);
            acc[j][4 * c4 + 3] = fmaf(xv[j], mv.w, acc[j][4 * c4 + 3]);
          }
        }
      }
    }
  }
  if (live) {
#pragma unroll
    for (int j = 0; j < CP; ++j) {
      float4* dst = reinterpret_cast<float4*>(part + static_cast<size_t>(col0 + j) * R);
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4)
        dst[c4] = make_float4(acc[j][4 * c4], acc[j][4 * c4 + 1], acc[j][4 * c4 + 2], acc[j][4 * c4 + 3]);
    }
  }
}

template <int R>
__global__ void __launch_bounds__(256) jd_cols_reduce(const __grid_constant__ JdBatch b, int which) {
  const JdProblem& p = b.pr[blockIdx.y];
  float* out = which == 0 ? p.U0 : p.V0;
  const int d = which == 0 ? p.d_out : p.d_in;
  const int K = p.n * p.ri;
  const int S = (K + kJdKSeg - 1) / kJdKSeg;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d * R; i += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int g = 0; g < S; ++g) s += p.part[static_cast<size_t>(g) * d * R + i];
    out[i] = s;
  }
}

// orthogonalize (U0 -> U, V0 -> V) by Cholesky-QR, twice, in three parallel steps per pass:
//   jd_gram:  partial Gram matrices X_b^T X_b of 256-row blocks b          (blockIdx.x = block)
//   jd_chol:  G = sum_b partials in block order (deterministic), Cholesky G = R^T R, R^-1
//   jd_apply: Y = X R^-1                                                   (rows in parallel)
// blockIdx.y = problem, blockIdx.z = matrix (0: U, 1: V).  Pass 0 maps X = U0 -> Y = U, pass 1
// maps U -> U in place (jd_apply: every thread reads its whole row before writing it).
constexpr int kJdGramRows = 256;

template <int R>
__device__ __forceinline__ void jd_orth_mats(const JdProblem& p, int z, int pass, const float*& src, float*& dst,
                                             int& d, float*& gram) {
  const bool u = z == 0;
  d = u ? p.d_out : p.d_in;
  float* X0 = u ? p.U0 : p.V0;
  float* X1 = u ? p.U : p.V;
  src = pass == 0 ? X0 : X1;
  dst = X1;
  gram = u ? p.Gu : p.Gv;
}

template <int R>
__global__ void __launch_bounds__(256) jd_gram(const __grid_constant__ JdBatch b, int pass) {
  const JdProblem& p = b.pr[blockIdx.y];
  const float* src;
  float* dst;
  int d;
  float* gram;
  jd_orth_mats<R>(p, blockIdx.z, pass, src, dst, d, gram);
  const int r0 = blockIdx.x * kJdGramRows;
  if (r0 >= d) return;
  // thread = (row a, 4 columns c4) of the R x R Gram block, GROUPS row groups split each 64-row chunk
  constexpr int CQ = R / 4, PAIRS = R * CQ;
  constexpr int GROUPS = PAIRS >= 256 ? 1 : 256 / PAIRS, PER = (PAIRS + 255) / 256;
  __shared__ float4 xs[64][CQ];
  __shared__ float4 red[GROUPS > 1 ? GROUPS : 1][GROUPS > 1 ? PAIRS : 1];
  const int grp = threadIdx.x / (PAIRS < 256 ? PAIRS : 256);
  float4 acc[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c0 = r0; c0 < min(d, r0 + kJdGramRows); c0 += 64) {
    for (int i = threadIdx.x; i < 64 * CQ; i += 256) {
      const int rr = i / CQ, cq = i % CQ;
      xs[rr][cq] = c0 + rr < d ? reinterpret_cast<const float4*>(src + static_cast<size_t>(c0 + rr) * R)[cq]
                               : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = (GROUPS > 1 ? threadIdx.x % PAIRS : threadIdx.x) + 256 * q;
      if (e < PAIRS) {
        const int a = e / CQ, c4 = e % CQ;
#pragma unroll 4
        for (int rr = grp; rr < 64; rr += GROUPS) {
          const float xa = reinterpret_cast<const float*>(&xs[rr][0])[a];
          const float4 xc = xs[rr][c4];
          acc[q].x = fmaf(xa, xc.x, acc[q].x);
          acc[q].y = fmaf(xa, xc.y, acc[q].y);
          acc[q].z = fmaf(xa, xc.z, acc[q].z);
          acc[q].w = fmaf(xa, xc.w, acc[q].w);
        }
      }
    }
    __syncthreads();
  }
  float4* out = reinterpret_cast<float4*>(gram + static_cast<size_t>(blockIdx.x) * R * R);
  if constexpr (GROUPS > 1) {
    red[grp][threadIdx.x % PAIRS] = acc[0];
    __syncthreads();
    if (threadIdx.x < PAIRS) {
      float4 t = red[0][threadIdx.x];
#pragma unroll
      for (int g = 1; g < GROUPS; ++g) {                  // fixed group order: deterministic
        const float4 u = red[g][threadIdx.x];
        t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
      }
      out[threadIdx.x] = t;                               // [a][c4] = row a, columns 4c4..4c4+3
    }
  } else {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = threadIdx.x + 256 * q;
      if (e < PAIRS) out[e] = acc[q];
    }
  }
}

// Rank collapse.  Column j of X is (numerically) in the span of columns 0..j-1 when its Cholesky
// pivot -- the squared norm of its residual after projecting out those columns -- falls below
// kJdCollapse of its squared norm: a cluster whose stacked LoRA rank n*r_i is below r, duplicate
// adapters, or an exactly rank-deficient iterate.  Plain Cholesky-QR would divide by ~0 and return
// Inf/NaN.  Instead that column of X is REPLACED by the first standard basis vector e_k (k in index
// order) whose residual is at least half its average, and the factorization continues: the result
// is a deterministic orthonormal completion with standard basis vectors in index order, as the
// oracle's _complete does for a span smaller than r (oracle/jd.py).  fp32 cancellation makes a
// residual below ~3e-3 of the column norm meaningless, hence the threshold.
constexpr float kJdCollapse = 1e-5f;

template <int R>
__global__ void __launch_bounds__(256) jd_chol(const __grid_constant__ JdBatch b, int pass) {
  const JdProblem& p = b.pr[blockIdx.y];
  const float* src;
  float* dst;
  int d;
  float* gram;
  jd_orth_mats<R>(p, blockIdx.z, pass, src, dst, d, gram);
  float* X = const_cast<float*>(src);               // a workspace iterate (U0/V0 or U/V): writable
  __shared__ float G[R][R + 1];
  __shared__ float diag0[R];
  __shared__ int sub_k;
  const int nb = (d + kJdGramRows - 1) / kJdGramRows;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < nb; ++k) s += gram[static_cast<size_t>(k) * R * R + e];   // block order
    G[e / R][e % R] = s;
    if (e / R == e % R) diag0[e / R] = s;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    // Cholesky G = L L^T (lower, in place), one column at a time; the warp splits each column's rows
    const int lane = threadIdx.x;
    for (int j = 0; j < R; ++j) {
      if (lane == 0) {
        float s = G[j][j];
        for (int k = 0; k < j; ++k) s -= G[j][k] * G[j][k];
        sub_k = -1;
        if (!(s > kJdCollapse * diag0[j])) {
          // column j collapsed: candidate e_k has Gram entries G[j][m] = X[k][m]; row j of L is
          // the forward substitution of those, its pivot 1 - |L[j][0..j-1]|^2
          const float need = 0.5f * static_cast<float>(d - j) / static_cast<float>(d);
          for (int k = 0; k < d; ++k) {
            float ss = 1.f;
            for (int m = 0; m < j; ++m) {
              float t = X[static_cast<size_t>(k) * R + m];
              for (int q = 0; q < m; ++q) t -= G[j][q] * G[m][q];
              t /= G[m][m];
              G[j][m] = t;
              ss -= t * t;
            }
            if (ss > need || k == d - 1) {
              sub_k = k;
              s = ss;
              break;
            }
          }
        }
        G[j][j] = sqrtf(fmaxf(s, 1e-30f));
      }
      __syncwarp();
      const int k = sub_k;
      if (k >= 0) {
        // X[:, j] := e_k; later columns' Gram entries with it are X[k][i]
        for (int i = j + 1 + lane; i < R; i += 32) G[i][j] = X[static_cast<size_t>(k) * R + i];
        __syncwarp();
        for (int row = lane; row < d; row += 32) X[static_cast<size_t>(row) * R + j] = row == k ? 1.f : 0.f;
      }
      __syncwarp();
      for (int i = j + 1 + lane; i < R; i += 32) {
        float t = G[i][j];
        for (int k2 = 0; k2 < j; ++k2) t -= G[i][k2] * G[j][k2];
        G[i][j] = t / G[j][j];
      }
      __syncwarp();
    }
    // R^-1 = (L^T)^-1, upper triangular: lane c solves L^T x = e_c for columns c = lane, lane+32
    float* Rinv = gram;                              // reuse partial slot 0 as [R][R] output
    for (int c = lane; c < R; c += 32) {
      float x[R];
#pragma unroll
      for (int i = R - 1; i >= 0; --i) {
        float t = i == c ? 1.f : 0.f;
#pragma unroll
        for (int k = i + 1; k < R; ++k) t -= G[k][i] * x[k];
        x[i] = i <= c ? t / G[i][i] : 0.f;
      }
#pragma unroll
      for (int i = 0; i < R; ++i) Rinv[i * R + c] = x[i];
    }
  }
}

// Y = X R^-1 (R^-1 upper triangular), thread = one row: the row is read whole into registers, so
// the in-place second pass is safe; R^-1 is read from shared memory as warp broadcasts.
template <int R>
__global__ void __launch_bounds__(256) jd_apply(const __grid_constant__ JdBatch b, int pass) {
  const JdProblem& p = b.pr[blockIdx.y];
  const float* src;
  float* dst;
  int d;
  float* gram;
  jd_orth_mats<R>(p, blockIdx.z, pass, src, dst, d, gram);
  __shared__ float Ri[R][R];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Ri[e / R][e % R] = gram[e];
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < d; r += gridDim.x * blockDim.x) {
    float x[R], y[R];
    const float4* row = reinterpret_cast<const float4*>(src + static_cast<size_t>(r) * R);
#pragma unroll
    for (int c4 = 0; c4 < R / 4; ++c4) {
      const float4 v = row[c4];
      x[4 * c4] = v.x; x[4 * c4 + 1] = v.y; x[4 * c4 + 2] = v.z; x[4 * c4 + 3] = v.w;
    }
#pragma unroll
    for (int c = 0; c < R; ++c) {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a <= c; ++a) s = fmaf(x[a], Ri[a][c], s);
      y[c] = s;
    }
    float4* out = reinterpret_cast<float4*>(dst + static_cast<size_t>(r) * R);
#pragma unroll
    for (int c4 = 0; c4 < R / 4; ++c4) out[c4] = make_float4(y[4 * c4], y[4 * c4 + 1], y[4 * c4 + 2], y[4 * c4 + 3]);
  }
}

// Sigma_i = Q_i^T P_i (R x R; row = out index); blockIdx.x = adapter
template <int R>
__global__ void __launch_bounds__(256) jd_sigma(const __grid_constant__ JdBatch b) {
  const JdProblem& p = b.pr[blockIdx.y];
  const int i = blockIdx.x;
  if (i >= p.n) return;
  const size_t base = static_cast<size_t>(i) * p.ri * R;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int o = e / R, k = e % R;
    float s = 0.f;
    for (int j = 0; j < p.ri; ++j) s = fmaf(p.Q[base + j * R + o], p.P[base + j * R + k], s);
    p.sigma[static_cast<size_t>(i) * R * R + e] = s;
  }
}

}  // namespace cts
