// Exact low-rank solve of the Gauss-Newton reduced system (PAPER Eq. 12,
// SPEC.md:292 solve_newton), replacing the O((mk)^3) dense Cholesky.
//
// With U = Y^T (x) I_k  (mk x k^2) and Zb[(a,p),(b,q)] = sum_i Rinv_i[a,b] x_ip x_iq,
// the reference's Schur correction is S = U Zb U^T (rank <= k^2), so
//
//     A = D - U Zb U^T,   D = blockdiag(X^T X + rho I + Diag(s_j / y_j)).
//
// Push-through: with w = Zb U^T dy,  dy = D^{-1}(rhs + U w)  and
// (I - Zb G) w = Zb U^T D^{-1} rhs,  G = U^T D^{-1} U = sum_j (y_j y_j^T) (x) D_j^{-1}.
// Symmetrised with G = L_G L_G^T:  H = I - L_G^T Zb L_G,  H v = L_G^T Zb u,
// w = L_G^{-T} v.  A is positive definite  <=>  H is (same nonzero spectrum as
// Zb G), so the Cholesky of H is also the exact PD test the reference's
// dense factorization performs.  Cost O(m k^3 + k^6) instead of O(m^3 k^3).
#include "common.cuh"
#include "nmfb200.h"

namespace {

__device__ __forceinline__ int pkx(int a, int b, int k) {
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
  return a * k - a * (a - 1) / 2 + (b - a);
}

// per column j: D_j = XtX + rho I + Diag(s_j / y_j) = L_j L_j^T;
// Dinv_pk = packed D_j^{-1}, YY_pk = packed y_j y_j^T
template <int K>
__global__ void __launch_bounds__(128) k_d_factor(const double* __restrict__ XtX,
                                                  const double* __restrict__ Yt,
                                                  const double* __restrict__ S, double rho,
                                                  long m, double* __restrict__ LD,
                                                  double* __restrict__ Dinvpk,
                                                  double* __restrict__ YYpk,
                                                  int* __restrict__ bad) {
  __shared__ double xx[K * K];
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) xx[e] = XtX[e];
  __syncthreads();
  const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double L[K][K], y[K];
#pragma unroll
  for (int p = 0; p < K; ++p) y[p] = Yt[j * K + p];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int c = 0; c < K; ++c) L[a][c] = (c <= a) ? xx[a * K + c] : 0.0;
#pragma unroll
  for (int p = 0; p < K; ++p) L[p][p] += rho + S[j * K + p] / y[p];
#pragma unroll
  for (int c = 0; c < K; ++c) {
    double s = L[c][c];
#pragma unroll
    for (int p = 0; p < c; ++p) s -= L[c][p] * L[c][p];
    if (!(s > 0.0)) {
      atomicMin(bad, (int)j);
      return;
    }
    const double d = sqrt(s);
    L[c][c] = d;
#pragma unroll
    for (int i = c + 1; i < K; ++i) {
      double t = L[i][c];
#pragma unroll
      for (int p = 0; p < c; ++p) t -= L[i][p] * L[c][p];
      L[i][c] = t / d;
    }
  }
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int c = 0; c < K; ++c) LD[(j * K + a) * K + c] = (c <= a) ? L[a][c] : 0.0;
  double Li[K][K];
#pragma unroll
  for (int c = 0; c < K; ++c)
#pragma unroll
    for (int a = 0; a < K; ++a) {
      if (a < c) {
        Li[a][c] = 0.0;
      } else {
        double s = (a == c) ? 1.0 : 0.0;
#pragma unroll
        for (int p = 0; p < a; ++p)
          if (p >= c) s -= L[a][p] * Li[p][c];
        Li[a][c] = s / L[a][a];
      }
    }
  constexpr int KK = K * (K + 1) / 2;
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int c = a; c < K; ++c) {
      double s = 0.0;
#pragma unroll
      for (int p = 0; p < K; ++p)
        if (p >= c) s = fma(Li[p][a], Li[p][c], s);
      const int e = a * K - a * (a - 1) / 2 + (c - a);
      Dinvpk[j * KK + e] = s;
      YYpk[j * KK + e] = y[a] * y[c];
    }
}

// t_j = D_j^{-1} b_j  (+ optional correction: t_j = base_j + D_j^{-1}(W^T y_j))
template <int K>
__global__ void k_d_solve(const double* __restrict__ LD, const double* __restrict__ b, long m,
                          double* __restrict__ t) {
  const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double L[K][K], v[K], z[K];
#pragma unroll
  for (int a = 0; a < K; ++a) {
    v[a] = b[j * K + a];
#pragma unroll
    for (int c = 0; c < K; ++c) L[a][c] = LD[(j * K + a) * K + c];
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double s = v[i];
#pragma unroll
    for (int p = 0; p < i; ++p) s -= L[i][p] * z[p];
    z[i] = s / L[i][i];
  }
#pragma unroll
  for (int i = K - 1; i >= 0; --i) {
    double s = z[i];
#pragma unroll
    for (int p = i + 1; p < K; ++p) s -= L[p][i] * v[p];
    v[i] = s / L[i][i];
  }
#pragma unroll
  for (int a = 0; a < K; ++a) t[j * K + a] = v[a];
}

template <int K>
__global__ void k_d_correct(const double* __restrict__ LD, const double* __restrict__ Yt,
                            const double* __restrict__ Wm, long m, double* __restrict__ t) {
  __shared__ double w[K * K];
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) w[e] = Wm[e];
  __syncthreads();
  const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double L[K][K], v[K], z[K];
#pragma unroll
  for (int p = 0; p < K; ++p) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < K; ++a) s = fma(Yt[j * K + a], w[a * K + p], s);
    v[p] = s;
#pragma unroll
    for (int c = 0; c < K; ++c) L[p][c] = LD[(j * K + p) * K + c];
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double s = v[i];
#pragma unroll
    for (int p = 0; p < i; ++p) s -= L[i][p] * z[p];
    z[i] = s / L[i][i];
  }
#pragma unroll
  for (int i = K - 1; i >= 0; --i) {
    double s = z[i];
#pragma unroll
    for (int p = i + 1; p < K; ++p) s -= L[p][i] * v[p];
    v[i] = s / L[i][i];
  }
#pragma unroll
  for (int a = 0; a < K; ++a) t[j * K + a] += v[a];
}

// in-place lower Cholesky of a Q x Q row-major matrix (smem or global) by one
// CTA, two barriers per column; warps own rows of the trailing update and lanes
// its columns (no integer division, contiguous accesses).  Returns the failing
// pivot column or -1 (in every thread).
__device__ int cta_cholesky(double* A, int Q, int* sfail) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int nw = nt >> 5;
  if (tid == 0) *sfail = -1;
  __syncthreads();
  for (int j = 0; j < Q; ++j) {
    const double pv = A[j * Q + j];
    if (!(pv > 0.0)) {
      if (tid == 0) *sfail = j;
      break;  // uniform: every thread read the same pivot
    }
    const double rd = 1.0 / sqrt(pv);
    for (int r = j + 1 + tid; r < Q; r += nt) A[r * Q + j] *= rd;
    __syncthreads();
    if (tid == 0) A[j * Q + j] = pv * rd;
    for (int r = j + 1 + wid; r < Q; r += nw) {
      const double lrj = A[r * Q + j];
      for (int c = j + 1 + lane; c <= r; c += 32) A[r * Q + c] -= lrj * A[c * Q + j];
    }
    __syncthreads();
  }
  __syncthreads();
  const int f = *sfail;
  __syncthreads();
  return f;
}

// C[r][c] (Q x Q) += sum over the lower-triangular factor, 2x2 register tiles:
//   mode 0: T1 = Zb L       (T1[r][c] = sum_{t >= c} Zb[r][t] L[t][c])
//   mode 1: H  = I - L^T T1 (H[r][c]  = delta - sum_{t >= r} L[t][r] T1[t][c], c <= r)
__device__ void cta_tri_gemm(const double* Zb_or_L, const double* Lm, double* out, int Q, int mode) {
  const int half = (Q + 1) / 2;
  for (int e = threadIdx.x; e < half * half; e += blockDim.x) {
    const int r0 = 2 * (e / half), c0 = 2 * (e % half);
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    if (mode == 0) {
      for (int t = c0; t < Q; ++t) {
        const double z0 = Zb_or_L[r0 * Q + t];
        const double z1 = (r0 + 1 < Q) ? Zb_or_L[(r0 + 1) * Q + t] : 0.0;
        const double l0 = Lm[t * Q + c0];
        const double l1 = (c0 + 1 < Q && t >= c0 + 1) ? Lm[t * Q + c0 + 1] : 0.0;
        acc[0][0] = fma(z0, l0, acc[0][0]);
        acc[0][1] = fma(z0, l1, acc[0][1]);
        acc[1][0] = fma(z1, l0, acc[1][0]);
        acc[1][1] = fma(z1, l1, acc[1][1]);
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
          if (r0 + a < Q && c0 + b < Q) out[(r0 + a) * Q + c0 + b] = acc[a][b];
    } else {
      if (c0 > r0 + 1) {  // strictly upper tile: zeros
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b)
            if (r0 + a < Q && c0 + b < Q) out[(r0 + a) * Q + c0 + b] = 0.0;
        continue;
      }
      for (int t = r0; t < Q; ++t) {
        const double l0 = Zb_or_L[t * Q + r0];
        const double l1 = (r0 + 1 < Q && t >= r0 + 1) ? Zb_or_L[t * Q + r0 + 1] : 0.0;
        const double t0 = Lm[t * Q + c0];
        const double t1 = (c0 + 1 < Q) ? Lm[t * Q + c0 + 1] : 0.0;
        acc[0][0] = fma(l0, t0, acc[0][0]);
        acc[0][1] = fma(l0, t1, acc[0][1]);
        acc[1][0] = fma(l1, t0, acc[1][0]);
        acc[1][1] = fma(l1, t1, acc[1][1]);
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int r = r0 + a, c = c0 + b;
          if (r < Q && c < Q) out[r * Q + c] = (c <= r) ? ((r == c ? 1.0 : 0.0) - acc[a][b]) : 0.0;
        }
    }
  }
}

// one CTA: LG = chol(G), H = I - LG^T Zb LG, LH = chol(H).  work: 2 Q^2 doubles
// (Zb kept in work[0, Q^2) for the solves).  Small Q works in shared memory.
__global__ void __launch_bounds__(1024) k_lowrank_factor(const double* __restrict__ Zpk,
                                                         const double* __restrict__ Gpk, int k,
                                                         double* __restrict__ LG,
                                                         double* __restrict__ LH,
                                                         double* __restrict__ Zb,
                                                         double* __restrict__ T1g,
                                                         int* __restrict__ info, int use_smem) {
  extern __shared__ double smf[];
  __shared__ int sfail;
  const int Q = k * k, KK = k * (k + 1) / 2;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* A = use_smem ? smf : LG;            // G -> L_G, later H -> L_H
  double* T1 = use_smem ? smf + Q * Q : T1g;  // Zb L_G
  for (int e = tid; e < Q * Q; e += nt) {
    const int r = e / Q, c = e % Q;
    const int a = r / k, p = r % k, b = c / k, q = c % k;
    const int ab = pkx(a, b, k), pq = pkx(p, q, k);
    Zb[e] = Zpk[ab * KK + pq];
    A[e] = (c <= r) ? Gpk[ab * KK + pq] : 0.0;
  }
  __syncthreads();
  int f = cta_cholesky(A, Q, &sfail);
  if (f >= 0) {
    if (tid == 0) *info = 1000000 + f;  // G singular: Y^T rank deficient
    return;
  }
  for (int e = tid; e < Q * Q; e += nt) {  // publish L_G (strict upper zero)
    const int r = e / Q, c = e % Q;
    const double v = (c <= r) ? A[e] : 0.0;
    A[e] = v;
    if (use_smem) LG[e] = v;
  }
  __syncthreads();
  // T1 = Zb L_G, then H = I - L_G^T T1 (lower part) -> LH (global)
  cta_tri_gemm(Zb, A, T1, Q, 0);
  __syncthreads();
  cta_tri_gemm(A, T1, LH, Q, 1);
  __syncthreads();
  double* B = use_smem ? smf : LH;
  if (use_smem)
    for (int e = tid; e < Q * Q; e += nt) B[e] = LH[e];
  __syncthreads();
  f = cta_cholesky(B, Q, &sfail);
  if (use_smem)
    for (int e = tid; e < Q * Q; e += nt) LH[e] = B[e];
  if (tid == 0) *info = f;  // -1: reduced system positive definite
}

// blocked in-CTA triangular solve with a row-major lower factor L (Q x Q):
// trans = 0: L z = b, trans = 1: L^T z = b; z overwrites b (shared memory).
__device__ void cta_trsv(const double* L, int Q, double* b, int trans) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int nblk = (Q + 31) / 32;
  for (int bb = 0; bb < nblk; ++bb) {
    const int blk = trans ? (nblk - 1 - bb) : bb;
    const int c0 = blk * 32, nc = min(32, Q - c0);
    if (wid == 0) {
      double v = lane < nc ? b[c0 + lane] : 0.0;
      if (!trans) {
        for (int j = 0; j < nc; ++j) {
          const double zj = __shfl_sync(0xffffffffu, v, j) / L[(c0 + j) * Q + c0 + j];
          if (lane == j) v = zj;
          if (lane > j && lane < nc) v -= L[(c0 + lane) * Q + c0 + j] * zj;
        }
      } else {
        for (int j = nc - 1; j >= 0; --j) {
          const double zj = __shfl_sync(0xffffffffu, v, j) / L[(c0 + j) * Q + c0 + j];
          if (lane == j) v = zj;
          if (lane < j) v -= L[(c0 + j) * Q + c0 + lane] * zj;
        }
      }
      if (lane < nc) b[c0 + lane] = v;
    }
    __syncthreads();
    if (!trans) {
      for (int r = c0 + nc + wid; r < Q; r += nw) {
        double acc = lane < nc ? L[r * Q + c0 + lane] * b[c0 + lane] : 0.0;
        acc = warp_sum(acc);
        if (lane == 0) b[r] -= acc;
      }
    } else {
      for (int c = tid; c < c0; c += blockDim.x) {
        double acc = 0.0;
        for (int r = 0; r < nc; ++r) acc = fma(L[(c0 + r) * Q + c], b[c0 + r], acc);
        b[c] -= acc;
      }
    }
    __syncthreads();
  }
}

// one CTA: w = LG^{-T} LH^{-T} LH^{-1} LG^T Zb u   (u, w: Q vectors).  With
// use_smem the two factors are staged in shared memory first (latency-bound
// substitution steps then hit smem instead of L2).
__global__ void __launch_bounds__(256) k_lowrank_apply(const double* __restrict__ LGg,
                                                       const double* __restrict__ LHg,
                                                       const double* __restrict__ Zb, int k,
                                                       const double* __restrict__ u,
                                                       double* __restrict__ w, int use_smem) {
  extern __shared__ double sm[];
  const int Q = k * k;
  double* a = sm;
  double* b = sm + Q;
  const double* LG = LGg;
  const double* LH = LHg;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  if (use_smem) {
    double* sg = sm + 2 * Q;
    double* shh = sg + Q * Q;
    for (int e = tid; e < Q * Q; e += blockDim.x) {
      sg[e] = LGg[e];
      shh[e] = LHg[e];
    }
    LG = sg;
    LH = shh;
  }
  for (int r = wid; r < Q; r += nw) {  // a = Zb u (warp per row, coalesced)
    double acc = 0.0;
    for (int c = lane; c < Q; c += 32) acc = fma(Zb[r * Q + c], u[c], acc);
    acc = warp_sum(acc);
    if (lane == 0) a[r] = acc;
  }
  __syncthreads();
  for (int r = tid; r < Q; r += blockDim.x) {  // b = LG^T a
    double acc = 0.0;
    for (int t = r; t < Q; ++t) acc = fma(LG[t * Q + r], a[t], acc);
    b[r] = acc;
  }
  __syncthreads();
  cta_trsv(LH, Q, b, 0);
  cta_trsv(LH, Q, b, 1);
  cta_trsv(LG, Q, b, 1);
  for (int r = tid; r < Q; r += blockDim.x) w[r] = b[r];
}

}  // namespace

#define NMFB_K_SWITCH(k, MACRO) \
  switch (k) {                  \
    MACRO(1) MACRO(2) MACRO(3) MACRO(4) MACRO(5) MACRO(6) MACRO(7) MACRO(8) MACRO(9) MACRO(10) \
    MACRO(11) MACRO(12) MACRO(13) MACRO(14) MACRO(15) MACRO(16) \
    default: return NMFB_EINVAL; \
  }

extern "C" int nmfb_d_factor(const double* XtX, const double* Yt, const double* S, double rho,
                             long m, long k, double* LD, double* Dinvpk, double* YYpk, int* bad,
                             void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (m <= 0) return NMFB_EINVAL;
  cudaMemsetAsync(bad, 0x7F, sizeof(int), st);
  const unsigned blocks = (unsigned)((m + 127) / 128);
#define CASE(KK)                                                                                 \
  case KK:                                                                                       \
    ++g_nmfb_launches, k_d_factor<KK><<<blocks, 128, 0, st>>>(XtX, Yt, S, rho, m, LD, Dinvpk,    \
                                                              YYpk, bad);                        \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_lowrank_factor(const double* Zpk, const double* Gpk, long k, double* LG,
                                   double* LH, double* work, int* info, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const long Q = k * k;
  const size_t smem = (size_t)2 * Q * Q * sizeof(double);
  const int use_smem = smem <= 200 * 1024;
  if (use_smem)
    cudaFuncSetAttribute(k_lowrank_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  ++g_nmfb_launches, k_lowrank_factor<<<1, 1024, use_smem ? smem : 0, st>>>(
      Zpk, Gpk, (int)k, LG, LH, work, work + Q * Q, info, use_smem);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// dy = A^{-1} rhs with A = D - U Zb U^T (factors from nmfb_d_factor / nmfb_lowrank_factor).
// Zb = work[0 .. Q^2) as left by nmfb_lowrank_factor; scratch: T (m,k), u, w (Q each).
extern "C" int nmfb_lowrank_solve(const double* LD, const double* Yt, const double* LG,
                                  const double* LH, const double* Zb, long m, long k,
                                  const double* rhs, double* dy, double* u, double* w,
                                  double* cwork, long cwork_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned blocks = (unsigned)((m + 127) / 128);
#define CASE(KK)                                                                           \
  case KK:                                                                                 \
    ++g_nmfb_launches, k_d_solve<KK><<<blocks, 128, 0, st>>>(LD, rhs, m, dy);              \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  int rc = nmfb_colprod(Yt, 0, m, k, dy, k, u, nullptr, 1.0, cwork, cwork_len, stream);
  if (rc != NMFB_OK) return rc;
  const long Q = k * k;
  const size_t sm_full = (size_t)(2 * Q + 2 * Q * Q) * sizeof(double);
  const int apply_smem = sm_full <= 200 * 1024;
  const size_t sm_apply = apply_smem ? sm_full : 2 * Q * sizeof(double);
  if (apply_smem)
    cudaFuncSetAttribute(k_lowrank_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_apply);
  ++g_nmfb_launches, k_lowrank_apply<<<1, 256, sm_apply, st>>>(LG, LH, Zb, (int)k, u, w, apply_smem);
#define CASE(KK)                                                                           \
  case KK:                                                                                 \
    ++g_nmfb_launches, k_d_correct<KK><<<blocks, 128, 0, st>>>(LD, Yt, w, m, dy);          \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}
