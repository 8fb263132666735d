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

// in-place lower Cholesky of a Q x Q row-major matrix by one CTA; returns pivot
// failure column or -1 (valid in every thread)
__device__ int cta_cholesky(double* A, int Q, int* sfail) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) *sfail = -1;
  __syncthreads();
  for (int j = 0; j < Q; ++j) {
    if (tid == 0) {
      const double d = A[j * Q + j];
      if (!(d > 0.0))
        *sfail = j;
      else
        A[j * Q + j] = sqrt(d);
    }
    __syncthreads();
    if (*sfail >= 0) break;
    const double djj = A[j * Q + j];
    for (int r = j + 1 + tid; r < Q; r += nt) A[r * Q + j] /= djj;
    __syncthreads();
    const int rem = Q - j - 1;
    for (int e = tid; e < rem * rem; e += nt) {
      const int r = j + 1 + e / rem, c = j + 1 + e % rem;
      if (c <= r) A[r * Q + c] -= A[r * Q + j] * A[c * Q + j];
    }
    __syncthreads();
  }
  const int f = *sfail;
  __syncthreads();
  return f;
}

// one CTA: LG = chol(G), H = I - LG^T Zb LG, LH = chol(H).  work: 3 Q^2 doubles.
__global__ void __launch_bounds__(1024) k_lowrank_factor(const double* __restrict__ Zpk,
                                                         const double* __restrict__ Gpk, int k,
                                                         double* __restrict__ LG,
                                                         double* __restrict__ LH,
                                                         double* __restrict__ Zb,
                                                         double* __restrict__ T1,
                                                         int* __restrict__ info) {
  __shared__ int sfail;
  const int Q = k * k, KK = k * (k + 1) / 2;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < Q * Q; e += nt) {
    const int r = e / Q, c = e % Q;
    const int a = r / k, p = r % k, b = c / k, q = c % k;
    const int ab = pkx(a, b, k), pq = pkx(p, q, k);
    Zb[e] = Zpk[ab * KK + pq];
    LG[e] = (c <= r) ? Gpk[ab * KK + pq] : 0.0;
  }
  __syncthreads();
  int f = cta_cholesky(LG, Q, &sfail);
  if (f >= 0) {
    if (tid == 0) *info = 1000000 + f;  // G singular: Y^T rank deficient
    return;
  }
  for (int e = tid; e < Q * Q; e += nt) {  // zero the strict upper part left by the factor
    const int r = e / Q, c = e % Q;
    if (c > r) LG[e] = 0.0;
  }
  __syncthreads();
  // T1 = Zb LG
  for (int e = tid; e < Q * Q; e += nt) {
    const int r = e / Q, c = e % Q;
    double s = 0.0;
    for (int t = c; t < Q; ++t) s = fma(Zb[r * Q + t], LG[t * Q + c], s);
    T1[e] = s;
  }
  __syncthreads();
  // H = I - LG^T T1 (lower part)
  for (int e = tid; e < Q * Q; e += nt) {
    const int r = e / Q, c = e % Q;
    if (c > r) {
      LH[e] = 0.0;
      continue;
    }
    double s = 0.0;
    for (int t = r; t < Q; ++t) s = fma(LG[t * Q + r], T1[t * Q + c], s);
    LH[e] = (r == c ? 1.0 : 0.0) - s;
  }
  __syncthreads();
  f = cta_cholesky(LH, Q, &sfail);
  if (tid == 0) *info = f;  // -1: reduced system positive definite
}

// one CTA: w = LG^{-T} LH^{-T} LH^{-1} LG^T Zb u   (u, w: Q vectors; scratch 2Q)
__global__ void __launch_bounds__(256) k_lowrank_apply(const double* __restrict__ LG,
                                                       const double* __restrict__ LH,
                                                       const double* __restrict__ Zb, int k,
                                                       const double* __restrict__ u,
                                                       double* __restrict__ w) {
  extern __shared__ double sm[];
  const int Q = k * k;
  double* a = sm;
  double* b = sm + Q;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int r = tid; r < Q; r += nt) {  // a = Zb u
    double s = 0.0;
    for (int c = 0; c < Q; ++c) s = fma(Zb[r * Q + c], u[c], s);
    a[r] = s;
  }
  __syncthreads();
  for (int r = tid; r < Q; r += nt) {  // b = LG^T a
    double s = 0.0;
    for (int t = r; t < Q; ++t) s = fma(LG[t * Q + r], a[t], s);
    b[r] = s;
  }
  __syncthreads();
  // a = LH^{-1} b (forward), then b = LH^{-T} a (backward), then a = LG^{-T} b
  if (tid < 32) {
    for (int i = 0; i < Q; ++i) {
      double s = 0.0;
      for (int p = tid; p < i; p += 32) s = fma(LH[i * Q + p], a[p], s);
      s = warp_sum(s);
      if (tid == 0) a[i] = (b[i] - s) / LH[i * Q + i];
      __syncwarp();
    }
    for (int i = Q - 1; i >= 0; --i) {
      double s = 0.0;
      for (int p = i + 1 + tid; p < Q; p += 32) s = fma(LH[p * Q + i], b[p], s);
      s = warp_sum(s);
      if (tid == 0) b[i] = (a[i] - s) / LH[i * Q + i];
      __syncwarp();
    }
    for (int i = Q - 1; i >= 0; --i) {
      double s = 0.0;
      for (int p = i + 1 + tid; p < Q; p += 32) s = fma(LG[p * Q + i], a[p], s);
      s = warp_sum(s);
      if (tid == 0) a[i] = (b[i] - s) / LG[i * Q + i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int r = tid; r < Q; r += nt) w[r] = a[r];
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
  ++g_nmfb_launches, k_lowrank_factor<<<1, 1024, 0, st>>>(Zpk, Gpk, (int)k, LG, LH, work,
                                                          work + Q * Q, info);
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
  ++g_nmfb_launches, k_lowrank_apply<<<1, 256, 2 * Q * sizeof(double), st>>>(LG, LH, Zb, (int)k, u, w);
#define CASE(KK)                                                                           \
  case KK:                                                                                 \
    ++g_nmfb_launches, k_d_correct<KK><<<blocks, 128, 0, st>>>(LD, Yt, w, m, dy);          \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}
