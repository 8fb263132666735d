// Fused small-problem interior-point iteration (configs c1-c3: k <= 4, m k <= 2048).
//
// At these sizes every matrix is L2-resident and the general pipeline
// (csrc/ipm.cu + csrc/lowrank.cu, ~34 launches per Gauss-Newton iteration) is
// bound by launch latency and by tiny grids.  The same mathematics is fused
// into six kernels per iteration; cross-CTA reductions use the "last CTA
// finishes" pattern (partials -> __threadfence -> atomic ticket -> the last
// CTA sums the partials in block order), so results stay deterministic and the
// whole iteration is graph-capturable (tickets are reset by the last CTA).
//
//   k_sx  : rows  -> R1 factors, h, g, and Z / H / X^T X
//   k_sy  : 1 CTA -> Y side: rhs, D_j factors, G, capacitance factors, dY, dS,
//           Gdy, Y-side scalars (PAPER Eq. 12 via the rank-k^2 identity)
//   k_sdir: rows  -> dX, dR (back substitution), gtp / fraction-to-boundary
//   k_sarm: quartic Armijo coefficients + the 61 barrier trial sums
//   k_sstep: device Armijo selection + update with nudge (+ factorization copy)
//   k_sres: F = XY - M, graX, graY, ||F||^2 and the KKT sums of Eq. (9)
#include "common.cuh"
#include "nmfb200.h"

namespace {

constexpr int SX_THREADS = 128;

__device__ __forceinline__ int pkx(int a, int b, int k) {
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
  return a * k - a * (a - 1) / 2 + (b - a);
}

// "last CTA finishes": returns true in every thread of the CTA that arrived last.
__device__ __forceinline__ bool last_cta(unsigned int* ticket) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

__device__ __forceinline__ void reset_ticket(unsigned int* ticket) {
  if (threadIdx.x == 0) *ticket = 0u;
}

// sum_b part[b * stride + e] in block order, with 16 loads in flight per batch
__device__ __forceinline__ double sum_over_blocks(const double* part, long nb, long stride, long e,
                                                  bool is_max = false) {
  double acc = is_max ? -1.0 / 0.0 : 0.0;
  long b = 0;
  for (; b + 16 <= nb; b += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = part[(b + u) * stride + e];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = is_max ? fmax(acc, v[u]) : acc + v[u];
  }
  for (; b < nb; ++b) {
    const double q = part[b * stride + e];
    acc = is_max ? fmax(acc, q) : acc + q;
  }
  return acc;
}

// ---------------------------------------------------------------------------
// k_sx: thread per row; partial reductions per CTA of Z (kk x kk), H (K x K),
// X^T X (K x K); the last CTA writes the totals.
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(SX_THREADS) k_sx(
    const double* __restrict__ X, const double* __restrict__ R, const double* __restrict__ gX,
    const double* __restrict__ Yt, long m, double mux, double rho, long n,
    double* __restrict__ Lout, double* __restrict__ hout, double* __restrict__ part,
    unsigned int* __restrict__ ticket, double* __restrict__ Zout, double* __restrict__ Hout,
    double* __restrict__ XtXout, int* __restrict__ bad) {
  constexpr int KK = K * (K + 1) / 2;
  constexpr int NOUT = KK * KK + 2 * K * K;
  __shared__ double gy[K * K];
  __shared__ double sA[SX_THREADS][KK], sXX[SX_THREADS][KK], sx[SX_THREADS][K], sg[SX_THREADS][K];
  const int tid = threadIdx.x;
  // Y Y^T (replicated, fixed order): warp per entry, lanes stride the columns
  {
    const int lane = tid & 31, wid = tid >> 5;
    for (int e = wid; e < K * K; e += SX_THREADS / 32) {
      const int a = e / K, b = e % K;
      double s = 0.0;
      for (long j = lane; j < m; j += 32) s = fma(Yt[j * K + a], Yt[j * K + b], s);
      s = warp_sum(s);
      if (lane == 0) gy[e] = s;
    }
  }
  __syncthreads();
  const long i = (long)blockIdx.x * SX_THREADS + tid;
  const int nrow = (int)min((long)SX_THREADS, n - (long)blockIdx.x * SX_THREADS);
  if (tid < nrow) {
    double x[K], L[K][K], b[K], hv[K], gv[K];
#pragma unroll
    for (int p = 0; p < K; ++p) x[p] = X[i * K + p];
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int c = 0; c < K; ++c) L[a][c] = (c <= a) ? gy[a * K + c] : 0.0;
#pragma unroll
    for (int p = 0; p < K; ++p) {
      L[p][p] += rho + R[i * K + p] / x[p];
      b[p] = mux / x[p] - gX[i * K + p];
    }
    bool ok = true;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double s = L[j][j];
#pragma unroll
      for (int p = 0; p < j; ++p) s -= L[j][p] * L[j][p];
      if (!(s > 0.0)) ok = false;
      const double d = sqrt(fmax(s, 1e-300));
      L[j][j] = d;
#pragma unroll
      for (int r = j + 1; r < K; ++r) {
        double t = L[r][j];
#pragma unroll
        for (int p = 0; p < j; ++p) t -= L[r][p] * L[j][p];
        L[r][j] = t / d;
      }
    }
    if (!ok) atomicMin(bad, (int)i);
#pragma unroll
    for (int a = 0; a < K; ++a) {
      double s = b[a];
#pragma unroll
      for (int p = 0; p < a; ++p) s -= L[a][p] * hv[p];
      hv[a] = s / L[a][a];
    }
#pragma unroll
    for (int a = K - 1; a >= 0; --a) {
      double s = hv[a];
#pragma unroll
      for (int p = a + 1; p < K; ++p) s -= L[p][a] * gv[p];
      gv[a] = s / L[a][a];
    }
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
#pragma unroll
    for (int a = 0; a < K; ++a) {
      hout[i * K + a] = hv[a];
      sx[tid][a] = x[a];
      sg[tid][a] = gv[a];
#pragma unroll
      for (int c = 0; c < K; ++c) Lout[(i * K + a) * K + c] = (c <= a) ? L[a][c] : 0.0;
#pragma unroll
      for (int c = a; c < K; ++c) {
        double s = 0.0;
#pragma unroll
        for (int p = 0; p < K; ++p)
          if (p >= c) s = fma(Li[p][a], Li[p][c], s);
        const int e = a * K - a * (a - 1) / 2 + (c - a);
        sA[tid][e] = s;
        sXX[tid][e] = x[a] * x[c];
      }
    }
  }
  __syncthreads();
  // per-CTA partials of Z, H = sum x g^T, X^T X (thread per output, rows in order)
  for (int e = tid; e < NOUT; e += blockDim.x) {
    double s = 0.0;
    if (e < KK * KK) {
      const int ab = e / KK, pq = e % KK;
      for (int r = 0; r < nrow; ++r) s = fma(sA[r][ab], sXX[r][pq], s);
    } else if (e < KK * KK + K * K) {
      const int q = e - KK * KK, p = q / K, a = q % K;
      for (int r = 0; r < nrow; ++r) s = fma(sx[r][p], sg[r][a], s);
    } else {
      const int q = e - KK * KK - K * K, p = q / K, a = q % K;
      for (int r = 0; r < nrow; ++r) s = fma(sx[r][p], sx[r][a], s);
    }
    part[(long)blockIdx.x * NOUT + e] = s;
  }
  if (last_cta(ticket)) {
    for (int e = tid; e < NOUT; e += blockDim.x) {
      const double s = sum_over_blocks(part, gridDim.x, NOUT, e);
      if (e < KK * KK)
        Zout[e] = s;
      else if (e < KK * KK + K * K)
        Hout[e - KK * KK] = s;
      else
        XtXout[e - KK * KK - K * K] = s;
    }
    reset_ticket(ticket);
  }
}

// in-smem right-looking Cholesky of a Q x Q row-major matrix (Q <= 32) by
// warp 0, lane = row; returns the failing pivot (-1: PD) in lane 0.  The strict
// upper triangle is zeroed.
__device__ int small_chol(double* A, int Q) {
  int fail = -1;
  if (threadIdx.x < 32) {
    const int r = threadIdx.x;
    for (int j = 0; j < Q; ++j) {
      const double pv = A[j * Q + j];
      if (!(pv > 0.0)) {
        fail = j;
        break;
      }
      const double d = sqrt(pv);
      __syncwarp();
      if (r > j && r < Q) A[r * Q + j] /= d;
      if (r == j) A[j * Q + j] = d;
      __syncwarp();
      if (r > j && r < Q) {
        const double lrj = A[r * Q + j];
        for (int c = j + 1; c <= r; ++c) A[r * Q + c] -= lrj * A[c * Q + j];
      }
      __syncwarp();
    }
    __syncwarp();
    if (r < Q)
      for (int c = r + 1; c < Q; ++c) A[r * Q + c] = 0.0;
  }
  return fail;
}

// ---------------------------------------------------------------------------
// k_sy: one CTA, the whole replicated Y side of the Gauss-Newton direction.
// Writes the same factor buffers as the general path (LD, LG, LH, Zb) so the
// predictor can reuse them through nmfb_lowrank_solve.
// ysc = [gtp_y, a1_y, a2_y]; info = -1 iff the reduced system is PD.
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(256) k_sy(
    const double* __restrict__ Yt, const double* __restrict__ S, const double* __restrict__ gY,
    const double* __restrict__ XtX, const double* __restrict__ H, const double* __restrict__ Zpk,
    double rho, double muy, double tau, long m, double* __restrict__ LDout,
    double* __restrict__ LGout, double* __restrict__ LHout, double* __restrict__ Zbout,
    double* __restrict__ dY, double* __restrict__ dS, double* __restrict__ Gdy,
    double* __restrict__ ysc, int* __restrict__ info, int* __restrict__ bad) {
  constexpr int KK = K * (K + 1) / 2, Q = K * K;
  extern __shared__ double sm[];
  double* rhs = sm;                 // m*K
  double* t = rhs + m * K;          // m*K
  double* dinv = t + m * K;         // m*KK
  double* yy = dinv + m * KK;       // m*KK
  __shared__ double G[Q * Q], Zb[Q * Q], T1[Q * Q], Hm[Q * Q], u[Q], w[Q], w2[Q];
  __shared__ double red[3][32];
  __shared__ int s_fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  // 1. rhs_j = muy / y - graY - H y_j; 2. D_j factors
  for (long j = tid; j < m; j += nt) {
    double y[K], L[K][K];
#pragma unroll
    for (int p = 0; p < K; ++p) y[p] = Yt[j * K + p];
#pragma unroll
    for (int p = 0; p < K; ++p) {
      double ra = 0.0;
#pragma unroll
      for (int a = 0; a < K; ++a) ra = fma(H[p * K + a], y[a], ra);
      rhs[j * K + p] = (muy / y[p] - gY[j * K + p]) - ra;
    }
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int c = 0; c < K; ++c) L[a][c] = (c <= a) ? XtX[a * K + c] : 0.0;
#pragma unroll
    for (int p = 0; p < K; ++p) L[p][p] += rho + S[j * K + p] / y[p];
    bool ok = true;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      double s = L[c][c];
#pragma unroll
      for (int p = 0; p < c; ++p) s -= L[c][p] * L[c][p];
      if (!(s > 0.0)) ok = false;
      const double d = sqrt(fmax(s, 1e-300));
      L[c][c] = d;
#pragma unroll
      for (int r = c + 1; r < K; ++r) {
        double tt = L[r][c];
#pragma unroll
        for (int p = 0; p < c; ++p) tt -= L[r][p] * L[c][p];
        L[r][c] = tt / d;
      }
    }
    if (!ok) atomicMin(bad, (int)j);
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
#pragma unroll
    for (int a = 0; a < K; ++a) {
#pragma unroll
      for (int c = 0; c < K; ++c) LDout[(j * K + a) * K + c] = (c <= a) ? L[a][c] : 0.0;
#pragma unroll
      for (int c = a; c < K; ++c) {
        double s = 0.0;
#pragma unroll
        for (int p = 0; p < K; ++p)
          if (p >= c) s = fma(Li[p][a], Li[p][c], s);
        const int e = a * K - a * (a - 1) / 2 + (c - a);
        dinv[j * KK + e] = s;
        yy[j * KK + e] = y[a] * y[c];
      }
    }
    // t_j = D_j^{-1} rhs_j
    double z[K], v[K];
#pragma unroll
    for (int a = 0; a < K; ++a) {
      double s = rhs[j * K + a];
#pragma unroll
      for (int p = 0; p < a; ++p) s -= L[a][p] * z[p];
      z[a] = s / L[a][a];
    }
#pragma unroll
    for (int a = K - 1; a >= 0; --a) {
      double s = z[a];
#pragma unroll
      for (int p = a + 1; p < K; ++p) s -= L[p][a] * v[p];
      v[a] = s / L[a][a];
    }
#pragma unroll
    for (int a = 0; a < K; ++a) t[j * K + a] = v[a];
  }
  __syncthreads();
  // 3. G = sum_j (y_j y_j^T) (x) D_j^{-1} (unpacked Q x Q), Zb unpacked, u = U^T t;
  //    warp per entry, lanes stride j, fixed butterfly -> deterministic
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int e = wid; e < KK * KK + Q; e += nw) {
    double s = 0.0;
    if (e < KK * KK) {
      const int ab = e / KK, pq = e % KK;
      for (long j = lane; j < m; j += 32) s = fma(yy[j * KK + ab], dinv[j * KK + pq], s);
    } else {
      const int q = e - KK * KK, a = q / K, p = q % K;
      for (long j = lane; j < m; j += 32) s = fma(Yt[j * K + a], t[j * K + p], s);
    }
    s = warp_sum(s);
    if (lane == 0) {
      if (e < KK * KK)
        T1[e] = s;  // packed G, unpacked below
      else
        u[e - KK * KK] = s;
    }
  }
  __syncthreads();
  for (int e = tid; e < Q * Q; e += nt) {
    const int r = e / Q, c = e % Q;
    const int a = r / K, p = r % K, b = c / K, q = c % K;
    const int ab = pkx(a, b, K), pq = pkx(p, q, K);
    G[e] = T1[ab * KK + pq];
    Zb[e] = Zpk[ab * KK + pq];
  }
  __syncthreads();
  // 4. LG = chol(G); H = I - LG^T Zb LG; LH = chol(H)
  int f = small_chol(G, Q);
  if (tid == 0) s_fail = f;
  __syncthreads();
  for (int e = tid; e < Q * Q; e += nt) {
    const int r = e / Q, c = e % Q;
    double s = 0.0;
    for (int q = c; q < Q; ++q) s = fma(Zb[r * Q + q], G[q * Q + c], s);
    T1[e] = s;
  }
  __syncthreads();
  for (int e = tid; e < Q * Q; e += nt) {
    const int r = e / Q, c = e % Q;
    double s = 0.0;
    for (int q = r; q < Q; ++q) s = fma(G[q * Q + r], T1[q * Q + c], s);
    Hm[e] = (r == c ? 1.0 : 0.0) - s;
  }
  __syncthreads();
  f = small_chol(Hm, Q);
  if (tid == 0 && s_fail < 0) s_fail = f;
  __syncthreads();
  for (int e = tid; e < Q * Q; e += nt) {
    LGout[e] = G[e];
    LHout[e] = Hm[e];
    Zbout[e] = Zb[e];
  }
  // 5. w = LG^{-T} LH^{-T} LH^{-1} LG^T Zb u (thread 0; Q <= 16)
  if (tid == 0) {
    for (int r = 0; r < Q; ++r) {
      double s = 0.0;
      for (int c = 0; c < Q; ++c) s = fma(Zb[r * Q + c], u[c], s);
      w[r] = s;
    }
    for (int r = 0; r < Q; ++r) {
      double s = 0.0;
      for (int q = r; q < Q; ++q) s = fma(G[q * Q + r], w[q], s);
      w2[r] = s;
    }
    for (int i = 0; i < Q; ++i) {
      double s = w2[i];
      for (int p = 0; p < i; ++p) s -= Hm[i * Q + p] * w[p];
      w[i] = s / Hm[i * Q + i];
    }
    for (int i = Q - 1; i >= 0; --i) {
      double s = w[i];
      for (int p = i + 1; p < Q; ++p) s -= Hm[p * Q + i] * w2[p];
      w2[i] = s / Hm[i * Q + i];
    }
    for (int i = Q - 1; i >= 0; --i) {
      double s = w2[i];
      for (int p = i + 1; p < Q; ++p) s -= G[p * Q + i] * w[p];
      w[i] = s / G[i * Q + i];
    }
    *info = s_fail;
  }
  __syncthreads();
  // 6. dY_j = t_j + D_j^{-1}(W^T y_j); dS; Y-side scalars
  double gtp = 0.0, a1 = 1.0 / 0.0, a2 = 1.0 / 0.0;
  for (long j = tid; j < m; j += nt) {
    double L[K][K], v[K], z[K];
#pragma unroll
    for (int p = 0; p < K; ++p) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < K; ++a) s = fma(Yt[j * K + a], w[a * K + p], s);
      v[p] = s;
#pragma unroll
      for (int c = 0; c < K; ++c) L[p][c] = LDout[(j * K + p) * K + c];
    }
#pragma unroll
    for (int a = 0; a < K; ++a) {
      double s = v[a];
#pragma unroll
      for (int p = 0; p < a; ++p) s -= L[a][p] * z[p];
      z[a] = s / L[a][a];
    }
#pragma unroll
    for (int a = K - 1; a >= 0; --a) {
      double s = z[a];
#pragma unroll
      for (int p = a + 1; p < K; ++p) s -= L[p][a] * v[p];
      v[a] = s / L[a][a];
    }
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const double d = t[j * K + a] + v[a];
      t[j * K + a] = d;
      dY[j * K + a] = d;
      const double y = Yt[j * K + a], s = S[j * K + a];
      const double ds = muy / y - s - (s / y) * d;
      dS[j * K + a] = ds;
      gtp = fma(d, gY[j * K + a] - muy / y, gtp);
      if (d < 0.0) a1 = fmin(a1, -tau * y / d);
      if (ds < 0.0) a2 = fmin(a2, -tau * s / ds);
    }
  }
  __syncthreads();
  for (int e = wid; e < K * K; e += nw) {  // Gdy = sum_j y_j dy_j^T
    const int a = e / K, b = e % K;
    double s = 0.0;
    for (long j = lane; j < m; j += 32) s = fma(Yt[j * K + a], t[j * K + b], s);
    s = warp_sum(s);
    if (lane == 0) Gdy[e] = s;
  }
  // fixed-tree block reductions of the Y-side scalars
  gtp = warp_sum(gtp);
  a1 = warp_min(a1);
  a2 = warp_min(a2);
  if (lane == 0) {
    red[0][wid] = gtp;
    red[1][wid] = a1;
    red[2][wid] = a2;
  }
  __syncthreads();
  if (tid == 0) {
    double g = 0.0, m1 = 1.0 / 0.0, m2 = 1.0 / 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      g += red[0][q];
      m1 = fmin(m1, red[1][q]);
      m2 = fmin(m2, red[2][q]);
    }
    ysc[0] = g;
    ysc[1] = m1;
    ysc[2] = m2;
  }
}

// ---------------------------------------------------------------------------
// k_sdir: rows -> dX, dR; combines with the Y-side scalars into
// out = [gtp, a1max, a2max, gtp_rows, gtp_cols] (same layout as nmfb_direction).
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(128) k_sdir(
    const double* __restrict__ Lin, const double* __restrict__ h, const double* __restrict__ Gdy,
    const double* __restrict__ X, const double* __restrict__ R, const double* __restrict__ gX,
    double mux, double tau, long n, double* __restrict__ dX, double* __restrict__ dR,
    const double* __restrict__ ysc, double* __restrict__ part, unsigned int* __restrict__ ticket,
    double* __restrict__ out) {
  __shared__ double gd[K * K];
  __shared__ double red[3][4];
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) gd[e] = Gdy[e];
  __syncthreads();
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  double gtp = 0.0, a1 = 1.0 / 0.0, a2 = 1.0 / 0.0;
  if (i < n) {
    double L[K][K], v[K], q[K], t[K], dx[K], x[K];
#pragma unroll
    for (int a = 0; a < K; ++a) {
      x[a] = X[i * K + a];
#pragma unroll
      for (int c = 0; c < K; ++c) L[a][c] = Lin[(i * K + a) * K + c];
    }
#pragma unroll
    for (int a = 0; a < K; ++a) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < K; ++b) s = fma(gd[a * K + b], x[b], s);
      v[a] = s;
    }
#pragma unroll
    for (int a = 0; a < K; ++a) {
      double s = v[a];
#pragma unroll
      for (int p = 0; p < a; ++p) s -= L[a][p] * q[p];
      q[a] = s / L[a][a];
    }
#pragma unroll
    for (int a = 0; a < K; ++a) t[a] = h[i * K + a] - q[a];
#pragma unroll
    for (int a = K - 1; a >= 0; --a) {
      double s = t[a];
#pragma unroll
      for (int p = a + 1; p < K; ++p) s -= L[p][a] * dx[p];
      dx[a] = s / L[a][a];
    }
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const double r = R[i * K + a], d = dx[a];
      const double dr = mux / x[a] - r - (r / x[a]) * d;
      dX[i * K + a] = d;
      dR[i * K + a] = dr;
      gtp = fma(d, gX[i * K + a] - mux / x[a], gtp);
      if (d < 0.0) a1 = fmin(a1, -tau * x[a] / d);
      if (dr < 0.0) a2 = fmin(a2, -tau * r / dr);
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  gtp = warp_sum(gtp);
  a1 = warp_min(a1);
  a2 = warp_min(a2);
  if (lane == 0) {
    red[0][wid] = gtp;
    red[1][wid] = a1;
    red[2][wid] = a2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double g = 0.0, m1 = 1.0 / 0.0, m2 = 1.0 / 0.0;
    for (int q = 0; q < 4; ++q) {
      g += red[0][q];
      m1 = fmin(m1, red[1][q]);
      m2 = fmin(m2, red[2][q]);
    }
    part[blockIdx.x * 3 + 0] = g;
    part[blockIdx.x * 3 + 1] = m1;
    part[blockIdx.x * 3 + 2] = m2;
  }
  if (last_cta(ticket)) {
    __shared__ double fin[3];
    if (threadIdx.x < 3) {
      // minima via max of negatives; sums in block order
      const int q = threadIdx.x;
      double v;
      if (q == 0) {
        v = sum_over_blocks(part, gridDim.x, 3, 0);
      } else {
        v = 1.0;
        long b = 0;
        const long nb = gridDim.x;
        for (; b + 16 <= nb; b += 16) {
          double w[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) w[u] = part[(b + u) * 3 + q];
#pragma unroll
          for (int u = 0; u < 16; ++u) v = fmin(v, w[u]);
        }
        for (; b < nb; ++b) v = fmin(v, part[b * 3 + q]);
      }
      fin[q] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      out[0] = fin[0] + ysc[0];
      out[1] = fmin(fin[1], ysc[1]);
      out[2] = fmin(fin[2], ysc[2]);
      out[3] = fin[0];
      out[4] = ysc[0];
      *ticket = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// k_sarm: blocks [0, ntr) compute one barrier trial each over all x and y
// entries; blocks [ntr, ntr + nq) the quartic partials over (i, j); the last
// CTA sums the quartic partials.  sc = scalar block (alpha max at sc[5]).
// ---------------------------------------------------------------------------
constexpr int SARM_TG = 16;   // trials per group (one accumulator pair each)
constexpr int SARM_CPG = 32;  // CTAs per trial group

template <int K>
__global__ void __launch_bounds__(256) k_sarm(
    const double* __restrict__ F, long n, long m, const double* __restrict__ X,
    const double* __restrict__ dX, const double* __restrict__ Yt, const double* __restrict__ dY,
    double* __restrict__ sc, int ntr, double* __restrict__ part,
    unsigned int* __restrict__ ticket) {
  __shared__ double sh[32];
  __shared__ double wred[8][2 * SARM_TG];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ngroups = (ntr + SARM_TG - 1) / SARM_TG;
  const int ntrial_ctas = ngroups * SARM_CPG;
  double* tpart = part + 6 * 256;  // trial partials after the quartic partials
  if ((int)blockIdx.x < ntrial_ctas) {
    const int grp = blockIdx.x / SARM_CPG, sub = blockIdx.x % SARM_CPG;
    const int t0 = grp * SARM_TG;
    const double amax = sc[5];
    double ax[SARM_TG], ay[SARM_TG];
#pragma unroll
    for (int q = 0; q < SARM_TG; ++q) ax[q] = ay[q] = 0.0;
    const long nx = n * K, ntot = n * K + m * K;
    for (long e = (long)sub * blockDim.x + tid; e < ntot; e += (long)SARM_CPG * blockDim.x) {
      const bool isx = e < nx;
      const double num = isx ? dX[e] : dY[e - nx], den = isx ? X[e] : Yt[e - nx];
#pragma unroll
      for (int q = 0; q < SARM_TG; ++q) {
        if (t0 + q < ntr) {  // (alpha dv) / v, the oracle's association
          const double v = log1p(ldexp(amax, -(t0 + q)) * num / den);
          if (isx)
            ax[q] += v;
          else
            ay[q] += v;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < SARM_TG; ++q) {
      const double vx = warp_sum(ax[q]), vy = warp_sum(ay[q]);
      if (lane == 0) {
        wred[wid][2 * q] = vx;
        wred[wid][2 * q + 1] = vy;
      }
    }
    __syncthreads();
    if (tid < 2 * SARM_TG) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += wred[w][tid];
      tpart[(long)blockIdx.x * 2 * SARM_TG + tid] = v;
    }
  } else {
    const long qb = blockIdx.x - ntrial_ctas, nq = gridDim.x - ntrial_ctas;
    double sq[6] = {0, 0, 0, 0, 0, 0};
    for (long e = qb * blockDim.x + tid; e < n * m; e += nq * blockDim.x) {
      const long i = e / m, j = e - i * m;
      const double a = F[e];
      double b = 0.0, c = 0.0;
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const double x = X[i * K + p], dx = dX[i * K + p];
        const double y = Yt[j * K + p], dy = dY[j * K + p];
        b = fma(dx, y, fma(x, dy, b));
        c = fma(dx, dy, c);
      }
      sq[0] = fma(a, a, sq[0]);
      sq[1] = fma(a, b, sq[1]);
      sq[2] = fma(b, b, sq[2]);
      sq[3] = fma(a, c, sq[3]);
      sq[4] = fma(b, c, sq[4]);
      sq[5] = fma(c, c, sq[5]);
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const double v = warp_sum(sq[q]);
      if (lane == 0) wred[wid][q] = v;
    }
    __syncthreads();
    if (tid < 6) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += wred[w][tid];
      part[qb * 6 + tid] = v;
    }
  }
  if (last_cta(ticket)) {
    const long nq = gridDim.x - ntrial_ctas;
    if (tid < 6) sc[10 + tid] = sum_over_blocks(part, nq, 6, tid);
    for (int e = tid; e < 2 * ntr; e += blockDim.x) {
      const int t = e >> 1, c = e & 1;
      const int grp = t / SARM_TG, q = t % SARM_TG;
      sc[32 + e] = sum_over_blocks(tpart + (long)grp * SARM_CPG * 2 * SARM_TG + 2 * q + c,
                                   SARM_CPG, 2 * SARM_TG, 0);
    }
    __syncthreads();
    reset_ticket(ticket);
  }
  (void)sh;
}

// ---------------------------------------------------------------------------
// k_sstep: device Armijo selection (every CTA, identical arithmetic to
// k_armijo_select / the host loop), then copy (Xf, Ytf) <- (X, Y) and the
// nudged update of X, Y (alpha1) and R, S (alpha2).
// ---------------------------------------------------------------------------
__device__ void armijo_pick(const double* sc, double mu, double wx, double wy, double eta,
                            int max_bt, double* a1o, double* a2o, int* to) {
  const double gtp = sc[4], a1max = sc[5];
  const double ab = sc[11], bb = sc[12], ac = sc[13], bc = sc[14], cc = sc[15];
  const double c2 = __dadd_rn(__dmul_rn(0.5, bb), ac);
  int t = 0;
  double a1 = a1max;
  for (;;) {
    a1 = a1max / ldexp(1.0, t);
    const double q2 = __dmul_rn(a1, a1), q3 = __dmul_rn(q2, a1), q4 = __dmul_rn(q3, a1);
    double quad = __dadd_rn(__dmul_rn(a1, ab), __dmul_rn(q2, c2));
    quad = __dadd_rn(quad, __dmul_rn(q3, bc));
    quad = __dadd_rn(quad, __dmul_rn(__dmul_rn(0.5, q4), cc));
    const double bar = __dadd_rn(__dmul_rn(wx, sc[32 + 2 * t]), __dmul_rn(wy, sc[33 + 2 * t]));
    const double dphi = __dsub_rn(quad, __dmul_rn(mu, bar));
    if (dphi <= __dmul_rn(__dmul_rn(eta, a1), gtp)) break;
    ++t;
    if (t > max_bt) {
      a1 = 0.0;
      break;
    }
  }
  *a1o = a1;
  *a2o = (t > max_bt) ? 0.0 : sc[6];
  *to = t;
}

__global__ void __launch_bounds__(256) k_sstep(double* __restrict__ sc, double mu, double wx,
                                               double wy, double eta, int max_bt, double tau,
                                               const int* __restrict__ fcodes,
                                               double* __restrict__ X, double* __restrict__ R,
                                               const double* __restrict__ dX,
                                               const double* __restrict__ dR, long nx,
                                               double* __restrict__ Yt, double* __restrict__ S,
                                               const double* __restrict__ dY,
                                               const double* __restrict__ dS, long ny,
                                               double* __restrict__ Xf, double* __restrict__ Ytf) {
  __shared__ double sa1, sa2;
  if (threadIdx.x == 0) {
    double a1, a2;
    int t;
    if (fcodes[0] != 0x7F7F7F7F || fcodes[1] >= 0 || fcodes[2] != 0x7F7F7F7F) {
      a1 = a2 = 0.0;  // factorization failed: no step, the host redoes it (dense)
      t = -2;
    } else {
      armijo_pick(sc, mu, wx, wy, eta, max_bt, &a1, &a2, &t);
    }
    sa1 = a1;
    sa2 = a2;
    if (blockIdx.x == 0) {
      sc[1] = a1;
      sc[2] = (double)t;
      sc[3] = a2;
    }
  }
  __syncthreads();
  const double a1 = sa1, a2 = sa2;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < nx + ny; e += stride) {
    double *v, *r, *vf;
    const double *dv, *dr;
    long q;
    if (e < nx) {
      q = e;
      v = X;
      r = R;
      vf = Xf;
      dv = dX;
      dr = dR;
    } else {
      q = e - nx;
      v = Yt;
      r = S;
      vf = Ytf;
      dv = dY;
      dr = dS;
    }
    const double old = v[q], nv = old + a1 * dv[q];
    vf[q] = old;
    v[q] = (nv > 0.0) ? nv : (1.0 - tau) * old;
    const double oldr = r[q], nr = oldr + a2 * dr[q];
    r[q] = (nr > 0.0) ? nr : (1.0 - tau) * oldr;
  }
}

// ---------------------------------------------------------------------------
// k_sres: CTA = row block of RB rows.  Phase 1 (warp per row): F = XY - M,
// graX, ||F||^2; phase 2 (thread per column): graY partial over the block.
// The last CTA sums graY / ||F||^2 and evaluates the 12 KKT sums of Eq. (9)
// over all of x, r, y, s (same layout as nmfb_kkt_sums).
// ---------------------------------------------------------------------------
template <int K, typename T>
__global__ void __launch_bounds__(256) k_sres(
    const T* __restrict__ M, long n, long m, const double* __restrict__ X,
    const double* __restrict__ Yt, double* __restrict__ F, double* __restrict__ gX,
    double* __restrict__ gY, const double* __restrict__ R, const double* __restrict__ S,
    double mux, double muy, int RB, double* __restrict__ part, unsigned int* __restrict__ ticket,
    double* __restrict__ sc) {
  extern __shared__ double tile[];  // RB x m
  __shared__ double sh[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long r0 = (long)blockIdx.x * RB;
  const int nr = (int)min((long)RB, n - r0);
  double fsq = 0.0;
  // X-part KKT terms (lane 0 of each row's warp): sums 0..3, maxes |g|, x
  double k0 = 0.0, k1 = 0.0, k2 = 0.0, k3 = 0.0, kg = -1.0 / 0.0, kx = -1.0 / 0.0;
  for (int rr = wid; rr < nr; rr += (int)(blockDim.x >> 5)) {
    const long i = r0 + rr;
    double x[K], g[K];
#pragma unroll
    for (int p = 0; p < K; ++p) {
      x[p] = X[i * K + p];
      g[p] = 0.0;
    }
    for (long j = lane; j < m; j += 32) {
      double f = -(double)M[i * m + j];
#pragma unroll
      for (int p = 0; p < K; ++p) f = fma(x[p], Yt[j * K + p], f);
      F[i * m + j] = f;
      tile[rr * m + j] = f;
      fsq = fma(f, f, fsq);
#pragma unroll
      for (int p = 0; p < K; ++p) g[p] = fma(f, Yt[j * K + p], g[p]);
    }
#pragma unroll
    for (int p = 0; p < K; ++p) g[p] = warp_sum(g[p]);
    if (lane == 0) {
#pragma unroll
      for (int p = 0; p < K; ++p) {
        gX[i * K + p] = g[p];
        const double r = R[i * K + p];
        const double xr = x[p] * r;
        k0 = fma(g[p] - r, g[p] - r, k0);
        k1 = fma(xr - mux, xr - mux, k1);
        k2 = fma(xr, xr, k2);
        k3 += xr;
        kg = fmax(kg, fabs(g[p]));
        kx = fmax(kx, x[p]);
      }
    }
  }
  __syncthreads();
  const long stride = m * K + 7;
  const long pbase = (long)blockIdx.x * stride;
  for (long j = tid; j < m; j += blockDim.x) {
    double acc[K];
#pragma unroll
    for (int p = 0; p < K; ++p) acc[p] = 0.0;
    for (int rr = 0; rr < nr; ++rr) {
      const double f = tile[rr * m + j];
#pragma unroll
      for (int p = 0; p < K; ++p) acc[p] = fma(f, X[(r0 + rr) * K + p], acc[p]);
    }
#pragma unroll
    for (int p = 0; p < K; ++p) part[pbase + j * K + p] = acc[p];
  }
  fsq = block_sum(fsq, sh);
  if (tid == 0) part[pbase + m * K] = fsq;
  __syncthreads();
  k0 = block_sum(k0, sh);
  if (tid == 0) part[pbase + m * K + 1] = k0;
  __syncthreads();
  k1 = block_sum(k1, sh);
  if (tid == 0) part[pbase + m * K + 2] = k1;
  __syncthreads();
  k2 = block_sum(k2, sh);
  if (tid == 0) part[pbase + m * K + 3] = k2;
  __syncthreads();
  k3 = block_sum(k3, sh);
  if (tid == 0) part[pbase + m * K + 4] = k3;
  __syncthreads();
  kg = block_max(kg, sh);
  if (tid == 0) part[pbase + m * K + 5] = kg;
  __syncthreads();
  kx = block_max(kx, sh);
  if (tid == 0) part[pbase + m * K + 6] = kx;
  if (last_cta(ticket)) {
    __shared__ double xs[7];
    for (long e = tid; e < stride; e += blockDim.x) {
      const bool mx = (e >= m * K + 5);
      const double v = sum_over_blocks(part, gridDim.x, stride, e, mx);
      if (e < m * K)
        gY[e] = v;
      else
        xs[e - m * K] = v;
    }
    __syncthreads();
    // Y-part KKT sums over the (replicated) y, s, graY
    double v4 = 0.0, v5 = 0.0, v6 = 0.0, v7 = 0.0, v9 = -1.0 / 0.0, v11 = -1.0 / 0.0;
    for (long e = tid; e < m * K; e += blockDim.x) {
      const double y = Yt[e], s = S[e], g = gY[e];
      const double ys = y * s;
      v4 = fma(g - s, g - s, v4);
      v5 = fma(ys - muy, ys - muy, v5);
      v6 = fma(ys, ys, v6);
      v7 += ys;
      v9 = fmax(v9, fabs(g));
      v11 = fmax(v11, y);
    }
    v4 = block_sum(v4, sh);
    __syncthreads();
    v5 = block_sum(v5, sh);
    __syncthreads();
    v6 = block_sum(v6, sh);
    __syncthreads();
    v7 = block_sum(v7, sh);
    __syncthreads();
    v9 = block_max(v9, sh);
    __syncthreads();
    v11 = block_max(v11, sh);
    if (tid == 0) {
      sc[0] = xs[0];
      sc[16] = xs[1];
      sc[17] = xs[2];
      sc[18] = xs[3];
      sc[19] = xs[4];
      sc[20] = v4;
      sc[21] = v5;
      sc[22] = v6;
      sc[23] = v7;
      sc[24] = xs[5];
      sc[25] = v9;
      sc[26] = xs[6];
      sc[27] = v11;
    }
    __syncthreads();
    reset_ticket(ticket);
  }
}

}  // namespace

// ============================================================================
// C-ABI
// ============================================================================
#define NMFB_K_SMALL(k, MACRO) \
  switch (k) {                 \
    MACRO(1) MACRO(2) MACRO(3) MACRO(4) \
    default: return NMFB_EUNSUPPORTED; \
  }

extern "C" int nmfb_small_supported(long n, long m, long k) {
  return (k >= 1 && k <= 4 && m * k <= 2048 && m >= 1 && n >= 1) ? 1 : 0;
}

// workspace sizes (doubles / tickets) for the fused small-problem iteration
extern "C" long nmfb_small_work_len(long n, long m, long k) {
  const long kk = k * (k + 1) / 2;
  const long sx = ((n + SX_THREADS - 1) / SX_THREADS) * (kk * kk + 2 * k * k);
  const long rb = 32;
  const long sres = ((n + rb - 1) / rb) * (m * k + 7);
  const long sdir = ((n + 127) / 128) * 3;
  const long sarm = 6 * 256 + 4 * 32 * 2 * 16;
  long w = sx;
  if (sres > w) w = sres;
  if (sdir > w) w = sdir;
  if (sarm > w) w = sarm;
  return w;
}

// One fused Gauss-Newton direction: rows (k_sx) -> Y side (k_sy) -> rows (k_sdir).
// Outputs: L, h (rows), LD, LG, LH, Zb (factors, general-path layout), Z, H, XtX,
// dX, dR, dY, dS, Gdy; sc[4..8] = [gtp, a1max, a2max, gtp_rows, gtp_cols];
// iscal: [0] R1 failing row (0x7F7F7F7F: none), [1] capacitance info (-1 ok),
// [2] D_j failing column.
extern "C" int nmfb_small_direction(const double* X, const double* R, const double* gX,
                                    const double* Yt, const double* S, const double* gY,
                                    long n, long m, long k, double mux, double muy, double rho,
                                    double tau, double* L, double* h, double* LD, double* LG,
                                    double* LH, double* Zb, double* Z, double* H, double* XtX,
                                    double* dX, double* dR, double* dY, double* dS, double* Gdy,
                                    double* sc, int* iscal, double* work, unsigned int* tickets,
                                    void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!nmfb_small_supported(n, m, k)) return NMFB_EUNSUPPORTED;
  cudaMemsetAsync(iscal, 0x7F, sizeof(int), st);
  cudaMemsetAsync(iscal + 2, 0x7F, sizeof(int), st);
  const unsigned bx = (unsigned)((n + SX_THREADS - 1) / SX_THREADS);
  const long kk = k * (k + 1) / 2;
  const size_t sy_smem = (size_t)m * (2 * k + 2 * kk) * sizeof(double);
  double* ysc = sc + 24 + 0;  // scratch inside the KKT area is free before k_sres rewrites it
#define CASE(KK_)                                                                                \
  case KK_:                                                                                      \
    ++g_nmfb_launches, k_sx<KK_><<<bx, SX_THREADS, 0, st>>>(X, R, gX, Yt, m, mux, rho, n, L, h,   \
                                                            work, tickets + 0, Z, H, XtX, iscal); \
    nmfb_smem_attr(k_sy<KK_>, (int)sy_smem);  \
    ++g_nmfb_launches, k_sy<KK_><<<1, 256, sy_smem, st>>>(Yt, S, gY, XtX, H, Z, rho, muy, tau, m, \
                                                          LD, LG, LH, Zb, dY, dS, Gdy, ysc,      \
                                                          iscal + 1, iscal + 2);                 \
    ++g_nmfb_launches, k_sdir<KK_><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(                 \
        L, h, Gdy, X, R, gX, mux, tau, n, dX, dR, ysc, work, tickets + 1, sc + 4);               \
    break;
  NMFB_K_SMALL(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// Armijo sums (quartic coefficients at sc[10..15], barrier trials at sc[32..]),
// device selection + update (+ factorization copy), then F/gradients/KKT at
// the new point (sc[0] = ||F||^2, sc[16..27] KKT sums).
extern "C" int nmfb_small_step_refresh(const void* M, int m_is_f32, long n, long m, long k,
                                       double* X, double* R, double* Yt, double* S,
                                       const double* dX, const double* dR, const double* dY,
                                       const double* dS, double* Xf, double* Ytf, double* Fold,
                                       double* Fnew, double* gX, double* gY, double mu, double wx,
                                       double wy, double eta, int max_bt, double tau, int ntrials,
                                       double* sc, const int* fcodes, double* work,
                                       unsigned int* tickets, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!nmfb_small_supported(n, m, k)) return NMFB_EUNSUPPORTED;
  const int nq = 64;
  const int ntc = ((ntrials + SARM_TG - 1) / SARM_TG) * SARM_CPG;
  const int RB = 32;
  const size_t tile = (size_t)RB * m * sizeof(double);
  const unsigned br = (unsigned)((n + RB - 1) / RB);
#define CASE(KK_)                                                                                   \
  case KK_:                                                                                         \
    ++g_nmfb_launches, k_sarm<KK_><<<ntc + nq, 256, 0, st>>>(Fold, n, m, X, dX, Yt, dY, sc,        \
                                                                 ntrials, work, tickets + 2);       \
    ++g_nmfb_launches, k_sstep<<<nmfb_blocks((n + m) * KK_, 256, 148 * 4), 256, 0, st>>>(           \
        sc, mu, wx, wy, eta, max_bt, tau, fcodes, X, R, dX, dR, n * KK_, Yt, S, dY, dS, m * KK_,   \
        Xf, Ytf);  \
    if (m_is_f32) {                                                                                 \
      nmfb_smem_attr(k_sres<KK_, float>, \
                           (int)tile);                                                              \
      ++g_nmfb_launches, k_sres<KK_, float><<<br, 256, tile, st>>>(                                 \
          (const float*)M, n, m, X, Yt, Fnew, gX, gY, R, S, wx * mu, wy * mu, RB, work,             \
          tickets + 3, sc);                                                                         \
    } else {                                                                                        \
      nmfb_smem_attr(k_sres<KK_, double>, \
                           (int)tile);                                                              \
      ++g_nmfb_launches, k_sres<KK_, double><<<br, 256, tile, st>>>(                                \
          (const double*)M, n, m, X, Yt, Fnew, gX, gY, R, S, wx * mu, wy * mu, RB, work,            \
          tickets + 3, sc);                                                                         \
    }                                                                                               \
    break;
  NMFB_K_SMALL(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}
