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
#include "chol_blk.cuh"

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
  for (int p = 0; p < K; ++p) L[p][p] += rho + S[j * K + p] * (1.0 / y[p]);
  double rd[K];  // reciprocal pivots (one rsqrt per column; multiplies below)
#pragma unroll
  for (int c = 0; c < K; ++c) {
    double s = L[c][c];
#pragma unroll
    for (int p = 0; p < c; ++p) s -= L[c][p] * L[c][p];
    if (!(s > 0.0)) {
      atomicMin(bad, (int)j);
      return;
    }
    const double di = rsqrt(s);
    L[c][c] = s * di;
    rd[c] = di;
#pragma unroll
    for (int i = c + 1; i < K; ++i) {
      double t = L[i][c];
#pragma unroll
      for (int p = 0; p < c; ++p) t -= L[i][p] * L[c][p];
      L[i][c] = t * di;
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
        Li[a][c] = s * rd[a];
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
  double rd[K];
#pragma unroll
  for (int i = 0; i < K; ++i) rd[i] = 1.0 / L[i][i];  // independent: off the solve chains
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double s = v[i];
#pragma unroll
    for (int p = 0; p < i; ++p) s -= L[i][p] * z[p];
    z[i] = s * rd[i];
  }
#pragma unroll
  for (int i = K - 1; i >= 0; --i) {
    double s = z[i];
#pragma unroll
    for (int p = i + 1; p < K; ++p) s -= L[p][i] * v[p];
    v[i] = s * rd[i];
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
  double rd[K];
#pragma unroll
  for (int i = 0; i < K; ++i) rd[i] = 1.0 / L[i][i];  // independent: off the solve chains
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double s = v[i];
#pragma unroll
    for (int p = 0; p < i; ++p) s -= L[i][p] * z[p];
    z[i] = s * rd[i];
  }
#pragma unroll
  for (int i = K - 1; i >= 0; --i) {
    double s = z[i];
#pragma unroll
    for (int p = i + 1; p < K; ++p) s -= L[p][i] * v[p];
    v[i] = s * rd[i];
  }
#pragma unroll
  for (int a = 0; a < K; ++a) t[j * K + a] += v[a];
}

// ---------------------------------------------------------------------------
// Blocked factorization path (nmfb_lowrank_factor): Q = k^2 up to 256.
// ---------------------------------------------------------------------------
// unpack packed Z and G into full Zb and lower G (Q x Q); info <- -1
__global__ void k_lr_unpack(const double* __restrict__ Zpk, const double* __restrict__ Gpk, int k,
                            double* __restrict__ Zb, double* __restrict__ Gl,
                            int* __restrict__ info) {
  const int Q = k * k, KK = k * (k + 1) / 2;
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e == 0) *info = -1;
  if (e >= (long)Q * Q) return;
  const int r = (int)(e / Q), c = (int)(e % Q);
  const int a = r / k, p = r % k, b = c / k, q = c % k;
  const int ab = pkx(a, b, k), pq = pkx(p, q, k);
  Zb[e] = Zpk[ab * KK + pq];
  Gl[e] = (c <= r) ? Gpk[ab * KK + pq] : 0.0;
}

// 32 x 32 output tile per CTA:
//   mode 0: C = Zb L            (T1)
//   mode 1: C = I - L^T T1      (H; only the lower triangle is consumed)
// Both operands' 32-row strips over the whole contraction are staged at once by cp.async
// (A as [row][t], B transposed as [column][t], leading dimension = 4 mod 16: conflict-free
// fragment loads), then the tile is 2 DMMA m8n8k4 chains per warp.
inline int lr_gemm_ld(int Q) {
  const int kp = (Q + 3) & ~3;
  return kp + ((4 - (kp & 15)) & 15);
}
__global__ void __launch_bounds__(256) k_lr_gemm(const double* __restrict__ Am,
                                                 const double* __restrict__ Bm, int Q, int mode,
                                                 double* __restrict__ C,
                                                 const int* __restrict__ info, int LDK) {
  extern __shared__ double gsm[];
  double* As = gsm;             // [32][LDK]
  double* Bt = gsm + 32 * LDK;  // [32][LDK]
  if (*info >= 1000000) return;  // G already failed
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const int Kp = (Q + 3) & ~3;
  for (int e = tid; e < 32 * Kp; e += 256) {
    // A: (i, t) with t fastest for mode 0 (rows of Zb), i fastest for mode 1 (L^T)
    const int i = mode == 0 ? e / Kp : e & 31;
    const int t = mode == 0 ? e - i * Kp : e >> 5;
    const int r = r0 + i;
    double* da = As + i * LDK + t;
    if (r < Q && t < Q)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(da)),
                   "l"(mode == 0 ? Am + (long)r * Q + t : Am + (long)t * Q + r)
                   : "memory");
    else
      *da = 0.0;
    // B: (t, j) with j fastest (rows of B), stored transposed
    const int jb = e & 31, tb = e >> 5;
    const int c = c0 + jb;
    double* db = Bt + jb * LDK + tb;
    if (tb < Q && c < Q)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(db)),
                   "l"(Bm + (long)tb * Q + c)
                   : "memory");
    else
      *db = 0.0;
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int g8 = lane >> 2, t4 = lane & 3;
  const int br = wid >> 1, bc0 = 2 * (wid & 1);
  const double* fa = As + (8 * br + g8) * LDK + t4;
  const double* fb0 = Bt + (8 * bc0 + g8) * LDK + t4;
  const double* fb1 = fb0 + 8 * LDK;
  double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
  for (int ks = 0; ks < Kp; ks += 4) {
    const double a = fa[ks];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c00), "+d"(c01)
                 : "d"(a), "d"(fb0[ks]));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c10), "+d"(c11)
                 : "d"(a), "d"(fb1[ks]));
  }
  const int r = r0 + 8 * br + g8;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int c = c0 + 8 * (bc0 + h) + 2 * t4 + v;
      const double acc = h ? (v ? c11 : c10) : (v ? c01 : c00);
      if (r < Q && c < Q) C[(long)r * Q + c] = mode == 0 ? acc : ((r == c ? 1.0 : 0.0) - acc);
    }
}

// blocked in-CTA triangular solve with a row-major lower factor L (Q x Q):
// trans = 0: L z = b, trans = 1: L^T z = b; z overwrites b (shared memory).
// The diagonal block's row (column) of each lane is loaded into registers before the
// sweep, so a column step is one shuffle + one FMA; the off-diagonal update is one
// thread per row (column) with a 32-term FMA chain instead of a warp reduction per row.
__device__ void cta_trsv(const double* L, int Q, double* b, int trans) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nblk = (Q + 31) / 32;
  for (int bb = 0; bb < nblk; ++bb) {
    const int blk = trans ? (nblk - 1 - bb) : bb;
    const int c0 = blk * 32, nc = min(32, Q - c0);
    if (wid == 0) {
      // the block's row (column) of this lane, strictly off the diagonal and pre-scaled by
      // 1 / L_ll: a sweep step is then one shuffle and one FMA (no multiply, no select on
      // the dependent chain)
      const double rl = lane < nc ? 1.0 / L[(c0 + lane) * Q + c0 + lane] : 0.0;
      double v = lane < nc ? b[c0 + lane] * rl : 0.0;
      double lr[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool in = lane < nc && j < nc && (trans ? j > lane : j < lane);
        lr[j] = in ? (trans ? L[(c0 + j) * Q + c0 + lane] : L[(c0 + lane) * Q + c0 + j]) * rl : 0.0;
      }
      if (!trans) {
#pragma unroll
        for (int j = 0; j < 31; ++j) v = fma(-lr[j], __shfl_sync(0xffffffffu, v, j), v);
      } else {
#pragma unroll
        for (int j = 31; j > 0; --j) v = fma(-lr[j], __shfl_sync(0xffffffffu, v, j), v);
      }
      if (lane < nc) b[c0 + lane] = v;
    }
    __syncthreads();
    if (!trans) {
      for (int r = c0 + nc + tid; r < Q; r += blockDim.x) {  // four partial sums: the FMA
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;         // chain is a quarter as deep
        const double* lp = L + r * Q + c0;
        int c = 0;
        for (; c + 3 < nc; c += 4) {
          s0 = fma(lp[c], b[c0 + c], s0);
          s1 = fma(lp[c + 1], b[c0 + c + 1], s1);
          s2 = fma(lp[c + 2], b[c0 + c + 2], s2);
          s3 = fma(lp[c + 3], b[c0 + c + 3], s3);
        }
        for (; c < nc; ++c) s0 = fma(lp[c], b[c0 + c], s0);
        b[r] -= (s0 + s1) + (s2 + s3);
      }
    } else {
      for (int c = tid; c < c0; c += blockDim.x) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        const double* lp = L + c0 * Q + c;
        int r = 0;
        for (; r + 3 < nc; r += 4) {
          s0 = fma(lp[r * Q], b[c0 + r], s0);
          s1 = fma(lp[(r + 1) * Q], b[c0 + r + 1], s1);
          s2 = fma(lp[(r + 2) * Q], b[c0 + r + 2], s2);
          s3 = fma(lp[(r + 3) * Q], b[c0 + r + 3], s3);
        }
        for (; r < nc; ++r) s0 = fma(lp[r * Q], b[c0 + r], s0);
        b[c] -= (s0 + s1) + (s2 + s3);
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
    double* shh = sg + ((Q * Q + 1) & ~1);  // 16-byte aligned for cp.async
    // both factors in flight at once (cp.async), instead of one dependent load per trip
    for (int e = 2 * tid; e < Q * Q; e += 2 * blockDim.x) {
      if (e + 1 < Q * Q) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(sg + e)), "l"(LGg + e) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(shh + e)), "l"(LHg + e) : "memory");
      } else {
        sg[e] = LGg[e];
        shh[e] = LHg[e];
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    LG = sg;
    LH = shh;
  }
  // a = Zb u: four threads per row, every load of a pass in flight at once (a warp per row
  // paid one L2 round trip per row: 11 us of the kernel's 36 at Q = 100)
  for (int e = tid; e < Q; e += blockDim.x) b[e] = u[e];
  __syncthreads();
  for (int r0 = 0; r0 < Q; r0 += (int)(blockDim.x >> 2)) {
    const int r = r0 + (tid >> 2), q = tid & 3;
    double s0 = 0.0, s1 = 0.0;
    if (r < Q) {
      const double* zr = Zb + (long)r * Q;
      int c = q;
      for (; c + 4 < Q; c += 8) {
        s0 = fma(__ldg(zr + c), b[c], s0);
        s1 = fma(__ldg(zr + c + 4), b[c + 4], s1);
      }
      if (c < Q) s0 = fma(__ldg(zr + c), b[c], s0);
    }
    double s = s0 + s1;
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (r < Q && q == 0) a[r] = s;
  }
  __syncthreads();
  for (int r = tid; r < Q; r += blockDim.x) {  // b = LG^T a (four partial sums)
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int t = r;
    for (; t + 3 < Q; t += 4) {
      s0 = fma(LG[t * Q + r], a[t], s0);
      s1 = fma(LG[(t + 1) * Q + r], a[t + 1], s1);
      s2 = fma(LG[(t + 2) * Q + r], a[t + 2], s2);
      s3 = fma(LG[(t + 3) * Q + r], a[t + 3], s3);
    }
    for (; t < Q; ++t) s0 = fma(LG[t * Q + r], a[t], s0);
    b[r] = (s0 + s1) + (s2 + s3);
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
  // unpack -> chol(G) -> T1 = Zb LG -> H = I - LG^T T1 -> chol(H); Zb stays in work[0, Q^2)
  cudaStream_t st = (cudaStream_t)stream;
  const long Q = k * k;
  if (Q > 256) return NMFB_EUNSUPPORTED;
  double* Zb = work;
  double* T1 = work + Q * Q;
  const size_t csm = chol_blk_smem(Q);
  ++g_nmfb_launches, k_lr_unpack<<<(unsigned)((Q * Q + 255) / 256), 256, 0, st>>>(Zpk, Gpk, (int)k, Zb, LG, info);
  (void)csm;
  launch_chol(LG, (int)Q, info, 1000000, 0, 0, st);
  const dim3 g((unsigned)((Q + 31) / 32), (unsigned)((Q + 31) / 32));
  const int ldk = lr_gemm_ld((int)Q);
  const size_t gsm = (size_t)2 * 32 * ldk * sizeof(double);
  nmfb_smem_attr(k_lr_gemm, gsm);
  ++g_nmfb_launches, k_lr_gemm<<<g, 256, gsm, st>>>(Zb, LG, (int)Q, 0, T1, info, ldk);
  ++g_nmfb_launches, k_lr_gemm<<<g, 256, gsm, st>>>(LG, T1, (int)Q, 1, LH, info, ldk);
  launch_chol(LH, (int)Q, info, 0, 1, 1, st);
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
  const size_t sm_full = (size_t)(2 * Q + 2 * Q * Q + 2) * sizeof(double);
  const int apply_smem = sm_full <= 200 * 1024;
  const size_t sm_apply = apply_smem ? sm_full : 2 * Q * sizeof(double);
  if (apply_smem)
    nmfb_smem_attr(k_lowrank_apply, (int)sm_apply);
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
