// Persistent stage 1 (warm-started ANLS, PAPER Alg. 1 / SPEC.md:209-242) for small
// problems: every sweep of run_stage1 in ONE cooperative launch.
//
// Per sweep (two grid barriers):
//   X half  (rows, CTA-local): Y Y^T (replicated), ctb = M_rows Y^T, the per-row
//           tolerance, the bit-exact warp NNLS per row (seeded from the previous
//           passive set), then partials of X^T X, X^T M (entry-major), ||dX||^2,
//           ||X||^2 -> barrier
//   Y half  (a slice of columns per CTA): fixed-order reduction of X^T X and of
//           the slice's X^T M, the bit-exact NNLS per column, new Y and passive
//           sets to global, ||dY||^2, ||Y||^2, sum r2 partials -> barrier
//   stats   every CTA reduces the sweep scalars in the same order, tests
//           ||d(x,y)|| <= eps_stol (1 + ||(x,y)||) and reloads Y.
// The NNLS is nnls_warp.cuh (the reference's bits; this file is compiled with
// -fmad=false).  Failures: per-rhs status codes land in stX / stY and the loop
// stops after the sweep in which one occurred (the host raises, as run_stage1).
#include <cooperative_groups.h>

#include "common.cuh"
#include "nmfb200.h"
#include "nnls_warp.cuh"

namespace {

constexpr int ST = 256;  // threads per CTA
constexpr int SNW = ST / 32;

struct S1Args {
  const void* M;
  long n, m;
  double *X, *Yt, *Xn, *Yn;
  uint8_t *pX, *pY;
  const double *row_n2, *col_n2;
  int8_t *stX, *stY;
  double tol_fixed;  // < 0: per-rhs 1e-12 max(1, ||ctb||_inf)
  int first_mode, max_sweeps, fixed;
  double eps_stol;
  double* logv;  // per sweep: [0.5 sum r2, step, nrm, -]
  int* status;   // [sweeps done, converged, failed]
  double* work;
  int m_in_smem;
  long long* prof;  // optional per-sweep phase clocks of CTA 0 (scripts/stage1_phases.py)
};

long long* g_s1_prof = nullptr;  // set by nmfb_stage1_set_prof (profiling only)

#define S1STAMP(i)                                                                  \
  do {                                                                              \
    if (a.prof && blockIdx.x == 0 && threadIdx.x < 32 && sweep < 512)               \
      a.prof[(long)sweep * 16 + (i)] = clock64();                                   \
  } while (0)

__device__ __forceinline__ void gsync() { cooperative_groups::this_grid().sync(); }

// sum over CTAs of entry-major partials part[e * G + c], lanes stride CTAs
__device__ __forceinline__ double s1_cta_sum(const double* part, int G, long e) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int c = lane; c < G; c += 32) s = s + __ldcg(part + e * G + c);
  return warp_sum(s);
}

template <int K, int W, typename T>
__global__ void __launch_bounds__(ST, 1) k_stage1_persist(S1Args a) {
  constexpr int SEGS = 32 / W;
  const long n = a.n, m = a.m, N = m * K;
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const long r0 = (long)cta * n / G, r1 = (long)(cta + 1) * n / G;
  const int nr = (int)(r1 - r0);
  const long nrm = (n + G - 1) / G;
  const long c0 = (long)cta * m / G, c1 = (long)(cta + 1) * m / G;
  const int nc = (int)(c1 - c0);
  // workspace: PA [K*K + N + 3][G] (GX, ctbY, dX2, X2, fail), PB [4][G]
  const long NA = (long)K * K + N + 3;
  double* PA = a.work;
  double* PB = PA + NA * G;

  const long ncm = (m + G - 1) / G;
  const long CB = nrm > ncm ? (nrm > 16 ? nrm : 16) : (ncm > 16 ? ncm : 16);
  extern __shared__ double sm[];
  double* Ys = sm;            // N (replicated Y)
  double* Xs = Ys + N;        // nrm * K (current X rows)
  double* Xn = Xs + nrm * K;  // nrm * K (new X rows)
  double* cb = Xn + nrm * K;  // CB * K: ctb rows, then the column slice's ctb
  double* tl = cb + CB * K;   // CB tolerances
  double* Ms = tl + CB;       // own rows of M (optional)
  __shared__ double gyy[K * K], gxx[K * K], scal[8], red[4 * SNW];
  // k <= 6: the passive factor of every subset (2^K), rebuilt per half sweep, and a
  // thread-per-rhs register NNLS (tnnls_solve) instead of warp segments
  constexpr bool TAB = K <= 6;
  constexpr int KT = TAB ? K : 1;
  __shared__ double tab[(1 << KT) * KT * KT + (1 << KT)];
  auto build_tab = [&](const double* C) {
    if constexpr (!TAB) return;
    const int seg = lane / W;
    WNnls<K, W> f;
    f.sl = lane % W;
    f.sm = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << (seg * W));
    const bool own = f.sl < K;
#pragma unroll
    for (int c = 0; c < K; ++c) f.C[c] = own ? C[f.sl * K + c] : 0.0;
    for (int pm = wid * SEGS + seg; pm < (1 << K); pm += SNW * SEGS) {  // segment-uniform
      const bool ok = f.factor((unsigned)pm);
      if (own)
#pragma unroll
        for (int c = 0; c < K; ++c) tab[(pm * K + f.sl) * K + c] = f.Lr[c];
      if (f.sl == 0) tab[(K * K << K) + pm] = ok ? 1.0 : 0.0;
    }
  };

  for (long e = tid; e < N; e += ST) Ys[e] = a.Yt[e];
  for (long e = tid; e < (long)nr * K; e += ST) Xs[e] = a.X[r0 * K + e];
  const T* Mg = (const T*)a.M;
  if (a.m_in_smem)
    for (long e = tid; e < (long)nr * m; e += ST) Ms[e] = (double)Mg[r0 * m + e];
  __syncthreads();
  const double* Mp = a.m_in_smem ? Ms : (const double*)a.M + r0 * m;

  int sweep = 0, converged = 0, failed = 0;
  for (;;) {
    const int mode = (sweep > 0) ? 2 : a.first_mode;
    S1STAMP(0);
    // ---------------- X half ----------------
    for (int e = wid; e < K * K; e += SNW) {  // Y Y^T, lanes stride the columns
      const int p = e / K, q = e % K;
      double s = 0.0;
      for (long j = lane; j < m; j += 32) s = s + Ys[j * K + p] * Ys[j * K + q];
      s = warp_sum(s);
      if (lane == 0) gyy[e] = s;
    }
    for (long e = tid; e < (long)nr * K; e += ST) {  // ctb = M_rows Y^T
      const int rr = (int)(e / K), p = (int)(e % K);
      double s = 0.0;
      for (long j = 0; j < m; ++j) s = s + Mp[(long)rr * m + j] * Ys[j * K + p];
      cb[e] = s;
    }
    __syncthreads();
    S1STAMP(1);
    for (int rr = tid; rr < nr; rr += ST) {
      double t = 0.0;
      for (int p = 0; p < K; ++p) t = fmax(t, fabs(cb[rr * K + p]));
      tl[rr] = a.tol_fixed >= 0.0 ? a.tol_fixed : 1e-12 * fmax(1.0, t);
    }
    __syncthreads();
    if constexpr (TAB) {
      build_tab(gyy);
      __syncthreads();
      for (int rr = tid; rr < nr; rr += ST) {
        const long i = r0 + rr;
        TNnls<K, false> ts;
        ts.C = gyy;
        unsigned seed = 0u;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          ts.d[j] = cb[rr * K + j];
          seed |= (mode == 2 && a.pX[i * K + j] != 0 ? 1u : 0u) << j;
        }
        double x[K], r2;
        unsigned pm;
        long nch;
        int st;
        tnnls_solve<K, false>(ts, tab, tab + (K * K << K), a.row_n2[i], tl[rr], mode == 2, seed,
                              3 * K, x, pm, nch, r2, st);
#pragma unroll
        for (int j = 0; j < K; ++j) {
          Xn[rr * K + j] = x[j];
          a.pX[i * K + j] = ((pm >> j) & 1u) ? 1 : 0;
        }
        a.stX[i] = (int8_t)st;
      }
    } else {
      const int seg = lane / W;
      WNnls<K, W> s;
      s.sl = lane % W;
      s.sm = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << (seg * W));
      const bool own = s.sl < K;
#pragma unroll
      for (int c = 0; c < K; ++c) s.C[c] = own ? gyy[s.sl * K + c] : 0.0;
      for (int rr = wid * SEGS + seg; rr < nr; rr += SNW * SEGS) {  // segment-uniform
        const long i = r0 + rr;
        const double d = own ? cb[rr * K + s.sl] : 0.0;
        const bool use_seed = mode == 2;
        const bool sp = use_seed && own && a.pX[i * K + s.sl] != 0;
        double x, r2;
        unsigned pm;
        long nch;
        int st;
        nnls_seg_solve<K, W>(s, d, a.row_n2[i], tl[rr], use_seed, sp, 3 * K, x, pm, nch, r2, st);
        if (own) {
          Xn[rr * K + s.sl] = x;
          a.pX[i * K + s.sl] = ((pm >> s.sl) & 1u) ? 1 : 0;
        }
        if (s.sl == 0) a.stX[i] = (int8_t)st;
      }
    }
    __syncthreads();
    S1STAMP(2);
    // partials: G_X = Xn^T Xn, ctbY = M_rows^T Xn, ||dX||^2, ||X||^2, failure flag
    for (long e = tid; e < NA; e += ST) {
      double s = 0.0;
      if (e < K * K) {
        const int p = (int)(e / K), q = (int)(e % K);
        for (int rr = 0; rr < nr; ++rr) s = s + Xn[rr * K + p] * Xn[rr * K + q];
      } else if (e < K * K + N) {
        const long f = e - K * K, j = f / K;
        const int p = (int)(f % K);
        for (int rr = 0; rr < nr; ++rr) s = s + Mp[(long)rr * m + j] * Xn[rr * K + p];
      } else if (e == K * K + N) {
        for (long q = 0; q < (long)nr * K; ++q) {
          const double dd = Xn[q] - Xs[q];
          s = s + dd * dd;
        }
      } else if (e == K * K + N + 1) {
        for (long q = 0; q < (long)nr * K; ++q) s = s + Xs[q] * Xs[q];
      } else {
        for (int rr = 0; rr < nr; ++rr)
          if (a.stX[r0 + rr] != 0) s = 1.0;
      }
      __stcg(PA + e * G + cta, s);
    }
    S1STAMP(3);
    gsync();
    S1STAMP(4);
    // ---------------- Y half (this CTA's column slice) ----------------
    for (int e = wid; e < K * K; e += SNW) {
      const double v = s1_cta_sum(PA, G, e);
      if (lane == 0) gxx[e] = v;
    }
    for (long e = wid; e < (long)nc * K; e += SNW) {
      const double v = s1_cta_sum(PA, G, K * K + c0 * K + e);
      if (lane == 0) cb[e] = v;
    }
    __syncthreads();
    for (int cc = tid; cc < nc; cc += ST) {
      double t = 0.0;
      for (int p = 0; p < K; ++p) t = fmax(t, fabs(cb[cc * K + p]));
      tl[cc] = a.tol_fixed >= 0.0 ? a.tol_fixed : 1e-12 * fmax(1.0, t);
    }
    __syncthreads();
    S1STAMP(5);
    double ydx = 0.0, yy = 0.0, yr2 = 0.0, yfail = 0.0;  // per-thread (segment lane 0)
    if constexpr (TAB) {
      build_tab(gxx);
      __syncthreads();
      for (int cc = tid; cc < nc; cc += ST) {
        const long j = c0 + cc;
        TNnls<K, false> ts;
        ts.C = gxx;
        unsigned seed = 0u;
#pragma unroll
        for (int q = 0; q < K; ++q) {
          ts.d[q] = cb[cc * K + q];
          seed |= (mode == 2 && a.pY[j * K + q] != 0 ? 1u : 0u) << q;
        }
        double y[K], r2;
        unsigned pm;
        long nch;
        int st;
        tnnls_solve<K, false>(ts, tab, tab + (K * K << K), a.col_n2[j], tl[cc], mode == 2, seed,
                              3 * K, y, pm, nch, r2, st);
#pragma unroll
        for (int q = 0; q < K; ++q) {
          a.Yn[j * K + q] = y[q];
          a.pY[j * K + q] = ((pm >> q) & 1u) ? 1 : 0;
          const double yo = Ys[j * K + q];
          ydx = ydx + (y[q] - yo) * (y[q] - yo);
          yy = yy + yo * yo;
        }
        a.stY[j] = (int8_t)st;
        yr2 = yr2 + r2;
        if (st != 0) yfail = 1.0;
      }
    } else {
      const int seg = lane / W;
      WNnls<K, W> s;
      s.sl = lane % W;
      s.sm = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << (seg * W));
      const bool own = s.sl < K;
#pragma unroll
      for (int c = 0; c < K; ++c) s.C[c] = own ? gxx[s.sl * K + c] : 0.0;
      for (int cc = wid * SEGS + seg; cc < nc; cc += SNW * SEGS) {
        const long j = c0 + cc;
        const double d = own ? cb[cc * K + s.sl] : 0.0;
        const bool use_seed = mode == 2;
        const bool sp = use_seed && own && a.pY[j * K + s.sl] != 0;
        double y, r2;
        unsigned pm;
        long nch;
        int st;
        nnls_seg_solve<K, W>(s, d, a.col_n2[j], tl[cc], use_seed, sp, 3 * K, y, pm, nch, r2, st);
        if (own) {
          a.Yn[j * K + s.sl] = y;
          a.pY[j * K + s.sl] = ((pm >> s.sl) & 1u) ? 1 : 0;
          const double yo = Ys[j * K + s.sl];
          ydx = ydx + (y - yo) * (y - yo);
          yy = yy + yo * yo;
        }
        if (s.sl == 0) {
          a.stY[j] = (int8_t)st;
          yr2 = yr2 + r2;
          if (st != 0) yfail = 1.0;
        }
      }
    }
    {
      double v0 = warp_sum(ydx), v1 = warp_sum(yy), v2 = warp_sum(yr2), v3 = warp_max(yfail);
      if (lane == 0) {
        red[0 * SNW + wid] = v0;
        red[1 * SNW + wid] = v1;
        red[2 * SNW + wid] = v2;
        red[3 * SNW + wid] = v3;
      }
      __syncthreads();
      if (tid < 4) {
        double s = 0.0;
        for (int w = 0; w < SNW; ++w) s = (tid == 3) ? fmax(s, red[tid * SNW + w]) : s + red[tid * SNW + w];
        __stcg(PB + (long)tid * G + cta, s);
      }
    }
    S1STAMP(6);
    gsync();
    S1STAMP(7);
    // ---------------- sweep statistics, convergence, reload ----------------
    for (int e = wid; e < 7; e += SNW) {
      double v;
      if (e < 2)
        v = s1_cta_sum(PA, G, K * K + N + e);  // dX^2, X^2
      else if (e == 2)
        v = s1_cta_sum(PA, G, K * K + N + 2);  // X failure flags
      else
        v = s1_cta_sum(PB, G, e - 3);  // dY^2, Y^2, r2, Y failure
      if (lane == 0) scal[e] = v;
    }
    __syncthreads();
    S1STAMP(8);
    const double step = sqrt(scal[0] + scal[3]);
    const double nrmv = sqrt(scal[1] + scal[4]);
    const double obj = 0.5 * scal[5];
    failed = (scal[2] > 0.0 || scal[6] > 0.0) ? 1 : 0;
    if (cta == 0 && tid == 0) {
      double* rec = a.logv + (long)sweep * 4;
      rec[0] = obj;
      rec[1] = step;
      rec[2] = nrmv;
    }
    ++sweep;
    converged = (!a.fixed && step <= a.eps_stol * (1.0 + nrmv)) ? 1 : 0;
    // X <- Xn (own rows), Y <- Yn (all)
    for (long e = tid; e < (long)nr * K; e += ST) Xs[e] = Xn[e];
    for (long e = tid; e < N; e += ST) Ys[e] = __ldcg(a.Yn + e);
    __syncthreads();
    if (a.prof && blockIdx.x == 0 && threadIdx.x < 32 && sweep - 1 < 512)
      a.prof[(long)(sweep - 1) * 16 + 9] = clock64();
    if (failed || converged || sweep >= a.max_sweeps) break;
  }
  for (long e = tid; e < (long)nr * K; e += ST) a.X[r0 * K + e] = Xs[e];
  if (cta == 0) {
    for (long e = tid; e < N; e += ST) a.Yt[e] = Ys[e];
    if (tid == 0) {
      a.status[0] = sweep;
      a.status[1] = converged;
      a.status[2] = failed;
    }
  }
}

int s1_grid(long n) {
  static int sms = 0;  // one CTA per SM (cooperative launch)
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1)
      sms = 1;
  }
  long g = (n + 15) / 16;
  if (g > sms) g = sms;
  return g < 1 ? 1 : (int)g;
}

template <int K>
long s1_smem(long n, long m, int G, bool with_m) {
  const long nrm = (n + G - 1) / G, ncm = (m + G - 1) / G;
  const long CB = nrm > ncm ? (nrm > 16 ? nrm : 16) : (ncm > 16 ? ncm : 16);
  long d = m * K + 2 * nrm * K + CB * (K + 1);
  if (with_m) d += nrm * m;
  return d * (long)sizeof(double);
}

constexpr long S1_SMEM_CAP = 200 * 1024;

}  // namespace

#define NMFB_S1_K(k, MACRO)                                                                      \
  switch (k) {                                                                                   \
    MACRO(1, 4) MACRO(2, 4) MACRO(3, 4) MACRO(4, 4) MACRO(5, 8) MACRO(6, 8) MACRO(7, 8) MACRO(8, 8) \
    default: return NMFB_EUNSUPPORTED;                                                           \
  }

extern "C" int nmfb_stage1_persist_supported(long n, long m, long k, int m_is_f32) {
  if (k < 1 || k > 8 || n < 1 || m < 1 || m * k > 4096) return 0;
  const int G = s1_grid(n);
  if ((n + G - 1) / G > 1024) return 0;
  // fp32 M is only read from shared memory (no fp32 global path): it must fit
#define CASE(KK_, WW_) \
  case KK_: return s1_smem<KK_>(n, m, G, m_is_f32 != 0) <= S1_SMEM_CAP ? 1 : 0;
  NMFB_S1_K(k, CASE)
#undef CASE
}

extern "C" long nmfb_stage1_persist_work_len(long n, long m, long k) {
  const int G = s1_grid(n);
  return ((long)k * k + m * k + 3) * G + 4L * G;
}

extern "C" int nmfb_stage1_persist(const void* M, int m_is_f32, long n, long m, long k, double* X,
                                   double* Yt, double* Xn, double* Yn, uint8_t* pX, uint8_t* pY,
                                   const double* row_n2, const double* col_n2, int8_t* stX,
                                   int8_t* stY, double tol_fixed, int first_mode, int max_sweeps,
                                   int fixed, double eps_stol, double* logv, int* status,
                                   double* work, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!nmfb_stage1_persist_supported(n, m, k, m_is_f32)) return NMFB_EUNSUPPORTED;
  if (max_sweeps < 1) return NMFB_EINVAL;
  const int G = s1_grid(n);
  S1Args a;
  a.M = M;
  a.n = n;
  a.m = m;
  a.X = X;
  a.Yt = Yt;
  a.Xn = Xn;
  a.Yn = Yn;
  a.pX = pX;
  a.pY = pY;
  a.row_n2 = row_n2;
  a.col_n2 = col_n2;
  a.stX = stX;
  a.stY = stY;
  a.tol_fixed = tol_fixed;
  a.first_mode = first_mode;
  a.max_sweeps = max_sweeps;
  a.fixed = fixed;
  a.eps_stol = eps_stol;
  a.logv = logv;
  a.status = status;
  a.work = work;
  a.prof = g_s1_prof;
  void* args[] = {&a};
  cudaError_t err = cudaSuccess;
#define LAUNCH(KK_, WW_, T_)                                                                     \
  {                                                                                              \
    const bool wm = s1_smem<KK_>(n, m, G, true) <= S1_SMEM_CAP;                                  \
    if (!wm && m_is_f32) return NMFB_EUNSUPPORTED;                                               \
    a.m_in_smem = wm ? 1 : 0;                                                                    \
    const long bytes = s1_smem<KK_>(n, m, G, wm);                                                \
    nmfb_smem_attr(k_stage1_persist<KK_, WW_, T_>, (size_t)bytes);                              \
    ++g_nmfb_launches;                                                                           \
    err = cudaLaunchCooperativeKernel((const void*)k_stage1_persist<KK_, WW_, T_>, dim3(G),      \
                                      dim3(ST), args, (size_t)bytes, st);                        \
  }
#define CASE(KK_, WW_)          \
  case KK_:                     \
    if (m_is_f32)               \
      LAUNCH(KK_, WW_, float)   \
    else                        \
      LAUNCH(KK_, WW_, double)  \
    break;
  NMFB_S1_K(k, CASE)
#undef CASE
#undef LAUNCH
  if (err != cudaSuccess) return NMFB_ELAUNCH;
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// profiling hook: per-sweep clock64 stamps of CTA 0 into prof[sweep * 16 + i] (NULL: off)
extern "C" int nmfb_stage1_set_prof(long long* prof) {
  g_s1_prof = prof;
  return NMFB_OK;
}
