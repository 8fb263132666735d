// Stage-2 (interior point) production kernels, SPEC.md:244-374 / PAPER
// Algorithm 2 and Eqs. 3-13.  Layouts: X, R, graX (n,k); Yt = Y^T, S, graY
// (m,k) (y = vec(Y) is Yt row-major); M, F (n,m) row-major; L (n,k,k);
// the reduced system A (mk,mk) row-major, index (j,p) = j*k + p.
//
// Key B200-first restructuring of the Schur reduction (PAPER.md:526 prices
// it at O(n m^2 k^2) and the reference kernel loops exactly that way,
// _kernels_numba.py:83-106):  with A_i = R1_i^{-1},
//
//   S_GN block (j,l) = sum_i (y_j^T A_i y_l) x_i x_i^T
//                    = sum_{a,b} y_ja y_lb Z_ab,   Z_ab = sum_i A_i[a,b] x_i x_i^T
//
// so the n-contraction collapses to ONE small reduction Z (k^2 x k^2, O(n k^4))
// followed by an O(m^2 k^3) expansion that streams A to HBM once.  The same
// identity gives r_acc_j = H y_j with H = sum_i x_i (L_i^{-T} h_i)^T and the
// back-substitution q_i = L_i^{-1} (sum_j y_j dy_j^T) x_i.  The full-Hessian
// extra terms use W = F^T P (m x k^3 GEMM) and a residual-weighted SYRK.

#include "common.cuh"
#include "nmfb200.h"

namespace {
__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
}  // namespace


// Barrier value source for CUDA-graph capture (nmfb_set_mu_source): while set,
// the mu-dependent launches below bake this device pointer ([mu, wx mu, wy mu]) into
// their arguments instead of the scalar values, so one captured iteration replays
// for any mu (the host rewrites the three doubles before a replay).
static const double* g_mu_dev = nullptr;

namespace {


__device__ __forceinline__ int pk(int a, int b, int k) {
  // packed index of (a, b), a <= b, row-major upper triangle
  return a * k - a * (a - 1) / 2 + (b - a);
}

// ---------------------------------------------------------------------------
// F = X Y - M, graX = F Y^T, fsq = ||F||^2 (partials per CTA)
// ---------------------------------------------------------------------------
template <int K, int R, typename T>
__global__ void __launch_bounds__(256) k_residual_rows(const T* __restrict__ M, long n, long m,
                                                       const double* __restrict__ X,
                                                       const double* __restrict__ Yt,
                                                       double* __restrict__ F,
                                                       double* __restrict__ gX,
                                                       double* __restrict__ part) {
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  double fsq = 0.0;
  for (long r0 = warp * R; r0 < n; r0 += nwarps * R) {
    double x[R][K], g[R][K];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int p = 0; p < K; ++p) {
        x[r][p] = (r0 + r < n) ? X[(r0 + r) * K + p] : 0.0;
        g[r][p] = 0.0;
      }
    for (long j = lane; j < m; j += 32) {
      double y[K];
#pragma unroll
      for (int p = 0; p < K; ++p) y[p] = __ldg(Yt + j * K + p);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r0 + r < n) {
          double f = -(double)M[(r0 + r) * m + j];
#pragma unroll
          for (int p = 0; p < K; ++p) f = fma(x[r][p], y[p], f);
          F[(r0 + r) * m + j] = f;
          fsq = fma(f, f, fsq);
#pragma unroll
          for (int p = 0; p < K; ++p) g[r][p] = fma(f, y[p], g[r][p]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const double v = warp_sum(g[r][p]);
        if (lane == 0 && r0 + r < n) gX[(r0 + r) * K + p] = v;
      }
  }
  fsq = block_sum(fsq, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = fsq;
}

// ---------------------------------------------------------------------------
// per-row small linear algebra (thread per row i)
// ---------------------------------------------------------------------------
// Reciprocal pivots: rd[j] = 1 / L[j][j] from one rsqrt per column, so the column
// scalings and the triangular solves multiply instead of dividing (K(K+1)/2 + 2K
// IEEE division sequences per row taken off the dependency chains).
template <int K>
__device__ __forceinline__ bool chol_row(double (&L)[K][K], double (&rd)[K]) {
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double s = L[j][j];
#pragma unroll
    for (int p = 0; p < j; ++p) s -= L[j][p] * L[j][p];
    if (!(s > 0.0)) return false;
    const double di = rsqrt(s);
    L[j][j] = s * di;
    rd[j] = di;
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      double t = L[i][j];
#pragma unroll
      for (int p = 0; p < j; ++p) t -= L[i][p] * L[j][p];
      L[i][j] = t * di;
    }
  }
  return true;
}

template <int K>
__device__ __forceinline__ void recip_diag(const double (&L)[K][K], double (&rd)[K]) {
#pragma unroll
  for (int i = 0; i < K; ++i) rd[i] = 1.0 / L[i][i];
}

template <int K>
__device__ __forceinline__ void fwd_row(const double (&L)[K][K], const double (&rd)[K],
                                        const double* b, double* z) {
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double s = b[i];
#pragma unroll
    for (int p = 0; p < i; ++p) s -= L[i][p] * z[p];
    z[i] = s * rd[i];
  }
}

template <int K>
__device__ __forceinline__ void bwd_row(const double (&L)[K][K], const double (&rd)[K],
                                        const double* b, double* z) {
#pragma unroll
  for (int i = K - 1; i >= 0; --i) {
    double s = b[i];
#pragma unroll
    for (int p = i + 1; p < K; ++p) s -= L[p][i] * z[p];
    z[i] = s * rd[i];
  }
}

// R1_i = YY^T + rho I + diag(r_i / x_i) = L_i L_i^T; h_i = L_i^{-1}(mux/x_i - graX_i);
// g_i = L_i^{-T} h_i; Apk_i = packed R1_i^{-1}; XXpk_i = packed x_i x_i^T.
// Thread per row (arithmetic unchanged); the five per-row outputs (K^2 + 2K + K(K+1)
// doubles) leave through a per-warp shared-memory stage so every global store of the warp
// is contiguous (thread-per-row stores directly would touch 32 lines per instruction).
constexpr int R1_THREADS = 64;
template <int K>
struct R1W {  // stage row pitch: K^2 (L) and K(K+1) (Apk | XXpk) doubles, + 1 against conflicts
  static constexpr int v = K * (K + 1) + 1;
};

template <int K>
__device__ __forceinline__ void r1_flush(double* __restrict__ stage, int lane, long row0, long n,
                                         int width, double* __restrict__ out) {
  __syncwarp();
  const long nrow = min(32L, n - row0);
  double* dst = out + row0 * width;
  for (int e = lane; e < nrow * width; e += 32) {
    const int r = e / width, c = e - (e / width) * width;
    dst[e] = stage[r * (R1W<K>::v) + c];
  }
  __syncwarp();
}

template <int K>
__global__ void __launch_bounds__(R1_THREADS) k_r1_factor(const double* __restrict__ GY,
                                                          const double* __restrict__ X,
                                                          const double* __restrict__ R,
                                                          const double* __restrict__ gX,
                                                          double mux, double rho, long n,
                                                          double* __restrict__ Lout,
                                                          double* __restrict__ h,
                                                          double* __restrict__ g,
                                                          double* __restrict__ Apk,
                                                          double* __restrict__ XXpk,
                                                          int* __restrict__ bad,
                                                          const double* __restrict__ mu_dev) {
  if (mu_dev != nullptr) mux = mu_dev[1];  // graph replays: barrier value from device memory
  extern __shared__ double r1s[];          // [warps][32][K^2 + 1] output stage
  __shared__ double gy[K * K];
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) gy[e] = GY[e];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* stage = r1s + (size_t)wid * 32 * (R1W<K>::v);
  double* srow = stage + lane * (R1W<K>::v);
  const long row0 = (long)blockIdx.x * blockDim.x + 32 * wid;
  if (row0 >= n) return;  // warp-uniform
  const long i = row0 + lane;
  const bool live = i < n;
  const long ii = live ? i : row0;  // tail lanes recompute row0 (never stored)
  double x[K], L[K][K], b[K], hv[K], gv[K];
#pragma unroll
  for (int p = 0; p < K; ++p) x[p] = X[ii * K + p];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int c = 0; c < K; ++c) L[a][c] = (c <= a) ? gy[a * K + c] : 0.0;
#pragma unroll
  for (int p = 0; p < K; ++p) {
    const double ix = 1.0 / x[p];
    L[p][p] += rho + R[ii * K + p] * ix;
    b[p] = mux * ix - gX[ii * K + p];
  }
  double rd[K];
  const bool ok = chol_row<K>(L, rd);
  if (live && !ok) atomicMin(bad, (int)i);
  if (__all_sync(0xffffffffu, !ok)) return;
  fwd_row<K>(L, rd, b, hv);
  bwd_row<K>(L, rd, hv, gv);
  // L (full K x K, zero upper)
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int c = 0; c < K; ++c) srow[a * K + c] = (c <= a) ? L[a][c] : 0.0;
  r1_flush<K>(stage, lane, row0, n, K * K, Lout);
#pragma unroll
  for (int a = 0; a < K; ++a) srow[a] = hv[a], srow[K + a] = gv[a];
  __syncwarp();
  {  // h and g (two K-wide arrays)
    const long nrow = min(32L, n - row0);
    for (int e = lane; e < nrow * K; e += 32) {
      const int r = e / K, c = e - (e / K) * K;
      h[row0 * K + e] = stage[r * (R1W<K>::v) + c];
      g[row0 * K + e] = stage[r * (R1W<K>::v) + K + c];
    }
    __syncwarp();
  }
  // Linv = L^{-1} (lower), then R1^{-1} = Linv^T Linv
  double Li[K][K];
#pragma unroll
  for (int c = 0; c < K; ++c) {
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
  }
  constexpr int KKc = K * (K + 1) / 2;
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int c = a; c < K; ++c) {
      double s = 0.0;
#pragma unroll
      for (int p = 0; p < K; ++p)
        if (p >= c) s = fma(Li[p][a], Li[p][c], s);
      const int e = a * K - a * (a - 1) / 2 + (c - a);
      srow[e] = s;
      srow[KKc + e] = x[a] * x[c];
    }
  __syncwarp();
  {  // Apk and XXpk (two K(K+1)/2-wide arrays)
    const long nrow = min(32L, n - row0);
    for (int e = lane; e < nrow * KKc; e += 32) {
      const int r = e / KKc, c = e - (e / KKc) * KKc;
      Apk[row0 * KKc + e] = stage[r * (R1W<K>::v) + c];
      XXpk[row0 * KKc + e] = stage[r * (R1W<K>::v) + KKc + c];
    }
  }
}

// h = L^{-1} b1, g = L^{-T} h for a given right-hand side (predictor reuse)
template <int K>
__global__ void k_hg_rows(const double* __restrict__ Lin, const double* __restrict__ b1,
                          double b1_scale, long n, double* __restrict__ h,
                          double* __restrict__ g) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double L[K][K], b[K], hv[K], gv[K];
#pragma unroll
  for (int a = 0; a < K; ++a) {
    b[a] = b1_scale * b1[i * K + a];
#pragma unroll
    for (int c = 0; c < K; ++c) L[a][c] = Lin[(i * K + a) * K + c];
  }
  double rd[K];
  recip_diag<K>(L, rd);
  fwd_row<K>(L, rd, b, hv);
  bwd_row<K>(L, rd, hv, gv);
#pragma unroll
  for (int a = 0; a < K; ++a) {
    h[i * K + a] = hv[a];
    g[i * K + a] = gv[a];
  }
}

// ---------------------------------------------------------------------------
// generic split-K C = A^T B:  part[s][a][b] = sum_{i in stripe s} A[i,a] B[i,b]
// A (rows x ca), B (rows x cb) row-major fp64; 32x32 output tiles.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_atb_partial(const double* __restrict__ A, long rows,
                                                     long ca, const double* __restrict__ B,
                                                     long cb, long stripe,
                                                     double* __restrict__ part) {
  __shared__ double sa[32][33];
  __shared__ double sb[32][33];
  const int tid = threadIdx.x;
  const long a0 = (long)blockIdx.x * 32, b0 = (long)blockIdx.y * 32;
  const long s = blockIdx.z;
  const long i_beg = s * stripe, i_end = min(rows, i_beg + stripe);
  const int ta = tid >> 3, tb = (tid & 7) * 4;  // 32 rows of a x (8 x 4) cols of b
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (long ib = i_beg; ib < i_end; ib += 32) {
    const int nr = (int)min(32L, i_end - ib);
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += 256) {
      const int r = e >> 5, c = e & 31;
      sa[r][c] = (r < nr && a0 + c < ca) ? A[(ib + r) * ca + a0 + c] : 0.0;
      sb[r][c] = (r < nr && b0 + c < cb) ? B[(ib + r) * cb + b0 + c] : 0.0;
    }
    __syncthreads();
    for (int r = 0; r < nr; ++r) {
      const double av = sa[r][ta];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(av, sb[r][tb + q], acc[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const long a = a0 + ta, b = b0 + tb + q;
    if (a < ca && b < cb) part[(s * ca + a) * cb + b] = acc[q];
  }
}

// out[e] = sum_s part[s][e]: one warp per entry, lanes stride the partials, fixed butterfly
__global__ void __launch_bounds__(256) k_sum_parts_warp(const double* __restrict__ part,
                                                        int nparts, long len,
                                                        double* __restrict__ out) {
  const long e = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= len) return;
  double v = 0.0;
  for (int s = lane; s < nparts; s += 32) v += part[(long)s * len + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) out[e] = v;
}

__global__ void k_sum_parts(const double* __restrict__ part, int nparts, long len,
                            double* __restrict__ out) {
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= len) return;
  double v = 0.0;
  for (int s = 0; s < nparts; ++s) v += part[(long)s * len + e];
  out[e] = v;
}

// ---------------------------------------------------------------------------
// out (ca x cb) = A^T B for tall operands (rows >> ca, cb): split-K over row stripes on
// the FP64 tensor pipe (DMMA m8n8k4).  CTA = 64 x 64 output tile x one row stripe; the
// stripe's rows are staged 32 at a time in shared memory (row pitch 72 doubles: the
// fragment reads of 4 rows x 8 columns hit each bank pair at most twice = 2 wavefronts);
// warp w owns output rows 8w..8w+7 (8 n-tiles).  Partials per stripe, fixed-order sum.
// Replaces cuBLAS DGEMM for the rank-k^2 capacitance Grams Z = sum_i Rinv_i (x) x_i x_i^T,
// G = sum_j y_j y_j^T (x) D_j^{-1} and the full-Hessian W = F^T P.
// ---------------------------------------------------------------------------
constexpr int ATB_T = 64, ATB_R = 32, ATB_LD = 72;

constexpr int ATB_S = 3;  // cp.async ring stages of ATB_R rows (both operands)
constexpr size_t ATB_SMEM = (size_t)ATB_S * 2 * ATB_R * ATB_LD * sizeof(double);

// flat != 0 (one 64 x 64 tile covers both operands, 16-byte aligned bases): a chunk of 32 rows
// is ONE contiguous run of 32 ca (32 cb) doubles, copied with 16-byte cp.async into a dense
// [row][ca] layout -- 7 copies per thread and chunk instead of 32 element copies with their
// address arithmetic (the element path spent ~1 us of a 2 us chunk issuing them at ca = 55)
__global__ void __launch_bounds__(256) k_atb_mma(const double* __restrict__ A, long rows, long ca,
                                                 const double* __restrict__ B, long cb,
                                                 long stripe, double* __restrict__ part, int flat) {
  extern __shared__ __align__(16) double atb_sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const long a0 = (long)blockIdx.x * ATB_T, b0 = (long)blockIdx.y * ATB_T;
  const long s = blockIdx.z;
  const long i_beg = s * stripe, i_end = min(rows, i_beg + stripe);
  const int nchunk = (int)((i_end - i_beg + ATB_R - 1) / ATB_R);
  // chunk c of the stripe into ring stage c % ATB_S: every element its own 8-byte cp.async
  // (rows of ca / cb doubles are not 16-byte aligned in general), zeros outside the operands
  auto issue = [&](int c) {
    if (c < nchunk) {
      double* sa = atb_sm + (size_t)(c % ATB_S) * 2 * ATB_R * ATB_LD;
      double* sb = sa + ATB_R * ATB_LD;
      const long ib = i_beg + (long)c * ATB_R;
      const int nr = (int)min((long)ATB_R, i_end - ib);
      if (flat) {
        const int na = nr * (int)ca, nb = nr * (int)cb;
        const double* ga = A + ib * ca;
        const double* gb = B + ib * cb;
        for (int e = 2 * tid; e < ATB_R * (int)ca; e += 512) {
          if (e + 1 < na)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(sa + e)), "l"(ga + e) : "memory");
          else {
            sa[e] = e < na ? ga[e] : 0.0;
            sa[e + 1] = 0.0;
          }
        }
        for (int e = 2 * tid; e < ATB_R * (int)cb; e += 512) {
          if (e + 1 < nb)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(sb + e)), "l"(gb + e) : "memory");
          else {
            sb[e] = e < nb ? gb[e] : 0.0;
            sb[e + 1] = 0.0;
          }
        }
      } else
#pragma unroll
      for (int q = 0; q < ATB_R * ATB_T / 256; ++q) {
        const int e = tid + 256 * q;
        const int r = e >> 6, cc = e & 63;
        double* da = sa + r * ATB_LD + cc;
        double* db = sb + r * ATB_LD + cc;
        if (r < nr && a0 + cc < ca)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(da)),
                       "l"(A + (ib + r) * ca + a0 + cc)
                       : "memory");
        else
          *da = 0.0;
        if (r < nr && b0 + cc < cb)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(db)),
                       "l"(B + (ib + r) * cb + b0 + cc)
                       : "memory");
        else
          *db = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
  for (int c = 0; c < ATB_S - 1; ++c) issue(c);
  for (int c = 0; c < nchunk; ++c) {
    issue(c + ATB_S - 1);  // the stage it overwrites was read two iterations ago (barrier below)
    asm volatile("cp.async.wait_group %0;" ::"n"(ATB_S - 1) : "memory");
    __syncthreads();
    const double* sa = atb_sm + (size_t)(c % ATB_S) * 2 * ATB_R * ATB_LD;
    const double* sb = sa + ATB_R * ATB_LD;
    if (flat) {
      const int lda = (int)ca, ldb = (int)cb;
      const bool va = 8 * warp + g < lda;
#pragma unroll
      for (int kk = 0; kk < ATB_R / 4; ++kk) {
        const double af = va ? sa[(4 * kk + t) * lda + 8 * warp + g] : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double bf = (8 * j + g < ldb) ? sb[(4 * kk + t) * ldb + 8 * j + g] : 0.0;
          dmma_f64(acc[j][0], acc[j][1], af, bf);
        }
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < ATB_R / 4; ++kk) {
        const double af = sa[(4 * kk + t) * ATB_LD + 8 * warp + g];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double bf = sb[(4 * kk + t) * ATB_LD + 8 * j + g];
          dmma_f64(acc[j][0], acc[j][1], af, bf);
        }
      }
    }
    __syncthreads();
  }
  const long a = a0 + 8 * warp + g;
  if (a >= ca) return;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const long b = b0 + 8 * j + 2 * t + c;
      if (b < cb) part[(s * ca + a) * cb + b] = acc[j][c];
    }
}

// ---------------------------------------------------------------------------
// Schur assembly: A = blockdiag(X^T X + rho I + Diag(s_j / y_j)) - S
// (lower block triangle j >= l written; diagonal blocks written in full)
// S_GN(j,l)[p,q] = sum_a y_ja V_l[a][p][q],  V_l[a][p][q] = sum_b y_lb Z[a,b][p,q]
// full: + sum_a y_ja W[l][p][q][a] + sum_a y_la W[j][q][p][a]   (term4 separate)
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(256) k_schur_assemble(
    const double* __restrict__ Yt, const double* __restrict__ S, long m,
    const double* __restrict__ Zpk, const double* __restrict__ XtX, double rho,
    const double* __restrict__ W, int TL, long jchunk, double* __restrict__ A) {
  extern __shared__ double V[];  // [TL][K][K][K]
  constexpr int KK = K * (K + 1) / 2;
  const long N = m * K;
  const long l0 = (long)blockIdx.x * TL;
  const int ntl = (int)min((long)TL, m - l0);
  const int tid = threadIdx.x;
  // V for the tile's columns l
  for (int e = tid; e < ntl * K * K * K; e += blockDim.x) {
    const int tl = e / (K * K * K);
    const int rem = e % (K * K * K);
    const int a = rem / (K * K), p = (rem / K) % K, q = rem % K;
    const long l = l0 + tl;
    double v = 0.0;
#pragma unroll
    for (int b = 0; b < K; ++b) {
      const int ab = a <= b ? pk(a, b, K) : pk(b, a, K);
      const int pq = p <= q ? pk(p, q, K) : pk(q, p, K);
      v = fma(Yt[l * K + b], Zpk[ab * KK + pq], v);
    }
    V[e] = v;
  }
  __syncthreads();
  const long j_beg = max(l0, (long)blockIdx.y * jchunk);
  const long j_end = min(m, ((long)blockIdx.y + 1) * jchunk);
  // each j contributes K rows (p) x ntl*K columns (tl, q)
  const int per_j = K * ntl * K;
  for (long e = tid; e < (j_end > j_beg ? (j_end - j_beg) : 0) * per_j; e += blockDim.x) {
    const long j = j_beg + e / per_j;
    const int rem = (int)(e % per_j);
    const int p = rem / (ntl * K);
    const int tl = (rem / K) % ntl;
    const int q = rem % K;
    const long l = l0 + tl;
    if (j < l) continue;
    double sv = 0.0;
    const double* Vl = V + (long)tl * K * K * K;
#pragma unroll
    for (int a = 0; a < K; ++a) sv = fma(Yt[j * K + a], Vl[(a * K + p) * K + q], sv);
    if (W) {
      const double* Wl = W + l * K * K * K;
      const double* Wj = W + j * K * K * K;
#pragma unroll
      for (int a = 0; a < K; ++a) {
        sv = fma(Yt[j * K + a], Wl[(p * K + q) * K + a], sv);
        sv = fma(Yt[l * K + a], Wj[(q * K + p) * K + a], sv);
      }
    }
    double v = -sv;
    if (j == l) {
      v += XtX[p * K + q];
      if (p == q) v += rho + S[j * K + p] / Yt[j * K + p];
    }
    A[(j * K + p) * N + l * K + q] = v;
  }
}

// full Hessian term 4: A[(j,p),(l,q)] -= sum_i f_ij f_il Ainv_i[p,q], j >= l.
// grid (tile j, tile l, pq chunk x row split).  nsplit == 1: subtract in place;
// else write part[split][j][l][pq] and k_term4_finish sums the splits in order.
template <int K, int PQC>
__global__ void __launch_bounds__(256) k_schur_term4(const double* __restrict__ F, long n, long m,
                                                     const double* __restrict__ Apk,
                                                     double* __restrict__ A, int nsplit,
                                                     double* __restrict__ part) {
  constexpr int KK = K * (K + 1) / 2;
  __shared__ double fj[32][16], fl[32][16], ap[32][PQC];
  const long tj = blockIdx.x, tl = blockIdx.y;
  if (tj < tl) return;
  const int zc = blockIdx.z / nsplit, zs = blockIdx.z % nsplit;
  const int pq0 = zc * PQC;
  const int npq = min(PQC, KK - pq0);
  const long rps = (n + nsplit - 1) / nsplit;
  const long i_beg = zs * rps, i_end = min(n, i_beg + rps);
  const int tid = threadIdx.x, jj = tid >> 4, ll = tid & 15;
  const long j = tj * 16 + jj, l = tl * 16 + ll;
  double acc[PQC];
#pragma unroll
  for (int c = 0; c < PQC; ++c) acc[c] = 0.0;
  for (long ib = i_beg; ib < i_end; ib += 32) {
    const int nr = (int)min(32L, i_end - ib);
    __syncthreads();
    for (int e = tid; e < 32 * 16; e += 256) {
      const int r = e >> 4, c = e & 15;
      const long jc = tj * 16 + c, lc = tl * 16 + c;
      fj[r][c] = (r < nr && jc < m) ? F[(ib + r) * m + jc] : 0.0;
      fl[r][c] = (r < nr && lc < m) ? F[(ib + r) * m + lc] : 0.0;
    }
    for (int e = tid; e < 32 * PQC; e += 256) {
      const int r = e / PQC, c = e % PQC;
      ap[r][c] = (r < nr && c < npq) ? Apk[(ib + r) * KK + pq0 + c] : 0.0;
    }
    __syncthreads();
    for (int r = 0; r < nr; ++r) {
      const double w = fj[r][jj] * fl[r][ll];
#pragma unroll
      for (int c = 0; c < PQC; ++c) acc[c] = fma(w, ap[r][c], acc[c]);
    }
  }
  if (j >= m || l >= m || j < l) return;
  if (nsplit > 1) {
    for (int c = 0; c < npq; ++c) part[((long)zs * m * m + j * m + l) * KK + pq0 + c] = acc[c];
    return;
  }
  const long N = m * K;
  for (int c = 0; c < npq; ++c) {
    // unpack pq0 + c -> (p, q), p <= q
    int e = pq0 + c, p = 0;
    while (e >= K - p) {
      e -= K - p;
      ++p;
    }
    const int q = p + e;
    A[(j * K + p) * N + l * K + q] -= acc[c];
    if (p != q) A[(j * K + q) * N + l * K + p] -= acc[c];
  }
}

// The same contraction on the FP64 tensor cores for K <= 4 (c1-c3, KK = K(K+1)/2 <= 10):
// per pq the tile is F_j^T diag(a_i[pq]) F_l, i.e. KK weighted SYRK/GEMMs that share both
// operand fragments.  CTA = 32 x 32 tile of (j, l) (lower tiles only) x a row split; warp =
// two 8 x 8 blocks x KK accumulator pairs; per contraction step of 4 rows: one fragment of
// F_j, two of F_l, KK weights, KK multiplies and 2 KK DMMA m8n8k4.  Rows staged in 32-row
// chunks by cp.async (double-buffered, leading dimension 36 = conflict-free fragments).
constexpr int T4M_LD = 36;
template <int K>
__global__ void __launch_bounds__(256) k_schur_term4_mma(const double* __restrict__ F, long n, long m,
                                                         const double* __restrict__ Apk,
                                                         double* __restrict__ A, int nsplit,
                                                         double* __restrict__ part) {
  constexpr int KK = K * (K + 1) / 2;
  constexpr int KP = (KK + 1) & ~1;  // padded weight row
  __shared__ __align__(16) double fj[2][32 * T4M_LD], fl[2][32 * T4M_LD], ap[2][32 * KP];
  const long tj = blockIdx.x, tl = blockIdx.y;
  if (tj < tl) return;
  const int zs = blockIdx.z;
  const long rps = (((n + nsplit - 1) / nsplit) + 31) / 32 * 32;
  const long i_beg = zs * rps, i_end = min(n, i_beg + rps);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int bj = wid >> 1, bl0 = 2 * (wid & 1);
  const long j0 = tj * 32, l0 = tl * 32;
  const int nchunk = i_end > i_beg ? (int)((i_end - i_beg + 31) / 32) : 0;
  auto issue = [&](int c) {
    if (c < nchunk) {
      const int st = c & 1;
      const long ib = i_beg + 32L * c;
      const int nr = (int)min(32L, i_end - ib);
      for (int e = tid; e < 32 * 32; e += 256) {
        const int r = e >> 5, cc = e & 31;
        double* dj = &fj[st][r * T4M_LD + cc];
        double* dl = &fl[st][r * T4M_LD + cc];
        if (r < nr && j0 + cc < m)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(dj)),
                       "l"(F + (ib + r) * m + j0 + cc)
                       : "memory");
        else
          *dj = 0.0;
        if (r < nr && l0 + cc < m)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(dl)),
                       "l"(F + (ib + r) * m + l0 + cc)
                       : "memory");
        else
          *dl = 0.0;
      }
      for (int e = tid; e < 32 * KK; e += 256) {
        const int r = e / KK, cc = e - r * KK;
        double* da = &ap[st][r * KP + cc];
        if (r < nr)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(da)),
                       "l"(Apk + (ib + r) * KK + cc)
                       : "memory");
        else
          *da = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[2][KK][2];
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int c = 0; c < KK; ++c) acc[b][c][0] = acc[b][c][1] = 0.0;
  issue(0);
  for (int c = 0; c < nchunk; ++c) {
    issue(c + 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const int st = c & 1;
    const double* pj = &fj[st][t4 * T4M_LD + 8 * bj + g8];
    const double* pl = &fl[st][t4 * T4M_LD + 8 * bl0 + g8];
    const double* pa = &ap[st][t4 * KP];
#pragma unroll 2
    for (int ks = 0; ks < 8; ++ks) {
      const double a = pj[4 * ks * T4M_LD];
      const double b0 = pl[4 * ks * T4M_LD], b1 = pl[4 * ks * T4M_LD + 8];
#pragma unroll
      for (int q = 0; q < KK; ++q) {
        const double aw = a * pa[4 * ks * KP + q];
        dmma_f64(acc[0][q][0], acc[0][q][1], aw, b0);
        dmma_f64(acc[1][q][0], acc[1][q][1], aw, b1);
      }
    }
    __syncthreads();
  }
  const long N = m * K;
  const long j = j0 + 8 * bj + g8;
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const long l = l0 + 8 * (bl0 + b) + 2 * t4 + v;
      if (j >= m || l >= m || j < l) continue;
      if (nsplit > 1) {
#pragma unroll
        for (int q = 0; q < KK; ++q) part[((long)zs * m * m + j * m + l) * KK + q] = acc[b][q][v];
      } else {
        int p = 0, e = 0;
#pragma unroll
        for (int q = 0; q < KK; ++q) {  // pq -> (p, qq), p <= qq, in packed order
          const int qq = p + e;
          A[(j * K + p) * N + l * K + qq] -= acc[b][q][v];
          if (p != qq) A[(j * K + qq) * N + l * K + p] -= acc[b][q][v];
          if (++e >= K - p) e = 0, ++p;
        }
      }
    }
}

template <int K>
__global__ void k_term4_finish(const double* __restrict__ part, long m, int nsplit,
                               double* __restrict__ A) {
  constexpr int KK = K * (K + 1) / 2;
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;  // (j, l, pq), j >= l
  if (e >= m * m * KK) return;
  const long jl = e / KK;
  const int pqi = (int)(e % KK);
  const long j = jl / m, l = jl % m;
  if (j < l) return;
  double s = 0.0;
  for (int z = 0; z < nsplit; ++z) s += part[(long)z * m * m * KK + e];
  int ee = pqi, p = 0;
  while (ee >= K - p) {
    ee -= K - p;
    ++p;
  }
  const int q = p + ee;
  const long N = m * K;
  A[(j * K + p) * N + l * K + q] -= s;
  if (p != q) A[(j * K + q) * N + l * K + p] -= s;
}

// P[i][(p,q,a)] = x_ip * Ainv_i[q,a]   (n x K^3, for W = F^T P)
template <int K>
__global__ void k_make_p(const double* __restrict__ X, const double* __restrict__ Apk, long n,
                         double* __restrict__ P) {
  constexpr int KK = K * (K + 1) / 2;
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * K * K * K) return;
  const long i = e / (K * K * K);
  const int rem = (int)(e % (K * K * K));
  const int p = rem / (K * K), q = (rem / K) % K, a = rem % K;
  const int qa = q <= a ? pk(q, a, K) : pk(a, q, K);
  P[e] = X[i * K + p] * Apk[i * KK + qa];
}

// rhs of the reduced system: muy/y - graY - H y_j - [full] (F^T g)_j
template <int K>
__global__ void k_schur_rhs(const double* __restrict__ Yt, const double* __restrict__ gY,
                            const double* __restrict__ H, const double* __restrict__ FtG,
                            double muy, long m, double* __restrict__ rhs,
    const double* __restrict__ mu_dev) {
  if (mu_dev != nullptr) muy = mu_dev[2];
  const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
#pragma unroll
  for (int p = 0; p < K; ++p) {
    double v = muy / Yt[j * K + p] - gY[j * K + p];
    double ra = 0.0;
#pragma unroll
    for (int a = 0; a < K; ++a) ra = fma(H[p * K + a], Yt[j * K + a], ra);
    if (FtG) ra += FtG[j * K + p];
    rhs[j * K + p] = v - ra;
  }
}

// ---------------------------------------------------------------------------
// back-substitution + dual directions + partial reductions (thread per row)
//   q_i = L_i^{-1}(Gdy x_i + [full] (F dY)_i), dx_i = L_i^{-T}(h_i - q_i)
//   dr = mux/x - r - (r/x) dx
// partials per CTA: [gtp, a1min, a2min]
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(128) k_dir_rows(const double* __restrict__ Lin,
                                                  const double* __restrict__ Xf,
                                                  const double* __restrict__ h,
                                                  const double* __restrict__ Gdy,
                                                  const double* __restrict__ FdY,
                                                  const double* __restrict__ X,
                                                  const double* __restrict__ R,
                                                  const double* __restrict__ gX, double mux,
                                                  double tau, long n, double* __restrict__ dX,
                                                  double* __restrict__ dR,
                                                  double* __restrict__ part,
    const double* __restrict__ mu_dev) {
  if (mu_dev != nullptr) mux = mu_dev[1];
  __shared__ double gd[K * K];
  __shared__ double sh[32];
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) gd[e] = Gdy[e];
  __syncthreads();
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  double gtp = 0.0, a1 = 1.0 / 0.0, a2 = 1.0 / 0.0;
  if (i < n) {
    double L[K][K], v[K], q[K], t[K], dx[K];
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int c = 0; c < K; ++c) L[a][c] = Lin[(i * K + a) * K + c];
#pragma unroll
    for (int a = 0; a < K; ++a) {
      double s = FdY ? FdY[i * K + a] : 0.0;
#pragma unroll
      for (int b = 0; b < K; ++b) s = fma(gd[a * K + b], Xf[i * K + b], s);
      v[a] = s;
    }
    double rd[K];
    recip_diag<K>(L, rd);
    fwd_row<K>(L, rd, v, q);
#pragma unroll
    for (int a = 0; a < K; ++a) t[a] = h[i * K + a] - q[a];
    bwd_row<K>(L, rd, t, dx);
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const double x = X[i * K + a], r = R[i * K + a];
      const double d = dx[a];
      const double dr = mux / x - r - (r / x) * d;
      dX[i * K + a] = d;
      dR[i * K + a] = dr;
      gtp = fma(d, gX[i * K + a] - mux / x, gtp);
      if (d < 0.0) a1 = fmin(a1, -tau * x / d);
      if (dr < 0.0) a2 = fmin(a2, -tau * r / dr);
    }
  }
  gtp = block_sum(gtp, sh);
  if (threadIdx.x == 0) part[blockIdx.x * 3 + 0] = gtp;
  __syncthreads();
  a1 = -block_max(-a1, sh);
  if (threadIdx.x == 0) part[blockIdx.x * 3 + 1] = a1;
  __syncthreads();
  a2 = -block_max(-a2, sh);
  if (threadIdx.x == 0) part[blockIdx.x * 3 + 2] = a2;
}

// Y side: ds = muy/y - s - (s/y) dy (dy already solved); partials [gtp, a1min, a2min]
__global__ void __launch_bounds__(256) k_dir_cols(const double* __restrict__ Yt,
                                                  const double* __restrict__ S,
                                                  const double* __restrict__ gY,
                                                  const double* __restrict__ dY, double muy,
                                                  double tau, long len,
                                                  double* __restrict__ dS,
                                                  double* __restrict__ part,
    const double* __restrict__ mu_dev) {
  if (mu_dev != nullptr) muy = mu_dev[2];
  __shared__ double sh[32];
  double gtp = 0.0, a1 = 1.0 / 0.0, a2 = 1.0 / 0.0;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (long)gridDim.x * blockDim.x) {
    const double y = Yt[e], s = S[e], d = dY[e];
    const double ds = muy / y - s - (s / y) * d;
    dS[e] = ds;
    gtp = fma(d, gY[e] - muy / y, gtp);
    if (d < 0.0) a1 = fmin(a1, -tau * y / d);
    if (ds < 0.0) a2 = fmin(a2, -tau * s / ds);
  }
  gtp = block_sum(gtp, sh);
  if (threadIdx.x == 0) part[blockIdx.x * 3 + 0] = gtp;
  __syncthreads();
  a1 = -block_max(-a1, sh);
  if (threadIdx.x == 0) part[blockIdx.x * 3 + 1] = a1;
  __syncthreads();
  a2 = -block_max(-a2, sh);
  if (threadIdx.x == 0) part[blockIdx.x * 3 + 2] = a2;
}

// out = [gtp, a1max, a2max] from row and column partials (fixed order)
__global__ void k_finish_dir(const double* __restrict__ prow, int nrow,
                             const double* __restrict__ pcol, int ncol,
                             double* __restrict__ out) {
  __shared__ double sh[32];
  double g = 0.0, a1 = 1.0, a2 = 1.0;
  for (int b = threadIdx.x; b < nrow; b += blockDim.x) {
    g += prow[b * 3];
    a1 = fmin(a1, prow[b * 3 + 1]);
    a2 = fmin(a2, prow[b * 3 + 2]);
  }
  double g2 = 0.0;
  for (int b = threadIdx.x; b < ncol; b += blockDim.x) {
    g2 += pcol[b * 3];
    a1 = fmin(a1, pcol[b * 3 + 1]);
    a2 = fmin(a2, pcol[b * 3 + 2]);
  }
  g = block_sum(g, sh);
  __syncthreads();
  g2 = block_sum(g2, sh);
  __syncthreads();
  a1 = -block_max(-a1, sh);
  __syncthreads();
  a2 = -block_max(-a2, sh);
  if (threadIdx.x == 0) {
    out[0] = g + g2;
    out[1] = a1;
    out[2] = a2;
    out[3] = g;   // row-block part (summed across ranks when M is row-sharded)
    out[4] = g2;  // column part (replicated)
  }
}

// ---------------------------------------------------------------------------
// Armijo: one pass over (i, j) for the six inner products of
//   A = F, B = dX Y + X dY, C = dX dY:  [AA, AB, BB, AC, BC, CC]
// ---------------------------------------------------------------------------
template <int K, int R>
__global__ void __launch_bounds__(256) k_quartic_rows(const double* __restrict__ F, long n,
                                                      long m, const double* __restrict__ X,
                                                      const double* __restrict__ dX,
                                                      const double* __restrict__ Yt,
                                                      const double* __restrict__ dYt,
                                                      double* __restrict__ part) {
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  double s[6] = {0, 0, 0, 0, 0, 0};
  for (long r0 = warp * R; r0 < n; r0 += nwarps * R) {
    double x[R][K], dx[R][K];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int p = 0; p < K; ++p) {
        x[r][p] = (r0 + r < n) ? X[(r0 + r) * K + p] : 0.0;
        dx[r][p] = (r0 + r < n) ? dX[(r0 + r) * K + p] : 0.0;
      }
    for (long j = lane; j < m; j += 32) {
      double y[K], dy[K];
#pragma unroll
      for (int p = 0; p < K; ++p) {
        y[p] = __ldg(Yt + j * K + p);
        dy[p] = __ldg(dYt + j * K + p);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r0 + r < n) {
          const double a = F[(r0 + r) * m + j];
          double b = 0.0, c = 0.0;
#pragma unroll
          for (int p = 0; p < K; ++p) {
            b = fma(dx[r][p], y[p], fma(x[r][p], dy[p], b));
            c = fma(dx[r][p], dy[p], c);
          }
          s[0] = fma(a, a, s[0]);
          s[1] = fma(a, b, s[1]);
          s[2] = fma(b, b, s[2]);
          s[3] = fma(a, c, s[3]);
          s[4] = fma(b, c, s[4]);
          s[5] = fma(c, c, s[5]);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const double v = block_sum(s[q], sh);
    if (threadIdx.x == 0) part[blockIdx.x * 6 + q] = v;
    __syncthreads();
  }
}

// barrier increments for every backtracking trial t (blockIdx.y):
//   part[t][b][0] = sum log1p(alpha_t dx/x), part[t][b][1] = same over y
// one CTA column per trial (blockIdx.y = t): the log1p are FP64-issue bound and one
// trial per CTA gives the most parallelism (batching trials per CTA with a shared
// division measured slower on B200); terms are the oracle's log1p((alpha dv) / v)
__global__ void __launch_bounds__(256) k_barrier_trials(const double* __restrict__ X,
                                                        const double* __restrict__ dX, long nx,
                                                        const double* __restrict__ Yt,
                                                        const double* __restrict__ dYt, long ny,
                                                        const double* __restrict__ alpha_max,
                                                        int ntrials, double* __restrict__ part,
                                                        int t0 = 0,
                                                        const double* __restrict__ skip = nullptr) {
  __shared__ double sh[32];
  if (skip != nullptr && *skip != 0.0) return;  // Armijo already decided (lazy batches)
  const int t = t0 + blockIdx.y;
  if (t >= ntrials) return;
  const double alpha = ldexp(*alpha_max, -t);
  double sx = 0.0, sy = 0.0;
  const long tid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long nt = (long)gridDim.x * blockDim.x;
  for (long e = tid; e < nx; e += nt) sx += log1p(alpha * dX[e] / X[e]);
  for (long e = tid; e < ny; e += nt) sy += log1p(alpha * dYt[e] / Yt[e]);
  sx = block_sum(sx, sh);
  __syncthreads();
  sy = block_sum(sy, sh);
  if (threadIdx.x == 0) {
    part[((long)t * gridDim.x + blockIdx.x) * 2 + 0] = sx;
    part[((long)t * gridDim.x + blockIdx.x) * 2 + 1] = sy;
  }
}

// out[t*2 + c] = sum_b part[t][b][c]  (one warp per (t, c), fixed order)
__global__ void k_finish_trials(const double* __restrict__ part, int nb, int nt,
                                double* __restrict__ out, int t0 = 0,
                                const double* __restrict__ skip = nullptr) {
  if (skip != nullptr && *skip != 0.0) return;
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int t = t0 + (w >> 1), c = w & 1;
  if (t >= nt) return;
  double v = 0.0;
  for (int b = lane; b < nb; b += 32) v += part[((long)t * nb + b) * 2 + c];
  v = warp_sum(v);
  if (lane == 0) out[t * 2 + c] = v;
}

// v <- v + alpha dv, entries that are not strictly positive become (1-tau) v
__global__ void k_step_nudge(double* __restrict__ v, const double* __restrict__ dv, long len,
                             double alpha, double tau) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (long)gridDim.x * blockDim.x) {
    const double old = v[e];
    const double nv = old + alpha * dv[e];
    v[e] = (nv > 0.0) ? nv : (1.0 - tau) * old;
  }
}

// KKT sums (PAPER Eq. 9) in one pass; partial layout per CTA (12 values):
//  sums: 0 ||gX-R||^2  1 ||x.r - mux||^2  2 ||x.r||^2  3 x^T r
//        4 ||gY-S||^2  5 ||y.s - muy||^2  6 ||y.s||^2  7 y^T s
//  maxes: 8 max|gX|  9 max|gY|  10 max x  11 max y
__global__ void __launch_bounds__(256) k_kkt_partial(const double* __restrict__ X,
                                                     const double* __restrict__ R,
                                                     const double* __restrict__ gX, long nx,
                                                     const double* __restrict__ Yt,
                                                     const double* __restrict__ S,
                                                     const double* __restrict__ gY, long ny,
                                                     double mux, double muy,
                                                     double* __restrict__ part,
    const double* __restrict__ mu_dev) {
  if (mu_dev != nullptr) {
    mux = mu_dev[1];
    muy = mu_dev[2];
  }
  __shared__ double sh[32];
  double v[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) v[q] = (q < 8) ? 0.0 : -1.0 / 0.0;
  const long tid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long nt = (long)gridDim.x * blockDim.x;
  if (R) {
    for (long e = tid; e < nx; e += nt) {
      const double x = X[e], r = R[e], g = gX[e];
      const double xr = x * r;
      v[0] = fma(g - r, g - r, v[0]);
      v[1] = fma(xr - mux, xr - mux, v[1]);
      v[2] = fma(xr, xr, v[2]);
      v[3] += xr;
      v[8] = fmax(v[8], fabs(g));
      v[10] = fmax(v[10], x);
    }
    for (long e = tid; e < ny; e += nt) {
      const double y = Yt[e], s = S[e], g = gY[e];
      const double ys = y * s;
      v[4] = fma(g - s, g - s, v[4]);
      v[5] = fma(ys - muy, ys - muy, v[5]);
      v[6] = fma(ys, ys, v[6]);
      v[7] += ys;
      v[9] = fmax(v[9], fabs(g));
      v[11] = fmax(v[11], y);
    }
  } else {  // primal-only scoring: r = max(gX,0), s = max(gY,0)
    for (long e = tid; e < nx; e += nt) {
      const double x = X[e], g = gX[e], r = fmax(g, 0.0);
      const double xr = x * r;
      v[0] = fma(g - r, g - r, v[0]);
      v[1] = fma(xr - mux, xr - mux, v[1]);
      v[2] = fma(xr, xr, v[2]);
      v[3] += xr;
      v[8] = fmax(v[8], fabs(g));
      v[10] = fmax(v[10], x);
    }
    for (long e = tid; e < ny; e += nt) {
      const double y = Yt[e], g = gY[e], s = fmax(g, 0.0);
      const double ys = y * s;
      v[4] = fma(g - s, g - s, v[4]);
      v[5] = fma(ys - muy, ys - muy, v[5]);
      v[6] = fma(ys, ys, v[6]);
      v[7] += ys;
      v[9] = fmax(v[9], fabs(g));
      v[11] = fmax(v[11], y);
    }
  }
#pragma unroll
  for (int q = 0; q < 12; ++q) {
    const double r = q < 8 ? block_sum(v[q], sh) : block_max(v[q], sh);
    if (threadIdx.x == 0) part[blockIdx.x * 12 + q] = r;
    __syncthreads();
  }
}

__global__ void k_finish_kkt(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double sh[32];
  for (int q = 0; q < 12; ++q) {
    double v = q < 8 ? 0.0 : -1.0 / 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
      v = q < 8 ? v + part[b * 12 + q] : fmax(v, part[b * 12 + q]);
    v = q < 8 ? block_sum(v, sh) : block_max(v, sh);
    if (threadIdx.x == 0) out[q] = v;
    __syncthreads();
  }
}

// mu_aff numerator: sum (x + a1 dx)(r + a2 dr) + sum (y + a1 dy)(s + a2 ds)
__global__ void __launch_bounds__(256) k_affine_partial(const double* __restrict__ X,
                                                        const double* __restrict__ dX,
                                                        const double* __restrict__ R,
                                                        const double* __restrict__ dR, long nx,
                                                        const double* __restrict__ Yt,
                                                        const double* __restrict__ dY,
                                                        const double* __restrict__ S,
                                                        const double* __restrict__ dS, long ny,
                                                        double a1, double a2,
                                                        double* __restrict__ part) {
  __shared__ double sh[32];
  double v = 0.0;
  const long tid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long nt = (long)gridDim.x * blockDim.x;
  for (long e = tid; e < nx; e += nt) v = fma(X[e] + a1 * dX[e], R[e] + a2 * dR[e], v);
  for (long e = tid; e < ny; e += nt) v = fma(Yt[e] + a1 * dY[e], S[e] + a2 * dS[e], v);
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// out[q] = sum_b part[b * nq + q]  (fixed order)
__global__ void k_finish_cols(const double* __restrict__ part, int nb, int nq,
                              double* __restrict__ out) {
  __shared__ double sh[32];
  for (int q = 0; q < nq; ++q) {
    double v = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) v += part[(long)b * nq + q];
    v = block_sum(v, sh);
    if (threadIdx.x == 0) out[q] = v;
    __syncthreads();
  }
}

__global__ void k_finish_sum1(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) v += part[b];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) *out = v;
}

__global__ void k_clamp_fill(double* __restrict__ v, long len, double lo) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (long)gridDim.x * blockDim.x)
    v[e] = fmax(v[e], lo);
}

__global__ void k_fill(double* __restrict__ v, long len, double c) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (long)gridDim.x * blockDim.x)
    v[e] = c;
}

// Armijo acceptance on the device (same arithmetic as the host loop in
// solver.run_ipm): first t with dphi(a1max 2^-t) <= eta a 2^-t gtp.
// sc layout: [4] gtp, [5] a1max, [6] a2max, [10..15] quartic, [32 + 2t (+1)] barrier sums.
// Writes sc[1] = alpha1 (0 when stalled), sc[2] = t (max_bt + 1 when stalled), sc[3] = alpha2.
// t_lim < 0: full search (t = 0 .. max_bt).  t_lim >= 0 (lazy pre-check): search
// t < t_lim only and record in sc[31] whether that decided (1) or the remaining
// trials are needed (0).  With sc[31] == 1 on entry to a full search, nothing to do.
__global__ void k_armijo_select(double* __restrict__ sc, double mu, double wx, double wy,
                                double eta, int max_bt, const int* __restrict__ fcodes,
                                int t_lim = -1, int honor_decided = 0,
                                const double* __restrict__ mu_dev = nullptr) {
  if (mu_dev != nullptr) mu = mu_dev[0];
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (honor_decided && sc[31] != 0.0) return;
  // fcodes = [R1 failing row, reduced-system info, D failing column]: on any
  // factorization failure take no step (t = -2) so the host can redo the
  // direction with the dense Schur solve
  if (fcodes && (fcodes[0] != 0x7F7F7F7F || fcodes[1] >= 0 || fcodes[2] != 0x7F7F7F7F)) {
    sc[1] = 0.0;
    sc[2] = -2.0;
    sc[3] = 0.0;
    if (t_lim >= 0) sc[31] = 1.0;
    return;
  }
  const double gtp = sc[4], a1max = sc[5];
  const double ab = sc[11], bb = sc[12], ac = sc[13], bc = sc[14], cc = sc[15];
  int t = 0;
  double a1 = a1max;
  // explicit _rn operations: no FMA contraction, same evaluation order as the host
  // expression a*ab + a*a*(0.5*bb + ac) + a*a*a*bc + 0.5*(a*a*a*a)*cc
  const double c2 = __dadd_rn(__dmul_rn(0.5, bb), ac);
  for (;;) {
    a1 = a1max / ldexp(1.0, t);
    const double a2 = __dmul_rn(a1, a1), a3 = __dmul_rn(a2, a1), a4 = __dmul_rn(a3, a1);
    double quad = __dadd_rn(__dmul_rn(a1, ab), __dmul_rn(a2, c2));
    quad = __dadd_rn(quad, __dmul_rn(a3, bc));
    quad = __dadd_rn(quad, __dmul_rn(__dmul_rn(0.5, a4), cc));
    const double bar = __dadd_rn(__dmul_rn(wx, sc[32 + 2 * t]), __dmul_rn(wy, sc[33 + 2 * t]));
    const double dphi = __dsub_rn(quad, __dmul_rn(mu, bar));
    if (dphi <= __dmul_rn(__dmul_rn(eta, a1), gtp)) break;
    ++t;
    if (t_lim >= 0 && t >= t_lim && t <= max_bt) {  // undecided within the first batch
      sc[31] = 0.0;
      return;
    }
    if (t > max_bt) {
      a1 = 0.0;
      break;
    }
  }
  if (t_lim >= 0) sc[31] = 1.0;
  sc[1] = a1;
  sc[2] = (double)t;
  sc[3] = (t > max_bt) ? 0.0 : sc[6];
}

// v += (*alpha) dv with the (1 - tau) nudge, alpha read from device memory
__global__ void k_step_nudge_dev(double* __restrict__ v, const double* __restrict__ dv, long len,
                                 const double* __restrict__ alpha, double tau) {
  const double a = *alpha;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (long)gridDim.x * blockDim.x) {
    const double old = v[e];
    const double nv = old + a * dv[e];
    v[e] = (nv > 0.0) ? nv : (1.0 - tau) * old;
  }
}

// step with the nudge rule that also reports whether any entry was nudged
// (flag: the residual-free refresh may then not advance M Y^T / M^T X incrementally)
__global__ void k_step_nudge_flag(double* __restrict__ v, const double* __restrict__ dv, long len,
                                  const double* __restrict__ alpha_dev, double alpha, double tau,
                                  int* __restrict__ flag) {
  const double a = alpha_dev ? *alpha_dev : alpha;
  int nudged = 0;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (long)gridDim.x * blockDim.x) {
    const double old = v[e];
    const double nv = old + a * dv[e];
    const bool ok = nv > 0.0;
    v[e] = ok ? nv : (1.0 - tau) * old;
    nudged |= !ok;
  }
  if (__syncthreads_or(nudged) && threadIdx.x == 0) atomicOr(flag, 1);
}

// residual-free refresh after a clean step: M Y'^T = M Y^T + a M dY^T and
// M^T X' = M^T X + a M^T dX (both products came from the Armijo pass at the
// previous point); a nudged step (flag != 0) leaves them for a full recompute
__global__ void k_ffree_advance(double* __restrict__ MY, const double* __restrict__ MdY, long nlen,
                                double* __restrict__ MX, const double* __restrict__ MtdX, long mlen,
                                const double* __restrict__ alpha_dev, double alpha,
                                const int* __restrict__ flag) {
  if (*flag) return;
  const double a = alpha_dev ? *alpha_dev : alpha;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < nlen + mlen;
       e += (long)gridDim.x * blockDim.x) {
    if (e < nlen)
      MY[e] = fma(a, MdY[e], MY[e]);
    else
      MX[e - nlen] = fma(a, MtdX[e - nlen], MX[e - nlen]);
  }
}

// The whole update (SPEC.md:359 nudge rule) in one launch: x, y += a1 (dx, dy) with the
// nudge flag, r, s += a2 (dr, ds), and (residual-free dual mode) the incremental advance of
// M Y^T / M^T X -- unconditional: a nudged step makes the host recompute both from M
// (solver.check_advance), which overwrites them.  Segments [X | Y | R | S | MY | MX].
struct StepAll {
  double* v[6];
  const double* dv[6];
  long len[6];
};
__global__ void __launch_bounds__(256) k_step_all(StepAll sa, const double* __restrict__ a1_dev,
                                                  double a1, const double* __restrict__ a2_dev,
                                                  double a2, double tau, int* __restrict__ flag) {
  const double s1 = a1_dev ? *a1_dev : a1, s2 = a2_dev ? *a2_dev : a2;
  const long o1 = sa.len[0], o2 = o1 + sa.len[1], o3 = o2 + sa.len[2], o4 = o3 + sa.len[3],
             o5 = o4 + sa.len[4], o6 = o5 + sa.len[5];
  int nudged = 0;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < o6;
       e += (long)gridDim.x * blockDim.x) {
    const int q = e < o1 ? 0 : e < o2 ? 1 : e < o3 ? 2 : e < o4 ? 3 : e < o5 ? 4 : 5;
    const long i = e - (q == 0 ? 0 : q == 1 ? o1 : q == 2 ? o2 : q == 3 ? o3 : q == 4 ? o4 : o5);
    double* v = sa.v[q];
    const double d = sa.dv[q][i];
    if (q >= 4) {
      v[i] = fma(s1, d, v[i]);
    } else {
      const double old = v[i];
      const double nv = old + (q < 2 ? s1 : s2) * d;
      const bool ok = nv > 0.0;
      v[i] = ok ? nv : (1.0 - tau) * old;
      nudged |= (q < 2) && !ok;
    }
  }
  if (flag != nullptr && __syncthreads_or(nudged) && threadIdx.x == 0) atomicOr(flag, 1);
}

constexpr int RED_BLOCKS = 296;  // fixed -> deterministic reductions

// ---------------------------------------------------------------------------
// Up to four k x k Grams A_q^T B_q over the same rows in one pass (the
// residual-free IPM's small contractions): CTA = row block, 32-row chunks
// staged in shared memory, thread per output; deterministic fixed-order finish.
// ---------------------------------------------------------------------------
struct GramSet {
  const double* A[4];
  const double* B[4];
  double* out[4];
  int count;
};

// One chunk of up to GR_CH rows per CTA: every A_q / B_q row segment of the chunk is
// copied to shared memory with cp.async in one round (all loads in flight), then
// thread per output entry.  (The 32-row double-barrier chunks of the first version
// paid three L2/HBM round trips per CTA: 10 us at c4's 20000 rows.)
constexpr int GR_CH = 128;

template <int K>
__global__ void __launch_bounds__(256) k_grams_partial(GramSet gs, long rows, long rows_per_cta,
                                                       double* __restrict__ part) {
  extern __shared__ __align__(16) double gsm[];  // [count][2][GR_CH][K]
  constexpr int KK = K * K;
  constexpr int U = (4 * KK + 255) / 256;
  const int nq = gs.count, NO = nq * KK, tid = threadIdx.x;
  const long i0 = (long)blockIdx.x * rows_per_cta, i1 = min(rows, i0 + rows_per_cta);
  double acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = 0.0;
  for (long ib = i0; ib < i1; ib += GR_CH) {
    const int nr = (int)min((long)GR_CH, i1 - ib);
    __syncthreads();
    for (int q = 0; q < nq; ++q) {
      double* sa = gsm + (long)(2 * q) * GR_CH * K;
      double* sb = sa + GR_CH * K;
      const double* ga = gs.A[q] + ib * K;
      const double* gb = gs.B[q] + ib * K;
      for (int e = tid; e < nr * K; e += 256) {
        const unsigned da = (unsigned)__cvta_generic_to_shared(sa + e);
        const unsigned db = (unsigned)__cvta_generic_to_shared(sb + e);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(da), "l"(ga + e) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(db), "l"(gb + e) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = tid + 256 * u;
      if (e < NO) {
        const int q = e / KK, a = (e / K) % K, b = e % K;
        const double* sa = gsm + (long)(2 * q) * GR_CH * K;
        const double* sb = sa + GR_CH * K;
        double s0 = acc[u];
        for (int r = 0; r < nr; ++r) s0 = fma(sa[r * K + a], sb[r * K + b], s0);
        acc[u] = s0;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int e = tid + 256 * u;
    if (e < NO) part[(long)blockIdx.x * NO + e] = acc[u];
  }
}

__global__ void __launch_bounds__(256) k_grams_finish(GramSet gs, int KK,
                                                      const double* __restrict__ part,
                                                      int nparts) {
  // one warp per output element, lanes stride the partials, fixed butterfly
  const int NO = gs.count * KK;
  const int e = (int)(((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= NO) return;
  double s = 0.0;
  for (int g = lane; g < nparts; g += 32) s += part[(long)g * NO + e];
  s = warp_sum(s);
  if (lane == 0) gs.out[e / KK][e % KK] = s;
}

}  // namespace

#define NMFB_K_SWITCH(k, MACRO) \
  switch (k) {                  \
    MACRO(1) MACRO(2) MACRO(3) MACRO(4) MACRO(5) MACRO(6) MACRO(7) MACRO(8) MACRO(9) MACRO(10) \
    MACRO(11) MACRO(12) MACRO(13) MACRO(14) MACRO(15) MACRO(16) \
    default: return NMFB_EINVAL; \
  }

extern "C" int nmfb_ipm_reduce_blocks(void) { return RED_BLOCKS; }

// F = X Y - M; graX = F Y^T; out[0] = ||F||^2.  work >= RED_BLOCKS.
extern "C" int nmfb_residual(const void* M, int m_is_f32, long n, long m, long k, const double* X,
                             const double* Yt, double* F, double* gX, double* out, double* work,
                             void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0 || m <= 0) return NMFB_EINVAL;
#define CASE(KK)                                                                          \
  case KK:                                                                                \
    if (m_is_f32)                                                                         \
      ++g_nmfb_launches, k_residual_rows<KK, 2, float><<<RED_BLOCKS, 256, 0, st>>>((const float*)M, n, m, X, \
                                                                Yt, F, gX, work);         \
    else                                                                                  \
      ++g_nmfb_launches, k_residual_rows<KK, 2, double><<<RED_BLOCKS, 256, 0, st>>>((const double*)M, n, m,  \
                                                                 X, Yt, F, gX, work);     \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  ++g_nmfb_launches, k_finish_sum1<<<1, 256, 0, st>>>(work, RED_BLOCKS, out);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_r1_factor(const double* GY, const double* X, const double* R,
                              const double* gX, double mux, double rho, long n, long k,
                              double* L, double* h, double* g, double* Apk, double* XXpk,
                              int* bad, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) return NMFB_EINVAL;
  cudaMemsetAsync(bad, 0x7F, sizeof(int), st);  // 0x7F7F7F7F: no failing row
  const int blocks = (int)((n + R1_THREADS - 1) / R1_THREADS);
#define CASE(KK)                                                                               \
  case KK: {                                                                                   \
    const size_t sm = (size_t)(R1_THREADS / 32) * 32 * R1W<KK>::v * sizeof(double);         \
    nmfb_smem_attr(k_r1_factor<KK>, sm);                                                       \
    ++g_nmfb_launches, k_r1_factor<KK><<<blocks, R1_THREADS, sm, st>>>(GY, X, R, gX, mux, rho, n, L, h, g, Apk, XXpk, bad, g_mu_dev); \
    break;                                                                                     \
  }
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_hg(const double* L, const double* b1, double b1_scale, long n, long k,
                       double* h, double* g, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) return NMFB_EINVAL;
  const int blocks = (int)((n + 127) / 128);
#define CASE(KK)                                                               \
  case KK:                                                                     \
    ++g_nmfb_launches, k_hg_rows<KK><<<blocks, 128, 0, st>>>(L, b1, b1_scale, n, h, g);           \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" long nmfb_atb_work_len(long rows, long ca, long cb) {
  const long tiles = ((ca + 31) / 32) * ((cb + 31) / 32);
  long ns = (148 * 4 + tiles - 1) / tiles;
  const long max_ns = (rows + 255) / 256;
  if (ns > max_ns) ns = max_ns;
  if (ns < 1) ns = 1;
  long len = ns * ca * cb;
  {  // k_atb_mma stripes (see nmfb_atb)
    const long t64 = ((ca + 63) / 64) * ((cb + 63) / 64);
    long n2 = (148 + t64 - 1) / t64;
    const long mx = (rows + 127) / 128;
    if (n2 > mx) n2 = mx;
    if (n2 < 1) n2 = 1;
    long stripe = (rows + n2 - 1) / n2;
    stripe = ((stripe + 31) / 32) * 32;
    n2 = stripe > 0 ? (rows + stripe - 1) / stripe : 1;
    if (n2 * ca * cb > len) len = n2 * ca * cb;
  }
  if (ca == cb && ca <= 16 && rows > 0) {  // small square products run as a Gram (nmfb_grams)
    const long g = nmfb_grams_work_len(rows, ca, 1);
    if (g > len) len = g;
  }
  return len;
}

// out (ca x cb) = A^T B; A (rows x ca), B (rows x cb).  No library GEMM: the large
// products run on k_atb_mma (FP64 tensor cores), the small square ones on nmfb_grams.
// Kept for ABI compatibility (it created the cuBLAS handle of earlier versions).
extern "C" int nmfb_blas_init(void* stream) {
  (void)stream;
  return NMFB_OK;
}

extern "C" int nmfb_atb(const double* A, long rows, long ca, const double* B, long cb,
                        double* out, double* work, long work_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (ca <= 0 || cb <= 0) return NMFB_EINVAL;
  if (rows <= 0) {
    cudaMemsetAsync(out, 0, sizeof(double) * ca * cb, st);
    return NMFB_OK;
  }
  // small square products (the packed k(k+1)/2-wide capacitance Grams of c1-c3): the
  // multi-Gram kernel (64 rows per CTA, warp-per-entry finish) instead of 32 x 32
  // tiles with 2 of 8 x 32 threads busy
  if (ca == cb && ca <= 16 && 2.0 * (double)rows * (double)ca * (double)cb < 1e7 &&
      nmfb_grams_work_len(rows, ca, 1) <= work_len)
    return nmfb_grams(1, A, B, out, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                      nullptr, nullptr, rows, ca, work, work_len, stream);
  // large products: split-K DMMA (k_atb_mma), fixed-order finish
  if (2.0 * (double)rows * (double)ca * (double)cb >= 1e6) {
    const long tiles = ((ca + ATB_T - 1) / ATB_T) * ((cb + ATB_T - 1) / ATB_T);
    long ns = (148 + tiles - 1) / tiles;  // one wave
    const long max_ns = (rows + 127) / 128;
    if (ns > max_ns) ns = max_ns;
    if (ns < 1) ns = 1;
    long stripe = (rows + ns - 1) / ns;
    stripe = ((stripe + ATB_R - 1) / ATB_R) * ATB_R;
    ns = (rows + stripe - 1) / stripe;
    if (ns * ca * cb <= work_len) {
      dim3 grid((unsigned)((ca + ATB_T - 1) / ATB_T), (unsigned)((cb + ATB_T - 1) / ATB_T),
                (unsigned)ns);
      nmfb_smem_attr(k_atb_mma, ATB_SMEM);
      const int flat = (ca <= ATB_T && cb <= ATB_T && (((uintptr_t)A | (uintptr_t)B) & 15) == 0) ? 1 : 0;
      ++g_nmfb_launches, k_atb_mma<<<grid, 256, ATB_SMEM, st>>>(A, rows, ca, B, cb, stripe, work, flat);
      ++g_nmfb_launches, k_sum_parts_warp<<<(unsigned)((ca * cb * 32 + 255) / 256), 256, 0, st>>>(
          work, (int)ns, ca * cb, out);
      NMFB_CHECK_LAUNCH();
      return NMFB_OK;
    }
  }
  const long tiles = ((ca + 31) / 32) * ((cb + 31) / 32);
  long ns = (148 * 4 + tiles - 1) / tiles;
  const long max_ns = (rows + 255) / 256;
  if (ns > max_ns) ns = max_ns;
  if (ns < 1) ns = 1;
  const long stripe = (rows + ns - 1) / ns;
  ns = (rows + stripe - 1) / stripe;
  dim3 grid((unsigned)((ca + 31) / 32), (unsigned)((cb + 31) / 32), (unsigned)ns);
  if (ns == 1) {
    ++g_nmfb_launches, k_atb_partial<<<grid, 256, 0, st>>>(A, rows, ca, B, cb, stripe, out);
  } else {
    if (ns * ca * cb > work_len) return NMFB_ENOMEM;
    ++g_nmfb_launches, k_atb_partial<<<grid, 256, 0, st>>>(A, rows, ca, B, cb, stripe, work);
    ++g_nmfb_launches, k_sum_parts<<<(unsigned)((ca * cb + 255) / 256), 256, 0, st>>>(work, (int)ns, ca * cb, out);
  }
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_make_p(const double* X, const double* Apk, long n, long k, double* P,
                           void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const long total = n * k * k * k;
  const unsigned blocks = (unsigned)((total + 255) / 256);
#define CASE(KK)                                                 \
  case KK:                                                       \
    ++g_nmfb_launches, k_make_p<KK><<<blocks, 256, 0, st>>>(X, Apk, n, P);          \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// Schur matrix assembly (lower block triangle).  W may be NULL (Gauss-Newton).
extern "C" int nmfb_schur_assemble(const double* Yt, const double* S, long m, long k,
                                   const double* Zpk, const double* XtX, double rho,
                                   const double* W, double* A, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (m <= 0) return NMFB_EINVAL;
  const long k3 = k * k * k;
  int TL = (int)(4096 / k3);  // <= 32 KB of V per CTA
  if (TL < 1) TL = 1;
  if (TL > 64) TL = 64;
  const size_t smem = (size_t)TL * k3 * sizeof(double);
  const long ltiles = (m + TL - 1) / TL;
  // split the j range so that there are enough CTAs
  long jsplit = (148 * 8 + ltiles - 1) / ltiles;
  if (jsplit < 1) jsplit = 1;
  long jchunk = (m + jsplit - 1) / jsplit;
  if (jchunk < 1) jchunk = 1;
  jsplit = (m + jchunk - 1) / jchunk;
  dim3 grid((unsigned)ltiles, (unsigned)jsplit);
#define CASE(KK)                                                                              \
  case KK:                                                                                    \
    nmfb_smem_attr(k_schur_assemble<KK>, \
                         (int)smem);                                                          \
    ++g_nmfb_launches, k_schur_assemble<KK><<<grid, 256, smem, st>>>(Yt, S, m, Zpk, XtX, rho, W, TL, jchunk, A); \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

static int term4_mma_nsplit(long n, long m) {
  const long t32 = (m + 31) / 32;
  const long active = t32 * (t32 + 1) / 2;
  long ns = (148 * 2 + active - 1) / active;
  const long maxs = (n + 255) / 256;
  if (ns > maxs) ns = maxs;
  if (ns > 32) ns = 32;
  return ns < 1 ? 1 : (int)ns;
}
static bool term4_use_mma(long k) {
  static const bool on = [] {
    const char* e = getenv("NMFB_TERM4_MMA");
    return !(e && e[0] == '0');
  }();
  return on && k <= 4;
}

static int term4_nsplit(long n, long m, long k) {
  const long kk = k * (k + 1) / 2;
  const long tiles = (m + 15) / 16;
  const long active = tiles * (tiles + 1) / 2 * ((kk + 15) / 16);
  long ns = (148 * 2 + active - 1) / active;
  const long maxs = (n + 255) / 256;
  if (ns > maxs) ns = maxs;
  if (ns > 32) ns = 32;
  return ns < 1 ? 1 : (int)ns;
}

extern "C" long nmfb_term4_work_len(long n, long m, long k) {
  int ns = term4_nsplit(n, m, k);
  if (k <= 4) ns = max(ns, term4_mma_nsplit(n, m));
  return ns > 1 ? (long)ns * m * m * (k * (k + 1) / 2) : 1;
}

extern "C" int nmfb_schur_term4(const double* F, long n, long m, long k, const double* Apk,
                                double* A, double* work, long work_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const long kk = k * (k + 1) / 2;
  if (term4_use_mma(k)) {  // K <= 4: weighted SYRKs on the FP64 tensor cores
    int ns = term4_mma_nsplit(n, m);
    if (ns > 1 && (long)ns * m * m * kk > work_len) ns = 1;
    const long t32 = (m + 31) / 32;
    dim3 grid((unsigned)t32, (unsigned)t32, (unsigned)ns);
#define CASEM(KK)                                                                              \
  case KK:                                                                                     \
    ++g_nmfb_launches, k_schur_term4_mma<KK><<<grid, 256, 0, st>>>(F, n, m, Apk, A, ns, work); \
    if (ns > 1)                                                                                \
      ++g_nmfb_launches, k_term4_finish<KK><<<(unsigned)((m * m * kk + 255) / 256), 256, 0, st>>>( \
          work, m, ns, A);                                                                     \
    break;
    switch (k) {
      CASEM(1) CASEM(2) CASEM(3) CASEM(4)
      default: return NMFB_EINVAL;
    }
#undef CASEM
    NMFB_CHECK_LAUNCH();
    return NMFB_OK;
  }
  const long tiles = (m + 15) / 16;
  int ns = term4_nsplit(n, m, k);
  if (ns > 1 && (long)ns * m * m * kk > work_len) ns = 1;
  const long nchunk = (kk + 15) / 16;
  dim3 grid((unsigned)tiles, (unsigned)tiles, (unsigned)(nchunk * ns));
#define CASE(KK)                                                                               \
  case KK: {                                                                                   \
    constexpr int PQ = (KK * (KK + 1) / 2) < 16 ? (KK * (KK + 1) / 2) : 16;                   \
    ++g_nmfb_launches, k_schur_term4<KK, PQ><<<grid, 256, 0, st>>>(F, n, m, Apk, A, ns, work); \
    if (ns > 1)                                                                                \
      ++g_nmfb_launches, k_term4_finish<KK><<<(unsigned)((m * m * kk + 255) / 256), 256, 0, st>>>( \
          work, m, ns, A);                                                                     \
    break;                                                                                     \
  }
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_schur_rhs(const double* Yt, const double* gY, const double* H,
                              const double* FtG, double muy, long m, long k, double* rhs,
                              void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned blocks = (unsigned)((m + 127) / 128);
#define CASE(KK)                                                                  \
  case KK:                                                                        \
    ++g_nmfb_launches, k_schur_rhs<KK><<<blocks, 128, 0, st>>>(Yt, gY, H, FtG, muy, m, rhs, g_mu_dev); \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// dx, dr, ds from dy; out = [gtp, a1max, a2max].  work >= 3*(ceil(n/128) + RED_BLOCKS)
extern "C" int nmfb_direction(const double* L, const double* Xf, const double* h,
                              const double* Gdy, const double* FdY, const double* X,
                              const double* R, const double* gX, double mux, const double* Yt,
                              const double* S, const double* gY, const double* dY, double muy,
                              double tau, long n, long m, long k, double* dX, double* dR,
                              double* dS, double* out, double* work, long work_len,
                              void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int rb = (int)((n + 127) / 128);
  if (work_len < 3L * (rb + RED_BLOCKS)) return NMFB_ENOMEM;
#define CASE(KK)                                                                              \
  case KK:                                                                                    \
    ++g_nmfb_launches, k_dir_rows<KK><<<rb, 128, 0, st>>>(L, Xf, h, Gdy, FdY, X, R, gX, mux, tau, n, dX, dR, work, g_mu_dev); \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  ++g_nmfb_launches, k_dir_cols<<<RED_BLOCKS, 256, 0, st>>>(Yt, S, gY, dY, muy, tau, m * k, dS, work + 3 * rb, g_mu_dev);
  ++g_nmfb_launches, k_finish_dir<<<1, 256, 0, st>>>(work, rb, work + 3 * rb, RED_BLOCKS, out);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// out[0..5] = [AA, AB, BB, AC, BC, CC]
extern "C" int nmfb_quartic(const double* F, long n, long m, long k, const double* X,
                            const double* dX, const double* Yt, const double* dYt, double* out,
                            double* work, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
#define CASE(KK)                                                                           \
  case KK:                                                                                 \
    ++g_nmfb_launches, k_quartic_rows<KK, 2><<<RED_BLOCKS, 256, 0, st>>>(F, n, m, X, dX, Yt, dYt, work);      \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  ++g_nmfb_launches, k_finish_cols<<<1, 256, 0, st>>>(work, RED_BLOCKS, 6, out);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// out[2t], out[2t+1] = barrier increments over X and Y for alpha_max / 2^t, t < ntrials
extern "C" int nmfb_barrier_trials(const double* X, const double* dX, long nx, const double* Yt,
                                   const double* dYt, long ny, const double* alpha_max, int ntrials,
                                   double* out, double* work, long work_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = 64;
  if (work_len < 2L * nb * ntrials) return NMFB_ENOMEM;
  dim3 grid(nb, ntrials);
  ++g_nmfb_launches, k_barrier_trials<<<grid, 256, 0, st>>>(X, dX, nx, Yt, dYt, ny, alpha_max, ntrials, work);
  ++g_nmfb_launches, k_finish_trials<<<(2 * ntrials * 32 + 255) / 256, 256, 0, st>>>(work, nb, ntrials, out);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_step_nudge(double* v, const double* dv, long len, double alpha, double tau,
                               void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (len <= 0) return NMFB_OK;
  ++g_nmfb_launches, k_step_nudge<<<nmfb_blocks(len, 256, 148 * 8), 256, 0, st>>>(v, dv, len, alpha, tau);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// out[12]: see k_kkt_partial.  R == NULL -> primal-only duals max(g, 0).
extern "C" int nmfb_kkt_sums(const double* X, const double* R, const double* gX, long nx,
                             const double* Yt, const double* S, const double* gY, long ny,
                             double mux, double muy, double* out, double* work, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  ++g_nmfb_launches, k_kkt_partial<<<RED_BLOCKS, 256, 0, st>>>(X, R, gX, nx, Yt, S, gY, ny, mux, muy, work, g_mu_dev);
  ++g_nmfb_launches, k_finish_kkt<<<1, 256, 0, st>>>(work, RED_BLOCKS, out);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_affine_mu(const double* X, const double* dX, const double* R,
                              const double* dR, long nx, const double* Yt, const double* dY,
                              const double* S, const double* dS, long ny, double a1, double a2,
                              double* out, double* work, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  ++g_nmfb_launches, k_affine_partial<<<RED_BLOCKS, 256, 0, st>>>(X, dX, R, dR, nx, Yt, dY, S, dS, ny, a1, a2, work);
  ++g_nmfb_launches, k_finish_sum1<<<1, 256, 0, st>>>(work, RED_BLOCKS, out);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_clamp_min(double* v, long len, double lo, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (len <= 0) return NMFB_OK;
  ++g_nmfb_launches, k_clamp_fill<<<nmfb_blocks(len, 256, 148 * 8), 256, 0, st>>>(v, len, lo);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_fill(double* v, long len, double c, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (len <= 0) return NMFB_OK;
  ++g_nmfb_launches, k_fill<<<nmfb_blocks(len, 256, 148 * 8), 256, 0, st>>>(v, len, c);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// Barrier trials + Armijo selection with lazy trial batches (graph-capturable): trials
// 0..7 first, a device pre-check of those, then trials 8.. only when it did not
// decide (the later launches return at once otherwise) and the full search.  The
// accepted t is the full search's: the pre-check runs the same arithmetic on the
// same sums, and the barrier sums of a trial do not depend on the batching.
extern "C" int nmfb_armijo_lazy(const double* X, const double* dX, long nx, const double* Yt,
                                const double* dYt, long ny, double* sc, int ntrials, double mu,
                                double wx, double wy, double eta, int max_backtracks,
                                const int* fcodes, double* work, long work_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = 64, TB = 8;
  if (ntrials < 1 || work_len < 2L * nb * ntrials) return NMFB_ENOMEM;
  const double* alpha_max = sc + 5;
  double* bars = sc + 32;
  const int tb = ntrials < TB ? ntrials : TB;
  ++g_nmfb_launches, k_barrier_trials<<<dim3(nb, tb), 256, 0, st>>>(X, dX, nx, Yt, dYt, ny,
                                                                    alpha_max, ntrials, work, 0, nullptr);
  ++g_nmfb_launches, k_finish_trials<<<(2 * tb * 32 + 255) / 256, 256, 0, st>>>(work, nb, tb, bars,
                                                                             0, nullptr);
  ++g_nmfb_launches, k_armijo_select<<<1, 32, 0, st>>>(sc, mu, wx, wy, eta, max_backtracks, fcodes,
                                                       tb, 0, g_mu_dev);
  if (ntrials > tb) {
    const int rest = ntrials - tb;
    ++g_nmfb_launches, k_barrier_trials<<<dim3(nb, rest), 256, 0, st>>>(
        X, dX, nx, Yt, dYt, ny, alpha_max, ntrials, work, tb, sc + 31);
    ++g_nmfb_launches, k_finish_trials<<<(2 * rest * 32 + 255) / 256, 256, 0, st>>>(
        work, nb, ntrials, bars, tb, sc + 31);
  }
  ++g_nmfb_launches, k_armijo_select<<<1, 32, 0, st>>>(sc, mu, wx, wy, eta, max_backtracks, fcodes,
                                                       -1, 1, g_mu_dev);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_armijo_select(double* sc, double mu, double wx, double wy, double eta,
                                  int max_backtracks, const int* fcodes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  ++g_nmfb_launches, k_armijo_select<<<1, 32, 0, st>>>(sc, mu, wx, wy, eta, max_backtracks, fcodes,
                                                       -1, 0, g_mu_dev);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_step_nudge_flag(double* v, const double* dv, long len, const double* alpha_dev,
                                    double alpha, double tau, int* flag, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (len <= 0) return NMFB_OK;
  ++g_nmfb_launches, k_step_nudge_flag<<<nmfb_blocks(len, 256, 148 * 8), 256, 0, st>>>(
      v, dv, len, alpha_dev, alpha, tau, flag);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_ffree_advance(double* MY, const double* MdY, long nlen, double* MX,
                                  const double* MtdX, long mlen, const double* alpha_dev,
                                  double alpha, const int* flag, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (nlen + mlen <= 0) return NMFB_OK;
  ++g_nmfb_launches, k_ffree_advance<<<nmfb_blocks(nlen + mlen, 256, 148 * 8), 256, 0, st>>>(
      MY, MdY, nlen, MX, MtdX, mlen, alpha_dev, alpha, flag);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_step_all(double* X, const double* dX, long nk, double* Y, const double* dY,
                             long mk, double* R, const double* dR, double* S, const double* dS,
                             double* MY, const double* MdY, double* MX, const double* MtdX,
                             const double* a1_dev, double a1, const double* a2_dev, double a2,
                             double tau, int* flag, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  StepAll sa;
  double* v[6] = {X, Y, R, S, MY, MX};
  const double* dv[6] = {dX, dY, dR, dS, MdY, MtdX};
  const long len[6] = {nk, mk, nk, mk, MY ? nk : 0, MX ? mk : 0};
  long tot = 0;
  for (int q = 0; q < 6; ++q) sa.v[q] = v[q], sa.dv[q] = dv[q], sa.len[q] = len[q], tot += len[q];
  if (tot <= 0) return NMFB_OK;
  ++g_nmfb_launches, k_step_all<<<nmfb_blocks(tot, 256, 148 * 8), 256, 0, st>>>(
      sa, a1_dev, a1, a2_dev, a2, tau, flag);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_step_nudge_dev(double* v, const double* dv, long len, const double* alpha,
                                   double tau, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (len <= 0) return NMFB_OK;
  ++g_nmfb_launches, k_step_nudge_dev<<<nmfb_blocks(len, 256, 148 * 8), 256, 0, st>>>(v, dv, len, alpha, tau);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// ---------------------------------------------------------------------------
// Residual-free ("F-free") gradients and Armijo coefficients for large M.
// With F = X Y - M (never formed):
//   graX = X (Y Y^T) - M Y^T,   graY = (X^T X) Y - X^T M   (rows of Y^T)
//   ||F||^2 = ||M||^2 - 2 <X, M Y^T> + <X^T X, Y Y^T>
// and, for A = F, B = dX Y + X dY, C = dX dY with the k x k Grams
//   A1 = dX^T dX, A2 = dX^T X, XX = X^T X, B1 = dY dY^T, B2 = Y dY^T, YY = Y Y^T:
//   AB = <dX, graX> + <dY, graY>            AC = tr(A2 B2) - <dX, M dY^T>
//   BB = tr(A1 YY) + tr(XX B1) + 2 tr(A2 B2^T)
//   BC = tr(A1 B2^T) + tr(A2^T B1)           CC = tr(A1 B1)
// so an IPM iteration streams M three times (M Y^T, X^T M, M dY^T) and needs
// no n x m workspace (64 GB at config c5).
// ---------------------------------------------------------------------------
template <int K>
__global__ void k_ffree_grad_rows(const double* __restrict__ V, const double* __restrict__ G,
                                  const double* __restrict__ MV, long rows,
                                  double* __restrict__ grad, double* __restrict__ part) {
  // grad[r] = V[r] G - MV[r]; part[block] = sum_r <V[r], MV[r]>
  __shared__ double g[K * K];
  __shared__ double sh[32];
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) g[e] = G[e];
  __syncthreads();
  double dot = 0.0;
  for (long r = (long)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (long)gridDim.x * blockDim.x) {
    double v[K];
#pragma unroll
    for (int p = 0; p < K; ++p) v[p] = V[r * K + p];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      double s = 0.0;
#pragma unroll
      for (int p = 0; p < K; ++p) s = fma(v[p], g[p * K + q], s);
      const double mv = MV[r * K + q];
      grad[r * K + q] = s - mv;
      dot = fma(v[q], mv, dot);
    }
  }
  dot = block_sum(dot, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = dot;
}

// sc[0] = ||M||^2 - 2 xm + <XX, YY>  (fsq)
__global__ void k_ffree_fsq(const double* __restrict__ part, int nb, double mnorm2,
                            const double* __restrict__ XX, const double* __restrict__ YY, int k,
                            double* __restrict__ sc, double* __restrict__ xm_out) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) v += part[b];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    double t = 0.0;
    if (XX && YY)  // the replicated <X^T X, Y Y^T> term (rank 0 only when row-sharded)
      for (int e = 0; e < k * k; ++e) t = fma(XX[e], YY[e], t);
    if (xm_out) *xm_out = v;
    sc[0] = mnorm2 - 2.0 * v + t;
  }
}

// quartic coefficients from Grams and dot products -> sc[10..15]
// dots: [0] <dX, graX>, [1] <dY, graY>, [2] <dX, M dY^T>  (traces of k x k products)
__global__ void k_ffree_quartic(const double* __restrict__ A1, const double* __restrict__ A2,
                                const double* __restrict__ XX, const double* __restrict__ B1,
                                const double* __restrict__ B2, const double* __restrict__ YY,
                                const double* __restrict__ Dgx, const double* __restrict__ Dgy,
                                const double* __restrict__ Dmd, int k, double* __restrict__ sc) {
  // one warp: lanes stride the k x k entries of every trace, fixed butterfly sums
  const int lane = threadIdx.x & 31;
  double t[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) t[q] = 0.0;
  for (int e = lane; e < k * k; e += 32) {
    const int a = e / k, b = e % k, et = b * k + a;
    t[0] = fma(A2[e], B2[et], t[0]);  // tr(A2 B2)
    t[1] = fma(A1[e], YY[et], t[1]);  // tr(A1 YY)
    t[2] = fma(XX[e], B1[et], t[2]);  // tr(XX B1)
    t[3] = fma(A2[e], B2[e], t[3]);   // tr(A2 B2^T)
    t[4] = fma(A1[e], B2[e], t[4]);   // tr(A1 B2^T)
    t[5] = fma(A2[e], B1[e], t[5]);   // tr(A2 B1^T)
    t[6] = fma(A1[e], B1[et], t[6]);  // tr(A1 B1)
  }
  for (int a = lane; a < k; a += 32) {
    t[7] += Dgx[a * k + a] + Dgy[a * k + a];
    t[8] += Dmd[a * k + a];
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) t[q] = warp_sum(t[q]);
  if (lane == 0) {
    sc[10] = sc[0];
    sc[11] = t[7];
    sc[12] = t[1] + t[2] + 2.0 * t[3];
    sc[13] = t[0] - t[8];
    sc[14] = t[4] + t[5];
    sc[15] = t[6];
  }
}

extern "C" int nmfb_ffree_grad_rows(const double* V, const double* G, const double* MV, long rows,
                                    long k, double* grad, double* part, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
#define CASE(KK)                                                                             \
  case KK:                                                                                   \
    ++g_nmfb_launches, k_ffree_grad_rows<KK><<<RED_BLOCKS, 256, 0, st>>>(V, G, MV, rows, grad, part); \
    break;
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_ffree_fsq(const double* part, double mnorm2, const double* XX,
                              const double* YY, long k, double* sc, double* xm_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  ++g_nmfb_launches, k_ffree_fsq<<<1, 256, 0, st>>>(part, RED_BLOCKS, mnorm2, XX, YY, (int)k, sc, xm_out);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_ffree_quartic(const double* A1, const double* A2, const double* XX,
                                  const double* B1, const double* B2, const double* YY,
                                  const double* Dgx, const double* Dgy, const double* Dmd, long k,
                                  double* sc, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  ++g_nmfb_launches, k_ffree_quartic<<<1, 32, 0, st>>>(A1, A2, XX, B1, B2, YY, Dgx, Dgy, Dmd, (int)k, sc);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// out_q = A_q^T B_q (k x k) for q < count <= 4; A_q, B_q (rows x k) row-major fp64.
// work >= nmfb_grams_work_len(rows, k, count).
static long grams_ctas(long rows) {
  long g = (rows + GR_CH - 1) / GR_CH;
  if (g > 296) g = 296;
  return g < 1 ? 1 : g;
}
extern "C" long nmfb_grams_work_len(long rows, long k, long count) {
  return grams_ctas(rows) * count * k * k;
}
extern "C" int nmfb_grams(int count, const double* A0, const double* B0, double* O0,
                          const double* A1, const double* B1, double* O1, const double* A2,
                          const double* B2, double* O2, const double* A3, const double* B3,
                          double* O3, long rows, long k, double* work, long work_len,
                          void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (count < 1 || count > 4 || k < 1 || k > 16) return NMFB_EINVAL;
  GramSet gs;
  const double* As[4] = {A0, A1, A2, A3};
  const double* Bs[4] = {B0, B1, B2, B3};
  double* Os[4] = {O0, O1, O2, O3};
  for (int q = 0; q < 4; ++q) {
    gs.A[q] = As[q];
    gs.B[q] = Bs[q];
    gs.out[q] = Os[q];
  }
  gs.count = count;
  if (rows <= 0) {
    for (int q = 0; q < count; ++q) cudaMemsetAsync(Os[q], 0, sizeof(double) * k * k, st);
    return NMFB_OK;
  }
  const long G = grams_ctas(rows);
  if (G * count * k * k > work_len) return NMFB_ENOMEM;
  const long rpc = (rows + G - 1) / G;
  static const bool attrs = [] {  // once, on the first (eager) call: 4 Grams of k = 16
#define SETA(KK_)                                                                             \
    nmfb_smem_attr(k_grams_partial<KK_>, \
                         (int)(8 * GR_CH * KK_ * sizeof(double)));
    SETA(1) SETA(2) SETA(3) SETA(4) SETA(5) SETA(6) SETA(7) SETA(8) SETA(9) SETA(10) SETA(11)
    SETA(12) SETA(13) SETA(14) SETA(15) SETA(16)
#undef SETA
    return true;
  }();
  (void)attrs;
#define CASE(KK_)                                                                             \
  case KK_: {                                                                                 \
    const size_t sm = (size_t)count * 2 * GR_CH * KK_ * sizeof(double);                       \
    ++g_nmfb_launches, k_grams_partial<KK_><<<(unsigned)G, 256, sm, st>>>(gs, rows, rpc, work); \
    break;                                                                                    \
  }
  NMFB_K_SWITCH(k, CASE)
#undef CASE
  const int NO = count * (int)(k * k);
  ++g_nmfb_launches, k_grams_finish<<<(NO + 7) / 8, 256, 0, st>>>(gs, (int)(k * k), work, (int)G);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_set_mu_source(const double* mu_dev) {
  g_mu_dev = mu_dev;
  return NMFB_OK;
}
