// Reference-surface kernels: the seven kernels of the reference's kernel
// module (/root/reference/pkg/src/nmfstream/_kernels_numba.py) as batched
// sm_100a kernels that are BIT-IDENTICAL to the reference.
//
// Every output element is produced by one thread that executes the exact
// operation sequence of the reference loop nest (same association order, no
// FMA contraction: this file is compiled with -fmad=false, sqrt and division
// are IEEE correctly rounded), so parallelism comes only from independent
// right-hand sides / blocks / output elements, never from reordering a sum.
//
//   nnls_batch           :277-477  one thread per rhs; warm modes 0/1/2
//                                  (mode 1, the sequential "streaming chain",
//                                  is resolved by a speculative fixed point)
//   block_cholesky       :12-29    one thread per block
//   block_solve_lower(_t):32-57    one thread per (block, rhs column)
//   schur_reduce         :72-143   one thread per output block pair (j, l)
//   rhs_reduce           :146-178  one thread per column j
//   back_substitute      :181-224  one thread per row i
//
// The production IPM path (ipm.cu, lowrank.cu, persist.cu) uses re-associated O(n k^4)
// formulations of the same quantities; these kernels are the parity surface.
#include "common.cuh"
#include "nmfb200.h"
#include "nnls_warp.cuh"

#include <climits>
#include <cstdlib>

namespace {

// packed lower-triangular index (i >= j)
__device__ __forceinline__ int tri(int i, int j) { return i * (i + 1) / 2 + j; }

// --------------------------------------------------------------------------
// nnls_batch
// --------------------------------------------------------------------------
template <int K>
struct NnlsScratch {
  double x[K], w[K], z[K], rbuf[K], dz[K], d[K];
  double L[K * (K + 1) / 2];
  int pidx[K];
};

// _passive_factor (:227-244); a_buf[a][b] == ctc[pidx[a]][pidx[b]] is read in place.
template <int K>
__device__ bool passive_factor(const double* ctc, int k, NnlsScratch<K>& s, int np) {
  for (int j = 0; j < np; ++j) {
    double acc = ctc[s.pidx[j] * k + s.pidx[j]];
    for (int p = 0; p < j; ++p) acc -= s.L[tri(j, p)] * s.L[tri(j, p)];
    if (acc <= 0.0) return false;
    s.L[tri(j, j)] = sqrt(acc);
    for (int i = j + 1; i < np; ++i) {
      double t = ctc[s.pidx[i] * k + s.pidx[j]];
      for (int p = 0; p < j; ++p) t -= s.L[tri(i, p)] * s.L[tri(j, p)];
      s.L[tri(i, j)] = t / s.L[tri(j, j)];
    }
  }
  return true;
}

// _chol_solve_small (:247-258): z <- (L L^T)^{-1} b
template <int K>
__device__ void chol_solve_small(const NnlsScratch<K>& s, const double* b, int np, double* z) {
  for (int i = 0; i < np; ++i) {
    double acc = b[i];
    for (int p = 0; p < i; ++p) acc -= s.L[tri(i, p)] * z[p];
    z[i] = acc / s.L[tri(i, i)];
  }
  for (int i = np - 1; i >= 0; --i) {
    double acc = z[i];
    for (int p = i + 1; p < np; ++p) acc -= s.L[tri(p, i)] * z[p];
    z[i] = acc / s.L[tri(i, i)];
  }
}

// _passive_solve_refined (:261-274)
template <int K>
__device__ void passive_solve_refined(const double* ctc, int k, NnlsScratch<K>& s, int np) {
  for (int a = 0; a < np; ++a) s.rbuf[a] = s.d[s.pidx[a]];
  chol_solve_small<K>(s, s.rbuf, np, s.z);
  for (int a = 0; a < np; ++a) {
    double acc = s.d[s.pidx[a]];
    for (int b = 0; b < np; ++b) acc -= ctc[s.pidx[a] * k + s.pidx[b]] * s.z[b];
    s.rbuf[a] = acc;
  }
  chol_solve_small<K>(s, s.rbuf, np, s.dz);
  for (int a = 0; a < np; ++a) s.z[a] += s.dz[a];
}

// seed_mode: 0 = no seed, 2 = seed every rhs from `seeds`, 1 = seed rhs t >= 1
// from `seeds` (the chain predecessor's passive set, supplied by the host-side
// fixed point).  ctc is staged in shared memory.
template <int K>
__global__ void __launch_bounds__(128) k_nnls(const double* __restrict__ ctc_g,
                                              const double* __restrict__ ctb,
                                              const double* __restrict__ btb,
                                              const uint8_t* __restrict__ seeds, int seed_mode,
                                              const double* __restrict__ tol, long max_changes,
                                              long nrhs, int k, double* __restrict__ x_out,
                                              uint8_t* __restrict__ p_out,
                                              long long* __restrict__ ch_out,
                                              double* __restrict__ r2_out,
                                              int8_t* __restrict__ st_out) {
  __shared__ double ctc[K * K];
  for (int i = threadIdx.x; i < k * k; i += blockDim.x) ctc[i] = ctc_g[i];
  __syncthreads();
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrhs) return;
  NnlsScratch<K> s;
  bool passive[K];
  for (int j = 0; j < k; ++j) s.d[j] = ctb[t * k + j];
  const double tol_t = tol[t];
  bool solved = false;
  long nch = 0;
  const bool use_seed = (seed_mode == 2) || (seed_mode == 1 && t > 0);
  if (use_seed) {
    for (int j = 0; j < k; ++j) passive[j] = seeds[t * k + j] != 0;
    int np = 0;
    for (int j = 0; j < k; ++j)
      if (passive[j]) s.pidx[np++] = j;
    if (np == 0) {
      bool ok = true;
      for (int j = 0; j < k; ++j)
        if (s.d[j] > tol_t) { ok = false; break; }
      if (ok) {
        for (int j = 0; j < k; ++j) s.x[j] = 0.0;
        solved = true;
      }
    } else if (passive_factor<K>(ctc, k, s, np)) {
      passive_solve_refined<K>(ctc, k, s, np);
      bool feas = true;
      for (int a = 0; a < np; ++a)
        if (s.z[a] < 0.0) { feas = false; break; }
      if (feas) {
        for (int j = 0; j < k; ++j) s.x[j] = 0.0;
        for (int a = 0; a < np; ++a) s.x[s.pidx[a]] = s.z[a];
        bool dual_ok = true;
        for (int j = 0; j < k; ++j) {
          double acc = s.d[j];
          for (int p = 0; p < k; ++p) acc -= ctc[j * k + p] * s.x[p];
          s.w[j] = acc;
          if (passive[j]) {
            if (fabs(acc) > tol_t) { dual_ok = false; break; }
          } else if (acc > tol_t) {
            dual_ok = false;
            break;
          }
        }
        solved = dual_ok;
      }
    }
  }
  int st = 0;
  if (!solved) {
    // cold Lawson-Hanson start (:377-461)
    for (int j = 0; j < k; ++j) {
      passive[j] = false;
      s.x[j] = 0.0;
      s.w[j] = s.d[j];
    }
    for (;;) {
      int jmax = -1;
      double wmax = tol_t;
      for (int j = 0; j < k; ++j)
        if (!passive[j] && s.w[j] > wmax) {
          wmax = s.w[j];
          jmax = j;
        }
      if (jmax < 0) break;
      passive[jmax] = true;
      nch += 1;
      if (nch > max_changes) { st = 1; break; }
      for (;;) {
        int np = 0;
        for (int j = 0; j < k; ++j)
          if (passive[j]) s.pidx[np++] = j;
        if (np == 0) break;
        if (!passive_factor<K>(ctc, k, s, np)) { st = 2; break; }
        passive_solve_refined<K>(ctc, k, s, np);
        bool all_pos = true;
        for (int a = 0; a < np; ++a)
          if (s.z[a] <= 0.0) { all_pos = false; break; }
        if (all_pos) {
          for (int j = 0; j < k; ++j) s.x[j] = 0.0;
          for (int a = 0; a < np; ++a) s.x[s.pidx[a]] = s.z[a];
          break;
        }
        double alpha = 1.0;
        for (int a = 0; a < np; ++a)
          if (s.z[a] <= 0.0) {
            const double xa = s.x[s.pidx[a]];
            const double ratio = xa / (xa - s.z[a]);
            if (ratio < alpha) alpha = ratio;
          }
        long ndrop = 0;
        for (int a = 0; a < np; ++a) {
          const int j = s.pidx[a];
          const double xa = s.x[j];
          const double newx = xa + alpha * (s.z[a] - xa);
          if (s.z[a] <= 0.0 && xa / (xa - s.z[a]) <= alpha) {
            s.x[j] = 0.0;
            passive[j] = false;
            ndrop += 1;
          } else {
            s.x[j] = newx > 0.0 ? newx : 0.0;
          }
        }
        nch += ndrop;
        if (nch > max_changes) { st = 1; break; }
      }
      if (st != 0) break;
      for (int j = 0; j < k; ++j) {
        double acc = s.d[j];
        for (int p = 0; p < k; ++p) acc -= ctc[j * k + p] * s.x[p];
        s.w[j] = acc;
      }
    }
  }
  double r2 = btb[t];
  for (int j = 0; j < k; ++j) {
    x_out[t * k + j] = s.x[j];
    p_out[t * k + j] = passive[j] ? 1 : 0;
    r2 -= 2.0 * s.x[j] * s.d[j];
  }
  for (int j = 0; j < k; ++j) {
    double acc = 0.0;
    for (int p = 0; p < k; ++p) acc += ctc[j * k + p] * s.x[p];
    r2 += s.x[j] * acc;
  }
  ch_out[t] = nch;
  r2_out[t] = r2 > 0.0 ? r2 : 0.0;
  st_out[t] = (int8_t)st;
}


// Passive Cholesky factors of every subset pm of {0..K-1}, one W-lane warp segment
// per subset running WNnls::factor (the bit-exact column-oriented factor of
// k_nnls_warp), scattered to global indices: T[(pm K + i) K + j], zero outside the
// passive rows/columns; okf[pm] = 1 when every pivot is positive.
template <int K, int W>
__global__ void __launch_bounds__(128) k_factor_table(const double* __restrict__ ctc_g,
                                                      double* __restrict__ T,
                                                      double* __restrict__ okf) {
  constexpr int SEGS = 32 / W;
  __shared__ double ctc[K * K];
  for (int i = threadIdx.x; i < K * K; i += blockDim.x) ctc[i] = ctc_g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, seg = lane / W;
  const long pm = ((long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * SEGS + seg;
  if (pm >= (1L << K)) return;  // segment-uniform
  WNnls<K, W> s;
  s.sl = lane % W;
  s.sm = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << (seg * W));
  const bool own = s.sl < K;
#pragma unroll
  for (int c = 0; c < K; ++c) s.C[c] = own ? ctc[s.sl * K + c] : 0.0;
  const bool ok = s.factor((unsigned)pm);
  if (own) {
    double* row = T + (pm * K + s.sl) * K;
#pragma unroll
    for (int c = 0; c < K; ++c) row[c] = s.Lr[c];
  }
  if (s.sl == 0) okf[pm] = ok ? 1.0 : 0.0;
}

// nnls_batch, one thread per rhs with every per-rhs vector in registers (exact K,
// fully unrolled) and the passive factors read from the subset table.  The
// passive set is a bit mask; loops run over all K indices in ascending order and
// skip non-passive terms with selects (acc stays bit-identical to the
// reference's loop over passive positions), so a warp stays converged inside a
// Lawson-Hanson trip and issues ~K^2 instructions per trip for 32 right-hand
// sides (the warp-per-rhs kernel issues that per rhs).
template <int K>
__global__ void __launch_bounds__(TabT<K>::v) k_nnls_tab(const double* __restrict__ ctc_g,
                                                  const double* __restrict__ ctb,
                                                  const double* __restrict__ btb,
                                                  const uint8_t* __restrict__ seeds, int seed_mode,
                                                  const double* __restrict__ tol, long max_changes,
                                                  long nrhs, double* __restrict__ x_out,
                                                  uint8_t* __restrict__ p_out,
                                                  long long* __restrict__ ch_out,
                                                  double* __restrict__ r2_out,
                                                  int8_t* __restrict__ st_out,
                                                  const double* __restrict__ T) {
  __shared__ double ctc[K * K];
  __shared__ double sLall[TNnls<K, true>::KT * TabT<K>::v];
  for (int i = threadIdx.x; i < K * K; i += blockDim.x) ctc[i] = ctc_g[i];
  __syncthreads();
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrhs) return;
  const double* okf = T + ((long)K * K << K);
  TNnls<K, true> s;
  s.C = ctc;
  s.sL = sLall + threadIdx.x;
#pragma unroll
  for (int j = 0; j < K; ++j) s.d[j] = ctb[t * K + j];
  const bool use_seed = (seed_mode == 2) || (seed_mode == 1 && t > 0);
  unsigned seed_pm = 0u;
  if (use_seed)
#pragma unroll
    for (int j = 0; j < K; ++j) seed_pm |= (seeds[t * K + j] != 0 ? 1u : 0u) << j;
  double x[K], r2;
  unsigned pm;
  long nch;
  int st;
  tnnls_solve<K, true>(s, T, okf, btb[t], tol[t], use_seed, seed_pm, max_changes, x, pm, nch, r2,
                       st);
#pragma unroll
  for (int j = 0; j < K; ++j) {
    x_out[t * K + j] = x[j];
    p_out[t * K + j] = TNnls<K, true>::bit(pm, j) ? 1 : 0;
  }
  ch_out[t] = nch;
  r2_out[t] = r2;
  st_out[t] = (int8_t)st;
}

template <int K, int W>
__global__ void __launch_bounds__(128) k_nnls_warp(const double* __restrict__ ctc_g,
                                                   const double* __restrict__ ctb,
                                                   const double* __restrict__ btb,
                                                   const uint8_t* __restrict__ seeds, int seed_mode,
                                                   const double* __restrict__ tol, long max_changes,
                                                   long nrhs, double* __restrict__ x_out,
                                                   uint8_t* __restrict__ p_out,
                                                   long long* __restrict__ ch_out,
                                                   double* __restrict__ r2_out,
                                                   int8_t* __restrict__ st_out,
                                                   const double* __restrict__ ftab = nullptr) {
  constexpr int SEGS = 32 / W;
  __shared__ double ctc[K * K];
  for (int i = threadIdx.x; i < K * K; i += blockDim.x) ctc[i] = ctc_g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, seg = lane / W;
  const long t = ((long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * SEGS + seg;
  if (t >= nrhs) return;  // segment-uniform
  WNnls<K, W> s;
  if (ftab != nullptr) {
    s.T = ftab;
    s.okf = ftab + ((long)K * K << K);
  }
  s.sl = lane % W;
  s.sm = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << (seg * W));
  const int sl = s.sl;
  const bool own = sl < K;
#pragma unroll
  for (int c = 0; c < K; ++c) s.C[c] = own ? ctc[sl * K + c] : 0.0;
  const double d = own ? ctb[t * K + sl] : 0.0;
  const bool use_seed = (seed_mode == 2) || (seed_mode == 1 && t > 0);
  const bool sp = use_seed && own && seeds[t * K + sl] != 0;
  double x, r2;
  unsigned pm;
  long nch;
  int st;
  nnls_seg_solve<K, W>(s, d, btb[t], tol[t], use_seed, sp, max_changes, x, pm, nch, r2, st);
  if (own) {
    x_out[t * K + sl] = x;
    p_out[t * K + sl] = ((pm >> sl) & 1u) ? 1 : 0;
  }
  if (sl == 0) {
    ch_out[t] = nch;
    r2_out[t] = r2;
    st_out[t] = (int8_t)st;
  }
}

__global__ void k_set_int(int* p, int v) { *p = v; }

// chain fixed point: seeds[t] <- passive[t-1]; flag if any seed changed.
__global__ void k_chain_update(const uint8_t* __restrict__ p_out, uint8_t* __restrict__ seeds,
                               long nrhs, int k, int* __restrict__ changed) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (t >= nrhs) return;
  bool diff = false;
  for (int j = 0; j < k; ++j) {
    const uint8_t v = p_out[(t - 1) * k + j];
    if (seeds[t * k + j] != v) {
      seeds[t * k + j] = v;
      diff = true;
    }
  }
  if (diff) atomicExch(changed, 1);
}

// --------------------------------------------------------------------------
// block_cholesky / block_solve_lower / block_solve_lower_t
// --------------------------------------------------------------------------
template <int K>
__global__ void k_block_chol(const double* __restrict__ blocks, long nb, int k,
                             double* __restrict__ out, int* __restrict__ bad) {
  const long b = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const double* A = blocks + b * k * k;
  double* L = out + b * k * k;
  double l[K * K];
  for (int j = 0; j < k; ++j) {
    double s = A[j * k + j];
    for (int p = 0; p < j; ++p) s -= l[j * K + p] * l[j * K + p];
    if (s <= 0.0) {
      atomicMin(bad, (int)b);
      return;  // entries not yet written stay zero, as in the reference
    }
    l[j * K + j] = sqrt(s);
    L[j * k + j] = l[j * K + j];
    for (int i = j + 1; i < k; ++i) {
      double t = A[i * k + j];
      for (int p = 0; p < j; ++p) t -= l[i * K + p] * l[j * K + p];
      l[i * K + j] = t / l[j * K + j];
      L[i * k + j] = l[i * K + j];
    }
  }
}

// the reference returns at the first failing block: blocks after it stay zero
__global__ void k_zero_after_bad(double* __restrict__ out, long nb, int k,
                                 const int* __restrict__ bad) {
  const long b0 = *bad;
  const long total = nb * k * k;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x)
    if (e / (k * k) > b0) out[e] = 0.0;
}

template <bool TRANS>
__global__ void k_block_trsm(const double* __restrict__ l, const double* __restrict__ b, long nb,
                             int k, int r, double* __restrict__ z) {
  const long id = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nb * r) return;
  const long t = id / r;
  const int c = (int)(id % r);
  const double* L = l + t * k * k;
  const double* B = b + t * k * r;
  double* Z = z + t * k * r;
  if (!TRANS) {
    for (int i = 0; i < k; ++i) {
      double s = B[i * r + c];
      for (int p = 0; p < i; ++p) s -= L[i * k + p] * Z[p * r + c];
      Z[i * r + c] = s / L[i * k + i];
    }
  } else {
    for (int i = k - 1; i >= 0; --i) {
      double s = B[i * r + c];
      for (int p = i + 1; p < k; ++p) s -= L[p * k + i] * Z[p * r + c];
      Z[i * r + c] = s / L[i * k + i];
    }
  }
}

// w = L^{-1} y_j for one column (the per-column body of _solve_lower_cols, :60-69)
template <int K>
__device__ __forceinline__ void lower_col(const double* L, int k, const double* yj, double* w) {
  for (int i = 0; i < k; ++i) {
    double s = yj[i];
    for (int p = 0; p < i; ++p) s -= L[i * k + p] * w[p];
    w[i] = s / L[i * k + i];
  }
}

// --------------------------------------------------------------------------
// back_substitute (:181-224): one thread per row i, streaming over j in the
// reference's order (w[:, j] is column-independent, so streaming is exact).
// --------------------------------------------------------------------------
template <int K>
__global__ void k_back_sub_exact(const double* __restrict__ x_rows,
                                 const double* __restrict__ y_cols, const double* __restrict__ l,
                                 const double* __restrict__ h, const double* __restrict__ dy,
                                 const double* __restrict__ resid, long n, long m, int k,
                                 int full, double* __restrict__ dx) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double Lr[K * K];
  for (int e = 0; e < k * k; ++e) Lr[(e / k) * K + (e % k)] = l[i * k * k + e];
  double u[K], q[K], w[K], fdy[K], extra[K], out[K];
  for (int p = 0; p < k; ++p) {
    u[p] = x_rows[i * k + p];
    q[p] = 0.0;
    fdy[p] = 0.0;
  }
  for (long j = 0; j < m; ++j) {
    for (int a = 0; a < k; ++a) {
      double s = y_cols[j * k + a];
      for (int p = 0; p < a; ++p) s -= Lr[a * K + p] * w[p];
      w[a] = s / Lr[a * K + a];
    }
    double t = 0.0;
    for (int p = 0; p < k; ++p) t += u[p] * dy[j * k + p];
    for (int p = 0; p < k; ++p) q[p] += w[p] * t;
    if (full) {
      const double f = resid[i * m + j];
      for (int p = 0; p < k; ++p) fdy[p] += f * dy[j * k + p];
    }
  }
  if (full) {
    for (int row = 0; row < k; ++row) {
      double s = fdy[row];
      for (int p = 0; p < row; ++p) s -= Lr[row * K + p] * extra[p];
      extra[row] = s / Lr[row * K + row];
    }
    for (int p = 0; p < k; ++p) q[p] += extra[p];
  }
  for (int row = k - 1; row >= 0; --row) {
    double s = h[i * k + row] - q[row];
    for (int p = row + 1; p < k; ++p) s -= Lr[p * K + row] * out[p];
    out[row] = s / Lr[row * K + row];
  }
  for (int p = 0; p < k; ++p) dx[i * k + p] = out[p];
}

// --------------------------------------------------------------------------
// rhs_reduce (:146-178): one thread per column j, sequential over rows i.
// --------------------------------------------------------------------------
template <int K>
__global__ void k_rhs_reduce_exact(const double* __restrict__ x_rows,
                                   const double* __restrict__ y_cols,
                                   const double* __restrict__ l, const double* __restrict__ h,
                                   const double* __restrict__ resid, long n, long m, int k,
                                   int full, double* __restrict__ r_acc) {
  const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double yj[K], w[K], g[K], acc[K];
  for (int p = 0; p < k; ++p) {
    yj[p] = y_cols[j * k + p];
    acc[p] = 0.0;
  }
  for (long i = 0; i < n; ++i) {
    const double* Li = l + i * k * k;
    const double* hi = h + i * k;
    lower_col<K>(Li, k, yj, w);
    double s = 0.0;
    for (int p = 0; p < k; ++p) s += w[p] * hi[p];
    for (int p = 0; p < k; ++p) acc[p] += s * x_rows[i * k + p];
    if (full) {
      for (int row = k - 1; row >= 0; --row) {
        double t = hi[row];
        for (int p = row + 1; p < k; ++p) t -= Li[p * k + row] * g[p];
        g[row] = t / Li[row * k + row];
      }
      const double f = resid[i * m + j];
      for (int p = 0; p < k; ++p) acc[p] += f * g[p];
    }
  }
  for (int p = 0; p < k; ++p) r_acc[j * k + p] = acc[p];
}

// --------------------------------------------------------------------------
// schur_reduce (:72-143): one thread per output block pair (j, l), sequential
// over rows i; the r_acc column j is produced by the (j, 0) thread.
// --------------------------------------------------------------------------
template <int K>
__global__ void k_schur_exact(const double* __restrict__ x_rows,
                              const double* __restrict__ y_cols, const double* __restrict__ l,
                              const double* __restrict__ h, const double* __restrict__ resid,
                              long n, long m, int k, int full, double* __restrict__ s_acc,
                              double* __restrict__ r_acc) {
  const long id = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= m * m) return;
  const long j = id / m, lc = id % m;
  const long mk = m * k;
  double yj[K], yl[K], wj[K], wl[K];
  double S[K * K], R[K];
  for (int p = 0; p < k; ++p) {
    yj[p] = y_cols[j * k + p];
    yl[p] = y_cols[lc * k + p];
    R[p] = 0.0;
    for (int q = 0; q < k; ++q) S[p * K + q] = 0.0;
  }
  double pinv[K * K], gj[K * K], gl[K * K];
  for (long i = 0; i < n; ++i) {
    const double* Li = l + i * k * k;
    const double* u = x_rows + i * k;
    const double* hi = h + i * k;
    lower_col<K>(Li, k, yj, wj);
    lower_col<K>(Li, k, yl, wl);
    if (!full) {
      if (lc == 0) {
        double s = 0.0;
        for (int p = 0; p < k; ++p) s += wj[p] * hi[p];
        for (int p = 0; p < k; ++p) R[p] += s * u[p];
      }
      double dot = 0.0;
      for (int p = 0; p < k; ++p) dot += wj[p] * wl[p];
      for (int p = 0; p < k; ++p) {
        const double up = dot * u[p];
        for (int q = 0; q < k; ++q) S[p * K + q] += up * u[q];
      }
    } else {
      // pinv = L^{-T} by back substitution on identity columns
      for (int c = 0; c < k; ++c)
        for (int row = k - 1; row >= 0; --row) {
          double s = (row == c) ? 1.0 : 0.0;
          for (int p = row + 1; p < k; ++p) s -= Li[p * k + row] * pinv[p * K + c];
          pinv[row * K + c] = s / Li[row * k + row];
        }
      const double fj = resid[i * m + j], fl = resid[i * m + lc];
      for (int p = 0; p < k; ++p)
        for (int q = 0; q < k; ++q) {
          gj[p * K + q] = u[p] * wj[q] + fj * pinv[p * K + q];
          gl[p * K + q] = u[p] * wl[q] + fl * pinv[p * K + q];
        }
      if (lc == 0) {
        for (int p = 0; p < k; ++p) {
          double s = 0.0;
          for (int q = 0; q < k; ++q) s += gj[p * K + q] * hi[q];
          R[p] += s;
        }
      }
      for (int p = 0; p < k; ++p)
        for (int q = 0; q < k; ++q) {
          double dot = 0.0;
          for (int c = 0; c < k; ++c) dot += gj[p * K + c] * gl[q * K + c];
          S[p * K + q] += dot;
        }
    }
  }
  for (int p = 0; p < k; ++p)
    for (int q = 0; q < k; ++q) s_acc[(j * k + p) * mk + lc * k + q] = S[p * K + q];
  if (lc == 0)
    for (int p = 0; p < k; ++p) r_acc[j * k + p] = R[p];
}

int kbucket(long k) { return k <= 4 ? 4 : (k <= 8 ? 8 : 16); }

}  // namespace

// ============================================================================
// C-ABI (declared in include/nmfb200.h)
// ============================================================================
#define NMFB_DISPATCH_K(k, CALL) \
  switch (kbucket(k)) {          \
    case 4: CALL(4); break;      \
    case 8: CALL(8); break;      \
    default: CALL(16); break;    \
  }

constexpr int FTAB_MAXK = 16;  // k = 12: 4096 subsets x 145 doubles = 4.8 MB; k = 16: 135 MB

static long ftab_len_k(long k) { return (k < 1 || k > FTAB_MAXK) ? 0 : (k * k + 1) << k; }

extern "C" long nmfb_nnls_ftab_len(long k) { return ftab_len_k(k); }

static int nnls_batch_impl(const double* ctc, const double* ctb, const double* btb,
                           const uint8_t* warm_passive, int warm_mode, const double* tol,
                           long max_changes, long nrhs, long k, double* x, uint8_t* passive,
                           long long* changes, double* resid2, int8_t* status,
                           uint8_t* seed_scratch, int* flag_scratch, double* ftab, long ftab_len,
                           void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (k < 1 || k > NMFB_MAX_K || nrhs < 0 || warm_mode < 0 || warm_mode > 2) return NMFB_EINVAL;
  if (nrhs == 0) return NMFB_OK;
  // factor table of every passive subset (k <= FTAB_MAXK, caller workspace); a negative
  // ftab_len means the table was already built for this ctc (nmfb_nnls_ftab_build)
  const double* ft = nullptr;
  if (ftab != nullptr && ftab_len < 0 && ftab_len_k(k) > 0 && -ftab_len >= ftab_len_k(k)) {
    ft = ftab;
  } else if (ftab != nullptr && ftab_len_k(k) > 0 && ftab_len >= ftab_len_k(k)) {
    const unsigned nsub = 1u << k;
#define FTCASE(KK)                                                                            \
  case KK: {                                                                                  \
    constexpr int WW = KK <= 4 ? 4 : (KK <= 8 ? 8 : 16);                                      \
    const unsigned per_blk = 4u * (32 / WW);                                                  \
    ++g_nmfb_launches, k_factor_table<KK, WW><<<(nsub + per_blk - 1) / per_blk, 128, 0,       \
                                                stream>>>(ctc, ftab, ftab + ((long)KK * KK << KK)); \
    break;                                                                                    \
  }
    switch (k) {
      FTCASE(1) FTCASE(2) FTCASE(3) FTCASE(4) FTCASE(5) FTCASE(6) FTCASE(7) FTCASE(8)
      FTCASE(9) FTCASE(10) FTCASE(11) FTCASE(12) FTCASE(13) FTCASE(14) FTCASE(15) FTCASE(16)
      default: break;
    }
#undef FTCASE
    ft = ftab;
  }
  const int threads = 128;
  const int blocks = (int)((nrhs + threads - 1) / threads);
  // Same bits either way.  Warp per rhs (k_nnls_warp) wins when the batch cannot
  // fill the GPU with one thread per rhs (B200: c4's 5000 Y columns 3.9x faster);
  // thread per rhs (k_nnls) wins on large batches and k >= 12 (c4's 20000 rows,
  // c5).  NMFB_NNLS_THREAD=1 / =0 forces one or the other.
  static const int force = [] {
    const char* e = getenv("NMFB_NNLS_THREAD");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  const bool thread_kernel =
      force >= 0 ? force == 1 : (ft == nullptr && !((nrhs <= 8192 && k <= 12) || nrhs <= 2048));
#define WCASE(KW, SEEDS, MODE)                                                                   \
  case KW: {                                                                                     \
    constexpr int WW = KW <= 4 ? 4 : (KW <= 8 ? 8 : 16);                                         \
    const long per_blk = 4L * (32 / WW);                                                         \
    ++g_nmfb_launches, k_nnls_warp<KW, WW><<<(unsigned)((nrhs + per_blk - 1) / per_blk), 128, 0, \
                                             stream>>>(ctc, ctb, btb, SEEDS, MODE, tol,           \
                                             max_changes, nrhs, x, passive, changes, resid2,     \
                                             status, ft);                                        \
    break;                                                                                       \
  }
#define TCASE(KT, SEEDS, MODE)                                                                  \
  case KT:                                                                                      \
    ++g_nmfb_launches, k_nnls_tab<KT><<<(unsigned)((nrhs + TabT<KT>::v - 1) / TabT<KT>::v), TabT<KT>::v, 0, stream>>>( \
        ctc, ctb, btb, SEEDS, MODE, tol, max_changes, nrhs, x, passive, changes, resid2, status, \
        ft);                                                                                    \
    break;
#define LAUNCH_NNLS(KK, SEEDS, MODE)                                                        \
  if (ft != nullptr && force < 0) {                                                         \
    switch (k) {                                                                            \
      TCASE(1, SEEDS, MODE) TCASE(2, SEEDS, MODE) TCASE(3, SEEDS, MODE) TCASE(4, SEEDS, MODE) \
      TCASE(5, SEEDS, MODE) TCASE(6, SEEDS, MODE) TCASE(7, SEEDS, MODE) TCASE(8, SEEDS, MODE) \
      TCASE(9, SEEDS, MODE) TCASE(10, SEEDS, MODE) TCASE(11, SEEDS, MODE) TCASE(12, SEEDS, MODE) \
      TCASE(13, SEEDS, MODE) TCASE(14, SEEDS, MODE) TCASE(15, SEEDS, MODE) TCASE(16, SEEDS, MODE) \
      default: return NMFB_EINVAL;                                                          \
    }                                                                                       \
  } else if (thread_kernel) {                                                               \
    ++g_nmfb_launches, k_nnls<KK><<<blocks, threads, 0, stream>>>(ctc, ctb, btb, SEEDS, MODE, tol, max_changes, \
                                             nrhs, (int)k, x, passive, changes, resid2, status); \
  } else {                                                                                  \
    switch (k) {                                                                            \
      WCASE(1, SEEDS, MODE) WCASE(2, SEEDS, MODE) WCASE(3, SEEDS, MODE) WCASE(4, SEEDS, MODE) \
      WCASE(5, SEEDS, MODE) WCASE(6, SEEDS, MODE) WCASE(7, SEEDS, MODE) WCASE(8, SEEDS, MODE) \
      WCASE(9, SEEDS, MODE) WCASE(10, SEEDS, MODE) WCASE(11, SEEDS, MODE) WCASE(12, SEEDS, MODE) \
      WCASE(13, SEEDS, MODE) WCASE(14, SEEDS, MODE) WCASE(15, SEEDS, MODE) WCASE(16, SEEDS, MODE) \
      default: return NMFB_EINVAL;                                                          \
    }                                                                                       \
  }
  if (warm_mode != 1) {
#define CALL(KK) LAUNCH_NNLS(KK, warm_passive, warm_mode)
    NMFB_DISPATCH_K(k, CALL);
#undef CALL
    NMFB_CHECK_LAUNCH();
    return NMFB_OK;
  }
  // warm_mode 1 (streaming chain, :312-315): rhs t is seeded with rhs t-1's
  // final passive set.  Speculate seeds = cold solution of t-1, then iterate
  // seeds[t] <- passive[t-1] until nothing changes.  Each pass fixes at least
  // the first inconsistent position, so the fixed point equals the sequential
  // chain exactly; on streaming data one extra pass is the norm.
  if (!seed_scratch || !flag_scratch) return NMFB_EINVAL;
#define CALL(KK) LAUNCH_NNLS(KK, warm_passive, 0)
  NMFB_DISPATCH_K(k, CALL);
#undef CALL
  NMFB_CHECK_LAUNCH();
  cudaMemsetAsync(seed_scratch, 0, (size_t)nrhs * k, stream);
  const int ub = (int)((nrhs + 255) / 256);
  for (long pass = 0; pass <= nrhs; ++pass) {
    cudaMemsetAsync(flag_scratch, 0, sizeof(int), stream);
    ++g_nmfb_launches, k_chain_update<<<ub, 256, 0, stream>>>(passive, seed_scratch, nrhs, (int)k, flag_scratch);
    int h_flag = 0;
    cudaMemcpyAsync(&h_flag, flag_scratch, sizeof(int), cudaMemcpyDeviceToHost, stream);
    if (cudaStreamSynchronize(stream) != cudaSuccess) return NMFB_ELAUNCH;
    if (!h_flag && pass > 0) break;
#define CALL(KK) LAUNCH_NNLS(KK, seed_scratch, 1)
    NMFB_DISPATCH_K(k, CALL);
#undef CALL
    NMFB_CHECK_LAUNCH();
  }
#undef LAUNCH_NNLS
#undef WCASE
#undef TCASE
  return NMFB_OK;
}

extern "C" int nmfb_surface_nnls_batch(const double* ctc, const double* ctb, const double* btb,
                                       const uint8_t* warm_passive, int warm_mode,
                                       const double* tol, long max_changes, long nrhs, long k,
                                       double* x, uint8_t* passive, long long* changes,
                                       double* resid2, int8_t* status, uint8_t* seed_scratch,
                                       int* flag_scratch, void* stream) {
  return nnls_batch_impl(ctc, ctb, btb, warm_passive, warm_mode, tol, max_changes, nrhs, k, x,
                         passive, changes, resid2, status, seed_scratch, flag_scratch, nullptr, 0,
                         stream);
}

// The subset factor table alone (for an NNLS batch launched later with -ftab_len): lets
// the host build it on a second stream while the streaming product computes ctb.
extern "C" int nmfb_nnls_ftab_build(const double* ctc, long k, double* ftab, long ftab_len,
                                    void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (ftab == nullptr || ftab_len_k(k) <= 0 || ftab_len < ftab_len_k(k)) return NMFB_EINVAL;
  const unsigned nsub = 1u << k;
#define FTCASE(KK)                                                                            \
  case KK: {                                                                                  \
    constexpr int WW = KK <= 4 ? 4 : (KK <= 8 ? 8 : 16);                                      \
    const unsigned per_blk = 4u * (32 / WW);                                                  \
    ++g_nmfb_launches, k_factor_table<KK, WW><<<(nsub + per_blk - 1) / per_blk, 128, 0,       \
                                                stream>>>(ctc, ftab, ftab + ((long)KK * KK << KK)); \
    break;                                                                                    \
  }
  switch (k) {
    FTCASE(1) FTCASE(2) FTCASE(3) FTCASE(4) FTCASE(5) FTCASE(6) FTCASE(7) FTCASE(8)
    FTCASE(9) FTCASE(10) FTCASE(11) FTCASE(12) FTCASE(13) FTCASE(14) FTCASE(15) FTCASE(16)
    default: return NMFB_EINVAL;
  }
#undef FTCASE
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_nnls_batch_ws(const double* ctc, const double* ctb, const double* btb,
                                  const uint8_t* warm_passive, int warm_mode, const double* tol,
                                  long max_changes, long nrhs, long k, double* x,
                                  uint8_t* passive, long long* changes, double* resid2,
                                  int8_t* status, uint8_t* seed_scratch, int* flag_scratch,
                                  double* ftab, long ftab_len, void* stream) {
  return nnls_batch_impl(ctc, ctb, btb, warm_passive, warm_mode, tol, max_changes, nrhs, k, x,
                         passive, changes, resid2, status, seed_scratch, flag_scratch, ftab,
                         ftab_len, stream);
}

extern "C" int nmfb_surface_block_cholesky(const double* blocks_in, long nb, long k,
                                           double* out, int* bad, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (k < 1 || k > NMFB_MAX_K || nb < 0) return NMFB_EINVAL;
  cudaMemsetAsync(out, 0, sizeof(double) * (size_t)nb * k * k, stream);
  ++g_nmfb_launches, k_set_int<<<1, 1, 0, stream>>>(bad, INT_MAX);
  if (nb == 0) return NMFB_OK;
  const int threads = 128;
  const int blocks = (int)((nb + threads - 1) / threads);
#define CALL(KK) ++g_nmfb_launches, k_block_chol<KK><<<blocks, threads, 0, stream>>>(blocks_in, nb, (int)k, out, bad)
  NMFB_DISPATCH_K(k, CALL);
#undef CALL
  ++g_nmfb_launches, k_zero_after_bad<<<nmfb_blocks(nb * k * k, 256), 256, 0, stream>>>(out, nb, (int)k, bad);
  NMFB_CHECK_LAUNCH();
  // the caller maps INT_MAX -> -1 (no failing block)
  return NMFB_OK;
}

extern "C" int nmfb_surface_block_solve_lower(const double* l, const double* b, long nb, long k,
                                              long r, int transposed, double* z, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (k < 1 || nb < 0 || r < 0) return NMFB_EINVAL;
  const long work = nb * r;
  if (work == 0) return NMFB_OK;
  const int threads = 128;
  const int blocks = (int)((work + threads - 1) / threads);
  if (transposed)
    ++g_nmfb_launches, k_block_trsm<true><<<blocks, threads, 0, stream>>>(l, b, nb, (int)k, (int)r, z);
  else
    ++g_nmfb_launches, k_block_trsm<false><<<blocks, threads, 0, stream>>>(l, b, nb, (int)k, (int)r, z);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_surface_back_substitute(const double* x_rows, const double* y_cols,
                                            const double* l, const double* h, const double* dy,
                                            const double* resid, long n, long m, long k,
                                            int full, double* dx, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (k < 1 || k > NMFB_MAX_K || n < 0 || m < 0) return NMFB_EINVAL;
  if (n == 0) return NMFB_OK;
  const int threads = 64;
  const int blocks = (int)((n + threads - 1) / threads);
#define CALL(KK)                                                                        \
  ++g_nmfb_launches, k_back_sub_exact<KK><<<blocks, threads, 0, stream>>>(x_rows, y_cols, l, h, dy, resid, n, \
                                                       m, (int)k, full, dx)
  NMFB_DISPATCH_K(k, CALL);
#undef CALL
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_surface_rhs_reduce(const double* x_rows, const double* y_cols,
                                       const double* l, const double* h, const double* resid,
                                       long n, long m, long k, int full, double* r_acc,
                                       void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (k < 1 || k > NMFB_MAX_K || n < 0 || m < 0) return NMFB_EINVAL;
  if (m == 0) return NMFB_OK;
  const int threads = 64;
  const int blocks = (int)((m + threads - 1) / threads);
#define CALL(KK)                                                                           \
  ++g_nmfb_launches, k_rhs_reduce_exact<KK><<<blocks, threads, 0, stream>>>(x_rows, y_cols, l, h, resid, n, m, \
                                                         (int)k, full, r_acc)
  NMFB_DISPATCH_K(k, CALL);
#undef CALL
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

extern "C" int nmfb_surface_schur_reduce(const double* x_rows, const double* y_cols,
                                         const double* l, const double* h, const double* resid,
                                         long n, long m, long k, int full, double* s_acc,
                                         double* r_acc, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (k < 1 || k > NMFB_MAX_K || n < 0 || m < 0) return NMFB_EINVAL;
  if (m == 0) return NMFB_OK;
  const long work = m * m;
  const int threads = 64;
  const int blocks = (int)((work + threads - 1) / threads);
#define CALL(KK)                                                                              \
  ++g_nmfb_launches, k_schur_exact<KK><<<blocks, threads, 0, stream>>>(x_rows, y_cols, l, h, resid, n, m, (int)k, \
                                                    full, s_acc, r_acc)
  NMFB_DISPATCH_K(k, CALL);
#undef CALL
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}
