// Single-CTA blocked Cholesky for small dense SPD matrices (N <= 800), shared by
// the rank-k^2 capacitance factors (lowrank.cu, N = k^2 <= 256) and the dense
// Gauss-Newton / full-Hessian Schur system of small problems (dense.cu).
//
// In place, lower, row-major, matrix in global memory (L2 resident), 32-column
// panels: warp 0 factors the diagonal block with its rows in registers (column
// j broadcast by shuffles), every warp solves panel rows (four in flight, one
// shuffle per column), and all threads apply the trailing update in 4 x 4
// register tiles read from a transposed shared-memory copy of the panel.
// Reciprocal pivots come from rsqrt; the strict upper triangle is zeroed.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace {

constexpr int CHOL_BLK_THREADS = 384;

inline size_t chol_blk_smem(long N) {  // diagonal block (32 x 33) + transposed panel (32 x N)
  return (size_t)(32 * 33 + 32 * (N + 2)) * sizeof(double);
}
// N <= CHOL_STAGE_MAX: the whole matrix is staged in shared memory for the factorization
// (every panel / trailing-update access hits shared memory instead of L2)
constexpr int CHOL_STAGE_MAX = 128;
inline size_t chol_blk_smem_staged(long N) {
  return chol_blk_smem(N) + (N <= CHOL_STAGE_MAX ? (size_t)N * N * sizeof(double) : 0);
}

template <int J, int C>
struct BCholUpd {
  static __device__ __forceinline__ void run(double (&a)[32], int r) {
    const double lcj = __shfl_sync(0xffffffffu, a[J], C);
    const double upd = a[C] - a[J] * lcj;
    a[C] = (r >= C) ? upd : a[C];
    BCholUpd<J, C + 1>::run(a, r);
  }
};
template <int J>
struct BCholUpd<J, 32> {
  static __device__ __forceinline__ void run(double (&)[32], int) {}
};
template <int J>
struct BCholStep {
  static __device__ __forceinline__ void run(double (&a)[32], int r, int& fail, double& di_r) {
    double pv = __shfl_sync(0xffffffffu, a[J], J);
    if (fail < 0 && !(pv > 0.0)) fail = J;
    if (fail >= 0) pv = 1.0;  // dummy pivot after a failure: no divergence, no break
    const double di = rsqrt(pv);
    a[J] = (r == J) ? pv * di : ((r > J) ? a[J] * di : a[J]);
    di_r = (r == J) ? di : di_r;
    BCholUpd<J, J + 1>::run(a, r);
    BCholStep<J + 1>::run(a, r, fail, di_r);
  }
};
template <>
struct BCholStep<32> {
  static __device__ __forceinline__ void run(double (&)[32], int, int&, double&) {}
};

// 32 x 32 diagonal factor, one warp, row r = lane in registers (the arithmetic of
// BCholStep, chol_blk.cuh, on the lower triangle) with the pivot chain software-pipelined:
// the next pivot a[J+1][J+1] - l^2 is formed from two shuffles issued before this step's
// column updates and its rsqrt is in flight while the remaining 30 - J updates issue.
template <int J>
struct FlowChol {
  static __device__ __forceinline__ void run(double (&a)[32], int r, double pv, double di,
                                             int& fail, double& di_r, int nb = 32) {
    a[J] = (r == J) ? pv * di : ((r > J) ? a[J] * di : a[J]);
    di_r = (r == J) ? di : di_r;
    if constexpr (J + 1 < 32) {
      // identity padding beyond an nb-wide block: nothing left to do.  Tested every eighth
      // column only -- a branch per column splits the unrolled chain into basic blocks and
      // the next pivot's rsqrt no longer overlaps this column's updates
      if constexpr ((J + 1) % 8 == 0) {
        if (J + 1 >= nb) {
          di_r = (r > J) ? 1.0 : di_r;
          return;
        }
      }
      const double l1 = __shfl_sync(0xffffffffu, a[J], J + 1);      // L[J+1][J]
      const double d1 = __shfl_sync(0xffffffffu, a[J + 1], J + 1);  // A[J+1][J+1] so far
      double pv1 = d1 - l1 * l1;
      if (fail < 0 && !(pv1 > 0.0)) fail = J + 1;
      if (fail >= 0) pv1 = 1.0;
      const double di1 = rsqrt(pv1);
      // column updates a[C] -= L[r][J] L[C][J], C > J: every broadcast first, then the
      // FMAs (entries above the diagonal, r < C, collect unused values)
      double l[32];
#pragma unroll
      for (int C = J + 2; C < 32; ++C) l[C] = __shfl_sync(0xffffffffu, a[J], C);
      a[J + 1] = a[J + 1] - a[J] * l1;
#pragma unroll
      for (int C = J + 2; C < 32; ++C) a[C] = a[C] - a[J] * l[C];
      FlowChol<J + 1>::run(a, r, pv1, di1, fail, di_r, nb);
    }
  }
};

// ---------------------------------------------------------------------------
// k_chol_one: N <= 128 (the k^2 x k^2 capacitance factors G and H of every c4 Gauss-Newton
// iteration, N = 100) with the whole matrix resident in shared memory, one CTA: staged by
// cp.async (every element in flight at once), per 32-column panel the diagonal block by one
// warp (FlowChol: pivot chain software-pipelined), the rows below by pre-scaled sweeps (one
// shuffle + one FMA per step, four rows per warp in flight) and the trailing update on the
// FP64 tensor cores (DMMA m8n8k4, 8 x 8 tiles of the lower triangle over the warps; leading
// dimension 132 = conflict-free fragment loads).
// ---------------------------------------------------------------------------
constexpr int CHOL_ONE_T = 256;
constexpr int CHOL_ONE_LD = 132;
inline size_t chol_one_smem() {
  return (size_t)(128 * CHOL_ONE_LD + 32 * 33 + 32) * sizeof(double);
}

__global__ void __launch_bounds__(CHOL_ONE_T) k_chol_one(double* __restrict__ Ag, int N,
                                                         int* __restrict__ info, int fail_base,
                                                         int skip_if_set, int set_ok) {
  extern __shared__ double so[];
  double* As = so;                       // [Np][LD], Np = N rounded up to 8
  double* lj = so + 128 * CHOL_ONE_LD;   // strictly lower diagonal block, rows scaled by 1/L_rr
  double* sdinv = lj + 32 * 33;
  __shared__ int sfail;
  if (skip_if_set && *info >= 0) return;
  constexpr int LD = CHOL_ONE_LD;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int Np = (N + 7) & ~7;
  // lower triangle (and the diagonal 32-blocks) in flight at once; one warp per row
  for (int r = wid; r < Np; r += CHOL_ONE_T / 32) {
    const int cend = min(Np, ((r >> 5) + 1) * 32);
    for (int cc = lane; cc < cend; cc += 32) {
      if (r < N && cc < N)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(As + r * LD + cc)),
                     "l"(Ag + (long)r * N + cc)
                     : "memory");
      else
        As[r * LD + cc] = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  if (tid == 0) sfail = -1;
  __syncthreads();
  const int g8 = lane >> 2, t4 = lane & 3;
  for (int p0 = 0; p0 < N; p0 += 32) {
    const int nb = min(32, N - p0);
    if (wid == 0) {
      double a[32];
#pragma unroll
      for (int c = 0; c < 32; ++c)
        a[c] = (lane < nb && c < nb) ? As[(p0 + lane) * LD + p0 + c] : (lane == c ? 1.0 : 0.0);
      int fail = -1;
      double di = 0.0;
      {
        double pv = __shfl_sync(0xffffffffu, a[0], 0);
        if (!(pv > 0.0)) fail = 0, pv = 1.0;
        FlowChol<0>::run(a, lane, pv, rsqrt(pv), fail, di, nb);
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const double v = (c <= lane) ? a[c] : 0.0;
        if (lane < nb && c < nb) As[(p0 + lane) * LD + p0 + c] = v;
        lj[lane * 33 + c] = (c < lane) ? v * di : 0.0;
      }
      sdinv[lane] = di;
      if (lane == 0 && fail >= 0 && fail < nb) sfail = p0 + fail;
    }
    __syncthreads();
    if (sfail >= 0) break;
    const int b0 = p0 + nb;
    if (b0 >= N) break;
    {  // rows below the block: x_c = a_c / L_cc - sum_{c' < c} x_c' L[c][c'] / L_cc
      const double dl = sdinv[lane];
      const double* lrow = lj + lane * 33;
      for (int rb = b0 + 4 * wid; rb < Np; rb += 4 * (CHOL_ONE_T / 32)) {
        double acc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = As[(rb + u) * LD + p0 + lane] * dl;
#pragma unroll 8
        for (int jj = 0; jj < 31; ++jj) {
          const double lcj = lrow[jj];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            acc[u] = fma(-lcj, __shfl_sync(0xffffffffu, acc[u], jj), acc[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) As[(rb + u) * LD + p0 + lane] = acc[u];
      }
    }
    __syncthreads();
    {  // trailing update of the lower triangle [b0, Np)^2 in 8 x 8 tiles
      const int nt = (Np - b0) >> 3;
      const int ntile = nt * (nt + 1) / 2;
      for (int tIdx = wid; tIdx < ntile; tIdx += CHOL_ONE_T / 32) {
        int ti = (int)((sqrtf(8.0f * (float)tIdx + 1.0f) - 1.0f) * 0.5f);
        while ((ti + 1) * (ti + 2) / 2 <= tIdx) ++ti;
        while (ti * (ti + 1) / 2 > tIdx) --ti;
        const int tj = tIdx - ti * (ti + 1) / 2;
        const int r0 = b0 + 8 * ti, c0 = b0 + 8 * tj;
        const double* fa = As + (r0 + g8) * LD + p0 + t4;
        const double* fb = As + (c0 + g8) * LD + p0 + t4;
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(d0), "+d"(d1)
              : "d"(fa[4 * ks]), "d"(fb[4 * ks]));
        double* o = As + (r0 + g8) * LD + c0 + 2 * t4;
        o[0] -= d0;
        o[1] -= d1;
      }
    }
    __syncthreads();
  }
  const int f = sfail;
  for (int r = wid; r < N; r += CHOL_ONE_T / 32)
    for (int cc = lane; cc < N; cc += 32) Ag[(long)r * N + cc] = cc <= r ? As[r * LD + cc] : 0.0;
  if (tid == 0) {
    if (f >= 0)
      *info = fail_base + f;
    else if (set_ok)
      *info = -1;
  }
}

// warp 0: the nb x nb diagonal block at (p0, p0), padded to 32 with identity
__device__ __noinline__ void chol_diag_block(double* A, long N, int p0, int nb, double* sd,
                                             double* dinv, int* sfail) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c)
    a[c] = (lane < nb && c < nb) ? A[(long)(p0 + lane) * N + p0 + c] : (lane == c ? 1.0 : 0.0);
  int fail = -1;
  double di = 0.0;
  BCholStep<0>::run(a, lane, fail, di);
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const double v = (c <= lane) ? a[c] : 0.0;
    if (lane < nb && c < nb) A[(long)(p0 + lane) * N + p0 + c] = v;
    sd[lane * 33 + c] = v;
  }
  dinv[lane] = di;
  if (lane == 0 && fail >= 0 && fail < nb) *sfail = p0 + fail;
}

// info: failure -> fail_base + pivot column; success -> -1 when set_ok.
// skip_if_set: do nothing if *info >= 0 on entry (an earlier factorization failed).
__global__ void __launch_bounds__(CHOL_BLK_THREADS) k_chol_blk(double* __restrict__ Ag, int N,
                                                               int* __restrict__ info,
                                                               int fail_base, int skip_if_set,
                                                               int set_ok) {
  extern __shared__ double smc[];
  double* sd = smc;              // diagonal block, 32 x 33
  double* pT = smc + 32 * 33;    // transposed panel: pT[i * LDT + (row - p0)]
  __shared__ double dinv[32];
  __shared__ int sfail;
  if (skip_if_set && *info >= 0) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nwarp = (int)(blockDim.x >> 5);
  const int LDT = N + 2;
  const bool staged = N <= CHOL_STAGE_MAX;
  double* A = Ag;
  if (staged) {  // the matrix into shared memory, all loads in flight
    A = pT + 32 * LDT;
    for (int e = tid; e < N * N; e += blockDim.x) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(A + e)),
                     "l"(Ag + e)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  }
  if (tid == 0) sfail = -1;
  __syncthreads();
  for (int p0 = 0; p0 < N; p0 += 32) {
    const int nb = min(32, N - p0);
    if (wid == 0) chol_diag_block(A, N, p0, nb, sd, dinv, &sfail);
    __syncthreads();
    if (sfail >= 0) break;
    // panel rows: L_rp = A_rp L_pp^{-T}, four rows per warp per column sweep
    {
      const double dl = dinv[lane];
      const double* lrow = sd + lane * 33;
      for (int rb = p0 + nb + 4 * wid; rb < N; rb += 4 * nwarp) {
        double acc[4], x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc[u] = (lane < nb && rb + u < N) ? A[(long)(rb + u) * N + p0 + lane] : 0.0;
          x[u] = 0.0;
        }
        for (int j = 0; j < nb; ++j) {
          const double lcj = (lane < nb) ? lrow[j] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double xj = __shfl_sync(0xffffffffu, acc[u] * dl, j);
            const double nacc = acc[u] - lcj * xj;
            x[u] = (lane == j) ? xj : x[u];
            acc[u] = (lane > j) ? nacc : acc[u];
          }
        }
        if (lane < nb) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (rb + u < N) {
              A[(long)(rb + u) * N + p0 + lane] = x[u];
              pT[lane * LDT + (rb + u - p0)] = x[u];
            }
        }
      }
    }
    __syncthreads();
    // trailing update of the lower triangle [b0, N)^2: row-major tile order, so a
    // warp shares its row tile (broadcast) and streams consecutive column tiles
    const int b0 = p0 + nb, n2 = N - b0;
    if (n2 > 0) {
      const int tt = (n2 + 3) >> 2;
      const int ntile = tt * (tt + 1) / 2;
      for (int t = tid; t < ntile; t += blockDim.x) {
        int ti = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
        while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
        while (ti * (ti + 1) / 2 > t) --ti;
        const int tj = t - ti * (ti + 1) / 2;
        const int r0 = b0 + 4 * ti, c0 = b0 + 4 * tj;
        const double* pr = pT + (r0 - p0);
        const double* pc = pT + (c0 - p0);
        double acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
        for (int i = 0; i < nb; ++i) {
          double ar[4], bc[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            ar[u] = pr[i * LDT + u];
            bc[u] = pc[i * LDT + u];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = fma(ar[u], bc[v], acc[u][v]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int r = r0 + u, c = c0 + v;
            if (r < N && c <= r) A[(long)r * N + c] -= acc[u][v];
          }
      }
    }
    __syncthreads();
  }
  const int f = sfail;
  if (staged) {
    __syncthreads();
    for (int e = tid; e < N * N; e += blockDim.x) {
      const int r = e / N, c = e - (e / N) * N;
      Ag[e] = c <= r ? A[e] : 0.0;
    }
  } else {
    for (int r = wid; r < N; r += nwarp)
      for (int c = r + 1 + lane; c < N; c += 32) A[(long)r * N + c] = 0.0;
  }
  if (tid == 0) {
    if (f >= 0)
      *info = fail_base + f;
    else if (set_ok)
      *info = -1;
  }
}


// ---------------------------------------------------------------------------
// Multi-CTA variant (cooperative launch) for 128 < N <= 4096: per 32-column panel
// the panel rows are solved by every CTA's warps (four rows per warp in flight)
// and the trailing update is split into 32 x 32 tiles over the CTAs; the CTA that
// owns the next diagonal tile factors it right after updating it, so a panel costs
// two grid barriers.  Same numerics as k_chol_blk's diagonal block and panel solve;
// the trailing update sums the panel's 32 products before subtracting.
// ---------------------------------------------------------------------------
constexpr int CHOL_COOP_THREADS = 256;

// 32 reciprocal pivots + the failure word of the cooperative factorization (a
// device global, so a launch inside CUDA-graph capture needs no allocation)
__device__ double g_coop_scratch[64];

__device__ __forceinline__ void coop_sync() {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
  }
  cooperative_groups::this_grid().sync();
}

__global__ void __launch_bounds__(CHOL_COOP_THREADS) k_chol_coop(double* __restrict__ A, int N,
                                                                 int* __restrict__ info,
                                                                 int fail_base, int set_ok,
                                                                 int skip_if_set) {
  double* dinv_g = g_coop_scratch;
  int* fail_g = reinterpret_cast<int*>(g_coop_scratch + 32);
  __shared__ double sd[32 * 33];   // diagonal block L_pp (row-major) for the panel solve
  __shared__ double pr[32][33], pc[32][33];
  __shared__ double dinv[32];
  __shared__ int sfail;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  constexpr int NWC = CHOL_COOP_THREADS / 32;
  if (skip_if_set && *info >= 0) return;  // every CTA sees the same word: uniform exit
  if (cta == 0 && tid == 0) *fail_g = -1;
  // first diagonal block
  if (cta == 0) {
    if (tid == 0) sfail = -1;
    __syncthreads();
    if (wid == 0) chol_diag_block(A, N, 0, min(32, N), sd, dinv, &sfail);
    __syncthreads();
    if (tid < 32) dinv_g[tid] = dinv[tid];
    if (tid == 0) *fail_g = sfail;
  }
  coop_sync();
  for (int p0 = 0; p0 < N; p0 += 32) {
    const int nb = min(32, N - p0);
    if (__ldcg(fail_g) >= 0) break;  // uniform
    // stage L_pp and 1/L_jj
    for (int e = tid; e < 32 * 32; e += CHOL_COOP_THREADS) {
      const int r = e >> 5, c = e & 31;
      sd[r * 33 + c] = (r < nb && c < nb) ? __ldcg(A + (long)(p0 + r) * N + p0 + c) : 0.0;
    }
    if (tid < 32) dinv[tid] = __ldcg(dinv_g + tid);
    __syncthreads();
    // panel rows [p0 + nb, N): warps across all CTAs, four rows each in flight
    {
      const double dl = dinv[lane];
      const double* lrow = sd + lane * 33;
      const long gw = (long)cta * NWC + wid, nwt = (long)G * NWC;
      for (long rb = p0 + nb + 4 * gw; rb < N; rb += 4 * nwt) {
        double acc[4], x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc[u] = (lane < nb && rb + u < N) ? __ldcg(A + (rb + u) * N + p0 + lane) : 0.0;
          x[u] = 0.0;
        }
        for (int j = 0; j < nb; ++j) {
          const double lcj = (lane < nb) ? lrow[j] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double xj = __shfl_sync(0xffffffffu, acc[u] * dl, j);
            const double nacc = acc[u] - lcj * xj;
            x[u] = (lane == j) ? xj : x[u];
            acc[u] = (lane > j) ? nacc : acc[u];
          }
        }
        if (lane < nb) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (rb + u < N) __stcg(A + (rb + u) * N + p0 + lane, x[u]);
        }
      }
    }
    coop_sync();
    // trailing update in 32 x 32 tiles (lower triangle of [b0, N)^2); tile 0 is the
    // next diagonal block: its owner (CTA 0) factors it right away
    const int b0 = p0 + nb, n2 = N - b0;
    if (n2 > 0) {
      const int T = (n2 + 31) / 32;
      const int ntile = T * (T + 1) / 2;
      for (int t = cta; t < ntile; t += G) {
        int ti = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
        while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
        while (ti * (ti + 1) / 2 > t) --ti;
        const int tj = t - ti * (ti + 1) / 2;
        const int R0 = b0 + 32 * ti, C0 = b0 + 32 * tj;
        __syncthreads();
        for (int e = tid; e < 32 * 32; e += CHOL_COOP_THREADS) {
          const int r = e >> 5, i = e & 31;
          pr[r][i] = (R0 + r < N && i < nb) ? __ldcg(A + (long)(R0 + r) * N + p0 + i) : 0.0;
          pc[r][i] = (C0 + r < N && i < nb) ? __ldcg(A + (long)(C0 + r) * N + p0 + i) : 0.0;
        }
        __syncthreads();
        const int ty = tid >> 4, tx = tid & 15;
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 8
        for (int i = 0; i < 32; ++i) {
          const double a0 = pr[2 * ty][i], a1 = pr[2 * ty + 1][i];
          const double c0v = pc[2 * tx][i], c1v = pc[2 * tx + 1][i];
          acc[0][0] = fma(a0, c0v, acc[0][0]);
          acc[0][1] = fma(a0, c1v, acc[0][1]);
          acc[1][0] = fma(a1, c0v, acc[1][0]);
          acc[1][1] = fma(a1, c1v, acc[1][1]);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int r = R0 + 2 * ty + u, c = C0 + 2 * tx + v;
            if (r < N && c <= r) {  // written by another CTA last panel: read through L2
              const long q = (long)r * N + c;
              A[q] = __ldcg(A + q) - acc[u][v];
            }
          }
        if (t == 0) {  // next diagonal block: factor it now (CTA 0)
          __syncthreads();
          __threadfence_block();
          if (tid == 0) sfail = -1;
          __syncthreads();
          if (wid == 0) chol_diag_block(A, N, b0, min(32, N - b0), sd, dinv, &sfail);
          __syncthreads();
          if (tid < 32) dinv_g[tid] = dinv[tid];
          if (tid == 0 && sfail >= 0) *fail_g = sfail;
        }
      }
    }
    coop_sync();
  }
  // zero the strict upper triangle, report
  const long gt = (long)cta * CHOL_COOP_THREADS + tid, nt = (long)G * CHOL_COOP_THREADS;
  for (long e = gt; e < (long)N * N; e += nt) {
    const int r = (int)(e / N), c = (int)(e % N);
    if (c > r) A[e] = 0.0;
  }
  if (cta == 0 && tid == 0) {
    const int f = __ldcg(fail_g);
    if (f >= 0)
      *info = fail_base + f;
    else if (set_ok)
      *info = -1;
  }
}

// launch helper: one CTA for N <= 128, cooperative panels above
inline int launch_chol(double* A, int N, int* info, int fail_base, int skip_if_set, int set_ok,
                       cudaStream_t st) {
  static const bool one = [] {
    const char* e = getenv("NMFB_CHOL_ONE");
    return !(e && e[0] == '0');
  }();
  if (N <= 128 && one) {
    const size_t sm = chol_one_smem();
    nmfb_smem_attr(k_chol_one, sm);
    ++g_nmfb_launches, k_chol_one<<<1, CHOL_ONE_T, sm, st>>>(A, N, info, fail_base, skip_if_set,
                                                              set_ok);
    return NMFB_OK;
  }
  if (N <= 128) {
    const size_t sm = chol_blk_smem_staged(N);
    nmfb_smem_attr(k_chol_blk, sm);
    ++g_nmfb_launches, k_chol_blk<<<1, CHOL_BLK_THREADS, sm, st>>>(A, N, info, fail_base,
                                                                   skip_if_set, set_ok);
    return NMFB_OK;
  }
  const int T = (N - 32 + 31) / 32;
  int G = T * (T + 1) / 2;
  if (G > 148) G = 148;
  if (G < 8) G = 8;
  void* args[] = {&A, &N, &info, &fail_base, &set_ok, &skip_if_set};
  ++g_nmfb_launches;
  if (cudaLaunchCooperativeKernel((const void*)k_chol_coop, dim3(G), dim3(CHOL_COOP_THREADS), args,
                                  0, st) != cudaSuccess)
    return NMFB_ELAUNCH;
  return NMFB_OK;
}

}  // namespace
