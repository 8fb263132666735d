// Dense SPD factor/solve of the mk x mk reduced (Schur) system
// spd_solve / PAPER.md:517-527 (Eq. 12).  Right-looking blocked Cholesky,
// lower, in place, row-major (lda = N), fp64:
//
//   for each 64-wide panel:  potrf of the diagonal tile in shared memory
//                            trsm of the tiles below (one CTA per 64 rows)
//                            syrk/gemm of the trailing lower triangle
//                            (64x64 tiles, 4x4 register micro-tiles)
//
// A non-positive pivot stores its global column in *info (first one wins,
// later kernels exit early); the host maps it to NotPositiveDefinite /
// SchurNotPositiveDefinite.  No pivoting, no silent regularisation.
// Triangular solves: a single-CTA blocked solver for small N, multi-CTA
// (diagonal solve + GEMV sweep) for large N.
#include <cooperative_groups.h>

#include "common.cuh"
#include "nmfb200.h"
#include "chol_blk.cuh"

namespace {

constexpr int NB = 64;

__global__ void __launch_bounds__(256) k_potrf_tile(double* __restrict__ A, long N, long k0,
                                                   int nb, int* __restrict__ info) {
  if (*info >= 0) return;
  __shared__ double t[NB][NB + 1];
  __shared__ int bad;
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += 256) {
    const int r = e / nb, c = e % nb;
    t[r][c] = (c <= r) ? A[(k0 + r) * N + k0 + c] : 0.0;
  }
  if (tid == 0) bad = -1;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (tid == 0) {
      const double d = t[j][j];
      if (!(d > 0.0)) {
        bad = j;
      } else {
        t[j][j] = sqrt(d);
      }
    }
    __syncthreads();
    if (bad >= 0) break;
    const double djj = t[j][j];
    for (int r = j + 1 + tid; r < nb; r += 256) t[r][j] /= djj;
    __syncthreads();
    // trailing update of the tile: t[r][c] -= t[r][j] * t[c][j], j < c <= r
    for (int e = tid; e < (nb - j - 1) * (nb - j - 1); e += 256) {
      const int r = j + 1 + e / (nb - j - 1), c = j + 1 + e % (nb - j - 1);
      if (c <= r) t[r][c] -= t[r][j] * t[c][j];
    }
    __syncthreads();
  }
  if (bad >= 0) {
    if (tid == 0) atomicCAS(info, -1, (int)(k0 + bad));
    return;
  }
  for (int e = tid; e < nb * nb; e += 256) {
    const int r = e / nb, c = e % nb;
    if (c <= r) A[(k0 + r) * N + k0 + c] = t[r][c];
  }
}

// rows [k0+nb, N) of the panel: L21 = A21 * L11^{-T}; one CTA per 64 rows
__global__ void __launch_bounds__(256) k_trsm_panel(double* __restrict__ A, long N, long k0,
                                                    int nb, const int* __restrict__ info) {
  if (*info >= 0) return;
  extern __shared__ double dsm[];
  double(*l11)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm);
  double(*x)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + NB * (NB + 1));
  const int tid = threadIdx.x;
  const long r0 = k0 + nb + (long)blockIdx.x * NB;
  const int nr = (int)min((long)NB, N - r0);
  for (int e = tid; e < nb * nb; e += 256) {
    const int r = e / nb, c = e % nb;
    l11[r][c] = (c <= r) ? A[(k0 + r) * N + k0 + c] : 0.0;
  }
  for (int e = tid; e < nr * nb; e += 256) {
    const int r = e / nb, c = e % nb;
    x[r][c] = A[(r0 + r) * N + k0 + c];
  }
  __syncthreads();
  // column-oriented forward substitution on every row at once: x L11^T = a
  for (int j = 0; j < nb; ++j) {
    const double d = l11[j][j];
    for (int r = tid; r < nr; r += 256) x[r][j] /= d;
    __syncthreads();
    for (int e = tid; e < nr * (nb - j - 1); e += 256) {
      const int r = e / (nb - j - 1), c = j + 1 + e % (nb - j - 1);
      x[r][c] -= x[r][j] * l11[c][j];
    }
    __syncthreads();
  }
  for (int e = tid; e < nr * nb; e += 256) {
    const int r = e / nb, c = e % nb;
    A[(r0 + r) * N + k0 + c] = x[r][c];
  }
}

// trailing lower triangle: A[i, j] -= sum_p L[i, k0+p] L[j, k0+p] for tiles bi >= bj
__global__ void __launch_bounds__(256) k_syrk_trailing(double* __restrict__ A, long N, long k0,
                                                       int nb, const int* __restrict__ info) {
  if (*info >= 0) return;
  extern __shared__ double dsm[];
  double(*li)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm);
  double(*lj)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + NB * (NB + 1));
  // map linear block id -> (bi, bj), bi >= bj, over the trailing tiles
  const long t = blockIdx.x;
  long bi = (long)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (bi * (bi + 1) / 2 > t) --bi;
  while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
  const long bj = t - bi * (bi + 1) / 2;
  const long base = k0 + nb;
  const long i0 = base + bi * NB, j0 = base + bj * NB;
  const int ni = (int)min((long)NB, N - i0), nj = (int)min((long)NB, N - j0);
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * nb; e += 256) {
    const int r = e / nb, c = e % nb;
    li[r][c] = r < ni ? A[(i0 + r) * N + k0 + c] : 0.0;
    lj[r][c] = r < nj ? A[(j0 + r) * N + k0 + c] : 0.0;
  }
  __syncthreads();
  const int tr = (tid >> 4) * 4, tc = (tid & 15) * 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int p = 0; p < nb; ++p) {
    double va[4], vb[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      va[a] = li[tr + a][p];
      vb[a] = lj[tc + a][p];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(va[a], vb[b], acc[a][b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = tr + a, c = tc + b;
      if (r < ni && c < nj && (i0 + r) >= (j0 + c)) A[(i0 + r) * N + j0 + c] -= acc[a][b];
    }
}

// ---------------------------------------------------------------------------
// triangular solves with the factor (lower, row-major): forward L z = b,
// backward L^T x = z, in place on b.  Single-CTA blocked variant.
// ---------------------------------------------------------------------------
// one warp solves the 32 x 32 diagonal block at c0 (nc <= 32 active columns):
// the block is staged in shared memory with reciprocal pivots first, so the
// column sweep is one shuffle + one FMA per step (no global loads or divides
// on the dependency chain).  v (lane = row) holds b on entry, z on exit.
__device__ __forceinline__ void trsv_load_blk(const double* __restrict__ L, long N, long c0,
                                              int nc, double* blk, int t0, int nt) {
  for (int e = t0; e < 32 * 32; e += nt) {
    const int r = e >> 5, c = e & 31;
    blk[r * 33 + c] = (r < nc && c < nc) ? L[(c0 + r) * N + c0 + c] : 0.0;
  }
}

// one warp solves the 32 x 32 diagonal block staged in blk (nc <= 32 active
// columns) with reciprocal pivots, so the column sweep is one shuffle + one FMA per
// step (no global loads or divides on the dependency chain).  v (lane = row) holds
// b on entry, z on exit.
__device__ __forceinline__ double trsv_diag_solve(int nc, int trans, double v, const double* blk,
                                                  double* rcp) {
  const int lane = threadIdx.x & 31;
  rcp[lane] = lane < nc ? 1.0 / blk[lane * 33 + lane] : 0.0;
  __syncwarp();
  const double rl = rcp[lane];
  if (!trans) {
    for (int j = 0; j < nc; ++j) {
      const double zj = __shfl_sync(0xffffffffu, v * rl, j);
      const double nv = v - blk[lane * 33 + j] * zj;
      v = (lane == j) ? zj : ((lane > j && lane < nc) ? nv : v);
    }
  } else {
    for (int j = nc - 1; j >= 0; --j) {
      const double zj = __shfl_sync(0xffffffffu, v * rl, j);
      const double nv = v - blk[j * 33 + lane] * zj;
      v = (lane == j) ? zj : (lane < j ? nv : v);
    }
  }
  return v;
}

__device__ __forceinline__ double trsv_diag_warp(const double* __restrict__ L, long N, long c0,
                                                 int nc, int trans, double v, double* blk,
                                                 double* rcp) {
  trsv_load_blk(L, N, c0, nc, blk, threadIdx.x & 31, 32);
  __syncwarp();
  return trsv_diag_solve(nc, trans, v, blk, rcp);
}

}  // namespace
#include "dense_flow.cuh"  // dataflow Cholesky / solves (uses trsv_diag_solve above)
namespace {

constexpr int TRSV_T = 256;  // 1024 threads spilled the 32-entry row to local memory

// Single-CTA blocked solve.  Per 32-column block: warp 0 solves the diagonal block
// (staged in shared memory one step ahead) while warps 1..7 load the next diagonal
// block and the L entries of their update rows into registers -- neither depends on
// the solution -- so after one barrier the update is 32 FMAs from registers.  The
// L2 round trips overlap the serial diagonal sweep instead of following it.
// The right-hand side lives in shared memory for the whole solve (dynamic, N doubles).
__global__ void __launch_bounds__(TRSV_T) k_trsv_single(const double* __restrict__ L, long N,
                                                      double* __restrict__ bg, int trans) {
  __shared__ double zb[32], sblk[2][32 * 33], srcp[32];
  extern __shared__ double b[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (long e = tid; e < N; e += TRSV_T) b[e] = bg[e];
  const long nblk = (N + 31) / 32;
  constexpr int UT = TRSV_T - 32;  // update threads (warps 1..7)
  {
    const long blk0 = trans ? (nblk - 1) : 0;
    trsv_load_blk(L, N, blk0 * 32, (int)min(32L, N - blk0 * 32), sblk[0], tid, TRSV_T);
  }
  __syncthreads();
  for (long bb = 0; bb < nblk; ++bb) {
    const long blk = trans ? (nblk - 1 - bb) : bb;
    const long c0 = blk * 32;
    const int nc = (int)min(32L, N - c0);
    const int cur = (int)(bb & 1);
    double l[32];
    long r_first = -1;  // the first update row (or column) of this thread, prefetched
    if (wid == 0) {
      double v = lane < nc ? b[c0 + lane] : 0.0;
      v = trsv_diag_solve(nc, trans, v, sblk[cur], srcp);
      if (lane < nc) b[c0 + lane] = v;
      zb[lane] = lane < nc ? v : 0.0;
    } else {
      if (bb + 1 < nblk) {
        const long nb = trans ? (blk - 1) : (blk + 1);
        trsv_load_blk(L, N, nb * 32, (int)min(32L, N - nb * 32), sblk[cur ^ 1], tid - 32, UT);
      }
      if (!trans) {
        const long r = c0 + nc + (tid - 32);
        if (r < N) {
          r_first = r;
#pragma unroll
          for (int c = 0; c < 32; ++c) l[c] = c < nc ? L[r * N + c0 + c] : 0.0;
        }
      } else {
        const long c = tid - 32;
        if (c < c0) {
          r_first = c;
#pragma unroll
          for (int r = 0; r < 32; ++r) l[r] = r < nc ? L[(c0 + r) * N + c] : 0.0;
        }
      }
    }
    __syncthreads();
    if (r_first >= 0) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 32; ++c) s = fma(l[c], zb[c], s);
      b[r_first] -= s;
    }
    // remaining update rows / columns (N > 256 + 32): all threads, loaded after the solve
    if (!trans) {
      for (long r = c0 + nc + UT + tid; r < N; r += TRSV_T) {
        double lr[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) lr[c] = c < nc ? L[r * N + c0 + c] : 0.0;
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < 32; ++c) s = fma(lr[c], zb[c], s);
        b[r] -= s;
      }
    } else {
      for (long c = UT + tid; c < c0; c += TRSV_T) {
        double lr[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) lr[r] = r < nc ? L[(c0 + r) * N + c] : 0.0;
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < 32; ++r) s = fma(lr[r], zb[r], s);
        b[c] -= s;
      }
    }
    __syncthreads();
  }
  for (long e = tid; e < N; e += TRSV_T) bg[e] = b[e];
}

// Cooperative solve for large N (mk up to 4096; c3's dense Schur fallbacks): ONE grid
// barrier per 32-column block.  Round b: CTA 0 applies z_b to block b+1's rows and
// solves block b+1's diagonal (a ~2 us chain) while CTAs 1..G-1 apply z_b to every
// row beyond block b+1 (all of L streams through the SMs once per solve); the
// transposed solve runs the same schedule on columns from the end.  The right-hand
// side stays in global memory (L2), read with ld.global.cg after each barrier.
__global__ void __launch_bounds__(256) k_trsv_coop(const double* __restrict__ L, long N,
                                                   double* __restrict__ b, int trans) {
  __shared__ double sblk[32 * 33], srcp[32], zs[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  const long nblk = (N + 31) / 32;
  auto blk_of = [&](long bb) { return trans ? (nblk - 1 - bb) : bb; };
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  if (cta == 0 && wid == 0) {  // block 0 (forward) / the last block (transposed)
    const long c0 = blk_of(0) * 32;
    const int nc = (int)min(32L, N - c0);
    double v = lane < nc ? b[c0 + lane] : 0.0;
    v = trsv_diag_warp(L, N, c0, nc, trans, v, sblk, srcp);
    if (lane < nc) b[c0 + lane] = v;
  }
  grid.sync();
  for (long bb = 0; bb + 1 < nblk; ++bb) {
    const long p0 = blk_of(bb) * 32;  // solved block
    const int np = (int)min(32L, N - p0);
    const long n0 = blk_of(bb + 1) * 32;  // next block
    const int nn = (int)min(32L, N - n0);
    if (tid < 32) zs[tid] = tid < np ? __ldcg(b + p0 + tid) : 0.0;
    __syncthreads();
    if (cta == 0) {
      if (wid == 0) {
        double v = lane < nn ? __ldcg(b + n0 + lane) : 0.0;
        double s = 0.0;
        if (lane < nn) {
          if (!trans) {
#pragma unroll 8
            for (int c = 0; c < np; ++c) s = fma(L[(n0 + lane) * N + p0 + c], zs[c], s);
          } else {
#pragma unroll 8
            for (int r = 0; r < np; ++r) s = fma(L[(p0 + r) * N + n0 + lane], zs[r], s);
          }
        }
        v -= s;
        v = trsv_diag_warp(L, N, n0, nn, trans, v, sblk, srcp);
        if (lane < nn) b[n0 + lane] = v;
      }
    } else {
      const long gt = (long)(cta - 1) * 256 + tid, gn = (long)(G - 1) * 256;
      if (!trans) {
        for (long r = n0 + nn + gt; r < N; r += gn) {
          double l[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) l[c] = c < np ? L[r * N + p0 + c] : 0.0;
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < 32; ++c) s = fma(l[c], zs[c], s);
          b[r] = __ldcg(b + r) - s;
        }
      } else {
        for (long c = gt; c < n0; c += gn) {
          double l[32];
#pragma unroll
          for (int r = 0; r < 32; ++r) l[r] = r < np ? L[(p0 + r) * N + c] : 0.0;
          double s = 0.0;
#pragma unroll
          for (int r = 0; r < 32; ++r) s = fma(l[r], zs[r], s);
          b[c] = __ldcg(b + c) - s;
        }
      }
    }
    grid.sync();
  }
}

// multi-CTA pieces for large N
__global__ void k_trsv_diag(const double* __restrict__ L, long N, double* __restrict__ b, long c0,
                            int nc, int trans) {
  __shared__ double sblk[32 * 33], srcp[32];
  const int lane = threadIdx.x;
  double v = lane < nc ? b[c0 + lane] : 0.0;
  v = trsv_diag_warp(L, N, c0, nc, trans, v, sblk, srcp);
  if (lane < nc) b[c0 + lane] = v;
}

__global__ void k_trsv_update(const double* __restrict__ L, long N, double* __restrict__ b,
                              long c0, int nc, int trans) {
  const int lane = threadIdx.x & 31;
  if (!trans) {
    const long r = c0 + nc + (((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (r >= N) return;
    double s = lane < nc ? L[r * N + c0 + lane] * b[c0 + lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) b[r] -= s;
  } else {
    const long c = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= c0) return;
    double s = 0.0;
    for (int r = 0; r < nc; ++r) s = fma(L[(c0 + r) * N + c], b[c0 + r], s);
    b[c] -= s;
  }
}

}  // namespace

constexpr size_t kTwoTiles = 2 * NB * (NB + 1) * sizeof(double);

extern "C" int nmfb_dense_solve_mode(const double* L, long N, double* b, int mode, void* stream);

extern "C" int nmfb_dense_cholesky(double* A, long N, int* info, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (N <= 0) return NMFB_EINVAL;
  static bool attr = false;
  if (!attr) {
    nmfb_smem_attr(k_trsm_panel, (int)kTwoTiles);
    nmfb_smem_attr(k_syrk_trailing, (int)kTwoTiles);
    attr = true;
  }
  if (flow_chol_eligible(A, N, nullptr)) {  // csrc/dense_flow.cuh: tile dataflow, DMMA
    const int rc = launch_chol_flow(A, (int)N, nullptr, info, 0, st);
    if (rc != NMFB_OK) return rc;
    NMFB_CHECK_LAUNCH();
    return NMFB_OK;
  }
  if (N <= 4096) {  // csrc/chol_blk.cuh: one CTA up to 128, cooperative panels above
    const int rc = launch_chol(A, (int)N, info, 0, 0, 1, st);
    if (rc != NMFB_OK) return rc;
    NMFB_CHECK_LAUNCH();
    return NMFB_OK;
  }
  cudaMemsetAsync(info, 0xFF, sizeof(int), st);  // -1: no failing pivot
  for (long k0 = 0; k0 < N; k0 += NB) {
    const int nb = (int)min((long)NB, N - k0);
    ++g_nmfb_launches, k_potrf_tile<<<1, 256, 0, st>>>(A, N, k0, nb, info);
    const long rest = N - k0 - nb;
    if (rest > 0) {
      const long tiles = (rest + NB - 1) / NB;
      ++g_nmfb_launches, k_trsm_panel<<<(unsigned)tiles, 256, kTwoTiles, st>>>(A, N, k0, nb, info);
      ++g_nmfb_launches, k_syrk_trailing<<<(unsigned)(tiles * (tiles + 1) / 2), 256, kTwoTiles, st>>>(A, N, k0, nb, info);
    }
  }
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// Factor A = L L^T in place and overwrite b with L^{-1} b in the same launch (the right-hand
// side rides along as one more tile row); finish with nmfb_dense_solve_back.  Falls back to
// the separate factorization + forward solve outside the dataflow kernel's range.
extern "C" int nmfb_dense_cholesky_rhs(double* A, long N, double* b, int* info, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (N <= 0 || b == nullptr) return NMFB_EINVAL;
  if (flow_chol_eligible(A, N, b)) {
    const int rc = launch_chol_flow(A, (int)N, b, info, 0, st);
    if (rc != NMFB_OK) return rc;
    NMFB_CHECK_LAUNCH();
    return NMFB_OK;
  }
  const int rc = nmfb_dense_cholesky(A, N, info, stream);
  if (rc != NMFB_OK) return rc;
  return nmfb_dense_solve_mode(A, N, b, 1, stream);
}

// profiling aid: 8 globaltimer stamps per tile of the dataflow factorization (null: off)
extern "C" int nmfb_flow_profile(long long* buf) {
  return cudaMemcpyToSymbol(g_flow_prof, &buf, sizeof(buf)) == cudaSuccess ? NMFB_OK : NMFB_ELAUNCH;
}

// b <- L^{-T} b (the second half of the solve after nmfb_dense_cholesky_rhs)
extern "C" int nmfb_dense_solve_back(const double* L, long N, double* b, void* stream) {
  return nmfb_dense_solve_mode(L, N, b, 2, stream);
}

// mode 1: b <- L^{-1} b, 2: b <- L^{-T} b, 3: both (the full solve)
extern "C" int nmfb_dense_solve_mode(const double* L, long N, double* b, int mode, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (N <= 0 || mode < 1 || mode > 3) return NMFB_EINVAL;
  if (flow_trsv_eligible(N)) {
    const int rc = launch_trsv_flow(L, (int)N, b, mode, st);
    if (rc != NMFB_OK) return rc;
    NMFB_CHECK_LAUNCH();
    return NMFB_OK;
  }
  if (N > 640 && N <= 65536) {
    int G = (int)((N - 32 + 255) / 256) + 1;
    if (G > 148) G = 148;
    if (G < 2) G = 2;
    for (int trans = 0; trans < 2; ++trans) {
      if (!(mode & (1 << trans))) continue;
      void* args[] = {(void*)&L, &N, &b, &trans};
      ++g_nmfb_launches;
      if (cudaLaunchCooperativeKernel((const void*)k_trsv_coop, dim3(G), dim3(256), args, 0, st) !=
          cudaSuccess)
        return NMFB_ELAUNCH;
    }
    NMFB_CHECK_LAUNCH();
    return NMFB_OK;
  }
  if (N > 4096) return mode == 3 ? nmfb_dense_solve(L, N, b, stream) : NMFB_EUNSUPPORTED;
  const size_t sm = (size_t)N * sizeof(double);
  nmfb_smem_attr(k_trsv_single, (int)(4096 * sizeof(double)));
  if (mode & 1) ++g_nmfb_launches, k_trsv_single<<<1, TRSV_T, sm, st>>>(L, N, b, 0);
  if (mode & 2) ++g_nmfb_launches, k_trsv_single<<<1, TRSV_T, sm, st>>>(L, N, b, 1);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// in-place solve (L L^T) x = b using the factor from nmfb_dense_cholesky
extern "C" int nmfb_dense_solve(const double* L, long N, double* b, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (N <= 0) return NMFB_EINVAL;
  if (flow_trsv_eligible(N)) return nmfb_dense_solve_mode(L, N, b, 3, stream);
  if (N > 640 && N <= 65536) {  // cooperative: one grid barrier per block
    int G = (int)((N - 32 + 255) / 256) + 1;
    if (G > 148) G = 148;
    if (G < 2) G = 2;
    for (int trans = 0; trans < 2; ++trans) {
      void* args[] = {(void*)&L, &N, &b, &trans};
      ++g_nmfb_launches;
      if (cudaLaunchCooperativeKernel((const void*)k_trsv_coop, dim3(G), dim3(256), args, 0, st) !=
          cudaSuccess)
        return NMFB_ELAUNCH;
    }
    NMFB_CHECK_LAUNCH();
    return NMFB_OK;
  }
  if (N <= 4096) {
    const size_t sm = (size_t)N * sizeof(double);
    static bool attr = false;
    if (!attr) {
      nmfb_smem_attr(k_trsv_single, (int)(4096 * sizeof(double)));
      attr = true;
    }
    ++g_nmfb_launches, k_trsv_single<<<1, TRSV_T, sm, st>>>(L, N, b, 0);
    ++g_nmfb_launches, k_trsv_single<<<1, TRSV_T, sm, st>>>(L, N, b, 1);
  } else {
    for (long c0 = 0; c0 < N; c0 += 32) {
      const int nc = (int)min(32L, N - c0);
      ++g_nmfb_launches, k_trsv_diag<<<1, 32, 0, st>>>(L, N, b, c0, nc, 0);
      const long rest = N - c0 - nc;
      if (rest > 0) ++g_nmfb_launches, k_trsv_update<<<(unsigned)((rest * 32 + 255) / 256), 256, 0, st>>>(L, N, b, c0, nc, 0);
    }
    const long nblk = (N + 31) / 32;
    for (long bb = nblk - 1; bb >= 0; --bb) {
      const long c0 = bb * 32;
      const int nc = (int)min(32L, N - c0);
      ++g_nmfb_launches, k_trsv_diag<<<1, 32, 0, st>>>(L, N, b, c0, nc, 1);
      if (c0 > 0) ++g_nmfb_launches, k_trsv_update<<<(unsigned)((c0 + 255) / 256), 256, 0, st>>>(L, N, b, c0, nc, 1);
    }
  }
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}
