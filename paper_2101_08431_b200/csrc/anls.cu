// Stage-1 (ANLS) production kernels: the HBM-streaming tall-skinny products
// around the batched NNLS (PAPER Algorithm 1).
//
//   X-update:  ctb = M Y^T      (n x k)   k_rowprod   one pass over M rows
//   Y-update:  ctb = (X^T M)^T  (m x k)   k_colprod   split-K partials over
//                                                     row stripes + fixed-order sum
//   Grams     YY^T, X^T X                 k_colprod on the factor itself
//   norms     ||M_i,:||^2, ||M_:,j||^2    once per problem (btb)
//   stats     step / norm / objective     fixed-tree block reductions
//
// All reductions use a fixed decomposition that depends only on the problem
// shape, so results are bit-reproducible run to run.  M may be float64 or
// float32 (config c5 stores M in fp32; products accumulate in fp64).
#include <cstdlib>

#include "common.cuh"
#include "nmfb200.h"
#include "tc_prod.cuh"
#include "tma_prod.cuh"

unsigned long long g_nmfb_launches = 0;

extern "C" unsigned long long nmfb_launch_count(void) { return g_nmfb_launches; }
int g_nmfb_last_cuda_error = 0;
extern "C" const char* nmfb_last_cuda_error(void) {
  return cudaGetErrorString((cudaError_t)g_nmfb_last_cuda_error);
}

namespace {

template <typename T>
struct Vec2;
template <>
struct Vec2<double> {
  using type = double2;
};
template <>
struct Vec2<float> {
  using type = float2;
};

// ---------------------------------------------------------------------------
// rowprod: out[i, :] = sum_j A[i, j] * B[j, :]   (A rows x cols, B cols x K)
// One warp per ROWS_PER_WARP rows; lanes stride the columns in pairs so each
// B row loaded into registers is reused for every row of the warp.
// Optional: tol[i] = 1e-12 * max(1, max_p |out[i,p]|)  (SPEC.md:147 default).
// ---------------------------------------------------------------------------
template <int K, int R, typename T>
__global__ void __launch_bounds__(256) k_rowprod(const T* __restrict__ A, long rows, long cols,
                                                 const double* __restrict__ B,
                                                 double* __restrict__ out,
                                                 double* __restrict__ tol, double alpha_scale) {
  const int lane = threadIdx.x & 31;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  for (long r0 = warp * R; r0 < rows; r0 += nwarps * R) {
    double acc[R][K];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int p = 0; p < K; ++p) acc[r][p] = 0.0;
    const bool pairs = (cols % 2 == 0);
    if (pairs) {
      using V = typename Vec2<T>::type;
      for (long j = 2 * lane; j < cols; j += 64) {
        double b0[K], b1[K];
#pragma unroll
        for (int p = 0; p < K; ++p) {
          b0[p] = __ldg(B + j * K + p);
          b1[p] = __ldg(B + (j + 1) * K + p);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (r0 + r < rows) {
            const V a = *reinterpret_cast<const V*>(A + (r0 + r) * cols + j);
            const double a0 = (double)a.x, a1 = (double)a.y;
#pragma unroll
            for (int p = 0; p < K; ++p) acc[r][p] = fma(a0, b0[p], fma(a1, b1[p], acc[r][p]));
          }
        }
      }
    } else {
      for (long j = lane; j < cols; j += 32) {
        double b0[K];
#pragma unroll
        for (int p = 0; p < K; ++p) b0[p] = __ldg(B + j * K + p);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (r0 + r < rows) {
            const double a0 = (double)A[(r0 + r) * cols + j];
#pragma unroll
            for (int p = 0; p < K; ++p) acc[r][p] = fma(a0, b0[p], acc[r][p]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double amax = 0.0;
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const double v = warp_sum(acc[r][p]) * alpha_scale;
        acc[r][p] = v;
        amax = fmax(amax, fabs(v));
      }
      if (lane == 0 && r0 + r < rows) {
#pragma unroll
        for (int p = 0; p < K; ++p) out[(r0 + r) * K + p] = acc[r][p];
        if (tol) tol[r0 + r] = 1e-12 * fmax(1.0, amax);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// colprod partials: part[s][j][p] = sum_{i in stripe s} A[i, j] * B[i, p]
// (A rows x cols, B rows x K).  A CTA owns a 64-column tile and one row
// stripe; B rows of the stripe are staged in shared memory and broadcast.
// ---------------------------------------------------------------------------
constexpr int CP_COLS = 64;   // columns per CTA (2 per thread, 32 threads per row group)
constexpr int CP_ROWS = 64;   // staged B rows per step

template <int K, typename T>
__global__ void __launch_bounds__(256) k_colprod_partial(const T* __restrict__ A, long rows,
                                                         long cols, const double* __restrict__ B,
                                                         long stripe, double* __restrict__ part) {
  __shared__ double sb[CP_ROWS * K];
  __shared__ double red[8][CP_COLS * K / 2 + 1];
  const int tid = threadIdx.x;
  const int cl = tid & 31;       // column pair within the tile
  const int rg = tid >> 5;       // row group (8 groups interleave the staged rows)
  const long j0 = (long)blockIdx.x * CP_COLS + 2 * cl;
  const long s = blockIdx.y;
  const long i_beg = s * stripe;
  const long i_end = min(rows, i_beg + stripe);
  double acc0[K], acc1[K];
#pragma unroll
  for (int p = 0; p < K; ++p) acc0[p] = acc1[p] = 0.0;
  for (long ib = i_beg; ib < i_end; ib += CP_ROWS) {
    const int nr = (int)min((long)CP_ROWS, i_end - ib);
    __syncthreads();
    for (int e = tid; e < nr * K; e += 256) sb[e] = B[ib * K + e];
    __syncthreads();
    for (int r = rg; r < nr; r += 8) {
      const long i = ib + r;
      double a0 = 0.0, a1 = 0.0;
      if (j0 + 1 < cols) {
        if ((cols & 1) == 0) {
          const typename Vec2<T>::type a = *reinterpret_cast<const typename Vec2<T>::type*>(A + i * cols + j0);
          a0 = (double)a.x;
          a1 = (double)a.y;
        } else {
          a0 = (double)A[i * cols + j0];
          a1 = (double)A[i * cols + j0 + 1];
        }
      } else if (j0 < cols) {
        a0 = (double)A[i * cols + j0];
      }
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const double b = sb[r * K + p];
        acc0[p] = fma(a0, b, acc0[p]);
        acc1[p] = fma(a1, b, acc1[p]);
      }
    }
  }
  // reduce the 8 row groups in a fixed order
  for (int half = 0; half < 2; ++half) {
    __syncthreads();
#pragma unroll
    for (int p = 0; p < K; ++p) red[rg][(cl)*K + p] = half == 0 ? acc0[p] : acc1[p];
    __syncthreads();
    for (int e = tid; e < 32 * K; e += 256) {
      double v = 0.0;
#pragma unroll
      for (int g = 0; g < 8; ++g) v += red[g][e];
      const int c = e / K, p = e % K;
      const long j = (long)blockIdx.x * CP_COLS + 2 * c + half;
      if (j < cols) part[(s * cols + j) * K + p] = v;
    }
  }
}


constexpr int CT_COLS = 128;  // column tile of the streaming column product

// ---------------------------------------------------------------------------
// v3 streaming products: no __syncthreads inside the streaming loops.
//
// k_rowprod_split: grid = (column chunks of CW) x (row splits).  The CTA stages
// its Y^T chunk once (transposed, conflict-free) and then every warp streams
// RW-row groups independently; per (row, chunk) partial sums go to `part`
// and a fixed-order k_sum_partials finishes (split-K over the columns).
// Accumulator type ACC: double for fp64 M; for fp32 M the per-(row, chunk)
// partial is accumulated in fp32 over CW/32 terms per lane and folded in fp64
// (c5 tolerance 1e-4; measured error ~1e-7).
// ---------------------------------------------------------------------------
template <typename T>
struct SplitCfg;
template <>
struct SplitCfg<double> {
  static constexpr int CW = 1024;
  using Y = double;
  using ACC = double;
};
template <>
struct SplitCfg<float> {
  static constexpr int CW = 2048;
  using Y = float;
  using ACC = float;
};

template <int K, int RW, typename T>
__global__ void __launch_bounds__(256, 2) k_rowprod_split(const T* __restrict__ A, long rows,
                                                          long cols, const double* __restrict__ B,
                                                          long rows_per_split,
                                                          double* __restrict__ part) {
  using C = SplitCfg<T>;
  using YT = typename C::Y;
  using ACC = typename C::ACC;
  using V = typename Vec2<T>::type;
  using VY = typename Vec2<YT>::type;
  constexpr int CW = C::CW;
  constexpr int UN = 2;  // column-pair iterations whose loads are issued together
  extern __shared__ __align__(16) unsigned char smraw[];
  YT* yT = reinterpret_cast<YT*>(smraw);  // [K][CW]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long j0 = (long)blockIdx.x * CW;
  const int cw = (int)min((long)CW, cols - j0);
  for (int e = tid; e < CW * K; e += 256) {
    const int jj = e / K, p = e - jj * K;
    yT[p * CW + jj] = (jj < cw) ? (YT)B[(j0 + jj) * K + p] : (YT)0;
  }
  __syncthreads();
  const long rb = (long)blockIdx.y * rows_per_split;
  const long re = min(rows, rb + rows_per_split);
  const bool vec = (cw == CW) && ((cols & 1) == 0);
  for (long r0 = rb + (long)warp * RW; r0 < re; r0 += 8 * RW) {
    ACC acc[RW][K];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int p = 0; p < K; ++p) acc[r][p] = (ACC)0;
    const T* arow[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) arow[r] = A + min(r0 + r, re - 1) * cols + j0;
    if (vec) {
      for (int u0 = 0; u0 < CW / 64; u0 += UN) {
        V a[UN][RW];
#pragma unroll
        for (int uu = 0; uu < UN; ++uu)
#pragma unroll
          for (int r = 0; r < RW; ++r)
            a[uu][r] = __ldg(reinterpret_cast<const V*>(arow[r] + 2 * lane + 64 * (u0 + uu)));
#pragma unroll
        for (int uu = 0; uu < UN; ++uu) {
          const int jj = 2 * lane + 64 * (u0 + uu);
#pragma unroll
          for (int p = 0; p < K; ++p) {
            const VY y = *reinterpret_cast<const VY*>(yT + p * CW + jj);
#pragma unroll
            for (int r = 0; r < RW; ++r)
              acc[r][p] = fma((ACC)a[uu][r].x, (ACC)y.x, fma((ACC)a[uu][r].y, (ACC)y.y, acc[r][p]));
          }
        }
      }
    } else {
      for (int jj = lane; jj < cw; jj += 32) {
        T a[RW];
#pragma unroll
        for (int r = 0; r < RW; ++r) a[r] = __ldg(arow[r] + jj);
#pragma unroll
        for (int p = 0; p < K; ++p) {
          const YT y = yT[p * CW + jj];
#pragma unroll
          for (int r = 0; r < RW; ++r) acc[r][p] = fma((ACC)a[r], (ACC)y, acc[r][p]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const double v = warp_sum((double)acc[r][p]);
        if (lane == 0 && r0 + r < re) part[((long)blockIdx.x * rows + r0 + r) * K + p] = v;
      }
  }
}

// k_colprod_warp: grid = (column tiles of 32*CPL) x (row splits); every warp
// streams its own interleaved rows (B row read as a warp broadcast through the
// read-only path, no shared-memory staging), one fixed-order smem reduction of
// the 8 warps at the end.
template <int K, int CPL, typename T>
__global__ void __launch_bounds__(256, 2) k_colprod_warp(const T* __restrict__ A, long rows,
                                                      long cols, const double* __restrict__ B,
                                                      long stripe, double* __restrict__ part) {
  __shared__ double red[8][32 * K + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long c0 = (long)blockIdx.x * (32 * CPL) + CPL * lane;
  const long s = blockIdx.y;
  const long i_beg = s * stripe, i_end = min(rows, i_beg + stripe);
  const bool inb = c0 + CPL <= cols;
  double acc[CPL][K];
#pragma unroll
  for (int c = 0; c < CPL; ++c)
#pragma unroll
    for (int p = 0; p < K; ++p) acc[c][p] = 0.0;
#pragma unroll 2
  for (long i = i_beg + warp; i < i_end; i += 8) {
    const T* arow = A + i * cols;
    double a[CPL];
    if (inb && (cols & 1) == 0) {
      using V = typename Vec2<T>::type;
#pragma unroll
      for (int c = 0; c < CPL; c += 2) {
        const V v = __ldg(reinterpret_cast<const V*>(arow + c0 + c));
        a[c] = (double)v.x;
        a[c + 1] = (double)v.y;
      }
    } else {
#pragma unroll
      for (int c = 0; c < CPL; ++c) a[c] = (c0 + c < cols) ? (double)arow[c0 + c] : 0.0;
    }
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const double b = __ldg(B + i * K + p);
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[c][p] = fma(a[c], b, acc[c][p]);
    }
  }
  for (int c = 0; c < CPL; ++c) {
    __syncthreads();
#pragma unroll
    for (int p = 0; p < K; ++p) red[warp][lane * K + p] = acc[c][p];
    __syncthreads();
    for (int e = tid; e < 32 * K; e += 256) {
      double v = 0.0;
#pragma unroll
      for (int g = 0; g < 8; ++g) v += red[g][e];
      const int l = e / K, p = e - l * K;
      const long j = (long)blockIdx.x * (32 * CPL) + CPL * l + c;
      if (j < cols) part[(s * cols + j) * K + p] = v;
    }
  }
}


// ---------------------------------------------------------------------------
// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) streaming products.
//
// The tall-skinny products are dense contractions over the long axis with an
// 8/16-wide output: on sm_100a the FP64 tensor pipe (DMMA) retires 256 MACs
// per warp instruction, so the SIMT issue/register pressure that kept the
// SIMT kernels latency-bound disappears and the loops become pure streams of
// 16-byte loads.  fp32 M (config c5) is widened to fp64 in registers.
//
// Fragment layout (PTX m8n8k4 .f64): lane = 4 g + t; A[g][t], B[t][g],
// C[g][2t + {0,1}].  Each lane loads a 2-wide vector of M and feeds it to two
// MMAs by permuting the contraction (row product) or the output rows (column
// product) inside each 8-column block, so every M byte is loaded once with
// 16-byte (fp64) / 8-byte (fp32) accesses.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <typename T>
__device__ __forceinline__ double2 ld2(const T* p);
template <>
__device__ __forceinline__ double2 ld2<double>(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}
template <>
__device__ __forceinline__ double2 ld2<float>(const float* p) {
  const float2 v = __ldg(reinterpret_cast<const float2*>(p));
  return make_double2((double)v.x, (double)v.y);
}

constexpr int MMA_CW = 512;  // row product: columns per chunk (multiple of 8)

// row product: part[chunk][row][p] = sum_{j in chunk} A[row][j] B[j][p]
// B fragments are pre-arranged in smem in fragment order (conflict-free).
template <int NT, typename T>
__global__ void __launch_bounds__(256, 2) k_rowprod_mma(const T* __restrict__ A, long rows,
                                                        long cols, const double* __restrict__ B,
                                                        int K, long rows_per_split,
                                                        double* __restrict__ part) {
  constexpr int RT = 2;  // 8-row tiles per warp
  extern __shared__ __align__(16) double sB[];  // [CW/8][2][NT][32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const long j0 = (long)blockIdx.x * MMA_CW;
  const int cw = (int)min((long)MMA_CW, cols - j0);
  const int npair = (cw + 7) >> 3;
  for (int e = tid; e < npair * 2 * NT * 32; e += 256) {
    const int l = e & 31, se = (e >> 5) / NT, nt = (e >> 5) % NT;
    const int sidx = se >> 1, ee = se & 1;
    const long col = j0 + 8 * sidx + 2 * (l & 3) + ee;
    const int pp = nt * 8 + (l >> 2);
    sB[e] = (col < cols && pp < K) ? B[col * K + pp] : 0.0;
  }
  __syncthreads();
  const long rb = (long)blockIdx.y * rows_per_split;
  const long re = min(rows, rb + rows_per_split);
  for (long r0 = rb + (long)warp * 8 * RT; r0 < re; r0 += 8 * 8 * RT) {
    double acc[RT][NT][2];
#pragma unroll
    for (int rt = 0; rt < RT; ++rt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[rt][nt][0] = acc[rt][nt][1] = 0.0;
    const T* arow[RT];
#pragma unroll
    for (int rt = 0; rt < RT; ++rt) arow[rt] = A + min(r0 + 8 * rt + g, re - 1) * cols + j0 + 2 * t;
    constexpr int UN = 8;
    const int nfull = cw >> 3;  // pairs whose 8 columns are all in range
    int sp = 0;
    for (; sp + UN <= nfull; sp += UN) {
      double2 a[UN][RT];
#pragma unroll
      for (int u = 0; u < UN; ++u)
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) a[u][rt] = ld2<T>(arow[rt] + 8 * (sp + u));
#pragma unroll
      for (int u = 0; u < UN; ++u)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double b0 = sB[((2 * (sp + u)) * NT + nt) * 32 + lane];
          const double b1 = sB[((2 * (sp + u) + 1) * NT + nt) * 32 + lane];
#pragma unroll
          for (int rt = 0; rt < RT; ++rt) {
            dmma(acc[rt][nt][0], acc[rt][nt][1], a[u][rt].x, b0);
            dmma(acc[rt][nt][0], acc[rt][nt][1], a[u][rt].y, b1);
          }
        }
    }
    for (; sp < npair; ++sp) {
      const bool ok = j0 + 8 * sp + 2 * t < cols;
      double2 a[RT];
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) a[rt] = ok ? ld2<T>(arow[rt] + 8 * sp) : make_double2(0.0, 0.0);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double b0 = sB[((2 * sp) * NT + nt) * 32 + lane];
        const double b1 = sB[((2 * sp + 1) * NT + nt) * 32 + lane];
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) {
          dmma(acc[rt][nt][0], acc[rt][nt][1], a[rt].x, b0);
          dmma(acc[rt][nt][0], acc[rt][nt][1], a[rt].y, b1);
        }
      }
    }
#pragma unroll
    for (int rt = 0; rt < RT; ++rt) {
      const long row = r0 + 8 * rt + g;
      if (row >= re) continue;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int pp = nt * 8 + 2 * t + c;
          if (pp < K) part[((long)blockIdx.x * rows + row) * K + pp] = acc[rt][nt][c];
        }
    }
  }
}

// column product: part[s][j][p] = sum_{i in stripe s} A[i][j] B[i][p].
// A warp owns 32 output columns (2 double2 loads per lane per 4-row k-step,
// each feeding an even- and an odd-column 8-row MMA tile).
template <int NT, typename T>
__global__ void __launch_bounds__(256, 2) k_colprod_mma(const T* __restrict__ A, long rows,
                                                        long cols, const double* __restrict__ B,
                                                        int K, long stripe,
                                                        double* __restrict__ part) {
  constexpr int RT2 = 2;  // 16-column groups per warp
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const long jw = (long)blockIdx.x * 256 + (long)warp * 32;  // warp's first column
  const long s = blockIdx.y;
  const long i_beg = s * stripe, i_end = min(rows, i_beg + stripe);
  double acc[RT2][2][NT][2];
#pragma unroll
  for (int r = 0; r < RT2; ++r)
#pragma unroll
    for (int par = 0; par < 2; ++par)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[r][par][nt][0] = acc[r][par][nt][1] = 0.0;
  bool colok[RT2];
#pragma unroll
  for (int r = 0; r < RT2; ++r) colok[r] = jw + 16 * r + 2 * g < cols;
  const bool bok0 = g < K, bok1 = 8 + g < K;
  constexpr int UN = 8;
  long i0 = i_beg;
  for (; i0 + 4 * UN <= i_end; i0 += 4 * UN) {
    double2 a[UN][RT2];
    double b[UN][NT];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const long i = i0 + 4 * u + t;
#pragma unroll
      for (int r = 0; r < RT2; ++r)
        a[u][r] = colok[r] ? ld2<T>(A + i * cols + jw + 16 * r + 2 * g) : make_double2(0.0, 0.0);
      b[u][0] = bok0 ? __ldg(B + i * K + g) : 0.0;
      if (NT > 1) b[u][NT - 1] = bok1 ? __ldg(B + i * K + 8 + g) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int r = 0; r < RT2; ++r) {
          dmma(acc[r][0][nt][0], acc[r][0][nt][1], a[u][r].x, b[u][nt]);
          dmma(acc[r][1][nt][0], acc[r][1][nt][1], a[u][r].y, b[u][nt]);
        }
  }
  for (; i0 < i_end; i0 += 4) {
    const long i = i0 + t;
    const bool rok = i < i_end;
    double2 a[RT2];
    double b[NT];
#pragma unroll
    for (int r = 0; r < RT2; ++r)
      a[r] = (rok && colok[r]) ? ld2<T>(A + i * cols + jw + 16 * r + 2 * g) : make_double2(0.0, 0.0);
    b[0] = (rok && bok0) ? __ldg(B + i * K + g) : 0.0;
    if (NT > 1) b[NT - 1] = (rok && bok1) ? __ldg(B + i * K + 8 + g) : 0.0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int r = 0; r < RT2; ++r) {
        dmma(acc[r][0][nt][0], acc[r][0][nt][1], a[r].x, b[nt]);
        dmma(acc[r][1][nt][0], acc[r][1][nt][1], a[r].y, b[nt]);
      }
  }
#pragma unroll
  for (int r = 0; r < RT2; ++r)
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      const long j = jw + 16 * r + 2 * g + par;
      if (j >= cols) continue;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int pp = nt * 8 + 2 * t + c;
          if (pp < K) part[(s * cols + j) * K + pp] = acc[r][par][nt][c];
        }
    }
}

// out[e] = scale * sum_{s < nparts} part[s][e]  (fixed order); optional per-row
// (of width K) tolerance as in k_rowprod.
template <int K>
__global__ void __launch_bounds__(256) k_sum_partials(const double* __restrict__ part, int nparts,
                                                      long len, double* __restrict__ out,
                                                      double* __restrict__ tol, double scale) {
  // element-parallel (coalesced) fixed-order sum; a CTA covers RB whole rows so
  // the per-row tolerance is finished from shared memory
  constexpr int RB = 256 / K;
  __shared__ double sv[RB * K];
  const long row0 = (long)blockIdx.x * RB;
  const long e0 = row0 * K;
  const int t = threadIdx.x;
  const long e = e0 + t;
  if (t < RB * K && e < len) {
    double v = 0.0;
    int s = 0;
    for (; s + 8 <= nparts; s += 8) {
      double w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) w[u] = part[(long)(s + u) * len + e];
#pragma unroll
      for (int u = 0; u < 8; ++u) v += w[u];
    }
    for (; s < nparts; ++s) v += part[(long)s * len + e];
    v *= scale;
    out[e] = v;
    sv[t] = v;
  }
  if (!tol) return;
  __syncthreads();
  const long r = row0 + t;
  if (t < RB && r * K < len) {
    double amax = 0.0;
#pragma unroll
    for (int p = 0; p < K; ++p) amax = fmax(amax, fabs(sv[t * K + p]));
    tol[r] = 1e-12 * fmax(1.0, amax);
  }
}

// grid for k_sum_partials over `rows` rows of width K
// short outputs (k x k Grams) over many partials: one warp per element, lanes
// stride the partials, fixed butterfly -> deterministic; all loads in flight
__global__ void __launch_bounds__(256) k_sum_partials_warp(const double* __restrict__ part,
                                                           int nparts, long len,
                                                           double* __restrict__ out,
                                                           double scale) {
  const long e = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= len) return;
  double v = 0.0;
  for (int s = lane; s < nparts; s += 32) v += part[(long)s * len + e];
  v = warp_sum(v);
  if (lane == 0) out[e] = v * scale;
}

template <int K>
inline unsigned sum_grid(long rows) {
  return (unsigned)((rows + (256 / K) - 1) / (256 / K));
}

// ---------------------------------------------------------------------------
// squared norms of rows and columns of M (btb; computed once per problem)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_row_sqnorm(const T* __restrict__ A, long rows, long cols,
                             double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  for (long i = warp; i < rows; i += nwarps) {
    double acc = 0.0;
    for (long j = lane; j < cols; j += 32) {
      const double a = (double)A[i * cols + j];
      acc = fma(a, a, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) out[i] = acc;
  }
}

template <typename T>
__global__ void k_col_sqnorm_partial(const T* __restrict__ A, long rows, long cols, long stripe,
                                     double* __restrict__ part) {
  const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long s = blockIdx.y;
  if (j >= cols) return;
  const long i_end = min(rows, (s + 1) * stripe);
  double acc = 0.0;
  for (long i = s * stripe; i < i_end; ++i) {
    const double a = (double)A[i * cols + j];
    acc = fma(a, a, acc);
  }
  part[s * cols + j] = acc;
}

// ---------------------------------------------------------------------------
// fixed-tree sums of several dot products in one pass (stage-1 statistics)
//   sums[0] = ||Xn - X||^2 + ||Yn - Y||^2, sums[1] = ||X||^2 + ||Y||^2,
//   sums[2] = sum resid2   (all partials per CTA, then one CTA finishes)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_stage1_stats_partial(
    const double* __restrict__ Xo, const double* __restrict__ Xn, long nx,
    const double* __restrict__ Yo, const double* __restrict__ Yn, long ny,
    const double* __restrict__ r2, long nr, double* __restrict__ part) {
  __shared__ double sh[32];
  double a = 0.0, b = 0.0, c = 0.0;
  const long tid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long nt = (long)gridDim.x * blockDim.x;
  for (long e = tid; e < nx; e += nt) {
    const double d = Xn[e] - Xo[e];
    a = fma(d, d, a);
    b = fma(Xo[e], Xo[e], b);
  }
  for (long e = tid; e < ny; e += nt) {
    const double d = Yn[e] - Yo[e];
    a = fma(d, d, a);
    b = fma(Yo[e], Yo[e], b);
  }
  for (long e = tid; e < nr; e += nt) c += r2[e];
  a = block_sum(a, sh);
  if (threadIdx.x == 0) part[blockIdx.x * 3 + 0] = a;
  b = block_sum(b, sh);
  if (threadIdx.x == 0) part[blockIdx.x * 3 + 1] = b;
  c = block_sum(c, sh);
  if (threadIdx.x == 0) part[blockIdx.x * 3 + 2] = c;
}

// one CTA: out[q] = sum_b part[b * nq + q] in a fixed tree
__global__ void __launch_bounds__(256) k_finish_sums(const double* __restrict__ part, int nblocks,
                                                     int nq, double* __restrict__ out) {
  __shared__ double sh[32];
  for (int q = 0; q < nq; ++q) {
    double v = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) v += part[(long)b * nq + q];
    v = block_sum(v, sh);
    if (threadIdx.x == 0) out[q] = v;
  }
}

__global__ void k_first_nonzero_i8(const int8_t* __restrict__ st, long len, int* __restrict__ out) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (long)gridDim.x * blockDim.x)
    if (st[e] != 0) atomicMin(out, (int)e);
}

constexpr int ROWPROD_R = 2;

bool rowprod_split(long rows, long cols) { return cols >= 2048 && rows >= 4096; }

template <typename T>
long rowprod_chunks(long cols) {
  return (cols + SplitCfg<T>::CW - 1) / SplitCfg<T>::CW;
}

template <int K, typename T>
int launch_rowprod(const T* A, long rows, long cols, const double* B, double* out, double* tol,
                   double scale, double* work, long work_len, cudaStream_t st) {
  static const bool f32_simt = [] {
    const char* e = getenv("NMFB_F32_SIMT");
    return e && e[0] == '1';
  }();
  const bool use_mma = !(sizeof(T) == 4 && f32_simt);
  if (rowprod_split(rows, cols) && K >= 5) {  // TMA-fed: DMMA (fp64 M) / tcgen05 tf32x3 (fp32 M)
    long nch = 0;
    const int rc = sizeof(T) == 8
                       ? tma_rowprod_f64((const double*)A, rows, cols, B, K, work, work_len, &nch, st)
                       : tc_rowprod_f32((const float*)A, rows, cols, B, K, work, work_len, &nch, st);
    if (rc == NMFB_OK) {
      if (!tol && rows * K <= 4096 && nch >= 32)
        ++g_nmfb_launches, k_sum_partials_warp<<<(unsigned)((rows * K + 7) / 8), 256, 0, st>>>(
            work, (int)nch, rows * K, out, scale);
      else
        ++g_nmfb_launches, k_sum_partials<K><<<sum_grid<K>(rows), 256, 0, st>>>(
            work, (int)nch, rows * K, out, tol, scale);
      NMFB_CHECK_LAUNCH();
      return NMFB_OK;
    }
    if (rc != NMFB_EUNSUPPORTED) return rc;
  }
  if (use_mma && rowprod_split(rows, cols) && (cols % 2 == 0) && K >= 5) {  // tensor-core streaming path
    constexpr int NT = (K + 7) / 8;
    const long nch = (cols + MMA_CW - 1) / MMA_CW;
    if (nch * rows * K > work_len) return NMFB_ENOMEM;
    const size_t smem = (size_t)MMA_CW * NT * 8 * sizeof(double);
    long nsplit = (148 * 2 * 4 + nch - 1) / nch;
    long rps = (rows + nsplit - 1) / nsplit;
    rps = ((rps + 127) / 128) * 128;
    nsplit = (rows + rps - 1) / rps;
    nmfb_smem_attr(k_rowprod_mma<NT, T>, (int)smem);
    dim3 grid((unsigned)nch, (unsigned)nsplit);
    ++g_nmfb_launches, k_rowprod_mma<NT, T><<<grid, 256, smem, st>>>(A, rows, cols, B, K, rps, work);
    if (!tol && rows * K <= 4096 && nch >= 32)
      ++g_nmfb_launches, k_sum_partials_warp<<<(unsigned)((rows * K + 7) / 8), 256, 0, st>>>(
          work, (int)nch, rows * K, out, scale);
    else
      ++g_nmfb_launches, k_sum_partials<K><<<sum_grid<K>(rows), 256, 0, st>>>(
          work, (int)nch, rows * K, out, tol, scale);
    NMFB_CHECK_LAUNCH();
    return NMFB_OK;
  }
  if (rowprod_split(rows, cols)) {  // HBM-streaming regime: split-K over column chunks
    constexpr int RW = (sizeof(T) == 4 || K <= 10) ? 4 : 2;
    constexpr int CW = SplitCfg<T>::CW;
    const long nch = rowprod_chunks<T>(cols);
    if (nch * rows * K > work_len) return NMFB_ENOMEM;
    const size_t smem = (size_t)K * CW * sizeof(typename SplitCfg<T>::Y);
    long nsplit = (148 * 2 * 4 + nch - 1) / nch;  // ~4 waves of 2 CTAs/SM: small tail
    long rps = (rows + nsplit - 1) / nsplit;
    rps = ((rps + 8 * RW - 1) / (8 * RW)) * (8 * RW);
    nsplit = (rows + rps - 1) / rps;
    nmfb_smem_attr(k_rowprod_split<K, RW, T>, (int)smem);
    dim3 grid((unsigned)nch, (unsigned)nsplit);
    ++g_nmfb_launches, k_rowprod_split<K, RW, T><<<grid, 256, smem, st>>>(A, rows, cols, B, rps, work);
    if (!tol && rows * K <= 4096 && nch >= 32)
      ++g_nmfb_launches, k_sum_partials_warp<<<(unsigned)((rows * K + 7) / 8), 256, 0, st>>>(
          work, (int)nch, rows * K, out, scale);
    else
      ++g_nmfb_launches, k_sum_partials<K><<<sum_grid<K>(rows), 256, 0, st>>>(
          work, (int)nch, rows * K, out, tol, scale);
    NMFB_CHECK_LAUNCH();
    return NMFB_OK;
  }
  const long warps = (rows + ROWPROD_R - 1) / ROWPROD_R;
  const int blocks = nmfb_blocks(warps * 32, 256, 148 * 16);
  ++g_nmfb_launches, k_rowprod<K, ROWPROD_R, T><<<blocks, 256, 0, st>>>(A, rows, cols, B, out, tol, scale);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

bool colprod_tiled(long rows, long cols) { return cols >= 1024 && rows >= 4096; }

long colprod_stripe(long rows, long cols) {
  // enough CTAs to cover the SMs several times, stripes of >= 256 rows
  const long col_tiles = (cols + (colprod_tiled(rows, cols) ? CT_COLS : CP_COLS) - 1) /
                         (colprod_tiled(rows, cols) ? CT_COLS : CP_COLS);
  long want = (148 * 8 + col_tiles - 1) / col_tiles;
  long stripe = (rows + want - 1) / want;
  if (stripe < 256) stripe = 256;
  return stripe;
}

template <int K, typename T>
int launch_colprod(const T* A, long rows, long cols, const double* B, double* out, double* tol,
                   double scale, double* work, long work_len, cudaStream_t st) {
  if (rows == 0) {
    cudaMemsetAsync(out, 0, sizeof(double) * cols * K, st);
    return NMFB_OK;
  }
  if (colprod_tiled(rows, cols) && K >= 5) {  // TMA-fed DMMA (tma_prod.cu)
    long ns = 0;
    int rc = NMFB_EUNSUPPORTED;
    if (sizeof(T) == 8)
      rc = tma_colprod_f64((const double*)A, rows, cols, B, K, work, work_len, &ns, st);
    else {
      rc = tc_colprod_f32((const float*)A, rows, cols, B, K, work, work_len, &ns, st);
      if (rc == NMFB_EUNSUPPORTED)
        rc = tma_colprod_f32((const float*)A, rows, cols, B, K, work, work_len, &ns, st);
    }
    if (rc == NMFB_OK) {
      if (!tol && cols * K <= 4096 && ns >= 32)
        ++g_nmfb_launches, k_sum_partials_warp<<<(unsigned)((cols * K + 7) / 8), 256, 0, st>>>(
            work, (int)ns, cols * K, out, scale);
      else
        ++g_nmfb_launches, k_sum_partials<K><<<sum_grid<K>(cols), 256, 0, st>>>(
            work, (int)ns, cols * K, out, tol, scale);
      NMFB_CHECK_LAUNCH();
      return NMFB_OK;
    }
    if (rc != NMFB_EUNSUPPORTED) return rc;
  }
  const long stripe = colprod_stripe(rows, cols);
  const long ns = (rows + stripe - 1) / stripe;
  if (ns * cols * K > work_len) return NMFB_ENOMEM;
  if (colprod_tiled(rows, cols) && (cols % 2 == 0) && K >= 5) {  // tensor-core streaming path
    constexpr int NT = (K + 7) / 8;
    dim3 gridm((unsigned)((cols + 255) / 256), (unsigned)ns);
    ++g_nmfb_launches, k_colprod_mma<NT, T><<<gridm, 256, 0, st>>>(A, rows, cols, B, K, stripe, work);
  } else if (colprod_tiled(rows, cols)) {
    dim3 grid((unsigned)((cols + CT_COLS - 1) / CT_COLS), (unsigned)ns);
    constexpr int CPL = K <= 10 ? 4 : 2;
    dim3 gridw((unsigned)((cols + 32 * CPL - 1) / (32 * CPL)), (unsigned)ns);
    ++g_nmfb_launches, k_colprod_warp<K, CPL, T><<<gridw, 256, 0, st>>>(A, rows, cols, B, stripe, work);
  } else {
    dim3 grid((unsigned)((cols + CP_COLS - 1) / CP_COLS), (unsigned)ns);
    ++g_nmfb_launches, k_colprod_partial<K, T><<<grid, 256, 0, st>>>(A, rows, cols, B, stripe, work);
  }
  if (!tol && cols * K <= 4096 && ns >= 32)  // Grams: warp per element
    ++g_nmfb_launches, k_sum_partials_warp<<<(unsigned)((cols * K + 7) / 8), 256, 0, st>>>(
        work, (int)ns, cols * K, out, scale);
  else
    ++g_nmfb_launches, k_sum_partials<K><<<sum_grid<K>(cols), 256, 0, st>>>(work, (int)ns, cols * K,
                                                                     out, tol, scale);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}


// ---------------------------------------------------------------------------
// Dual streaming product: ONE pass over M gives both
//     outR = M B1   (rows x K; B1: cols x K, e.g. M dY^T)
//     outC = M^T B2 (cols x K; B2: rows x K, e.g. M^T dX)
// The stage-2 Armijo pass and the incremental refresh (M Y'^T = M Y^T + a M dY^T,
// M^T X' = M^T X + a M^T dX, paper_2101_08431_b200/solver.py) need exactly these two.
//
// CTA = 256-column chunk x row split; warp w owns columns [32w, 32w+32) of the chunk
// and walks the split's rows in 8-row tiles.  For every 8 x 32 region the warp issues
// the column-product loads (lane = 4g+t: rows {t, 4+t}, columns 16h + 2g, +1) and the
// row-product loads (row g, columns 8q + 2t, +1) of the same 2 KB (the second set is
// an L1 hit), so every byte of M comes from HBM once and both products run on the FP64
// tensor pipe (DMMA m8n8k4, fragment conventions as k_rowprod_mma / k_colprod_mma).
// Column partials stay in registers for the whole split; row partials (8 tiles = 64
// rows per warp) are exchanged through shared memory and summed over the 8 warps in a
// fixed order, so the result is deterministic.  Partials: partR[chunk][row][p],
// partC[split][col][p]; the fixed-order k_sum_partials finishes both.
// ---------------------------------------------------------------------------
constexpr int DP_CW = 256;  // columns per chunk (8 warps x 32)
constexpr int DP_RB = 64;   // rows per exchange block (8 tiles of 8)

template <int NT>
struct DualTile {
  double2 ac[2][2];  // column-product layout: rows {t, 4+t}, columns 16h + 2g (+1)
  double b2[2][NT];  // B2 rows {t, 4+t}, p = 8 nt + g
};

template <int NT, typename T>
__device__ __forceinline__ void dual_load(DualTile<NT>& d, const T* __restrict__ A,
                                          const double* __restrict__ B2, long cols, int K,
                                          long rbase, long re, long jw, const bool (&cok)[2],
                                          int g, int t) {
  const double2 z2 = make_double2(0.0, 0.0);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const long i = rbase + 4 * u + t;
    const bool ok = i < re;
#pragma unroll
    for (int h = 0; h < 2; ++h)
      d.ac[u][h] = (ok && cok[h]) ? ld2<T>(A + i * cols + jw + 16 * h + 2 * g) : z2;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      d.b2[u][nt] = (ok && nt * 8 + g < K) ? __ldg(B2 + i * K + nt * 8 + g) : 0.0;
  }
}

template <int NT, typename T>
__global__ void __launch_bounds__(256, 2) k_dualprod_mma(const T* __restrict__ A, long rows,
                                                         long cols, const double* __restrict__ B1,
                                                         const double* __restrict__ B2, int K,
                                                         long rows_per_split,
                                                         double* __restrict__ partR,
                                                         double* __restrict__ partC) {
  extern __shared__ __align__(16) double dsm[];
  double* sB = dsm;                            // [CW/8][2][NT][32] B1 fragments of the chunk
  double* xb = dsm + DP_CW / 8 * 2 * NT * 32;  // [8 warps][DP_RB][NT*8] row-partial exchange
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const long j0 = (long)blockIdx.x * DP_CW;
  for (int e = tid; e < DP_CW / 8 * 2 * NT * 32; e += 256) {
    const int l = e & 31, se = (e >> 5) / NT, nt = (e >> 5) % NT;
    const int sidx = se >> 1, ee = se & 1;
    const long col = j0 + 8 * sidx + 2 * (l & 3) + ee;
    const int pp = nt * 8 + (l >> 2);
    sB[e] = (col < cols && pp < K) ? B1[col * K + pp] : 0.0;
  }
  __syncthreads();
  const long jw = j0 + 32 * warp;  // this warp's first column
  const long rb = (long)blockIdx.y * rows_per_split;
  const long re = min(rows, rb + rows_per_split);
  bool cok[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) cok[h] = jw + 16 * h + 2 * g < cols;
  double accC[2][2][NT][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int par = 0; par < 2; ++par)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) accC[h][par][nt][0] = accC[h][par][nt][1] = 0.0;
  double* xw = xb + (long)warp * DP_RB * NT * 8;
  const bool hi = (g >> 2) != 0;
  // software pipeline: the operands of tile i+1 are in flight while tile i is computed
  DualTile<NT> cur, nxt;
  const long ntile = (re - rb + 7) / 8;
  if (ntile > 0) dual_load<NT, T>(cur, A, B2, cols, K, rb, re, jw, cok, g, t);
  for (long it = 0; it < ntile; ++it) {
    const long rbase = rb + 8 * it;
    if (it + 1 < ntile) dual_load<NT, T>(nxt, A, B2, cols, K, rbase + 8, re, jw, cok, g, t);
    // column product: D(8 cols x 8 p) += M^T(8 cols x 4 rows) B2(4 rows x 8 p)
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          dmma(accC[h][0][nt][0], accC[h][0][nt][1], cur.ac[u][h].x, cur.b2[u][nt]);
          dmma(accC[h][1][nt][0], accC[h][1][nt][1], cur.ac[u][h].y, cur.b2[u][nt]);
        }
    // row product: the fragments (row g, columns 8q + 2t, +1) are permuted out of the
    // column-product registers: lane 16(q&1) + 4t + (g&3) holds them in ac[g>>2][q>>1]
    double accR[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) accR[nt][0] = accR[nt][1] = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int src = 16 * (q & 1) + 4 * t + (g & 3);
      const double x0 = __shfl_sync(0xffffffffu, cur.ac[0][q >> 1].x, src);
      const double y0 = __shfl_sync(0xffffffffu, cur.ac[0][q >> 1].y, src);
      const double x1 = __shfl_sync(0xffffffffu, cur.ac[1][q >> 1].x, src);
      const double y1 = __shfl_sync(0xffffffffu, cur.ac[1][q >> 1].y, src);
      const double ax = hi ? x1 : x0, ay = hi ? y1 : y0;
      const int grp = 4 * warp + q;  // 8-column group inside the chunk
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double b0 = sB[((2 * grp) * NT + nt) * 32 + lane];
        const double b1 = sB[((2 * grp + 1) * NT + nt) * 32 + lane];
        dmma(accR[nt][0], accR[nt][1], ax, b0);
        dmma(accR[nt][0], accR[nt][1], ay, b1);
      }
    }
    // this warp's 32-column share of the tile's row products -> exchange buffer
    const int rt = (int)(it & (DP_RB / 8 - 1));
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      *reinterpret_cast<double2*>(xw + (8 * rt + g) * NT * 8 + nt * 8 + 2 * t) =
          make_double2(accR[nt][0], accR[nt][1]);
    if (rt == DP_RB / 8 - 1 || it + 1 == ntile) {
      // fixed-order sum of the 8 warps' shares of the block's rows
      __syncthreads();
      const long r0 = rbase - 8 * rt;
      for (int e = tid; e < DP_RB * K; e += 256) {
        const int rr = e / K, pp = e - rr * K;
        const long row = r0 + rr;
        if (row >= re) continue;
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) v += xb[((long)w * DP_RB + rr) * NT * 8 + pp];
        partR[((long)blockIdx.x * rows + row) * K + pp] = v;
      }
      __syncthreads();
    }
    cur = nxt;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      const long j = jw + 16 * h + 2 * g + par;
      if (j >= cols) continue;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int pp = nt * 8 + 2 * t + c;
          if (pp < K) partC[((long)blockIdx.y * cols + j) * K + pp] = accC[h][par][nt][c];
        }
    }
}

struct DualGrid {
  long nch, nsplit, rps;
};

inline DualGrid dual_grid(long rows, long cols) {
  DualGrid d;
  d.nch = (cols + DP_CW - 1) / DP_CW;
  long nsplit = (148 * 2 * 2 + d.nch - 1) / d.nch;  // ~2 waves of 2 CTAs per SM
  long rps = (rows + nsplit - 1) / nsplit;
  rps = ((rps + DP_RB - 1) / DP_RB) * DP_RB;
  d.rps = rps;
  d.nsplit = (rows + rps - 1) / rps;
  return d;
}

template <int K, typename T>
int launch_dualprod(const T* A, long rows, long cols, const double* B1, const double* B2,
                    double* outR, double* outC, double* work, long work_len, cudaStream_t st) {
  static_assert(K >= 1 && K <= 16, "K");
  constexpr int NT = (K + 7) / 8;
  // measured on B200 (scripts/bench_dual.py): the fused pass wins for K <= 8 (c4 shape,
  // k = 4: 276 us vs 331 us for the two streams); for 8 < K <= 16 its 8-warp row-partial
  // exchange stalls the stream (357 vs 347 us at k = 10), so the two streaming products
  // (each ~70 % of HBM) run back to back instead
  if (sizeof(T) == 8 && K >= 5) {  // one TMA-fed pass (tma_prod.cu)
    const int rc = tma_dualprod_f64((const double*)A, rows, cols, B1, B2, K, outR, outC, work,
                                    work_len, st);
    if (rc == NMFB_OK) {
      const long nch = (cols + TMA_RP_CW - 1) / TMA_RP_CW;
      ++g_nmfb_launches, k_sum_partials<K><<<sum_grid<K>(rows), 256, 0, st>>>(
          work, (int)nch, rows * K, outR, nullptr, 1.0);
      NMFB_CHECK_LAUNCH();
      return NMFB_OK;
    }
    if (rc != NMFB_EUNSUPPORTED) return rc;
  }
  if (K > 8) {
    int rc = launch_rowprod<K, T>(A, rows, cols, B1, outR, nullptr, 1.0, work, work_len, st);
    if (rc != NMFB_OK) return rc;
    return launch_colprod<K, T>(A, rows, cols, B2, outC, nullptr, 1.0, work, work_len, st);
  }
  const DualGrid d = dual_grid(rows, cols);
  const long needR = d.nch * rows * K, needC = d.nsplit * cols * K;
  if (needR + needC > work_len) return NMFB_ENOMEM;
  double* partR = work;
  double* partC = work + needR;
  const size_t smem = (size_t)(DP_CW / 8 * 2 * NT * 32 + 8 * DP_RB * NT * 8) * sizeof(double);
  dim3 grid((unsigned)d.nch, (unsigned)d.nsplit);
  nmfb_smem_attr(k_dualprod_mma<NT, T>, (int)smem);
  ++g_nmfb_launches, k_dualprod_mma<NT, T><<<grid, 256, smem, st>>>(A, rows, cols, B1, B2, K,
                                                                      d.rps, partR, partC);
  ++g_nmfb_launches, k_sum_partials<K><<<sum_grid<K>(rows), 256, 0, st>>>(partR, (int)d.nch,
                                                                         rows * K, outR, nullptr, 1.0);
  ++g_nmfb_launches, k_sum_partials<K><<<sum_grid<K>(cols), 256, 0, st>>>(partC, (int)d.nsplit,
                                                                         cols * K, outC, nullptr, 1.0);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

}  // namespace

#define NMFB_K_SWITCH(k, MACRO) \
  switch (k) {                  \
    MACRO(1) MACRO(2) MACRO(3) MACRO(4) MACRO(5) MACRO(6) MACRO(7) MACRO(8) MACRO(9) MACRO(10) \
    MACRO(11) MACRO(12) MACRO(13) MACRO(14) MACRO(15) MACRO(16) \
    default: return NMFB_EINVAL; \
  }

extern "C" long nmfb_colprod_work_len(long rows, long cols, long k) {
  if (rows <= 0) return 1;
  const long stripe = colprod_stripe(rows, cols);
  long ns = (rows + stripe - 1) / stripe;
  if (colprod_tiled(rows, cols)) {
    const long nt = 2 * tma_colprod_splits(rows, cols);  // fp32: two row halves per split
    if (nt > ns) ns = nt;
  }
  return ns * cols * k;
}

extern "C" long nmfb_rowprod_work_len(long rows, long cols, long k, int a_is_f32) {
  if (!rowprod_split(rows, cols)) return 1;
  const long mma = (cols + MMA_CW - 1) / MMA_CW;
  const long simt = a_is_f32 ? rowprod_chunks<float>(cols) : rowprod_chunks<double>(cols);
  return (mma > simt ? mma : simt) * rows * k;
}

extern "C" int nmfb_rowprod(const void* A, int a_is_f32, long rows, long cols, const double* B,
                            long k, double* out, double* tol, double scale, double* work,
                            long work_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (rows < 0 || cols < 0) return NMFB_EINVAL;
  if (rows == 0) return NMFB_OK;
#define CASE(KK)                                                                               \
  case KK:                                                                                     \
    return a_is_f32 ? launch_rowprod<KK, float>((const float*)A, rows, cols, B, out, tol, scale, \
                                                work, work_len, st)                            \
                    : launch_rowprod<KK, double>((const double*)A, rows, cols, B, out, tol,    \
                                                 scale, work, work_len, st);
  NMFB_K_SWITCH(k, CASE)
#undef CASE
}

extern "C" int nmfb_colprod(const void* A, int a_is_f32, long rows, long cols, const double* B,
                            long k, double* out, double* tol, double scale, double* work,
                            long work_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (rows < 0 || cols < 0) return NMFB_EINVAL;
  if (cols == 0) return NMFB_OK;
  // k x k Grams (X^T X, Y Y^T, X^T g, Y dY^T ...): one pass of the multi-Gram kernel
  // (csrc/ipm.cu nmfb_grams, 64 rows per CTA + warp-per-entry finish) instead of the
  // column-tiled split-K product, whose 64-column tiles run 2 of 32 lanes at cols = k
  if (!a_is_f32 && cols == k && tol == nullptr && scale == 1.0 && rows > 0 &&
      nmfb_grams_work_len(rows, k, 1) <= work_len)
    return nmfb_grams(1, (const double*)A, B, out, nullptr, nullptr, nullptr, nullptr, nullptr,
                      nullptr, nullptr, nullptr, nullptr, rows, k, work, work_len, stream);
#define CASE(KK)                                                                                \
  case KK:                                                                                      \
    return a_is_f32 ? launch_colprod<KK, float>((const float*)A, rows, cols, B, out, tol, scale, \
                                                work, work_len, st)                             \
                    : launch_colprod<KK, double>((const double*)A, rows, cols, B, out, tol,     \
                                                 scale, work, work_len, st);
  NMFB_K_SWITCH(k, CASE)
#undef CASE
}

extern "C" long nmfb_dualprod_work_len(long rows, long cols, long k) {
  if (rows <= 0 || cols <= 0) return 1;
  const DualGrid d = dual_grid(rows, cols);
  long len = d.nch * rows * k + d.nsplit * cols * k;
  const long r = nmfb_rowprod_work_len(rows, cols, k, 0), r32 = nmfb_rowprod_work_len(rows, cols, k, 1);
  const long c = nmfb_colprod_work_len(rows, cols, k);
  const long tm = tma_dualprod_work_len(rows, cols, k);
  if (tm > len) len = tm;
  if (r > len) len = r;
  if (r32 > len) len = r32;
  if (c > len) len = c;
  return len;
}

extern "C" int nmfb_dualprod(const void* A, int a_is_f32, long rows, long cols, const double* B1,
                             const double* B2, long k, double* outR, double* outC, double* work,
                             long work_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (rows < 0 || cols < 0) return NMFB_EINVAL;
  if (rows == 0 || cols == 0) {
    if (rows) cudaMemsetAsync(outR, 0, sizeof(double) * rows * k, st);
    if (cols) cudaMemsetAsync(outC, 0, sizeof(double) * cols * k, st);
    return NMFB_OK;
  }
  if (cols % 2) return NMFB_EUNSUPPORTED;  // 2-wide vector loads of M rows
#define CASE(KK)                                                                                \
  case KK:                                                                                      \
    return a_is_f32 ? launch_dualprod<KK, float>((const float*)A, rows, cols, B1, B2, outR, outC, \
                                                 work, work_len, st)                            \
                    : launch_dualprod<KK, double>((const double*)A, rows, cols, B1, B2, outR,   \
                                                  outC, work, work_len, st);
  NMFB_K_SWITCH(k, CASE)
#undef CASE
}

extern "C" int nmfb_sqnorms(const void* A, int a_is_f32, long rows, long cols, double* row_out,
                            double* col_out, double* work, long work_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (rows <= 0 || cols <= 0) return NMFB_EINVAL;
  const int blocks = nmfb_blocks(rows * 32, 256, 148 * 16);
  const long stripe = colprod_stripe(rows, cols);
  const long ns = (rows + stripe - 1) / stripe;
  if (ns * cols > work_len) return NMFB_ENOMEM;
  dim3 grid((unsigned)((cols + 127) / 128), (unsigned)ns);
  if (a_is_f32) {
    ++g_nmfb_launches, k_row_sqnorm<float><<<blocks, 256, 0, st>>>((const float*)A, rows, cols, row_out);
    ++g_nmfb_launches, k_col_sqnorm_partial<float><<<grid, 128, 0, st>>>((const float*)A, rows, cols, stripe, work);
  } else {
    ++g_nmfb_launches, k_row_sqnorm<double><<<blocks, 256, 0, st>>>((const double*)A, rows, cols, row_out);
    ++g_nmfb_launches, k_col_sqnorm_partial<double><<<grid, 128, 0, st>>>((const double*)A, rows, cols, stripe, work);
  }
  ++g_nmfb_launches, k_sum_partials<1><<<sum_grid<1>(cols), 256, 0, st>>>(work, (int)ns, cols, col_out,
                                                                   nullptr, 1.0);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// stats[0] = ||dX||^2 + ||dY||^2, stats[1] = ||X_old||^2 + ||Y_old||^2, stats[2] = sum r2
extern "C" int nmfb_stage1_stats(const double* Xo, const double* Xn, long nx, const double* Yo,
                                 const double* Yn, long ny, const double* r2, long nr,
                                 double* stats, double* work, long work_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int blocks = 296;
  if (work_len < blocks * 3) return NMFB_ENOMEM;
  ++g_nmfb_launches, k_stage1_stats_partial<<<blocks, 256, 0, st>>>(Xo, Xn, nx, Yo, Yn, ny, r2, nr, work);
  ++g_nmfb_launches, k_finish_sums<<<1, 256, 0, st>>>(work, blocks, 3, stats);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

__global__ void k_row_tol(const double* __restrict__ c, long rows, int k, double* __restrict__ tol) {
  const long r = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double a = 0.0;
  for (int p = 0; p < k; ++p) a = fmax(a, fabs(c[r * k + p]));
  tol[r] = 1e-12 * fmax(1.0, a);
}

// tol[r] = 1e-12 max(1, ||c_r||_inf), for products reduced across ranks
extern "C" int nmfb_row_tol(const double* c, long rows, long k, double* tol, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (rows <= 0) return NMFB_OK;
  ++g_nmfb_launches, k_row_tol<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(c, rows, (int)k, tol);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// acc = min(acc, (tag << 40) | (i << 8) | st[i]) over the i with st[i] != 0: the first
// failing rhs of the earliest tagged batch, with its status code (fixed-sweep stage 1
// checks failures once at the end instead of synchronising every sweep)
__global__ void k_first_failure_i8(const int8_t* __restrict__ st, long len, unsigned long long tag,
                                   unsigned long long* __restrict__ acc) {
  unsigned long long best = ~0ull;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (long)gridDim.x * blockDim.x) {
    const int8_t v = st[i];
    if (v != 0) {
      const unsigned long long key = (tag << 40) | ((unsigned long long)i << 8) | (unsigned char)v;
      best = key < best ? key : best;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t < best ? t : best;
  }
  if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(acc, best);
}

extern "C" int nmfb_first_failure_i8(const int8_t* st, long len, long tag, unsigned long long* acc,
                                     void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (len <= 0) return NMFB_OK;
  if (tag < 0 || tag >= (1L << 24) || len >= (1L << 32)) return NMFB_EINVAL;
  ++g_nmfb_launches, k_first_failure_i8<<<nmfb_blocks(len, 256, 148 * 4), 256, 0, s>>>(
      st, len, (unsigned long long)tag, acc);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// *out = first index with st != 0 (0x7F7F7F7F when none); out is set, not accumulated
extern "C" int nmfb_first_nonzero_i8(const int8_t* st, long len, int* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(out, 0x7F, sizeof(int), s);
  if (len <= 0) return NMFB_OK;
  ++g_nmfb_launches, k_first_nonzero_i8<<<nmfb_blocks(len, 256, 148 * 4), 256, 0, s>>>(st, len, out);
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}
