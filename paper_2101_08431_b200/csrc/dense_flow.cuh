// Dataflow dense Cholesky and triangular solves for the mk x mk reduced (Schur) system,
// 128 < N <= 4096 (SPEC.md:68 spd_solve / PAPER.md:517-527, Eq. 12): the full-coupling
// directions of c2 / c3 factor one such matrix per inertia try.
//
// k_chol_flow: left-looking tile Cholesky (32 x 32 tiles, lower, in place, row-major) with
// NO grid barriers.  Tiles are taken in column-major order, round-robin over the co-resident
// CTAs; tile (i, j) accumulates sum_q L_iq L_jq^T on the FP64 tensor cores (DMMA m8n8k4 from
// double-buffered cp.async.cg tiles) as soon as the tiles of its two tile rows exist, then
// the diagonal tile is factored by one warp (rows in registers) and an off-diagonal tile is
// solved against L_jj by row sweeps.  Readiness is one counter per tile row (prog[i] = number
// of finished tiles of row i; tiles of a row finish in order), published with a release
// store after the tile is written and read with acquire loads -- a CTA far from the
// wavefront polls once per tile, one near it works ahead on the terms that exist.  An
// optional right-hand side rides along as one more tile row, so the forward substitution
// L z = b costs one tile per column instead of a second kernel.
//
// k_trsv_flow: forward / backward substitution with one CTA per 32-row block.  Block j
// streams its tiles of L (prefetched: they do not depend on the solution) against the solved
// blocks, which it receives by polling the solution vector itself (8-byte stores of finished
// entries over an all-ones pattern), so a hop costs one L2 write and one L2 read; the
// 32 x 32 diagonal solve is the warp sweep of dense.cu.
//
// Every spin is bounded (clock64 budget): a broken dependency raises the abort word and
// the factorization reports failure instead of hanging the device.
//
// The progress counters, reciprocal pivots and solution scratch are device globals (as
// g_coop_scratch of the panel kernel: no allocation inside CUDA-graph capture), re-armed by
// stream-ordered memsets before each launch: launches on ONE stream at a time per process.
#pragma once
#include <cooperative_groups.h>

#include "chol_blk.cuh"
#include "common.cuh"

namespace {

constexpr int FLOW_T = 256;
constexpr int FLOW_MAXT = 128;  // tile rows (N <= 4096)
constexpr int FLOW_LDM = 36;    // DMMA operand tiles (conflict-free fragment loads)
constexpr int FLOW_LDS = 33;    // row-sweep tiles (lane = row)
constexpr int FLOW_NONE = 0x7f7f7f7f;
constexpr long long FLOW_SPIN = 3000000000ll;  // ~1.5 s of SM clocks

__device__ int g_flow_prog[FLOW_MAXT + 4];  // [FLOW_MAXT + 2]: abort word
__device__ int g_flow_fail;                 // first failing pivot column (FLOW_NONE: none)
__device__ double g_flow_dinv[FLOW_MAXT * 32];
__device__ double g_flow_z[FLOW_MAXT * 32], g_flow_x[FLOW_MAXT * 32];
// optional phase stamps of the factorization (scripts/flow_phases.py): 8 globaltimer values
// per tile in global tile order; null = off
__device__ long long* g_flow_prof;
__device__ __forceinline__ void flow_stamp(long long* pr, long g, int slot) {
  if (pr != nullptr && threadIdx.x == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    pr[g * 8 + slot] = t;
  }
}

__device__ __forceinline__ int flow_ld(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void flow_st(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void flow_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// min(prog[i], prog[j]) seen by thread 0, broadcast; < 0: abort
__device__ __forceinline__ int flow_peek(int i, int j, int* sh) {
  if (threadIdx.x == 0) {
    const int a = flow_ld(g_flow_prog + i);
    const int b = (j == i) ? a : flow_ld(g_flow_prog + j);
    int v = min(a, b);
    if (flow_ld(g_flow_prog + FLOW_MAXT + 2)) v = -1;
    *sh = v;
  }
  __syncthreads();
  const int v = *sh;
  __syncthreads();
  return v;
}
// wait until min(prog[i], prog[j]) >= need (a failed pivot ends every wait: the results
// are discarded by the caller); < 0: abort
__device__ __noinline__ int flow_wait(int i, int j, int need, int* sh) {
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    int v;
    for (;;) {
      const int a = flow_ld(g_flow_prog + i);
      const int b = (j == i) ? a : flow_ld(g_flow_prog + j);
      v = min(a, b);
      if (v >= need) break;
      if (flow_ld(g_flow_prog + FLOW_MAXT + 2)) {
        v = -1;
        break;
      }
      if (flow_ld(&g_flow_fail) != FLOW_NONE) {
        v = need;
        break;
      }
      if (clock64() - t0 > FLOW_SPIN) {
        flow_st(g_flow_prog + FLOW_MAXT + 2, 1);
        v = -1;
        break;
      }
    }
    *sh = v;
  }
  __syncthreads();
  const int v = *sh;
  __syncthreads();
  return v;
}

// rows [I0, I0 + 32) x columns [32 q, 32 q + 32) of A into dst (leading dimension FLOW_LDM)
// with 16-byte cp.async.cg (L2 only: the tile was written by another SM); rows beyond N are
// zero.  rrow: the right-hand-side tile row (row 0 = rhs[32 q ..], the rest zero).
__device__ __forceinline__ void flow_issue(double* dst, const double* __restrict__ A, int N,
                                           int I0, int q, bool rrow,
                                           const double* __restrict__ rhs) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int ch = tid + h * FLOW_T;
    const int r = ch >> 4, c2 = (ch & 15) * 2;
    double* d = dst + r * FLOW_LDM + c2;
    if (rrow) {
      double2 v = make_double2(0.0, 0.0);
      if (r == 0) {
        v.x = __ldcg(rhs + q * 32 + c2);
        v.y = __ldcg(rhs + q * 32 + c2 + 1);
      }
      *reinterpret_cast<double2*>(d) = v;
    } else if (I0 + r < N) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(d)),
                   "l"(A + (long)(I0 + r) * N + q * 32 + c2)
                   : "memory");
    } else {
      *reinterpret_cast<double2*>(d) = make_double2(0.0, 0.0);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

constexpr size_t FLOW_SMEM = (size_t)(4 * 32 * FLOW_LDM + 2 * 32 * FLOW_LDS) * sizeof(double);

__global__ void __launch_bounds__(FLOW_T) k_chol_flow(double* __restrict__ A, int N,
                                                      double* __restrict__ rhs,
                                                      int* __restrict__ info, int fail_base) {
  extern __shared__ double fsm[];
  double* bA = fsm;                      // [2][32 * FLOW_LDM] tiles (i, q)
  double* bB = bA + 2 * 32 * FLOW_LDM;   // [2][32 * FLOW_LDM] tiles (j, q)
  double* tl = bB + 2 * 32 * FLOW_LDM;   // the tile being finished
  double* lj = tl + 32 * FLOW_LDS;       // L_jj for the row sweeps
  __shared__ double sdinv[32];
  __shared__ int sh_v, sfail;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  const int T = (N + 31) / 32;
  const int R = T + (rhs != nullptr ? 1 : 0);
  // strict upper triangle outside the diagonal tiles (never read by the factorization)
  for (int r = cta * (FLOW_T / 32) + wid; r < N; r += G * (FLOW_T / 32))
    for (int c = ((r >> 5) + 1) * 32 + lane; c < N; c += 32) A[(long)r * N + c] = 0.0;
  const long ntiles = (long)T * R - (long)T * (T - 1) / 2;
  long long* prof = g_flow_prof;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int br = wid >> 1, bc0 = 2 * (wid & 1);
  int j = 0;
  long base = 0;
  for (long g = cta; g < ntiles; g += G) {
    while (g >= base + (R - j)) {
      base += R - j;
      ++j;
    }
    const int i = j + (int)(g - base);
    const bool diag = (i == j), rrow = (i == T);
    const int I0 = 32 * i, J0 = 32 * j;
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
    bool dead = false;
    flow_stamp(prof, g, 0);
    // A_ij itself (untouched input) on its way while the products accumulate; identity
    // padding beyond N keeps the padded factor trivial
    double aij[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int e = tid + h * FLOW_T, r = e >> 5, c = e & 31;
      if (rrow)
        aij[h] = (r == 0 && J0 + c < N) ? __ldcg(rhs + J0 + c) : 0.0;
      else if (I0 + r < N && J0 + c < N)
        aij[h] = __ldcg(A + (long)(I0 + r) * N + J0 + c);
      else
        aij[h] = (diag && r == c) ? 1.0 : 0.0;
    }
    if (j > 0) {
      int known = flow_peek(i, j, &sh_v);
      dead = known < 0;
      int loaded = -1;
      for (int q = 0; q < j && !dead; ++q) {
        if (loaded < q) {
          if (known < q + 1) known = flow_wait(i, j, q + 1, &sh_v);
          if (known < 0) {
            dead = true;
            break;
          }
          flow_issue(bA + (q & 1) * 32 * FLOW_LDM, A, N, I0, q, rrow, rhs);
          if (!diag) flow_issue(bB + (q & 1) * 32 * FLOW_LDM, A, N, J0, q, false, rhs);
          loaded = q;
        }
        if (q + 1 < j) {
          if (known < q + 2) known = flow_peek(i, j, &sh_v);
          if (known < 0) {
            dead = true;
            break;
          }
          if (known >= q + 2) {
            flow_issue(bA + ((q + 1) & 1) * 32 * FLOW_LDM, A, N, I0, q + 1, rrow, rhs);
            if (!diag) flow_issue(bB + ((q + 1) & 1) * 32 * FLOW_LDM, A, N, J0, q + 1, false, rhs);
            loaded = q + 1;
          }
        }
        if (loaded > q) {
          if (diag)
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          else
            asm volatile("cp.async.wait_group 2;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double* pa = bA + (q & 1) * 32 * FLOW_LDM;
        const double* pb = diag ? pa : bB + (q & 1) * 32 * FLOW_LDM;
        const double* fa = pa + (8 * br + g8) * FLOW_LDM + t4;
        const double* fb0 = pb + (8 * bc0 + g8) * FLOW_LDM + t4;
        const double* fb1 = fb0 + 8 * FLOW_LDM;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const double a = fa[4 * ks];
          flow_dmma(c00, c01, a, fb0[4 * ks]);
          flow_dmma(c10, c11, a, fb1[4 * ks]);
        }
        __syncthreads();
      }
    }
    if (dead) break;
    flow_stamp(prof, g, 1);
    // tl = A_ij - sum
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int e = tid + h * FLOW_T;
      tl[(e >> 5) * FLOW_LDS + (e & 31)] = aij[h];
    }
    __syncthreads();
    {
      double* o = tl + (8 * br + g8) * FLOW_LDS + 8 * bc0 + 2 * t4;
      o[0] -= c00;
      o[1] -= c01;
      o[8] -= c10;
      o[9] -= c11;
    }
    __syncthreads();
    flow_stamp(prof, g, 2);
    if (diag) {
      const int nb = min(32, N - J0);
      if (wid == 0) {
        double a[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) a[c] = tl[lane * FLOW_LDS + c];
        int fail = -1;
        double di = 0.0;
        {
          double pv = __shfl_sync(0xffffffffu, a[0], 0);
          if (!(pv > 0.0)) fail = 0, pv = 1.0;
          FlowChol<0>::run(a, lane, pv, rsqrt(pv), fail, di, nb);
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) tl[lane * FLOW_LDS + c] = (c <= lane) ? a[c] : 0.0;
        sdinv[lane] = di;
        if (lane == 0) sfail = (fail >= 0 && fail < nb) ? fail : -1;
      }
      __syncthreads();
      flow_stamp(prof, g, 5);
      for (int e = tid; e < 1024; e += FLOW_T) {
        const int r = e >> 5, c = e & 31;
        if (r < nb && c < nb) __stcg(A + (long)(J0 + r) * N + J0 + c, tl[r * FLOW_LDS + c]);
      }
      if (tid < 32) __stcg(g_flow_dinv + J0 + tid, sdinv[tid]);
      if (tid == 0 && sfail >= 0) atomicMin(&g_flow_fail, J0 + sfail);
    } else {
      // L_jj must exist (prog[j] > j); a failed pivot or an abort ends the wait
      if (flow_wait(j, j, j + 1, &sh_v) < 0) break;
      flow_stamp(prof, g, 3);
      for (int e = tid; e < 1024; e += FLOW_T) {
        const int r = e >> 5, c = e & 31;
        // strictly lower part only: the sweeps scale by 1 / L_cc (sdinv) and must leave
        // an entry alone once its column is reached
        // and rows pre-scaled by 1 / L_rr, which takes the multiply off the sweep's chain
        lj[r * FLOW_LDS + c] = (c < r && J0 + r < N) ? __ldcg(A + (long)(J0 + r) * N + J0 + c) *
                                                           __ldcg(g_flow_dinv + J0 + r)
                                                     : 0.0;
      }
      if (tid < 32) sdinv[tid] = __ldcg(g_flow_dinv + J0 + tid);
      __syncthreads();
      flow_stamp(prof, g, 4);
      {
        const double dl = sdinv[lane];
        const double* lrow = lj + lane * FLOW_LDS;
        // x_c = a_c / L_cc - sum_{c' < c} x_c' (L[c][c'] / L_cc): lane c stops changing once
        // the sweep passes column c (the staged copy is strictly lower)
        double acc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = tl[(4 * wid + u) * FLOW_LDS + lane] * dl;
#pragma unroll 8
        for (int jj = 0; jj < 31; ++jj) {
          const double lcj = lrow[jj];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            acc[u] = fma(-lcj, __shfl_sync(0xffffffffu, acc[u], jj), acc[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) tl[(4 * wid + u) * FLOW_LDS + lane] = acc[u];
      }
      __syncthreads();
      flow_stamp(prof, g, 5);
      for (int e = tid; e < 1024; e += FLOW_T) {
        const int r = e >> 5, c = e & 31;
        if (J0 + c < N) {
          if (rrow) {
            if (r == 0) __stcg(rhs + J0 + c, tl[c]);
          } else if (I0 + r < N) {
            __stcg(A + (long)(I0 + r) * N + J0 + c, tl[r * FLOW_LDS + c]);
          }
        }
      }
    }
    __syncthreads();
    flow_stamp(prof, g, 6);
    if (tid == 0) {
      flow_st(g_flow_prog + i, j + 1);  // release: orders the CTA's writes (bar.sync above)
      flow_stamp(prof, g, 7);
      if (g == ntiles - 1) {  // the last tile depends on every diagonal tile
        const int f = flow_ld(&g_flow_fail);
        *info = (f != FLOW_NONE) ? fail_base + f : -1;
      }
    }
  }
  if (tid == 0 && flow_ld(g_flow_prog + FLOW_MAXT + 2)) *info = fail_base;  // aborted
}

// one double of the solution vector, polled until it differs from the all-ones pattern
__device__ __forceinline__ double flow_poll(const double* p, bool& dead) {
  unsigned long long bits;
  long long t0 = 0;
  int spins = 0;
  for (;;) {
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(bits) : "l"(p) : "memory");
    if (bits != 0xffffffffffffffffull) break;
    if ((++spins & 1023) == 0) {
      if (t0 == 0) t0 = clock64();
      if (flow_ld(g_flow_prog + FLOW_MAXT + 2) || clock64() - t0 > FLOW_SPIN) {
        flow_st(g_flow_prog + FLOW_MAXT + 2, 1);
        dead = true;
        bits = 0;
        break;
      }
    }
  }
  return __longlong_as_double((long long)bits);
}

// mode 1: b <- L^{-1} b; 2: b <- L^{-T} b; 3: b <- (L L^T)^{-1} b.  One CTA per 32-row block.
__global__ void __launch_bounds__(FLOW_T) k_trsv_flow(const double* __restrict__ L, int N,
                                                      double* __restrict__ b, int mode) {
  __shared__ double blk[32 * 33], bF[32 * 33], bT[32 * 33], rcp[32], red[8][33], zs[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int T = (N + 31) / 32, j = blockIdx.x, J0 = 32 * j;
  const int nc = min(32, N - J0);
  bool dead = false;
  for (int e = tid; e < 32 * 32; e += FLOW_T) {
    const int r = e >> 5, c = e & 31;
    blk[r * 33 + c] = (r < nc && c < nc) ? L[(long)(J0 + r) * N + J0 + c] : 0.0;
  }
  if (tid < 32) zs[tid] = tid < nc ? b[J0 + tid] : 0.0;
  __syncthreads();
  if (tid < 32) rcp[tid] = tid < nc ? 1.0 / blk[tid * 33 + tid] : 0.0;
  __syncthreads();
  // strictly lower block scaled by rows (forward) and, transposed, by columns (backward):
  // the sweeps are then one shuffle and one FMA per step
  for (int e = tid; e < 32 * 32; e += FLOW_T) {
    const int r = e >> 5, c = e & 31;
    const double v = c < r ? blk[r * 33 + c] : 0.0;
    bF[r * 33 + c] = v * rcp[r];
    bT[c * 33 + r] = v * rcp[c];
  }
  __syncthreads();
  if (mode & 1) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0}, cur[4], nxt[4];
    const bool rv[4] = {J0 + 4 * wid < N, J0 + 4 * wid + 1 < N, J0 + 4 * wid + 2 < N,
                        J0 + 4 * wid + 3 < N};
    const double* lr = L + (long)(J0 + 4 * wid) * N + lane;
#pragma unroll
    for (int u = 0; u < 4; ++u) nxt[u] = (j > 0 && rv[u]) ? __ldg(lr + (long)u * N) : 0.0;
    for (int i = 0; i < j; ++i) {
#pragma unroll
      for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
      if (i + 1 < j) {
#pragma unroll
        for (int u = 0; u < 4; ++u) nxt[u] = rv[u] ? __ldg(lr + (long)u * N + 32 * (i + 1)) : 0.0;
      }
      const double zi = flow_poll(g_flow_z + 32 * i + lane, dead);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = fma(cur[u], zi, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double s = warp_sum(acc[u]);
      if (lane == 0) red[0][4 * wid + u] = s;
    }
    __syncthreads();
    if (wid == 0) {
      double v = lane < nc ? (zs[lane] - red[0][lane]) * rcp[lane] : 0.0;
#pragma unroll 8
      for (int jj = 0; jj < 31; ++jj)
        v = fma(-bF[lane * 33 + jj], __shfl_sync(0xffffffffu, v, jj), v);
      v = lane < nc ? v : 0.0;
      __stcg(g_flow_z + J0 + lane, v);
      zs[lane] = v;
      if (mode == 1 && lane < nc) b[J0 + lane] = v;
    }
    __syncthreads();
  }
  if (mode & 2) {
    double acc = 0.0, cur[4], nxt[4];
    const bool cv = J0 + lane < N;
    const double* lc = L + (long)(4 * wid) * N + J0 + lane;
    auto ld_tile = [&](int i, double (&o)[4]) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        o[u] = (cv && 32 * i + 4 * wid + u < N) ? __ldg(lc + (long)(32 * i + u) * N) : 0.0;
    };
    if (j + 1 < T) ld_tile(T - 1, nxt);
    for (int i = T - 1; i > j; --i) {
#pragma unroll
      for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
      if (i - 1 > j) ld_tile(i - 1, nxt);
      const double xi = flow_poll(g_flow_x + 32 * i + lane, dead);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        acc = fma(cur[u], __shfl_sync(0xffffffffu, xi, 4 * wid + u), acc);
    }
    red[wid][lane] = acc;
    __syncthreads();
    if (wid == 0) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += red[w][lane];
      double v = lane < nc ? (zs[lane] - s) * rcp[lane] : 0.0;
#pragma unroll 8
      for (int jj = 31; jj > 0; --jj)
        v = fma(-bT[lane * 33 + jj], __shfl_sync(0xffffffffu, v, jj), v);
      v = lane < nc ? v : 0.0;
      __stcg(g_flow_x + J0 + lane, v);
      if (lane < nc) b[J0 + lane] = v;
    }
  }
  (void)dead;
}

inline bool flow_enabled() {
  static int v = [] {
    const char* e = getenv("NMFB_DENSE_FLOW");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v != 0;
}

inline bool flow_chol_eligible(const double* A, long N, const double* rhs) {
  return flow_enabled() && N > 128 && N <= 32 * FLOW_MAXT && (N % 2) == 0 &&
         ((uintptr_t)A & 15) == 0 && ((uintptr_t)rhs & 7) == 0;
}
inline bool flow_trsv_eligible(long N) { return flow_enabled() && N > 64 && N <= 32 * FLOW_MAXT; }

inline int launch_chol_flow(double* A, int N, double* rhs, int* info, int fail_base,
                            cudaStream_t st) {
  static int* prog = nullptr;
  static int* fail = nullptr;
  static int occ = 0;
  if (!prog) {
    cudaGetSymbolAddress((void**)&prog, g_flow_prog);
    cudaGetSymbolAddress((void**)&fail, g_flow_fail);
    nmfb_smem_attr(k_chol_flow, FLOW_SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_chol_flow, FLOW_T, FLOW_SMEM);
    if (occ < 1) occ = 1;
    if (occ > 2) occ = 2;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int T = (N + 31) / 32, R = T + (rhs ? 1 : 0);
  const long ntiles = (long)T * R - (long)T * (T - 1) / 2;
  int G = sms * occ;
  if (G > ntiles) G = (int)ntiles;
  cudaMemsetAsync(prog, 0, sizeof(int) * (FLOW_MAXT + 4), st);
  cudaMemsetAsync(fail, 0x7f, sizeof(int), st);
  void* args[] = {&A, &N, &rhs, &info, &fail_base};
  ++g_nmfb_launches;
  if (cudaLaunchCooperativeKernel((const void*)k_chol_flow, dim3(G), dim3(FLOW_T), args, FLOW_SMEM,
                                  st) != cudaSuccess)
    return NMFB_ELAUNCH;
  return NMFB_OK;
}

inline int launch_trsv_flow(const double* L, int N, double* b, int mode, cudaStream_t st) {
  static double* z = nullptr;
  static double* x = nullptr;
  static int* prog = nullptr;
  if (!z) {
    cudaGetSymbolAddress((void**)&z, g_flow_z);
    cudaGetSymbolAddress((void**)&x, g_flow_x);
    cudaGetSymbolAddress((void**)&prog, g_flow_prog);
  }
  const int T = (N + 31) / 32;
  if (mode & 1) cudaMemsetAsync(z, 0xff, sizeof(double) * 32 * T, st);
  if (mode & 2) cudaMemsetAsync(x, 0xff, sizeof(double) * 32 * T, st);
  cudaMemsetAsync(prog + FLOW_MAXT + 2, 0, sizeof(int), st);
  void* args[] = {(void*)&L, &N, &b, &mode};
  ++g_nmfb_launches;
  if (cudaLaunchCooperativeKernel((const void*)k_trsv_flow, dim3(T), dim3(FLOW_T), args, 0, st) !=
      cudaSuccess)
    return NMFB_ELAUNCH;
  return NMFB_OK;
}

}  // namespace
