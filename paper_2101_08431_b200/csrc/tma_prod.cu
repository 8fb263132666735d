// TMA-fed streaming products over an fp64 M (configs c2-c4 and the fp64 streaming
// session): ctb = M Y^T of the X-update and X^T M of the Y-update,
// and the same two products in the residual-free stage 2 (M dY^T, M^T dX).
//
// Design (B200, sm_100a):
//   * persistent grid, one CTA per SM; a static, contiguous range of work items per CTA
//     (the decomposition depends only on the shape, so the split-K partials and their
//     fixed-order sum are bit-reproducible run to run);
//   * one producer warp issues cp.async.bulk.tensor (TMA) loads of 128-byte-wide boxes
//     of M, 128B-swizzled, into a 4-stage shared-memory ring with full/empty mbarriers
//     (128 KB in flight per SM: enough to cover HBM latency at the full rate without
//     any register staging);
//   * eight consumer warps read the fragments of FP64 tensor-core MMAs (DMMA m8n8k4)
//     straight from the ring.  The swizzle (16-byte chunk c of 128-byte line r lives at
//     c ^ (r & 7)) together with the lane -> row map below makes every 16-byte fragment
//     load conflict-free: row product: lanes 4g..4g+3 read line sigma(g) = (g >> 1) |
//     ((g & 1) << 2), so the two rows of a quarter-warp differ in bit 2; column product:
//     the contraction rows of one MMA are the even (then the odd) lines 2t, so the eight
//     lanes of a quarter-warp hit chunks g ^ 2t, all distinct.
//
// The row product accumulates each row's chunk in the same order as k_rowprod_mma
// (csrc/anls.cu: ascending 8-column groups, the even then the odd column of each lane's
// pair), so its partials are bit-identical to the register-direct kernel's.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "tma_prod.cuh"

namespace {

constexpr int NCW = 8;                  // consumer warps
constexpr int NTHREADS = (NCW + 1) * 32;  // + one producer warp
constexpr int STAGES = 4;
constexpr int STAGE_BYTES = 32 * 1024;

// ---- PTX helpers ------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(su32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ double2 lds128(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(su32(p)));
  return v;
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ring / barrier carving of the dynamic shared memory (1024-byte aligned for the swizzle)
struct Carve {
  double* ring;
  uint64_t* full;
  uint64_t* empty;
  double* extra;
};
__device__ __forceinline__ Carve carve(uint8_t* raw) {
  const uint32_t base = su32(raw);
  const uint32_t pad = ((base + 1023u) & ~1023u) - base;
  uint8_t* p = raw + pad;
  Carve c;
  c.ring = reinterpret_cast<double*>(p);
  c.full = reinterpret_cast<uint64_t*>(p + STAGES * STAGE_BYTES);
  c.empty = c.full + STAGES;
  c.extra = reinterpret_cast<double*>(c.empty + STAGES);
  return c;
}

__device__ __forceinline__ void init_barriers(const Carve& c) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&c.full[s], 1);
      mbar_init(&c.empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

// ---- row product ------------------------------------------------------------
// item = (chunk of TMA_RP_CW columns, band of RP_BR rows), chunk-major.  A stage is
// RP_SBOX boxes of 16 columns x RP_BR rows; consumer warp w owns rows [16 w, 16 w + 16)
// of the band (two 8-row MMA tiles) and accumulates them over the chunk.
//
// NT = 8-wide output tiles on the tensor pipe.  TL > 0 (K = 8 + TL, 9 <= K <= 12): the
// first 8 outputs go to DMMA and the last TL to the FP64 SIMT pipe (DFMA), a separate
// pipe on sm_100a, instead of a second, mostly-padding DMMA tile: at K = 10 a quarter
// of the products' tensor work disappears (the kernels run close to the DMMA limit).
// The TL columns of every lane's row partials are summed over the four lanes of a
// quad (fixed shuffle tree) when the band finishes.
constexpr int RP_RT = 2;
constexpr int RP_BR = NCW * 8 * RP_RT;       // 128 rows per band
constexpr int RP_BOX = RP_BR * 16;           // doubles per box (16 KB)
constexpr int RP_SBOX = STAGE_BYTES / (RP_BOX * 8);  // boxes per stage (2)
constexpr int RP_NGRP = TMA_RP_CW / 8;       // 8-column groups per chunk

template <int TL>
struct TailPitch {
  static constexpr int v = TL <= 2 ? 2 : 4;  // doubles per (group, t, ee) tail record
};

__device__ __forceinline__ double quad_sum(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

template <int NT, int TL>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_rowprod_tma(const __grid_constant__ CUtensorMap map, long rows, long cols,
                  const double* __restrict__ B, int K, long nitems, long nbands,
                  double* __restrict__ part) {
  static_assert(TL == 0 || NT == 1, "DFMA tail only after one DMMA tile");
  constexpr int TP = TailPitch<TL>::v;
  extern __shared__ uint8_t smem_raw[];
  const Carve c = carve(smem_raw);
  double* sB = c.extra;  // [RP_NGRP][2][NT][32] fragment order (as k_rowprod_mma)
  double* sT = sB + RP_NGRP * 2 * NT * 32;  // [RP_NGRP][4 t][2 ee][TP]: B[8q+2t+ee][8+j]
  init_barriers(c);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long i_beg = (long)blockIdx.x * nitems / gridDim.x;
  const long i_end = (long)(blockIdx.x + 1) * nitems / gridDim.x;

  if (warp == NCW) {  // ===== TMA producer =====
    if (lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      for (long it = i_beg; it < i_end; ++it) {
        const long chunk = it / nbands, band = it - chunk * nbands;
        const long j0 = chunk * TMA_RP_CW;
        const int cw = (int)min((long)TMA_RP_CW, cols - j0);
        const int nbox = (cw + 15) >> 4;
        for (int b0 = 0; b0 < nbox; b0 += RP_SBOX) {
          const int nb = min(RP_SBOX, nbox - b0);
          mbar_wait(&c.empty[stage], phase ^ 1u);
          mbar_expect_tx(&c.full[stage], (unsigned)(nb * RP_BOX * 8));
          for (int b = 0; b < nb; ++b)
            tma_load_2d(c.ring + ((size_t)stage * RP_SBOX + b) * RP_BOX, &map, &c.full[stage],
                        (int)(j0 + 16 * (b0 + b)), (int)(band * RP_BR));
          if (++stage == STAGES) stage = 0, phase ^= 1u;
        }
      }
    }
    return;
  }

  // ===== consumers =====
  const int g = lane >> 2, t = lane & 3;
  const int sig = (g >> 1) | ((g & 1) << 2);  // line of this lane's A-fragment row
  int stage = 0;
  unsigned phase = 0;
  long cur_chunk = -1;
  for (long it = i_beg; it < i_end; ++it) {
    const long chunk = it / nbands, band = it - chunk * nbands;
    const long j0 = chunk * TMA_RP_CW;
    const int cw = (int)min((long)TMA_RP_CW, cols - j0);
    const int nbox = (cw + 15) >> 4;
    if (chunk != cur_chunk) {  // stage this chunk's B fragments (zero beyond cols / K)
      consumers_sync();
      const int ngrp = 2 * nbox;  // 8-column groups
      // asynchronous 8-byte gathers (cp.async, zero-filled out of range): every element
      // of the chunk is in flight at once instead of one dependent load per trip
      for (int e = threadIdx.x; e < ngrp * 2 * NT * 32; e += NCW * 32) {
        const int l = e & 31, se = (e >> 5) / NT, nt = (e >> 5) % NT;
        const int sidx = se >> 1, ee = se & 1;
        const long col = j0 + 8 * sidx + 2 * (l & 3) + ee;
        const int pp = nt * 8 + (l >> 2);
        const bool ok = col < cols && pp < K;
        cp_async8(sB + e, ok ? B + col * K + pp : B, ok ? 8 : 0);
      }
      if (TL > 0)
        for (int e = threadIdx.x; e < ngrp * 8 * TP; e += NCW * 32) {
          const int j = e % TP, rec = e / TP;  // rec = (q * 4 + t) * 2 + ee
          const long col = j0 + 8 * (rec >> 3) + 2 * ((rec >> 1) & 3) + (rec & 1);
          const bool ok = col < cols && j < TL;
          cp_async8(sT + e, ok ? B + col * K + 8 + j : B, ok ? 8 : 0);
        }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      consumers_sync();
      cur_chunk = chunk;
    }
    double acc[RP_RT][NT][2];
    double tacc[RP_RT][TL > 0 ? TL : 1];
#pragma unroll
    for (int rt = 0; rt < RP_RT; ++rt) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[rt][nt][0] = acc[rt][nt][1] = 0.0;
#pragma unroll
      for (int j = 0; j < (TL > 0 ? TL : 1); ++j) tacc[rt][j] = 0.0;
    }
    for (int b0 = 0; b0 < nbox; b0 += RP_SBOX) {
      const int nb = min(RP_SBOX, nbox - b0);
      mbar_wait(&c.full[stage], phase);
#pragma unroll
      for (int b = 0; b < RP_SBOX; ++b) {
        if (b < nb) {
          const double* box = c.ring + ((size_t)stage * RP_SBOX + b) * RP_BOX;
          double2 a[2][RP_RT];
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
#pragma unroll
            for (int rt = 0; rt < RP_RT; ++rt) {
              const int r = 8 * (RP_RT * warp + rt) + sig;
              a[kk][rt] = lds128(box + r * 16 + (((4 * kk + t) ^ sig) << 1));
            }
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int q = 2 * (b0 + b) + kk;  // 8-column group within the chunk
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const double bx = sB[((2 * q) * NT + nt) * 32 + lane];
              const double by = sB[((2 * q + 1) * NT + nt) * 32 + lane];
#pragma unroll
              for (int rt = 0; rt < RP_RT; ++rt) dmma(acc[rt][nt][0], acc[rt][nt][1], a[kk][rt].x, bx);
#pragma unroll
              for (int rt = 0; rt < RP_RT; ++rt) dmma(acc[rt][nt][0], acc[rt][nt][1], a[kk][rt].y, by);
            }
            if (TL > 0) {
              const double* tr = sT + ((q * 4 + t) * 2) * TP;
              double tx[TP], ty[TP];
#pragma unroll
              for (int j = 0; j < TP; j += 2) {
                const double2 u = lds128(tr + j), v = lds128(tr + TP + j);
                tx[j] = u.x, tx[j + 1] = u.y, ty[j] = v.x, ty[j + 1] = v.y;
              }
#pragma unroll
              for (int rt = 0; rt < RP_RT; ++rt)
#pragma unroll
                for (int j = 0; j < (TL > 0 ? TL : 1); ++j)
                  tacc[rt][j] = fma(a[kk][rt].y, ty[j], fma(a[kk][rt].x, tx[j], tacc[rt][j]));
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.empty[stage]);
      if (++stage == STAGES) stage = 0, phase ^= 1u;
    }
#pragma unroll
    for (int rt = 0; rt < RP_RT; ++rt) {
      const long row = band * RP_BR + 8 * (RP_RT * warp + rt) + sig;
      double tsum[TL > 0 ? TL : 1];
#pragma unroll
      for (int j = 0; j < (TL > 0 ? TL : 1); ++j) tsum[j] = TL > 0 ? quad_sum(tacc[rt][j]) : 0.0;
      if (row >= rows) continue;
      double* dst = part + (chunk * rows + row) * K;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int pp = nt * 8 + 2 * t + e;
          if (pp < K) dst[pp] = acc[rt][nt][e];
        }
      if (TL > 0 && t == 0)
#pragma unroll
        for (int j = 0; j < (TL > 0 ? TL : 1); ++j) dst[8 + j] = tsum[j];
    }
  }
}

// ---- column product ---------------------------------------------------------
// item = (chunk of 128 columns, split of CP_BR-aligned rows), chunk-major.  A stage is
// 8 boxes of 16 columns x 32 rows plus the stage's 32 rows of B (one bulk copy); consumer
// warp w owns box w (16 columns of the chunk) and accumulates them over the split.  NT /
// TL as in the row product (the TL tail columns summed over the quad at the item end).
constexpr int CP_CW = 128;
constexpr int CP_BR = 32;
constexpr int CP_BOX = CP_BR * 16;  // doubles per box (4 KB)

template <int NT, int TL, bool FULL>
__device__ __forceinline__ void colprod_stage(const double* __restrict__ box,
                                              const double* __restrict__ xs,
                                              const double* __restrict__ B, int K, long r0,
                                              long re, int g, int t, double (&acc)[2][NT][2],
                                              double (&tacc)[2][TL > 0 ? TL : 1]) {
#pragma unroll
  for (int blk = 0; blk < CP_BR / 8; ++blk) {
    const int ra = 8 * blk + 2 * t, rbb = ra + 1;  // lines 2t, 2t + 1 of the 8-row block
    const double2 a0 = lds128(box + ra * 16 + ((g ^ (ra & 7)) << 1));
    const double2 a1 = lds128(box + rbb * 16 + ((g ^ (rbb & 7)) << 1));
    const long ia = r0 + ra, ib = ia + 1;
    double b0[NT], b1[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int pp = nt * 8 + g;
      if (FULL) {
        b0[nt] = pp < K ? xs[ra * K + pp] : 0.0;
        b1[nt] = pp < K ? xs[rbb * K + pp] : 0.0;
      } else {
        b0[nt] = (ia < re && pp < K) ? __ldg(B + ia * K + pp) : 0.0;
        b1[nt] = (ib < re && pp < K) ? __ldg(B + ib * K + pp) : 0.0;
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      dmma(acc[0][nt][0], acc[0][nt][1], a0.x, b0[nt]);
      dmma(acc[1][nt][0], acc[1][nt][1], a0.y, b0[nt]);
      dmma(acc[0][nt][0], acc[0][nt][1], a1.x, b1[nt]);
      dmma(acc[1][nt][0], acc[1][nt][1], a1.y, b1[nt]);
    }
    if (TL > 0) {
#pragma unroll
      for (int j = 0; j < (TL > 0 ? TL : 1); ++j) {
        double xa, xb;
        if (FULL) {
          xa = xs[ra * K + 8 + j];
          xb = xs[rbb * K + 8 + j];
        } else {
          xa = ia < re ? __ldg(B + ia * K + 8 + j) : 0.0;
          xb = ib < re ? __ldg(B + ib * K + 8 + j) : 0.0;
        }
        tacc[0][j] = fma(a1.x, xb, fma(a0.x, xa, tacc[0][j]));
        tacc[1][j] = fma(a1.y, xb, fma(a0.y, xa, tacc[1][j]));
      }
    }
  }
}

template <int NT, int TL>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_colprod_tma(const __grid_constant__ CUtensorMap map, long rows, long cols,
                  const double* __restrict__ B, int K, long nitems, long nsplit, long split_rows,
                  double* __restrict__ part) {
  static_assert(TL == 0 || NT == 1, "DFMA tail only after one DMMA tile");
  extern __shared__ uint8_t smem_raw[];
  const Carve c = carve(smem_raw);
  double* sXs = c.extra;  // [STAGES][CP_BR][<= 16]: the stage's rows of B, dense (row pitch K)
  init_barriers(c);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long i_beg = (long)blockIdx.x * nitems / gridDim.x;
  const long i_end = (long)(blockIdx.x + 1) * nitems / gridDim.x;

  if (warp == NCW) {  // ===== TMA producer =====
    if (lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      for (long it = i_beg; it < i_end; ++it) {
        const long chunk = it / nsplit, s = it - chunk * nsplit;
        const long rb = s * split_rows, re = min(rows, rb + split_rows);
        for (long r0 = rb; r0 < re; r0 += CP_BR) {
          // the stage's rows of B (contiguous rows x K doubles) ride on the same barrier
          // when the whole 32-row block lies inside the split; otherwise consumers read them
          // from global memory (split / matrix tail)
          const bool bfull = r0 + CP_BR <= re;
          const unsigned bbytes = bfull ? (unsigned)(CP_BR * K * 8) : 0u;
          mbar_wait(&c.empty[stage], phase ^ 1u);
          mbar_expect_tx(&c.full[stage], (unsigned)STAGE_BYTES + bbytes);
          for (int b = 0; b < NCW; ++b)
            tma_load_2d(c.ring + ((size_t)stage * NCW + b) * CP_BOX, &map, &c.full[stage],
                        (int)(chunk * CP_CW + 16 * b), (int)r0);
          if (bfull) bulk_load(sXs + (size_t)stage * CP_BR * 16, B + r0 * K, bbytes, &c.full[stage]);
          if (++stage == STAGES) stage = 0, phase ^= 1u;
        }
      }
    }
    return;
  }

  const int g = lane >> 2, t = lane & 3;
  int stage = 0;
  unsigned phase = 0;
  for (long it = i_beg; it < i_end; ++it) {
    const long chunk = it / nsplit, s = it - chunk * nsplit;
    const long rb = s * split_rows, re = min(rows, rb + split_rows);
    double acc[2][NT][2];  // [column parity][n tile][2]
    double tacc[2][TL > 0 ? TL : 1];
#pragma unroll
    for (int par = 0; par < 2; ++par) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[par][nt][0] = acc[par][nt][1] = 0.0;
#pragma unroll
      for (int j = 0; j < (TL > 0 ? TL : 1); ++j) tacc[par][j] = 0.0;
    }
    for (long r0 = rb; r0 < re; r0 += CP_BR) {
      mbar_wait(&c.full[stage], phase);
      const double* box = c.ring + ((size_t)stage * NCW + warp) * CP_BOX;
      const double* xs = sXs + (size_t)stage * CP_BR * 16;
      if (r0 + CP_BR <= re)
        colprod_stage<NT, TL, true>(box, xs, B, K, r0, re, g, t, acc, tacc);
      else
        colprod_stage<NT, TL, false>(box, xs, B, K, r0, re, g, t, acc, tacc);
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.empty[stage]);
      if (++stage == STAGES) stage = 0, phase ^= 1u;
    }
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      const long col = chunk * CP_CW + 16 * warp + 2 * g + par;
      double tsum[TL > 0 ? TL : 1];
#pragma unroll
      for (int j = 0; j < (TL > 0 ? TL : 1); ++j) tsum[j] = TL > 0 ? quad_sum(tacc[par][j]) : 0.0;
      if (col >= cols) continue;
      double* dst = part + (s * cols + col) * K;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int pp = nt * 8 + 2 * t + e;
          if (pp < K) dst[pp] = acc[par][nt][e];
        }
      if (TL > 0 && t == 0)
#pragma unroll
        for (int j = 0; j < (TL > 0 ? TL : 1); ++j) dst[8 + j] = tsum[j];
    }
  }
}

// ---- column product, fp32 M (config c5) --------------------------------------
// Same item / split scheme as k_colprod_tma; a stage is 4 boxes of 32 fp32 columns x 32
// rows (16 KB) + the stage's 32 rows of B.  Warp w owns box (w & 3) and the row half
// (w >> 2) of every stage; lane (g, t) reads a float4 (columns 4g .. 4g + 3) of the lines
// 2t and 2t + 1 of each 8-row block -- under the 128B swizzle the eight lanes of a
// quarter-warp hit the chunks g ^ 2t, all distinct -- and feeds four column parities to
// the FP64 tensor cores (fp32 -> fp64 exactly).  The two row halves write separate
// partials (2 per split), summed with the rest in k_sum_partials' fixed order.
constexpr int CP32_CW = 128;
constexpr int CP32_BR = 32;
constexpr int CP32_BOX = CP32_BR * 32;  // floats per box (4 KB)

template <int NT>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_colprod_tma_f32(const __grid_constant__ CUtensorMap map, long rows, long cols,
                      const double* __restrict__ B, int K, long nitems, long nsplit,
                      long split_rows, double* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  const Carve c = carve(smem_raw);
  double* sXs = c.extra;  // [STAGES][CP32_BR][<= 16]
  init_barriers(c);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long i_beg = (long)blockIdx.x * nitems / gridDim.x;
  const long i_end = (long)(blockIdx.x + 1) * nitems / gridDim.x;
  float* ring = reinterpret_cast<float*>(c.ring);
  constexpr int SBYTES = 4 * CP32_BOX * 4;  // 16 KB of M per stage

  if (warp == NCW) {  // ===== TMA producer =====
    if (lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      for (long it = i_beg; it < i_end; ++it) {
        const long chunk = it / nsplit, s = it - chunk * nsplit;
        const long rb = s * split_rows, re = min(rows, rb + split_rows);
        for (long r0 = rb; r0 < re; r0 += CP32_BR) {
          const bool bfull = r0 + CP32_BR <= re;
          const unsigned bbytes = bfull ? (unsigned)(CP32_BR * K * 8) : 0u;
          mbar_wait(&c.empty[stage], phase ^ 1u);
          mbar_expect_tx(&c.full[stage], (unsigned)SBYTES + bbytes);
          for (int b = 0; b < 4; ++b)
            tma_load_2d(ring + ((size_t)stage * 4 + b) * CP32_BOX, &map, &c.full[stage],
                        (int)(chunk * CP32_CW + 32 * b), (int)r0);
          if (bfull) bulk_load(sXs + (size_t)stage * CP32_BR * 16, B + r0 * K, bbytes, &c.full[stage]);
          if (++stage == STAGES) stage = 0, phase ^= 1u;
        }
      }
    }
    return;
  }

  const int g = lane >> 2, t = lane & 3;
  const int bx = warp & 3, rh = warp >> 2;  // box, row half of the stage
  int stage = 0;
  unsigned phase = 0;
  for (long it = i_beg; it < i_end; ++it) {
    const long chunk = it / nsplit, s = it - chunk * nsplit;
    const long rb = s * split_rows, re = min(rows, rb + split_rows);
    double acc[4][NT][2];  // [column parity][n tile][2]
#pragma unroll
    for (int par = 0; par < 4; ++par)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[par][nt][0] = acc[par][nt][1] = 0.0;
    for (long r0 = rb; r0 < re; r0 += CP32_BR) {
      mbar_wait(&c.full[stage], phase);
      const float* box = ring + ((size_t)stage * 4 + bx) * CP32_BOX;
      const double* xs = sXs + (size_t)stage * CP32_BR * 16;
      const bool bfull = r0 + CP32_BR <= re;
#pragma unroll
      for (int bl = 0; bl < 2; ++bl) {
        const int blk = 2 * rh + bl;
        const int ra = 8 * blk + 2 * t, rbb = ra + 1;
        const float4 f0 = *reinterpret_cast<const float4*>(box + ra * 32 + ((g ^ (ra & 7)) << 2));
        const float4 f1 = *reinterpret_cast<const float4*>(box + rbb * 32 + ((g ^ (rbb & 7)) << 2));
        const long ia = r0 + ra, ib = ia + 1;
        double b0[NT], b1[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int pp = nt * 8 + g;
          if (bfull) {
            b0[nt] = pp < K ? xs[ra * K + pp] : 0.0;
            b1[nt] = pp < K ? xs[rbb * K + pp] : 0.0;
          } else {
            b0[nt] = (ia < re && pp < K) ? __ldg(B + ia * K + pp) : 0.0;
            b1[nt] = (ib < re && pp < K) ? __ldg(B + ib * K + pp) : 0.0;
          }
        }
        const double a0[4] = {(double)f0.x, (double)f0.y, (double)f0.z, (double)f0.w};
        const double a1[4] = {(double)f1.x, (double)f1.y, (double)f1.z, (double)f1.w};
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
          for (int par = 0; par < 4; ++par) dmma(acc[par][nt][0], acc[par][nt][1], a0[par], b0[nt]);
#pragma unroll
          for (int par = 0; par < 4; ++par) dmma(acc[par][nt][0], acc[par][nt][1], a1[par], b1[nt]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.empty[stage]);
      if (++stage == STAGES) stage = 0, phase ^= 1u;
    }
    // D row g of parity par <-> column 32 bx + 4 g + par of the chunk
#pragma unroll
    for (int par = 0; par < 4; ++par) {
      const long col = chunk * CP32_CW + 32 * bx + 4 * g + par;
      if (col >= cols) continue;
      double* dst = part + ((2 * s + rh) * cols + col) * K;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int pp = nt * 8 + 2 * t + e;
          if (pp < K) dst[pp] = acc[par][nt][e];
        }
    }
  }
}

// ---- dual product -----------------------------------------------------------
// ONE pass over M for both outR = M B1 (rows x K, B1: cols x K, e.g. M dY^T) and
// outC = M^T B2 (cols x K, B2: rows x K, e.g. M^T dX) -- the two products of every
// residual-free IPM iteration (solver.py _armijo_free + the incremental refresh).
// item = (chunk of TMA_RP_CW columns, band of 64 rows), chunk-major, contiguous ranges per
// CTA.  A stage is 8 boxes of 16 columns x 64 rows (64 KB, 2-stage ring).  Row part:
// warp w owns rows [8 w, 8 w + 8) of the band (one MMA tile; B1 fragments resident per
// chunk) and writes partR[chunk][row] when the band's chunk is done.  Column part: warp w
// owns box w of every stage (columns 16 w .. 16 w + 15 of the stage's 128), i.e. boxes
// {8 s + w} of the chunk, accumulated over the CTA's bands of the chunk in registers and
// flushed to partC[cta][segment] when the chunk changes.  Both parts: one DMMA tile
// (outputs 0..7) + the DFMA tail for K = 9..12, so the pass stays HBM-bound.
constexpr int DU_BR = 64;
constexpr int DU_BOX = DU_BR * 16;  // doubles per box (8 KB)
constexpr int DU_STAGES = 2;
constexpr int DU_STAGE_BYTES = NCW * DU_BOX * 8;  // 64 KB
constexpr int DU_SEGS = 4;                        // chunk segments per CTA range
constexpr int DU_CBOX = TMA_RP_CW / 16 / NCW;     // column boxes per warp per chunk (4)

struct DualCarve {
  double* ring;
  uint64_t* full;
  uint64_t* empty;
  double* sB;   // [RP_NGRP][2][NT][32]
  double* sT;   // [RP_NGRP][4][2][TP]
  double* sX;   // [DU_STAGES][DU_BR][16]
};

template <int NT, int TL>
__device__ __forceinline__ DualCarve dual_carve(uint8_t* raw) {
  const uint32_t base = su32(raw);
  const uint32_t pad = ((base + 1023u) & ~1023u) - base;
  uint8_t* p = raw + pad;
  DualCarve c;
  c.ring = reinterpret_cast<double*>(p);
  c.full = reinterpret_cast<uint64_t*>(p + DU_STAGES * DU_STAGE_BYTES);
  c.empty = c.full + DU_STAGES;
  c.sB = reinterpret_cast<double*>(c.empty + DU_STAGES);
  c.sT = c.sB + RP_NGRP * 2 * NT * 32;
  c.sX = c.sT + RP_NGRP * 8 * 4;
  return c;
}

template <int NT, int TL>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_dualprod_tma(const __grid_constant__ CUtensorMap map, long rows, long cols,
                   const double* __restrict__ B1, const double* __restrict__ B2, int K,
                   long nitems, long nbands, double* __restrict__ partR,
                   double* __restrict__ partC) {
  static_assert(TL == 0 || NT == 1, "DFMA tail only after one DMMA tile");
  constexpr int TP = TailPitch<TL>::v;
  constexpr int TLA = TL > 0 ? TL : 1;
  extern __shared__ uint8_t smem_raw[];
  const DualCarve c = dual_carve<NT, TL>(smem_raw);
  if (threadIdx.x == 0) {
    for (int s = 0; s < DU_STAGES; ++s) {
      mbar_init(&c.full[s], 1);
      mbar_init(&c.empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long i_beg = (long)blockIdx.x * nitems / gridDim.x;
  const long i_end = (long)(blockIdx.x + 1) * nitems / gridDim.x;
  constexpr int SCOLS = NCW * 16;  // columns per stage (128)

  if (warp == NCW) {  // ===== TMA producer =====
    if (lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      for (long it = i_beg; it < i_end; ++it) {
        const long chunk = it / nbands, band = it - chunk * nbands;
        const long j0 = chunk * TMA_RP_CW, r0 = band * DU_BR;
        const int cw = (int)min((long)TMA_RP_CW, cols - j0);
        const int nst = (cw + SCOLS - 1) / SCOLS;
        const bool bfull = r0 + DU_BR <= rows;
        for (int sidx = 0; sidx < nst; ++sidx) {
          const int nbox = min(NCW, (cw - sidx * SCOLS + 15) >> 4);
          const unsigned bbytes = bfull ? (unsigned)(DU_BR * K * 8) : 0u;
          mbar_wait(&c.empty[stage], phase ^ 1u);
          mbar_expect_tx(&c.full[stage], (unsigned)(nbox * DU_BOX * 8) + bbytes);
          for (int b = 0; b < nbox; ++b)
            tma_load_2d(c.ring + ((size_t)stage * NCW + b) * DU_BOX, &map, &c.full[stage],
                        (int)(j0 + sidx * SCOLS + 16 * b), (int)r0);
          if (bfull) bulk_load(c.sX + (size_t)stage * DU_BR * 16, B2 + r0 * K, bbytes, &c.full[stage]);
          if (++stage == DU_STAGES) stage = 0, phase ^= 1u;
        }
      }
    }
    return;
  }

  // ===== consumers =====
  const int g = lane >> 2, t = lane & 3;
  const int sig = (g >> 1) | ((g & 1) << 2);
  int stage = 0;
  unsigned phase = 0;
  long cur_chunk = -1;
  int seg = -1;
  double cacc[DU_CBOX][2][NT][2];  // column part: [box of this warp][parity][tile][2]
  double ctacc[DU_CBOX][2][TLA];
  auto zero_cols = [&]() {
#pragma unroll
    for (int q = 0; q < DU_CBOX; ++q)
#pragma unroll
      for (int par = 0; par < 2; ++par) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) cacc[q][par][nt][0] = cacc[q][par][nt][1] = 0.0;
#pragma unroll
        for (int j = 0; j < TLA; ++j) ctacc[q][par][j] = 0.0;
      }
  };
  auto flush_cols = [&](long chunk) {  // partC[cta][seg][local column][p]
    double* base = partC + ((long)blockIdx.x * DU_SEGS + seg) * (long)TMA_RP_CW * K;
#pragma unroll
    for (int q = 0; q < DU_CBOX; ++q)
#pragma unroll
      for (int par = 0; par < 2; ++par) {
        double ts[TLA];
#pragma unroll
        for (int j = 0; j < TLA; ++j) ts[j] = TL > 0 ? quad_sum(ctacc[q][par][j]) : 0.0;
        const int lc = (q * NCW + warp) * 16 + 2 * g + par;  // local column in the chunk
        double* dst = base + (long)lc * K;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int pp = nt * 8 + 2 * t + e;
            if (pp < K) dst[pp] = cacc[q][par][nt][e];
          }
        if (TL > 0 && t == 0)
#pragma unroll
          for (int j = 0; j < TLA; ++j) dst[8 + j] = ts[j];
      }
    (void)chunk;
  };
  zero_cols();
  for (long it = i_beg; it < i_end; ++it) {
    const long chunk = it / nbands, band = it - chunk * nbands;
    const long j0 = chunk * TMA_RP_CW, r0 = band * DU_BR;
    const int cw = (int)min((long)TMA_RP_CW, cols - j0);
    const int nst = (cw + SCOLS - 1) / SCOLS;
    const bool bfull = r0 + DU_BR <= rows;
    if (chunk != cur_chunk) {
      if (cur_chunk >= 0) {
        flush_cols(cur_chunk);
        zero_cols();
      }
      ++seg;
      consumers_sync();
      const int ngrp = 2 * ((cw + 15) >> 4);
      for (int e = threadIdx.x; e < ngrp * 2 * NT * 32; e += NCW * 32) {
        const int l = e & 31, se = (e >> 5) / NT, nt = (e >> 5) % NT;
        const int sidx = se >> 1, ee = se & 1;
        const long col = j0 + 8 * sidx + 2 * (l & 3) + ee;
        const int pp = nt * 8 + (l >> 2);
        const bool ok = col < cols && pp < K;
        cp_async8(c.sB + e, ok ? B1 + col * K + pp : B1, ok ? 8 : 0);
      }
      if (TL > 0)
        for (int e = threadIdx.x; e < ngrp * 8 * TP; e += NCW * 32) {
          const int j = e % TP, rec = e / TP;
          const long col = j0 + 8 * (rec >> 3) + 2 * ((rec >> 1) & 3) + (rec & 1);
          const bool ok = col < cols && j < TL;
          cp_async8(c.sT + e, ok ? B1 + col * K + 8 + j : B1, ok ? 8 : 0);
        }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      consumers_sync();
      cur_chunk = chunk;
    }
    // two independent accumulator sets per tile (even / odd column of each lane's pair):
    // the DMMA chains are half as deep; summed when the band's chunk is done
    double racc[NT][2], racc2[NT][2], rtacc[TLA], rtacc2[TLA];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) racc[nt][0] = racc[nt][1] = racc2[nt][0] = racc2[nt][1] = 0.0;
#pragma unroll
    for (int j = 0; j < TLA; ++j) rtacc[j] = rtacc2[j] = 0.0;
    for (int sidx = 0; sidx < nst; ++sidx) {
      const int nbox = min(NCW, (cw - sidx * SCOLS + 15) >> 4);
      mbar_wait(&c.full[stage], phase);
      const double* ring = c.ring + (size_t)stage * NCW * DU_BOX;
      // -- row part: rows 8 warp + sig over the stage's boxes
      for (int b = 0; b < nbox; ++b) {
        const double* box = ring + (size_t)b * DU_BOX;
        const int r = 8 * warp + sig;
        const double2 a0 = lds128(box + r * 16 + ((t ^ sig) << 1));
        const double2 a1 = lds128(box + r * 16 + (((4 + t) ^ sig) << 1));
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const double2 a = kk ? a1 : a0;
          const int q = 2 * (sidx * NCW + b) + kk;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const double bx = c.sB[((2 * q) * NT + nt) * 32 + lane];
            const double by = c.sB[((2 * q + 1) * NT + nt) * 32 + lane];
            dmma(racc[nt][0], racc[nt][1], a.x, bx);
            dmma(racc2[nt][0], racc2[nt][1], a.y, by);
          }
          if (TL == 2) {  // both tail records of the pair in two 16-byte loads (TP = 2)
            const double* tr = c.sT + ((q * 4 + t) * 2) * TP;
            const double2 t0 = lds128(tr), t1 = lds128(tr + 2);
            rtacc[0] = fma(a.x, t0.x, rtacc[0]);
            rtacc[1 % TLA] = fma(a.x, t0.y, rtacc[1 % TLA]);
            rtacc2[0] = fma(a.y, t1.x, rtacc2[0]);
            rtacc2[1 % TLA] = fma(a.y, t1.y, rtacc2[1 % TLA]);
          } else if (TL > 0) {
            const double* tr = c.sT + ((q * 4 + t) * 2) * TP;
#pragma unroll
            for (int j = 0; j < TLA; ++j) {
              rtacc[j] = fma(a.x, tr[j], rtacc[j]);
              rtacc2[j] = fma(a.y, tr[TP + j], rtacc2[j]);
            }
          }
        }
      }
      // -- column part: box `warp` of the stage over its 64 rows
      if (warp < nbox) {
        const int q = sidx;  // this warp's column box index within the chunk = sidx * NCW + warp
        const double* box = ring + (size_t)warp * DU_BOX;
        const double* xs = c.sX + (size_t)stage * DU_BR * 16;
#pragma unroll
        for (int qq = 0; qq < DU_CBOX; ++qq) {
          if (qq != q) continue;  // registers stay statically indexed
          // the odd contraction rows accumulate into per-stage temporaries (independent
          // DMMA chains), folded into the chunk accumulators after the stage
          double u[2][NT][2], ut[2][TLA];
#pragma unroll
          for (int par = 0; par < 2; ++par) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) u[par][nt][0] = u[par][nt][1] = 0.0;
#pragma unroll
            for (int j = 0; j < TLA; ++j) ut[par][j] = 0.0;
          }
#pragma unroll 2
          for (int blk = 0; blk < DU_BR / 8; ++blk) {
            const int ra = 8 * blk + 2 * t, rbb = ra + 1;
            const double2 a0 = lds128(box + ra * 16 + ((g ^ (ra & 7)) << 1));
            const double2 a1 = lds128(box + rbb * 16 + ((g ^ (rbb & 7)) << 1));
            const long ia = r0 + ra, ib = ia + 1;
            double b0[NT], b1[NT];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const int pp = nt * 8 + g;
              if (bfull) {
                b0[nt] = pp < K ? xs[ra * K + pp] : 0.0;
                b1[nt] = pp < K ? xs[rbb * K + pp] : 0.0;
              } else {
                b0[nt] = (ia < rows && pp < K) ? __ldg(B2 + ia * K + pp) : 0.0;
                b1[nt] = (ib < rows && pp < K) ? __ldg(B2 + ib * K + pp) : 0.0;
              }
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              dmma(cacc[qq][0][nt][0], cacc[qq][0][nt][1], a0.x, b0[nt]);
              dmma(cacc[qq][1][nt][0], cacc[qq][1][nt][1], a0.y, b0[nt]);
              dmma(u[0][nt][0], u[0][nt][1], a1.x, b1[nt]);
              dmma(u[1][nt][0], u[1][nt][1], a1.y, b1[nt]);
            }
            if (TL == 2 && bfull) {  // K = 10: the two tail entries of a row in one 16-byte load
              const double2 xa = lds128(xs + ra * K + 8), xb = lds128(xs + rbb * K + 8);
              ctacc[qq][0][0] = fma(a0.x, xa.x, ctacc[qq][0][0]);
              ctacc[qq][1][0] = fma(a0.y, xa.x, ctacc[qq][1][0]);
              ut[0][0] = fma(a1.x, xb.x, ut[0][0]);
              ut[1][0] = fma(a1.y, xb.x, ut[1][0]);
              ctacc[qq][0][1 % TLA] = fma(a0.x, xa.y, ctacc[qq][0][1 % TLA]);
              ctacc[qq][1][1 % TLA] = fma(a0.y, xa.y, ctacc[qq][1][1 % TLA]);
              ut[0][1 % TLA] = fma(a1.x, xb.y, ut[0][1 % TLA]);
              ut[1][1 % TLA] = fma(a1.y, xb.y, ut[1][1 % TLA]);
            } else if (TL > 0) {
#pragma unroll
              for (int j = 0; j < TLA; ++j) {
                double xa, xb;
                if (bfull) {
                  xa = xs[ra * K + 8 + j];
                  xb = xs[rbb * K + 8 + j];
                } else {
                  xa = ia < rows ? __ldg(B2 + ia * K + 8 + j) : 0.0;
                  xb = ib < rows ? __ldg(B2 + ib * K + 8 + j) : 0.0;
                }
                ctacc[qq][0][j] = fma(a0.x, xa, ctacc[qq][0][j]);
                ctacc[qq][1][j] = fma(a0.y, xa, ctacc[qq][1][j]);
                ut[0][j] = fma(a1.x, xb, ut[0][j]);
                ut[1][j] = fma(a1.y, xb, ut[1][j]);
              }
            }
          }
#pragma unroll
          for (int par = 0; par < 2; ++par) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              cacc[qq][par][nt][0] += u[par][nt][0], cacc[qq][par][nt][1] += u[par][nt][1];
#pragma unroll
            for (int j = 0; j < TLA; ++j) ctacc[qq][par][j] += ut[par][j];
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.empty[stage]);
      if (++stage == DU_STAGES) stage = 0, phase ^= 1u;
    }
    {  // row partials of this (chunk, band)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) racc[nt][0] += racc2[nt][0], racc[nt][1] += racc2[nt][1];
      double ts[TLA];
#pragma unroll
      for (int j = 0; j < TLA; ++j) ts[j] = TL > 0 ? quad_sum(rtacc[j] + rtacc2[j]) : 0.0;
      const long row = r0 + 8 * warp + sig;
      if (row < rows) {
        double* dst = partR + (chunk * rows + row) * K;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int pp = nt * 8 + 2 * t + e;
            if (pp < K) dst[pp] = racc[nt][e];
          }
        if (TL > 0 && t == 0)
#pragma unroll
          for (int j = 0; j < TLA; ++j) dst[8 + j] = ts[j];
      }
    }
  }
  if (cur_chunk >= 0) flush_cols(cur_chunk);
}

// outC[j][p] = sum over the CTAs whose item range meets column j's chunk (ascending CTA
// order, fixed) of partC[cta][segment of that chunk][local column][p].  One block row per
// chunk (blockIdx.y): thread 0 lists the contributing (CTA, segment) slots once.
__global__ void __launch_bounds__(256) k_sum_dual_cols(const double* __restrict__ partC, long cols,
                                                       int K, long nitems, long nbands, int G,
                                                       double* __restrict__ out) {
  __shared__ int slot[256];
  __shared__ int wcnt[8];
  __shared__ int nslot;
  const long chunk = blockIdx.y;
  {  // thread b tests CTA b (G <= 256); ballot prefix keeps ascending CTA order
    const int b = threadIdx.x, lane = b & 31, w = b >> 5;
    const long lo = chunk * nbands, hi = lo + nbands;  // the chunk's items [lo, hi)
    bool hit = false;
    int sl = 0;
    if (b < G) {
      const long first = ((long)b * nitems) / G, fend = ((long)(b + 1) * nitems) / G;
      hit = fend > first && fend > lo && first < hi;
      if (hit) sl = (int)((long)b * DU_SEGS + (max(lo, first) / nbands - first / nbands));
    }
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wcnt[w] = __popc(m);
    __syncthreads();
    int base = 0;
    for (int i = 0; i < w; ++i) base += wcnt[i];
    if (hit) slot[base + __popc(m & ((1u << lane) - 1u))] = sl;
    if (b == 255) {
      int n = 0;
      for (int i = 0; i < 8; ++i) n += wcnt[i];
      nslot = n;
    }
  }
  __syncthreads();
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;  // element within the chunk
  const long cw = min((long)TMA_RP_CW, cols - chunk * TMA_RP_CW);
  if (e >= cw * K) return;
  double v = 0.0;
  for (int i = 0; i < nslot; ++i) v += partC[(long)slot[i] * TMA_RP_CW * K + e];
  out[chunk * TMA_RP_CW * K + e] = v;
}

// ---- host side ----------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
  }();
  return fn;
}

bool make_map(CUtensorMap* m, const double* A, long rows, long cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(double)};
  const cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  static const CUtensorMapL2promotion promo = [] {
    const char* e = getenv("NMFB_TMA_L2P");  // L2 fetch granularity (experiments)
    const int v = e ? atoi(e) : 0;
    return v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
         : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
         : v == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                    : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  }();
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)A, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() {
  static int sms = [] {
    int d = 0, v = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return v > 0 ? v : 148;
  }();
  return sms;
}

bool shape_ok(const double* A, long rows, long cols) {
  // TMA: 16-byte aligned base and row pitch, coordinates in int32
  return ((uintptr_t)A % 16 == 0) && (cols % 2 == 0) && rows < (1L << 31) && cols < (1L << 31);
}

}  // namespace

static int g_tma_prod = -1;  // -1: from NMFB_TMA_PROD (default on)

bool tma_prod_enabled() {
  if (g_tma_prod < 0) {
    const char* e = getenv("NMFB_TMA_PROD");
    g_tma_prod = (e && e[0] == '0') ? 0 : 1;
  }
  return g_tma_prod != 0;
}

extern "C" int nmfb_tma_products(int on) {
  const int prev = tma_prod_enabled() ? 1 : 0;
  if (on >= 0) g_tma_prod = on ? 1 : 0;
  return prev;
}

int tma_rowprod_f64(const double* A, long rows, long cols, const double* B, int K, double* work,
                    long work_len, long* nparts, cudaStream_t st) {
  if (!tma_prod_enabled() || K < 1 || K > 16 || !shape_ok(A, rows, cols)) return NMFB_EUNSUPPORTED;
  const long nch = (cols + TMA_RP_CW - 1) / TMA_RP_CW;
  if (nch * rows * K > work_len) return NMFB_ENOMEM;
  CUtensorMap map;
  if (!make_map(&map, A, rows, cols, RP_BR)) return NMFB_EUNSUPPORTED;
  const long nbands = (rows + RP_BR - 1) / RP_BR;
  const long nitems = nch * nbands;
  const int grid = (int)min((long)num_sms(), nitems);
  const int NT = (K + 7) / 8;
  const size_t smem = 1024 + STAGES * STAGE_BYTES + 2 * STAGES * 8 +
                      (size_t)RP_NGRP * 2 * NT * 32 * sizeof(double) +
                      (size_t)RP_NGRP * 8 * 4 * sizeof(double);
#define RP_LAUNCH(NT_, TL_)                                                                     \
  nmfb_smem_attr(k_rowprod_tma<NT_, TL_>, smem);                                                \
  ++g_nmfb_launches, k_rowprod_tma<NT_, TL_><<<grid, NTHREADS, smem, st>>>(map, rows, cols, B, K, \
                                                                           nitems, nbands, work)
  switch (K) {
    case 9: RP_LAUNCH(1, 1); break;
    case 10: RP_LAUNCH(1, 2); break;
    case 11: RP_LAUNCH(1, 3); break;
    case 12: RP_LAUNCH(1, 4); break;
    default:
      if (NT == 1) {
        RP_LAUNCH(1, 0);
      } else {
        RP_LAUNCH(2, 0);
      }
  }
#undef RP_LAUNCH
  *nparts = nch;
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

long tma_colprod_splits(long rows, long cols) {
  const long nch = (cols + CP_CW - 1) / CP_CW;
  // about 8 items per CTA over the whole grid, splits of whole 32-row boxes
  long want = (8L * num_sms() + nch - 1) / nch;
  if (want < 1) want = 1;
  long sr = (rows + want - 1) / want;
  sr = ((sr + CP_BR - 1) / CP_BR) * CP_BR;
  if (sr < 4 * CP_BR) sr = 4 * CP_BR;
  return (rows + sr - 1) / sr;
}

int tma_colprod_f64(const double* A, long rows, long cols, const double* B, int K, double* work,
                    long work_len, long* nparts, cudaStream_t st) {
  if (!tma_prod_enabled() || K < 1 || K > 16 || !shape_ok(A, rows, cols)) return NMFB_EUNSUPPORTED;
  const long nch = (cols + CP_CW - 1) / CP_CW;
  long ns = tma_colprod_splits(rows, cols);
  long sr = (rows + ns - 1) / ns;
  sr = ((sr + CP_BR - 1) / CP_BR) * CP_BR;
  ns = (rows + sr - 1) / sr;
  if (ns * cols * K > work_len) return NMFB_ENOMEM;
  CUtensorMap map;
  if (!make_map(&map, A, rows, cols, CP_BR)) return NMFB_EUNSUPPORTED;
  const long nitems = nch * ns;
  const int grid = (int)min((long)num_sms(), nitems);
  const size_t smem = 1024 + STAGES * STAGE_BYTES + 2 * STAGES * 8 +
                      (size_t)STAGES * CP_BR * 16 * sizeof(double);
  if ((uintptr_t)B % 16) return NMFB_EUNSUPPORTED;  // bulk copies of B rows
#define CP_LAUNCH(NT_, TL_)                                                                     \
  nmfb_smem_attr(k_colprod_tma<NT_, TL_>, smem);                                                \
  ++g_nmfb_launches, k_colprod_tma<NT_, TL_><<<grid, NTHREADS, smem, st>>>(map, rows, cols, B, K, \
                                                                           nitems, ns, sr, work)
  switch (K) {
    case 9: CP_LAUNCH(1, 1); break;
    case 10: CP_LAUNCH(1, 2); break;
    case 11: CP_LAUNCH(1, 3); break;
    case 12: CP_LAUNCH(1, 4); break;
    default:
      if (K <= 8) {
        CP_LAUNCH(1, 0);
      } else {
        CP_LAUNCH(2, 0);
      }
  }
#undef CP_LAUNCH
  *nparts = ns;
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

long tma_dualprod_work_len(long rows, long cols, long k) {
  const long nch = (cols + TMA_RP_CW - 1) / TMA_RP_CW;
  return nch * rows * k + (long)num_sms() * DU_SEGS * TMA_RP_CW * k;
}

int tma_dualprod_f64(const double* A, long rows, long cols, const double* B1, const double* B2,
                     int K, double* outR, double* outC, double* work, long work_len,
                     cudaStream_t st) {
  if (!tma_prod_enabled() || K < 5 || K > 16 || !shape_ok(A, rows, cols) || (uintptr_t)B2 % 16)
    return NMFB_EUNSUPPORTED;
  const long nch = (cols + TMA_RP_CW - 1) / TMA_RP_CW;
  const long nbands = (rows + DU_BR - 1) / DU_BR;
  const long nitems = nch * nbands;
  const int G = (int)min((long)num_sms(), nitems);
  // every CTA range must meet at most DU_SEGS chunks
  if ((nitems + G - 1) / G + 1 > (long)(DU_SEGS - 1) * nbands + 1) return NMFB_EUNSUPPORTED;
  if (tma_dualprod_work_len(rows, cols, K) > work_len) return NMFB_ENOMEM;
  if (G > 256) return NMFB_EUNSUPPORTED;  // k_sum_dual_cols: one thread per CTA
  CUtensorMap map;
  if (!make_map(&map, A, rows, cols, DU_BR)) return NMFB_EUNSUPPORTED;
  double* partR = work;
  double* partC = work + nch * rows * K;
  const int NT = (K + 7) / 8;
  const size_t smem = 1024 + DU_STAGES * DU_STAGE_BYTES + 2 * DU_STAGES * 8 +
                      (size_t)RP_NGRP * 2 * NT * 32 * sizeof(double) +
                      (size_t)RP_NGRP * 8 * 4 * sizeof(double) +
                      (size_t)DU_STAGES * DU_BR * 16 * sizeof(double);
#define DU_LAUNCH(NT_, TL_)                                                                      \
  nmfb_smem_attr(k_dualprod_tma<NT_, TL_>, smem);                                                \
  ++g_nmfb_launches, k_dualprod_tma<NT_, TL_><<<G, NTHREADS, smem, st>>>(map, rows, cols, B1, B2, \
                                                                         K, nitems, nbands,      \
                                                                         partR, partC)
  static const int no_tail = [] {
    const char* e = getenv("NMFB_DUAL_NOTAIL");
    return e && e[0] == '1';
  }();
  switch (no_tail ? 0 : K) {
    case 9: DU_LAUNCH(1, 1); break;
    case 10: DU_LAUNCH(1, 2); break;  // K = 11, 12: two DMMA tiles (a 3-4 wide tail spills)
    default:
      if (NT == 1) {
        DU_LAUNCH(1, 0);
      } else {
        DU_LAUNCH(2, 0);
      }
  }
#undef DU_LAUNCH
  ++g_nmfb_launches, k_sum_dual_cols<<<dim3((unsigned)((TMA_RP_CW * K + 255) / 256), (unsigned)nch),
                                        256, 0, st>>>(partC, cols, K, nitems, nbands, G, outC);
  (void)outR;  // the caller sums the row partials (fixed order, with its k_sum_partials)
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

// fp32 M: the FP64 tensor-core column product fed by TMA (c5's M^T X / M^T dX)
int tma_colprod_f32(const float* A, long rows, long cols, const double* B, int K, double* work,
                    long work_len, long* nparts, cudaStream_t st) {
  if (!tma_prod_enabled() || K < 1 || K > 16 || (uintptr_t)A % 16 || cols % 4 ||
      rows >= (1L << 31) || cols >= (1L << 31) || (uintptr_t)B % 16)
    return NMFB_EUNSUPPORTED;
  const long nch = (cols + CP32_CW - 1) / CP32_CW;
  long ns = tma_colprod_splits(rows, cols);
  long sr = (rows + ns - 1) / ns;
  sr = ((sr + CP32_BR - 1) / CP32_BR) * CP32_BR;
  ns = (rows + sr - 1) / sr;
  if (2 * ns * cols * K > work_len) return NMFB_ENOMEM;
  auto fn = encode_fn();
  if (!fn) return NMFB_EUNSUPPORTED;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(float)};
  const cuuint32_t box[2] = {32, (cuuint32_t)CP32_BR};
  const cuuint32_t es[2] = {1, 1};
  if (fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)A, dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return NMFB_EUNSUPPORTED;
  const long nitems = nch * ns;
  const int grid = (int)min((long)num_sms(), nitems);
  const size_t smem = 1024 + STAGES * STAGE_BYTES + 2 * STAGES * 8 +
                      (size_t)STAGES * CP32_BR * 16 * sizeof(double);
  if (K <= 8) {
    nmfb_smem_attr(k_colprod_tma_f32<1>, smem);
    ++g_nmfb_launches, k_colprod_tma_f32<1><<<grid, NTHREADS, smem, st>>>(map, rows, cols, B, K,
                                                                          nitems, ns, sr, work);
  } else {
    nmfb_smem_attr(k_colprod_tma_f32<2>, smem);
    ++g_nmfb_launches, k_colprod_tma_f32<2><<<grid, NTHREADS, smem, st>>>(map, rows, cols, B, K,
                                                                          nitems, ns, sr, work);
  }
  *nparts = 2 * ns;
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}
