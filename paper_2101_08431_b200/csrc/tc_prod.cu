// tcgen05 (5th-generation tensor core) streaming products for an fp32 M (config c5:
// 200000 x 40000, k = 16, fp32 storage with fp64 solves).  At k = 16 the products do
// 8 flops per byte of fp32 M, which puts the FP64 DMMA kernels at the FP64 tensor limit
// (csrc/anls.cu, 8.3 / 11.5 ms per pass); the tf32 tensor cores have > 20x that rate, so
// the pass becomes HBM-bound even with a 3-term split:
//
//   M = Mh + Ml,  Y = Yh + Yl  (tf32 parts: Mh = M with the low 13 mantissa bits cleared,
//   Ml = M - Mh exactly, Yh / Yl likewise from the fp64 factor)
//   M Y ~= Mh Yh + Mh Yl + Ml Yh        (relative error ~2^-21 per term)
//
// accumulated in fp32 in tensor memory over one 512-column chunk (ctb of a 128-row band)
// and written as fp64 split-K partials that the fixed-order k_sum_partials finishes.
//
// Row product (ctb = M Y^T, X-update / M dY^T):
//   warp 0      TMA producer: one 128-row x 32-column box of M per stage, 128B-swizzled,
//               which is exactly the canonical K-major SW128 UMMA operand layout;
//   warp 1      TMEM allocator + single-thread MMA issuer (tcgen05.mma.cta_group::1.kind::tf32,
//               M = 128, N = 16, K = 8; 3 MMAs per K step), tcgen05.commit -> mbarriers;
//   warps 4..7  converters (Mh in place, Ml to a twin buffer, fence.proxy.async) and the
//               epilogue (tcgen05.ld 32x32b: thread = row, 16 fp32 columns -> fp64 partials),
//               which runs on the double-buffered accumulator while the next item's MMAs go.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "tc_prod.cuh"

namespace {

constexpr int TC_STAGES = 8;                // TMA ring of M tiles: 128 KB in flight per SM
constexpr int TC_LO = 3;                    // Ml buffers in tensor memory (convert -> MMA)
constexpr int TC_BR = 128;                  // rows per band (UMMA M)
constexpr int TC_BC = 32;                   // columns per stage (one 128-byte swizzle atom)
constexpr int TC_TILE = TC_BR * TC_BC * 4;  // bytes per M tile (16 KB)
constexpr int TC_N = 16;                    // outputs (K <= 16 zero-padded)
constexpr int TC_SUB = 4;                   // stages per accumulator flush (128 columns)
constexpr int TC_EPI_LAG = 2;               // stages converted before an accumulator's epilogue
constexpr int TC_NCONV = 8;                // converter warps (4 .. 11); 4 .. 7 also run the epilogue
constexpr int TC_THREADS = (4 + TC_NCONV) * 32;
__host__ __device__ constexpr uint32_t tc_idesc(int n) {
  return (1u << 4)       // D fp32
         | (2u << 7)     // A tf32
         | (2u << 10)    // B tf32
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TC_BR >> 4) << 24);
}

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
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void converters_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(TC_NCONV * 32) : "memory");
}

// K-major, 128B-swizzled UMMA shared-memory descriptor (sm_100: version 1, layout 2):
// 8-row core groups 1024 bytes apart (SBO), LBO unused for swizzled K-major operands
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}
template <int N>
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(tc_idesc(N)), "r"(accumulate)
      : "memory");
}
// A operand from tensor memory (lane = row, one 32-bit column per K element)
template <int N>
__device__ __forceinline__ void umma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(tc_idesc(N)), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
      "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

// tf32 split of an fp32 value: hi = value with the low 13 mantissa bits cleared, lo = rest
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
}

// byte offset of element (row r, k-element e) of a K-major SW128 operand with `rows`
// rows per 32-element atom column (atom column a = e / 32 occupies rows * 128 bytes)
__device__ __forceinline__ uint32_t sw128_off(int r, int e, int rows) {
  const int a = e >> 5, ee = e & 31;
  const int ch = ee >> 2, w = ee & 3;
  return (uint32_t)(a * rows * 128 + r * 128 + (((ch ^ (r & 7)) << 4) | (w << 2)));
}

struct TcSmem {
  float* hi;        // [TC_STAGES][TC_TILE]  M tiles as landed by TMA (the tensor core reads
                    // them as tf32, i.e. truncated to Mh)
  float* bcat;      // [CW / 32 atoms][32 rows: Yh p = 0..15, Yl p = 0..15][128 B]
  uint64_t* full;   // TMA landed
  uint64_t* conv;   // converters done (Ml of the stage in tensor memory)
  uint64_t* empty;  // MMAs of the stage done
  uint64_t* accf;   // [2] accumulator ready
  uint64_t* acce;   // [2] accumulator drained
  uint64_t* bready; // B chunk converted
  uint64_t* loe;    // [TC_LO] Ml buffer consumed by the MMAs
  uint32_t* tmem_base;
};

__device__ __forceinline__ TcSmem tc_carve(uint8_t* raw, int cw) {
  const uint32_t base = su32(raw);
  uint8_t* p = raw + (((base + 1023u) & ~1023u) - base);
  TcSmem s;
  s.hi = reinterpret_cast<float*>(p);
  s.bcat = reinterpret_cast<float*>(p + TC_STAGES * TC_TILE);
  uint64_t* b = reinterpret_cast<uint64_t*>(p + TC_STAGES * TC_TILE + cw * 2 * TC_N * 4);
  s.full = b;
  s.conv = b + TC_STAGES;
  s.empty = b + 2 * TC_STAGES;
  s.accf = b + 3 * TC_STAGES;
  s.acce = s.accf + 2;
  s.bready = s.acce + 2;
  s.loe = s.bready + 1;
  s.tmem_base = reinterpret_cast<uint32_t*>(s.loe + TC_LO);
  return s;
}

// TMEM columns: [0, 64) two 32-column fp32 accumulators, [64, 64 + 32 TC_LO) Ml buffers
constexpr uint32_t TC_TMEM_COLS = 256;
constexpr uint32_t TC_LO_COL = 64;

// item = (chunk of TC_RP_CW columns, band of 128 rows), chunk-major, contiguous per CTA.
// Within an item the accumulator is flushed every TC_SUB stages (128 columns: the tensor
// core's fp32 accumulation truncates, so shorter runs keep it at ~2e-6 relative) into fp64
// registers of the epilogue threads (thread = row).
// Per K step (8 columns): D[:, 0:32] += Mh [Yh | Yl] (A = the TMA tile in shared memory,
// N = 32) and D[:, 0:16] += Ml Yh (A = Ml in tensor memory, N = 16); the epilogue adds
// D[:, p] + D[:, 16 + p].  Shared-memory traffic per 16 KB of M: the TMA write, one
// converter read and one tensor-core read (Ml never touches shared memory).
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_rowprod_tc(const __grid_constant__ CUtensorMap map, long rows, long cols,
                 const double* __restrict__ B, int K, long nitems, long nbands,
                 double* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  const TcSmem s = tc_carve(smem_raw, TC_RP_CW);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < TC_STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.conv[i], 4);  // one converter group per stage
      mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s.accf[i], 1);
      mbar_init(&s.acce[i], 4);
    }
    mbar_init(s.bready, TC_NCONV);
    for (int i = 0; i < TC_LO; ++i) mbar_init(&s.loe[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(s.tmem_base)),
                 "n"(TC_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s.tmem_base;
  const long i_beg = (long)blockIdx.x * nitems / gridDim.x;
  const long i_end = (long)(blockIdx.x + 1) * nitems / gridDim.x;

  if (warp == 0) {  // ===== TMA producer =====
    if (lane == 0) {
      int st = 0;
      unsigned ph = 0;
      for (long it = i_beg; it < i_end; ++it) {
        const long chunk = it / nbands, band = it - chunk * nbands;
        const long j0 = chunk * TC_RP_CW;
        const int nst = (int)((min((long)TC_RP_CW, cols - j0) + TC_BC - 1) / TC_BC);
        for (int k = 0; k < nst; ++k) {
          mbar_wait(&s.empty[st], ph ^ 1u);
          mbar_expect_tx(&s.full[st], TC_TILE);
          tma_load_2d(s.hi + (size_t)st * (TC_TILE / 4), &map, &s.full[st], (int)(j0 + k * TC_BC),
                      (int)(band * TC_BR));
          if (++st == TC_STAGES) st = 0, ph ^= 1u;
        }
      }
    }
  } else if (warp == 1) {  // ===== MMA issuer =====
    if (lane == 0) {
      int st = 0, lo_i = 0;
      unsigned ph = 0, bph = 0;
      long cur_chunk = -1;
      int acc = 0;
      unsigned aph[2] = {0u, 0u};
      const uint32_t bcat = su32(s.bcat);
      for (long it = i_beg; it < i_end; ++it) {
        const long chunk = it / nbands;
        const long j0 = chunk * TC_RP_CW;
        const int nst = (int)((min((long)TC_RP_CW, cols - j0) + TC_BC - 1) / TC_BC);
        if (chunk != cur_chunk) {  // the converters staged this chunk's B
          mbar_wait(s.bready, bph);
          bph ^= 1u;
          cur_chunk = chunk;
        }
        for (int k0 = 0; k0 < nst; k0 += TC_SUB) {
          mbar_wait(&s.acce[acc], aph[acc] ^ 1u);  // the epilogue drained this accumulator
          aph[acc] ^= 1u;
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(acc * 2 * TC_N);
          const int k1 = min(nst, k0 + TC_SUB);
          for (int k = k0; k < k1; ++k) {
            mbar_wait(&s.conv[st], ph);
            tc_fence_after();
            const uint32_t ah = su32(s.hi) + st * TC_TILE;
            const uint32_t al = tmem + TC_LO_COL + (uint32_t)(lo_i * TC_BC);
#pragma unroll
            for (int kk = 0; kk < TC_BC / 8; ++kk) {
              const uint64_t db = umma_desc(bcat + (uint32_t)(k * 2 * TC_N * 128 + kk * 32));
              umma_tf32<2 * TC_N>(d, umma_desc(ah + kk * 32), db, (k > k0 || kk) ? 1u : 0u);
              umma_tf32_ta<TC_N>(d, al + kk * 8, db, 1u);
            }
            umma_commit(&s.empty[st]);  // frees the stage once these MMAs have read it
            umma_commit(&s.loe[lo_i]);
            if (++lo_i == TC_LO) lo_i = 0;
            if (++st == TC_STAGES) st = 0, ph ^= 1u;
          }
          umma_commit(&s.accf[acc]);
          acc ^= 1;
        }
      }
    }
  } else if (warp >= 4) {  // ===== converters + epilogue =====
    const int ct = threadIdx.x - 128;  // 0 .. 32 TC_NCONV - 1
    const bool epi = warp < 8;         // warps 4..7: one per TMEM lane quadrant
    const int q = warp & 3;            // TMEM lane quadrant of this warp
    const int grp = (warp - 4) >> 2;   // converter group: stages alternate between the two groups
    const int r = 32 * q + lane;       // tile row (= TMEM lane) this thread converts
    unsigned gcnt = 0;
    int st = 0, lo_i = 0;
    unsigned ph = 0;
    unsigned lo_ph[TC_LO] = {};
    long cur_chunk = -1;
    int acc = 0;
    unsigned aph[2] = {0u, 0u};
    double a64[TC_N];
    long pend_chunk = -1, pend_band = -1;
    int pend_acc = 0;
    bool pend_last = false;
    int pend_age = 0;
    auto epilogue = [&]() {
      const int a = pend_acc;
      mbar_wait(&s.accf[a], aph[a]);
      aph[a] ^= 1u;
      tc_fence_after();
      uint32_t v[2 * TC_N];
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * 2 * TC_N);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
          "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
            "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
            "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
            "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.acce[a]);
#pragma unroll
      for (int p = 0; p < TC_N; ++p)
        a64[p] += (double)__uint_as_float(v[p]) + (double)__uint_as_float(v[TC_N + p]);
      if (pend_last) {
        const long row = pend_band * TC_BR + 32 * q + lane;
        if (row < rows) {
          double* dst = part + (pend_chunk * rows + row) * K;
#pragma unroll
          for (int p = 0; p < TC_N; ++p)
            if (p < K) dst[p] = a64[p];
        }
#pragma unroll
        for (int p = 0; p < TC_N; ++p) a64[p] = 0.0;
      }
      pend_chunk = -1;
    };
#pragma unroll
    for (int p = 0; p < TC_N; ++p) a64[p] = 0.0;
    for (long it = i_beg; it < i_end; ++it) {
      const long chunk = it / nbands, band = it - chunk * nbands;
      const long j0 = chunk * TC_RP_CW;
      const int cw = (int)min((long)TC_RP_CW, cols - j0);
      const int nst = (cw + TC_BC - 1) / TC_BC;
      if (chunk != cur_chunk) {
        // B chunk (cols x K fp64) -> [Yh | Yl] tf32, K-major SW128 [atom][32 rows][128 B];
        // the MMAs of the previous chunk must be done with the old B: drain them first
        if (pend_chunk >= 0) {
          if (epi) epilogue();
          pend_chunk = -1;
        }
        converters_sync();
        const int natoms = (cw + 31) >> 5;
        uint8_t* bb = reinterpret_cast<uint8_t*>(s.bcat);
        // 16 independent loads in flight per thread, then the conversions / stores
        for (int e0 = ct; e0 < natoms * 32 * TC_N; e0 += TC_NCONV * 32 * 16) {
          double y[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int e = e0 + TC_NCONV * 32 * u;
            const int p = e & (TC_N - 1), c = e >> 4;  // p fastest: coalesced B[col][p] reads
            const long col = j0 + c;
            y[u] = (e < natoms * 32 * TC_N && col < cols && p < K) ? __ldg(B + col * K + p) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int e = e0 + TC_NCONV * 32 * u;
            if (e >= natoms * 32 * TC_N) break;
            const int p = e & (TC_N - 1), c = e >> 4;
            const float yh = __uint_as_float(__float_as_uint((float)y[u]) & 0xFFFFE000u);
            const float yl = (float)(y[u] - (double)yh);
            *reinterpret_cast<float*>(bb + sw128_off(p, c, 2 * TC_N)) = yh;
            *reinterpret_cast<float*>(bb + sw128_off(TC_N + p, c, 2 * TC_N)) = yl;
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(s.bready);
        cur_chunk = chunk;
      }
      for (int k = 0; k < nst; ++k) {
        const bool mine = (gcnt++ & 1) == grp;
        lo_ph[lo_i] ^= 1u;
        if (mine) {
          mbar_wait(&s.full[st], ph);
          mbar_wait(&s.loe[lo_i], lo_ph[lo_i]);  // the MMAs TC_LO conversions back are done
          tc_fence_after();
          // this thread's row r: all 32 columns (8 swizzled 16-byte chunks)
          const uint8_t* row = reinterpret_cast<const uint8_t*>(s.hi + (size_t)st * (TC_TILE / 4)) + r * 128;
          uint32_t lo[32];
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            const float4 x = *reinterpret_cast<const float4*>(row + ((c4 ^ (r & 7)) << 4));
            float h_, l_;
            split_tf32(x.x, h_, l_), lo[4 * c4 + 0] = __float_as_uint(l_);
            split_tf32(x.y, h_, l_), lo[4 * c4 + 1] = __float_as_uint(l_);
            split_tf32(x.z, h_, l_), lo[4 * c4 + 2] = __float_as_uint(l_);
            split_tf32(x.w, h_, l_), lo[4 * c4 + 3] = __float_as_uint(l_);
          }
          const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + TC_LO_COL + (uint32_t)(lo_i * TC_BC);
          tmem_st32(taddr, lo);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s.conv[st]);
        }
        if (++lo_i == TC_LO) lo_i = 0;
        if (++st == TC_STAGES) st = 0, ph ^= 1u;
        // the previous accumulator's epilogue, TC_EPI_LAG stages behind its last MMAs (they
        // have finished by then; the other accumulator keeps the tensor core busy)
        if (pend_chunk >= 0 && ++pend_age > TC_EPI_LAG) {
          if (epi) epilogue();
          pend_chunk = -1;
        }
        if (k % TC_SUB == TC_SUB - 1 || k == nst - 1) {
          if (pend_chunk >= 0) {  // (short items) never more than one accumulator pending
            if (epi) epilogue();
            pend_chunk = -1;
          }
          pend_chunk = chunk, pend_band = band, pend_acc = acc, pend_last = (k == nst - 1);
          pend_age = 0;
          acc ^= 1;
        }
      }
    }
    if (epi && pend_chunk >= 0) epilogue();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TC_TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// Column product for an fp32 M: part[split][col][p] = sum_{i in split} M[i][col] X[i][p]
// (Y-update X^T M, graY, the IPM's M^T dX).  D = M^T X: the UMMA M dimension is 128
// columns of M (TMEM lanes), K runs down the rows.  A stage is 32 rows x 128 columns:
// four TMA boxes of 32 columns x 32 rows (128B swizzle), which is the canonical
// MN-major SW128 operand (LBO = 4 KB between the 32-column boxes, SBO = 1 KB between
// 8-row groups), plus the stage's 32 rows of X by one bulk copy.  Converters (8 warps)
// write Ml (thread = column, 16 rows each) to tensor memory and [Xh | Xl]^T as the
// K-major SW128 B operand of the stage; MMAs per 8 rows: Mh^T [Xh | Xl] (N = 32, A
// MN-major from shared memory) and Ml^T Xh (N = 16, A from tensor memory).  Item =
// (128-column chunk, row split), chunk-major, contiguous per CTA; accumulators flushed to
// fp64 every TC_SUB stages (128 rows) like the row product.
// ---------------------------------------------------------------------------
constexpr int CT_BR = 32;                    // rows per stage (= K per stage)
static_assert(64 + TC_LO * 2 * 32 <= 256, "TMEM columns: accumulators + Mh / Ml buffers");
constexpr int CT_CW = 128;                   // columns per item (UMMA M)
constexpr int CT_TILE = CT_BR * CT_CW * 4;   // 16 KB of M per stage
constexpr int CT_XB = CT_BR * TC_N * 8;      // raw X rows per stage (<= 4 KB)
constexpr int CT_BB = 2 * TC_N * CT_BR * 4;  // [Xh | Xl]^T tile per stage (4 KB)

__host__ __device__ constexpr uint32_t ct_idesc_mn(int n) { return tc_idesc(n) | (1u << 15); }

__device__ __forceinline__ uint64_t umma_desc_mn(uint32_t saddr, uint32_t lbo = 4096u,
                                                  uint32_t sbo = 1024u) {  // MN-major SW128
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}
__device__ __forceinline__ void umma_tf32_mn32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(ct_idesc_mn(2 * TC_N)), "r"(accumulate)
      : "memory");
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    k_colprod_tc(const __grid_constant__ CUtensorMap map, long rows, long cols,
                 const double* __restrict__ X, int K, long nitems, long nsplit, long split_rows,
                 double* __restrict__ part, int dbg) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = su32(smem_raw);
  uint8_t* sp = smem_raw + (((base + 1023u) & ~1023u) - base);
  float* tiles = reinterpret_cast<float*>(sp);                                   // [ST][4 boxes]
  uint8_t* bcat = sp + TC_STAGES * CT_TILE;                                       // [ST][4 KB]
  double* xraw = reinterpret_cast<double*>(sp + TC_STAGES * (CT_TILE + CT_BB));  // [ST][<=4 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sp + TC_STAGES * (CT_TILE + CT_BB + CT_XB));
  uint64_t* full = bars;
  uint64_t* conv = bars + TC_STAGES;
  uint64_t* empty = bars + 2 * TC_STAGES;
  uint64_t* accf = bars + 3 * TC_STAGES;
  uint64_t* acce = accf + 2;
  uint64_t* loe = acce + 2;
  uint32_t* tmem_base = reinterpret_cast<uint32_t*>(loe + TC_LO);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < TC_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&conv[i], 4);  // one converter group per stage
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], 4);
    }
    for (int i = 0; i < TC_LO; ++i) mbar_init(&loe[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_base)),
                 "n"(TC_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base;
  const long i_beg = (long)blockIdx.x * nitems / gridDim.x;
  const long i_end = (long)(blockIdx.x + 1) * nitems / gridDim.x;

  if (warp == 0) {  // ===== TMA producer =====
    if (lane == 0) {
      int st = 0;
      unsigned ph = 0;
      for (long it = i_beg; it < i_end; ++it) {
        const long chunk = it / nsplit, s = it - chunk * nsplit;
        const long rb = s * split_rows, re = min(rows, rb + split_rows);
        for (long r0 = rb; r0 < re; r0 += CT_BR) {
          const bool xfull = r0 + CT_BR <= rows;
          const unsigned xbytes = xfull ? (unsigned)(CT_BR * K * 8) : 0u;
          mbar_wait(&empty[st], ph ^ 1u);
          mbar_expect_tx(&full[st], (unsigned)CT_TILE + xbytes);
          for (int b = 0; b < 4; ++b)
            tma_load_2d(tiles + (size_t)st * (CT_TILE / 4) + b * (CT_BR * 32), &map, &full[st],
                        (int)(chunk * CT_CW + 32 * b), (int)r0);
          if (xfull)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
                "[%3];" ::"r"(su32(xraw + (size_t)st * (CT_XB / 8))),
                "l"(X + r0 * K), "r"(xbytes), "r"(su32(&full[st]))
                : "memory");
          if (++st == TC_STAGES) st = 0, ph ^= 1u;
        }
      }
    }
  } else if (warp == 1) {  // ===== MMA issuer =====
    if (lane == 0) {
      int st = 0, lo_i = 0, acc = 0;
      unsigned ph = 0;
      unsigned aph[2] = {0u, 0u};
      for (long it = i_beg; it < i_end; ++it) {
        const long s = it % nsplit;
        const long rb = s * split_rows, re = min(rows, rb + split_rows);
        const int nst = (int)((re - rb + CT_BR - 1) / CT_BR);
        for (int k0 = 0; k0 < nst; k0 += TC_SUB) {
          mbar_wait(&acce[acc], aph[acc] ^ 1u);
          aph[acc] ^= 1u;
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(acc * 2 * TC_N);
          const int k1 = min(nst, k0 + TC_SUB);
          for (int k = k0; k < k1; ++k) {
            mbar_wait(&conv[st], ph);
            tc_fence_after();
            const uint32_t bt = su32(bcat) + st * CT_BB;
            const uint32_t ah = tmem + TC_LO_COL + (uint32_t)(lo_i * 2 * CT_BR);  // Mh | Ml
#pragma unroll
            for (int kk = 0; kk < CT_BR / 8; ++kk) {
              const uint64_t db = umma_desc(bt + kk * 32);
              umma_tf32_ta<2 * TC_N>(d, ah + kk * 8, db, (k > k0 || kk) ? 1u : 0u);
              if (!(dbg & 1)) umma_tf32_ta<TC_N>(d, ah + CT_BR + kk * 8, db, 1u);
            }
            umma_commit(&empty[st]);
            umma_commit(&loe[lo_i]);
            if (++lo_i == TC_LO) lo_i = 0;
            if (++st == TC_STAGES) st = 0, ph ^= 1u;
          }
          umma_commit(&accf[acc]);
          acc ^= 1;
        }
      }
    }
  } else if (warp >= 4) {  // ===== converters + epilogue =====
    const int ct = threadIdx.x - 128;
    const bool epi = warp < 8;
    const int q = warp & 3;            // TMEM lane quadrant = box of the stage
    const int grp = (warp - 4) >> 2;   // converter group: stages alternate between the two groups
    const int gt = threadIdx.x - 128 - 128 * grp;  // thread within the group (0..127)
    unsigned gcnt = 0;
    int st = 0, lo_i = 0, acc = 0;
    unsigned ph = 0;
    unsigned lo_ph[TC_LO] = {};
    unsigned aph[2] = {0u, 0u};
    double a64[TC_N];
    long pend_chunk = -1, pend_s = -1;
    int pend_acc = 0, pend_age = 0;
    bool pend_last = false;
    auto epilogue = [&]() {
      const int a = pend_acc;
      mbar_wait(&accf[a], aph[a]);
      aph[a] ^= 1u;
      tc_fence_after();
      uint32_t v[2 * TC_N];
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * 2 * TC_N);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
          "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
            "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
            "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
            "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[a]);
#pragma unroll
      for (int p = 0; p < TC_N; ++p)
        a64[p] += (double)__uint_as_float(v[p]) + (double)__uint_as_float(v[TC_N + p]);
      if (pend_last) {
        const long col = pend_chunk * CT_CW + 32 * q + lane;
        if (col < cols) {
          double* dst = part + (pend_s * cols + col) * K;
#pragma unroll
          for (int p = 0; p < TC_N; ++p)
            if (p < K) dst[p] = a64[p];
        }
#pragma unroll
        for (int p = 0; p < TC_N; ++p) a64[p] = 0.0;
      }
    };
#pragma unroll
    for (int p = 0; p < TC_N; ++p) a64[p] = 0.0;
    for (long it = i_beg; it < i_end; ++it) {
      const long chunk = it / nsplit, s = it - chunk * nsplit;
      const long rb = s * split_rows, re = min(rows, rb + split_rows);
      const int nst = (int)((re - rb + CT_BR - 1) / CT_BR);
      for (int k = 0; k < nst; ++k) {
        const long r0 = rb + (long)k * CT_BR;
        const bool mine = (gcnt++ & 1) == grp;
        lo_ph[lo_i] ^= 1u;
        if (mine) {
          mbar_wait(&full[st], ph);
          mbar_wait(&loe[lo_i], lo_ph[lo_i]);
          tc_fence_after();
          // Mh / Ml: this thread's column (lane of box q), the stage's 32 rows
          const uint8_t* box = reinterpret_cast<const uint8_t*>(tiles + (size_t)st * (CT_TILE / 4)) +
                               q * (CT_BR * 128);
          uint32_t hi[32], lo[32];
#pragma unroll
          for (int r = 0; r < CT_BR; ++r) {
            const float x = *reinterpret_cast<const float*>(
                box + r * 128 + ((((lane >> 2) ^ (r & 7)) << 4) | ((lane & 3) << 2)));
            float h_, l_;
            split_tf32(x, h_, l_);
            hi[r] = __float_as_uint(h_);
            lo[r] = __float_as_uint(l_);
          }
          const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + TC_LO_COL +
                                 (uint32_t)(lo_i * 2 * CT_BR);
          tmem_st32(taddr, hi);
          tmem_st32(taddr + CT_BR, lo);
          // [Xh | Xl]^T: B operand rows p (hi) and 16 + p (lo), K = the stage's 32 rows
          const double* xs = xraw + (size_t)st * (CT_XB / 8);
          const bool xfull = r0 + CT_BR <= rows;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = gt + 128 * u;  // (r, p), p fastest
            const int r = e >> 4, p = e & 15;
            double xv = 0.0;
            if (p < K) xv = xfull ? xs[r * K + p] : (r0 + r < rows ? __ldg(X + (r0 + r) * K + p) : 0.0);
            const float xh = __uint_as_float(__float_as_uint((float)xv) & 0xFFFFE000u);
            const float xl = (float)(xv - (double)xh);
            uint8_t* bb = bcat + st * CT_BB;
            *reinterpret_cast<float*>(bb + sw128_off(p, r, 2 * TC_N)) = xh;
            *reinterpret_cast<float*>(bb + sw128_off(TC_N + p, r, 2 * TC_N)) = xl;
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          fence_async_smem();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv[st]);
        }
        if (++lo_i == TC_LO) lo_i = 0;
        if (++st == TC_STAGES) st = 0, ph ^= 1u;
        if (pend_chunk >= 0 && ++pend_age > TC_EPI_LAG) {
          if (epi) epilogue();
          pend_chunk = -1;
        }
        if (k % TC_SUB == TC_SUB - 1 || k == nst - 1) {
          if (pend_chunk >= 0) {
            if (epi) epilogue();
            pend_chunk = -1;
          }
          pend_chunk = chunk, pend_s = s, pend_acc = acc, pend_last = (k == nst - 1);
          pend_age = 0;
          acc ^= 1;
        }
      }
    }
    if (epi && pend_chunk >= 0) epilogue();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TC_TMEM_COLS)
                 : "memory");
  }
}

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

int num_sms() {
  static int sms = [] {
    int d = 0, v = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return v > 0 ? v : 148;
  }();
  return sms;
}

}  // namespace

static int g_tc_prod = -1;

bool tc_prod_enabled() {
  if (g_tc_prod < 0) {
    const char* e = getenv("NMFB_TC_PROD");
    g_tc_prod = (e && e[0] == '0') ? 0 : 1;
  }
  return g_tc_prod != 0;
}

extern "C" int nmfb_tc_products(int on) {
  const int prev = tc_prod_enabled() ? 1 : 0;
  if (on >= 0) g_tc_prod = on ? 1 : 0;
  return prev;
}

static CUtensorMapL2promotion tc_promo() {
  static const CUtensorMapL2promotion p = [] {
    const char* e = getenv("NMFB_TC_L2P");  // L2 fetch granularity (default 256 B)
    const int v = e ? atoi(e) : 256;
    return v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
         : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
         : v == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                    : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  }();
  return p;
}

int tc_rowprod_f32(const float* A, long rows, long cols, const double* B, int K, double* work,
                   long work_len, long* nparts, cudaStream_t st) {
  if (!tc_prod_enabled() || K < 1 || K > TC_N || (uintptr_t)A % 16 || cols % 4 ||
      rows >= (1L << 31) || cols >= (1L << 31))
    return NMFB_EUNSUPPORTED;
  const long nch = (cols + TC_RP_CW - 1) / TC_RP_CW;
  if (nch * rows * K > work_len) return NMFB_ENOMEM;
  auto fn = encode_fn();
  if (!fn) return NMFB_EUNSUPPORTED;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(float)};
  const cuuint32_t box[2] = {TC_BC, TC_BR};
  const cuuint32_t es[2] = {1, 1};
  if (fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)A, dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, tc_promo(),
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return NMFB_EUNSUPPORTED;
  const long nbands = (rows + TC_BR - 1) / TC_BR;
  const long nitems = nch * nbands;
  const int grid = (int)min((long)num_sms(), nitems);
  const size_t smem = 1024 + TC_STAGES * TC_TILE + 2 * (size_t)TC_RP_CW * TC_N * 4 + 256;
  nmfb_smem_attr(k_rowprod_tc, smem);
  ++g_nmfb_launches, k_rowprod_tc<<<grid, TC_THREADS, smem, st>>>(map, rows, cols, B, K, nitems,
                                                                  nbands, work);
  *nparts = nch;
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}

int tc_colprod_f32(const float* A, long rows, long cols, const double* X, int K, double* work,
                   long work_len, long* nparts, cudaStream_t st) {
  if (!tc_prod_enabled() || K < 1 || K > TC_N || (uintptr_t)A % 16 || (uintptr_t)X % 16 ||
      cols % 4 || rows >= (1L << 31) || cols >= (1L << 31))
    return NMFB_EUNSUPPORTED;
  const long nch = (cols + CT_CW - 1) / CT_CW;
  // about 8 items per CTA, splits of whole 128-row accumulator runs
  long want = (8L * num_sms() + nch - 1) / nch;
  if (want < 1) want = 1;
  long sr = (rows + want - 1) / want;
  sr = ((sr + 4 * CT_BR - 1) / (4 * CT_BR)) * (4 * CT_BR);
  const long ns = (rows + sr - 1) / sr;
  if (ns * cols * K > work_len) return NMFB_ENOMEM;
  auto fn = encode_fn();
  if (!fn) return NMFB_EUNSUPPORTED;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(float)};
  const cuuint32_t box[2] = {32, CT_BR};
  const cuuint32_t es[2] = {1, 1};
  if (fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)A, dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return NMFB_EUNSUPPORTED;
  const long nitems = nch * ns;
  const int grid = (int)min((long)num_sms(), nitems);
  const size_t smem = 1024 + TC_STAGES * (CT_TILE + CT_BB + CT_XB) + 256;
  nmfb_smem_attr(k_colprod_tc, smem);
  static const int dbg = [] {
    const char* e = getenv("NMFB_CT_DBG");
    return e ? atoi(e) : 0;
  }();
  ++g_nmfb_launches, k_colprod_tc<<<grid, TC_THREADS, smem, st>>>(map, rows, cols, X, K, nitems, ns,
                                                                  sr, work, dbg);
  *nparts = ns;
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}
