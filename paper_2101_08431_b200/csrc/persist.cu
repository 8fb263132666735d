// Persistent interior-point inner loop for small problems (configs c1-c3).
//
// csrc/small.cu runs one Gauss-Newton iteration as six kernels replayed from a
// CUDA graph, with one host synchronisation per iteration; at c2 sizes every
// launch is latency-bound.  Here ONE cooperative launch runs the whole inner
// loop of Algorithm 2 (PAPER Alg. 2 / SPEC.md:337-345: direction -> Armijo ->
// nudged update -> gradients/KKT, repeated while E(.;mu) > eps_mu):
//
//   * every CTA owns a contiguous block of rows of M (kept in shared memory
//     when it fits), X, R, graX and the row factors L_i, h_i;
//   * the Y side (m x k: Y, S, graY, dY, D_j^{-1}) and every k/k^2-sized object
//     are replicated in every CTA's shared memory and computed redundantly with
//     identical arithmetic, so all CTAs take the same branch without a broadcast;
//   * cross-CTA sums are written as per-CTA partials and, after a grid barrier,
//     reduced by every CTA in a fixed lane/CTA order (bit-identical everywhere);
//   * four grid barriers per iteration: R1/Z partials | direction + quartic
//     partials | barrier-trial partials (8 trials per batch, batches only while
//     Armijo keeps backtracking) | residual + graY partials.
//
// Exits (status): 0 inner loop done (E(.;mu) <= eps_mu or the iteration budget),
// 1 factorization failure at the current point (no step taken; the host redoes
// the iteration eagerly with the dense Schur system or raises), 2 Armijo stall.
// The state left in global memory is what the host path leaves after the same
// iterations: X, R, graX, Y, S, graY, F (into Fout), R1 factors L, the
// factorization copy (Xf, Ytf) and the low-rank factors (LD, LG, LH, Zb) for the
// predictor, and the KKT sums at sc[16..27], ||F||^2 at sc[0].
#include <cooperative_groups.h>

#include "common.cuh"
#include "nmfb200.h"

namespace {

constexpr int PT = 256;      // threads per CTA
constexpr int NW = PT / 32;  // warps per CTA
constexpr int TB = 8;        // barrier trials per batch
constexpr int LOGW = 8;      // doubles per iteration record
static_assert(TB == NW, "one warp per barrier trial");

struct PArgs {
  const void* M;
  long n, m;
  double *X, *R, *gX, *Yt, *S, *gY, *Fout, *L, *Xf, *Ytf, *LD, *LG, *LH, *Zb;
  double *sc, *logv, *work;
  int *fcodes, *status;
  unsigned int* bar;
  double mu, wx, wy, rho, tau, eta, eps_mu, tol0;
  int max_bt, ntrials, max_iters, m_in_smem;
  long long* prof;  // optional per-iteration phase clocks of CTA 0 (16 per iteration)
};

// all lanes of warp 0 store the same stamp: no intra-warp divergence (a lane-0-only
// store left the warp diverged at the next shuffles and distorted what it measured)
#define STAMP(i)                                                            \
  do {                                                                      \
    if (a.prof && blockIdx.x == 0 && threadIdx.x < 32 && it < 4096)         \
      a.prof[(long)it * 40 + (i)] = clock64();                              \
  } while (0)

// Grid barrier: cooperative-groups grid sync (measured on B200 with 148 CTAs:
// 1.3 us, against 1.8 us for an atomic counter and 2.8 us for per-CTA flags polled
// by every CTA; scripts/micro/bar.cu).  `epoch` counts barriers (debugging aid).
__device__ __forceinline__ void grid_barrier(unsigned* flags, unsigned& epoch) {
  (void)flags;
  ++epoch;
  cooperative_groups::this_grid().sync();
}

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

// Reduce entries [e0, e1) of an entry-major partial array part[e * G + c] over
// the G CTAs: warp w takes chunks of EB consecutive entries, each lane issues all
// of its loads (CTAs lane, lane+32, ..) before reducing; fixed order -> the same
// bits in every lane of every CTA.  kind 0 sum, 1 min, 2 max.  G <= 160.
template <int KD>
__device__ __forceinline__ double op2(double a, double b) {
  return KD == 0 ? a + b : (KD == 1 ? fmin(a, b) : fmax(a, b));
}
template <int KD>
__device__ __forceinline__ double warp_op(double v) {
  return KD == 0 ? warp_sum(v) : (KD == 1 ? warp_min(v) : warp_max(v));
}
template <int KD>
__device__ __forceinline__ double op_id() {
  return KD == 0 ? 0.0 : (KD == 1 ? 1.0 / 0.0 : -1.0 / 0.0);
}

template <int EB, int KD>
__device__ __forceinline__ void reduce_entries(const double* part, int G, long e0, long e1,
                                               double* out, bool out_global = false) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll 1
  for (long eb = e0 + (long)wid * EB; eb < e1; eb += (long)NW * EB) {
    double v[EB][5];
#pragma unroll
    for (int b = 0; b < EB; ++b)
#pragma unroll
      for (int u = 0; u < 5; ++u) {
        const int c = lane + 32 * u;
        v[b][u] = (eb + b < e1 && c < G) ? ldcg(part + (eb + b) * G + c) : op_id<KD>();
      }
    __syncwarp();
    double s[EB];
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      s[b] = v[b][0];
#pragma unroll
      for (int u = 1; u < 5; ++u) s[b] = op2<KD>(s[b], v[b][u]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // level-major: the EB shuffles issue together
      double t[EB];
#pragma unroll
      for (int b = 0; b < EB; ++b) t[b] = __shfl_xor_sync(0xffffffffu, s[b], o);
#pragma unroll
      for (int b = 0; b < EB; ++b) s[b] = op2<KD>(s[b], t[b]);
    }
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      if (lane == 0 && eb + b < e1) {
        if (out_global)
          __stcg(out + (eb + b - e0), s[b]);
        else
          out[eb + b - e0] = s[b];
      }
    }
  }
}

// As reduce_entries, with the reduction kind chosen per entry (kind_of(e): 0 sum,
// 1 min, 2 max) so differently-typed partials share one round trip to L2.
template <int EB, typename KF, bool OUTG = false>
__device__ __forceinline__ void reduce_mixed(const double* part, int G, long e0, long e1,
                                             double* out, KF kind_of, int warp_lo = 0,
                                             int warp_n = NW) {
  const int lane = threadIdx.x & 31, wid = (threadIdx.x >> 5) - warp_lo;
  if (wid < 0 || wid >= warp_n) return;
#pragma unroll 1
  for (long eb = e0 + (long)wid * EB; eb < e1; eb += (long)warp_n * EB) {
    double v[EB][5];
    int kd[EB];
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      kd[b] = (eb + b < e1) ? kind_of(eb + b) : 0;
      const double idv = kd[b] == 0 ? 0.0 : (kd[b] == 1 ? 1.0 / 0.0 : -1.0 / 0.0);
#pragma unroll
      for (int u = 0; u < 5; ++u) {
        const int c = lane + 32 * u;
        v[b][u] = (eb + b < e1 && c < G) ? ldcg(part + (eb + b) * G + c) : idv;
      }
    }
    __syncwarp();
    double s[EB];
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      s[b] = v[b][0];
#pragma unroll
      for (int u = 1; u < 5; ++u)
        s[b] = kd[b] == 0 ? s[b] + v[b][u] : (kd[b] == 1 ? fmin(s[b], v[b][u]) : fmax(s[b], v[b][u]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // level-major: the EB shuffles issue together
      double t[EB];
#pragma unroll
      for (int b = 0; b < EB; ++b) t[b] = __shfl_xor_sync(0xffffffffu, s[b], o);
#pragma unroll
      for (int b = 0; b < EB; ++b)
        s[b] = kd[b] == 0 ? s[b] + t[b] : (kd[b] == 1 ? fmin(s[b], t[b]) : fmax(s[b], t[b]));
    }
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      if (lane == 0 && eb + b < e1) {
        if (OUTG)
          __stcg(out + (eb + b - e0), s[b]);
        else
          out[eb + b - e0] = s[b];
      }
    }
  }
}

// Cholesky of a Q x Q smem matrix by warp 0 with the rows in registers (lane = row,
// column j broadcast by shuffles); the strict upper triangle is zeroed and the
// reciprocal diagonal 1/L_jj stored in dinv[Q].  Returns the failing pivot (-1: PD)
// in every lane of warp 0.
// (compile-time recursion keeps every row element in a register even where the
// unroller would give up inside this large kernel)
template <int J, int C, int Q>
struct CholUpd {
  static __device__ __forceinline__ void run(double (&a)[Q], int r) {
    const double lcj = __shfl_sync(0xffffffffu, a[J], C);
    const double upd = a[C] - a[J] * lcj;
    a[C] = (r >= C) ? upd : a[C];
    CholUpd<J, C + 1, Q>::run(a, r);
  }
};
template <int J, int Q>
struct CholUpd<J, Q, Q> {
  static __device__ __forceinline__ void run(double (&)[Q], int) {}
};
template <int J, int Q>
struct CholStep {
  static __device__ __forceinline__ void run(double (&a)[Q], int r, int& fail, double& di_r) {
    double pv = __shfl_sync(0xffffffffu, a[J], J);
    if (fail < 0 && !(pv > 0.0)) fail = J;  // continue on a dummy pivot after a failure
    if (fail >= 0) pv = 1.0;
    const double di = rsqrt(pv);
    // selects, not branches: the warp stays converged for the shuffles
    a[J] = (r == J) ? pv * di : ((r > J) ? a[J] * di : a[J]);
    di_r = (r == J) ? di : di_r;
    CholUpd<J, J + 1, Q>::run(a, r);
    CholStep<J + 1, Q>::run(a, r, fail, di_r);
  }
};
template <int Q>
struct CholStep<Q, Q> {
  static __device__ __forceinline__ void run(double (&)[Q], int, int&, double&) {}
};

template <int Q>
__device__ __forceinline__ int warp_chol(double* A, double* dinv) {
  const int r = threadIdx.x & 31;
  __syncwarp();
  double a[Q];
#pragma unroll
  for (int c = 0; c < Q; ++c) a[c] = (r < Q) ? A[r * Q + c] : 0.0;
  int fail = -1;
  double di_r = 0.0;
  CholStep<0, Q>::run(a, r, fail, di_r);
  if (r < Q) {
#pragma unroll
    for (int c = 0; c < Q; ++c) A[r * Q + c] = (c <= r) ? a[c] : 0.0;
    dinv[r] = di_r;
  }
  return fail;
}

// Block reductions of NV values with the result in EVERY thread (fixed order).
// Value q is min-reduced if bit q of MINM is set, max-reduced for MAXM, else summed.
// The warp stage is level-major so the NV independent shuffles of a level issue
// back to back (value-major chains ran one after another: 1.5 us for 9 values);
// per value the arithmetic is warp_sum / warp_min / warp_max's exactly.
template <int NV, int MINM, int MAXM>
__device__ __forceinline__ void warp_reduce_multi(double (&v)[NV]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double t[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) t[q] = __shfl_xor_sync(0xffffffffu, v[q], o);
#pragma unroll
    for (int q = 0; q < NV; ++q)
      v[q] = ((MINM >> q) & 1) ? fmin(v[q], t[q]) : (((MAXM >> q) & 1) ? fmax(v[q], t[q]) : v[q] + t[q]);
  }
}

// Warp stage of block_reduce_all: recursive halving over NP = 2^LG >= NV slots
// (at offset o a lane keeps one half of its slots and ships the other half to lane
// ^ o), then plain butterflies over the remaining lane bits: NP - 1 + 5 - LG
// shuffles instead of 5 NV.  Afterwards lane l holds the warp total of value
// (l >> (5 - LG)) in v[0].  Deterministic and identical in every CTA.
template <int NV, int MINM, int MAXM>
struct WarpHalve {
  static constexpr int LG = NV <= 1 ? 0 : NV <= 2 ? 1 : NV <= 4 ? 2 : NV <= 8 ? 3 : NV <= 16 ? 4 : 5;
  static constexpr int NP = 1 << LG;
  static __device__ __forceinline__ double opk(int idx, double a, double b) {
    return ((MINM >> idx) & 1) ? fmin(a, b) : (((MAXM >> idx) & 1) ? fmax(a, b) : a + b);
  }
  static __device__ __forceinline__ double run(const double (&in)[NV]) {
    const int lane = threadIdx.x & 31;
    double v[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) v[q] = q < NV ? in[q] : 0.0;
    int base = 0;
#pragma unroll
    for (int st = 0; st < LG; ++st) {
      const int o = 16 >> st, c = NP >> (st + 1);  // slots kept after this step
      const bool up = (lane & o) != 0;
      if (up) base += c;
#pragma unroll
      for (int i = 0; i < c; ++i) {
        const double send = up ? v[i] : v[i + c];
        const double keep = up ? v[i + c] : v[i];
        const double recv = __shfl_xor_sync(0xffffffffu, send, o);
        v[i] = opk(base + i, keep, recv);
      }
    }
#pragma unroll
    for (int o = 16 >> LG; o > 0; o >>= 1) v[0] = opk(base, v[0], __shfl_xor_sync(0xffffffffu, v[0], o));
    return v[0];
  }
};

// Block reduction of NV values with the result in EVERY thread (fixed order).
// Value q is min-reduced if bit q of MINM is set, max-reduced for MAXM, else summed.
// sh: two buffers of 16 NW + 16 doubles, alternated by `phase` (every thread toggles it
// identically): a buffer is rewritten two reductions later, after the intermediate
// reduction's barriers, which every thread reaches only once it has read it.
// (The previous form - value-major warp_sum chains, then every thread folding all
// NV x NW warp partials - was bound by shuffle and LDS issue: 1.5 us for 9 values.)
template <int NV, int MINM = 0, int MAXM = 0>
__device__ __forceinline__ void block_reduce_all(double (&v)[NV], double* sh, int& phase) {
  static_assert(NV <= 16, "block_reduce_all: NV <= 16");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  using WH = WarpHalve<NV, MINM, MAXM>;
  double* b = sh + phase * (16 * NW + 16);
  double* res = b + 16 * NW;
  phase ^= 1;
  __syncwarp();
  const double wv = WH::run(v);
  constexpr int SH = 5 - WH::LG;
  const int idx = lane >> SH;
  if ((lane & ((1 << SH) - 1)) == 0 && idx < NV) b[idx * NW + wid] = wv;
  __syncthreads();
  if (threadIdx.x < NV) {
    const int q = threadIdx.x;
    double r = b[q * NW];
#pragma unroll
    for (int w = 1; w < NW; ++w) r = WH::opk(q, r, b[q * NW + w]);
    res[q] = r;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = res[q];
}

__device__ __forceinline__ int pk(int a, int b, int k) {
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
  return a * k - a * (a - 1) / 2 + (b - a);
}

// Cholesky of a K x K SPD matrix in registers (lower), ok flag; small.cu order.
// rd[j] = 1 / L[j][j] (one rsqrt per pivot): every later "/ L[j][j]" of the row and
// column factors becomes a multiply, which takes the IEEE division sequences (and
// their slow-path calls) off the per-iteration dependency chains.
template <int K>
__device__ __forceinline__ bool reg_chol(double (&L)[K][K], double (&rd)[K]) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double s = L[j][j];
#pragma unroll
    for (int p = 0; p < j; ++p) s -= L[j][p] * L[j][p];
    if (!(s > 0.0)) ok = false;
    const double sp = fmax(s, 1e-300);
    const double di = rsqrt(sp);
    L[j][j] = sp * di;
    rd[j] = di;
#pragma unroll
    for (int r = j + 1; r < K; ++r) {
      double t = L[r][j];
#pragma unroll
      for (int p = 0; p < j; ++p) t -= L[r][p] * L[j][p];
      L[r][j] = t * di;
    }
  }
  return ok;
}

template <int K>
__device__ __forceinline__ void reg_inv_lower(const double (&L)[K][K], const double (&rd)[K],
                                              double (&Li)[K][K]) {
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
}

template <int K>
__device__ __forceinline__ void reg_solve(const double (&L)[K][K], const double (&rd)[K],
                                          const double (&b)[K], double (&out)[K]) {
  double z[K];
#pragma unroll
  for (int a = 0; a < K; ++a) {
    double s = b[a];
#pragma unroll
    for (int p = 0; p < a; ++p) s -= L[a][p] * z[p];
    z[a] = s * rd[a];
  }
#pragma unroll
  for (int a = K - 1; a >= 0; --a) {
    double s = z[a];
#pragma unroll
    for (int p = a + 1; p < K; ++p) s -= L[p][a] * out[p];
    out[a] = s * rd[a];
  }
}

__device__ __forceinline__ double nudge(double old, double d, double a, double tau) {
  const double nv = old + a * d;
  return (nv > 0.0) ? nv : (1.0 - tau) * old;
}

// per-CTA workspace layout (doubles) in PArgs::work
struct WLayout {
  long pa, pb, pc, pd, pg, total;
};
__host__ __device__ inline WLayout wlayout(long G, long m, int K) {
  const long KK = K * (K + 1) / 2, N = m * K;
  WLayout w;
  const long sa = KK * KK + 2 * K * K + 1;
  w.pa = 0;
  w.pb = w.pa + G * sa;
  w.pc = w.pb + G * (9 + 2 * TB);  // 9 direction/quartic sums + the speculative trial batch
  w.pd = w.pc + 2 * G * 2 * TB;
  w.pg = w.pd + G * 8;
  w.total = w.pg + G * N;
  return w;
}

template <int K>
__host__ __device__ inline long smem_doubles(long nrm, long m, bool with_m) {
  const long KK = K * (K + 1) / 2, N = m * K;
  long d = 4 * N + m * KK + nrm * (10 * K + 2 * K * K + KK);  // + double-buffered row-factor snapshots
  if (with_m) d += nrm * m;
  return d;
}

template <int K, typename T>
__global__ void __launch_bounds__(PT, 1) k_ipm_persist(PArgs a) {
  constexpr int KK = K * (K + 1) / 2, Q = K * K;
  constexpr int SA = KK * KK + 2 * K * K + 1;  // phase-A partial stride
  const long n = a.n, m = a.m, N = m * K;
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const long r0 = (long)cta * n / G, r1 = (long)(cta + 1) * n / G;
  const int nr = (int)(r1 - r0);
  const long nrm = (n + G - 1) / G;
  // this CTA's slice of the m k Y-side entries (barrier trials, graY totals)
  const long y0 = (long)cta * (m * K) / G, y1 = (long)(cta + 1) * (m * K) / G;
  const double mux = a.wx * a.mu, muy = a.wy * a.mu;
  // column-per-thread passes over the own rows: q_rs threads per column when m < PT
  const int q_rs = m >= PT ? 1 : PT / (int)m;
  const long q_j0 = m >= PT ? tid : tid % (int)m;
  const int q_roff = m >= PT ? 0 : tid / (int)m;
  const WLayout wl = wlayout(G, m, K);
  double* PA = a.work + wl.pa;
  double* PB = a.work + wl.pb;
  double* PC = a.work + wl.pc;
  double* PD = a.work + wl.pd;
  double* PG = a.work + wl.pg;

  extern __shared__ double sm[];
  double* Ys = sm;
  double* Ss = Ys + N;
  double* gYs = Ss + N;
  double* Ts = gYs + N;  // t_j, then dY
  double* dinv = Ts + N;
  // Y-side arrays live in shared memory component-major (SoA: entry (j, p) at p m + j)
  // so lanes striding j read consecutive words; global Y^T / S / graY stay (m, k)
  // row-major.  dinv (packed D_j^{-1}) likewise: entry (j, c) at c m + j.
#define YI(j, p) ((long)(p) * m + (j))
#define DI(j, c) ((long)(c) * m + (j))
  double* xs = dinv + m * KK;
  double* rs = xs + nrm * K;
  double* gxs = rs + nrm * K;
  double* dxs = gxs + nrm * K;
  double* drs = dxs + nrm * K;
  double* hs = drs + nrm * K;
  double* gs = hs + nrm * K;
  // row factors and the factorization point (X rows, Y) double-buffered by iteration
  // parity: the last step's factorization is committed to global memory once, at exit
  double* Lsb = gs + nrm * K;
  double* xsnap = Lsb + 2 * nrm * K * K;
  double* As = xsnap + 2 * nrm * K;
  double* rds = As + nrm * KK;  // 1 / L_i,pp of the row factors
  double* Ms = rds + nrm * K;   // own rows of M (when m_in_smem)

  __shared__ double ZHX[SA];  // Z (packed kk x kk), H, X^T X, failing R1 row
  double* Zs = ZHX;
  double* Hs = Zs + KK * KK;
  double* XtXs = Hs + K * K;
  __shared__ double Gdy[K * K], gy[K * K], dGi[Q], dHi[Q];
  __shared__ double Gm[Q * Q], Zbm[Q * Q], T1[Q * Q], Hm[Q * Q], u[Q], w[Q];
  __shared__ double red[2 * (16 * NW + 16)];
  int rph = 0;  // block_reduce_all buffer phase
  __shared__ double scal[24];  // [0..2] ysc, [3..5] gtp,a1max,a2max, [6..11] quartic
  __shared__ double kx[8];     // X-part KKT sums + fsq (after phase E)
  __shared__ double bars[2 * TB];
  __shared__ double pbv[9 + 2 * TB];  // reduced phase-B partials (+ speculative trial sums)
  __shared__ int s_fail, s_t;
  __shared__ int ia[KK], ic[KK];

  // ---- load the state --------------------------------------------------------
  #pragma unroll 1
  for (int e = tid; e < KK; e += PT) {
    for (int p = 0; p < K; ++p)
      for (int q = p; q < K; ++q)
        if (pk(p, q, K) == e) {
          ia[e] = p;
          ic[e] = q;
        }
  }
  #pragma unroll 1
  for (long e = tid; e < N; e += PT) {
    const long so = YI(e / K, e % K);
    Ys[so] = a.Yt[e];
    Ss[so] = a.S[e];
    gYs[so] = a.gY[e];
  }
  #pragma unroll 1
  for (long e = tid; e < (long)nr * K; e += PT) {
    xs[e] = a.X[r0 * K + e];
    rs[e] = a.R[r0 * K + e];
    gxs[e] = a.gX[r0 * K + e];
  }
  const T* Mg = (const T*)a.M;
  if (a.m_in_smem)
    #pragma unroll 1
    for (long e = tid; e < (long)nr * m; e += PT) Ms[e] = (double)Mg[r0 * m + e];
  __syncthreads();
  // own rows of M through one generic pointer (shared memory when staged, else the
  // fp64 global rows; the host only allows fp32 M when it is staged)
  const double* Mp = a.m_in_smem ? Ms : (const double*)a.M + r0 * m;

  // Partial barrier sums of trial tq over this CTA's x entries and its slice of y
  // (warp-uniform tq; lanes stride the entries).  (2^-t a1m num) / den ==
  // 2^-t ((a1m num) / den) exactly, so one division per entry gives the oracle's
  // (alpha dv) / v bit for bit.
  auto trial_sums = [&](int tq, double a1m, double& ax, double& ay) {
    ax = 0.0;
    ay = 0.0;
    if (tq < a.ntrials) {
      #pragma unroll 1
      for (long e = lane; e < (long)nr * K; e += 32) ax += log1p(ldexp((a1m * dxs[e]) / xs[e], -tq));
      #pragma unroll 1
      for (long e = y0 + lane; e < y1; e += 32) ay += log1p(ldexp((a1m * Ts[e]) / Ys[e], -tq));
    }
    double axy[2] = {ax, ay};
    warp_reduce_multi<2, 0, 0>(axy);
    ax = axy[0];
    ay = axy[1];
  };

  unsigned epoch = 0;
  int it = 0;
  int status = 0;
  int fact_it = -1;  // iteration whose factorization (L, X rows, Y) is committed at exit
  for (;;) {
    // ======== phase A: rows -> R1 factors, h, g; partials of Z, H, X^T X ========
    STAMP(0);
    double* Ls = Lsb + (long)(it & 1) * nrm * K * K;
    {
      double* xsn = xsnap + (long)(it & 1) * nrm * K;
      #pragma unroll 1
      for (long e = tid; e < (long)nr * K; e += PT) xsn[e] = xs[e];
    }
    #pragma unroll 1
    for (int e = wid; e < K * K; e += NW) {
      const int p = e / K, q = e % K;
      double s = 0.0;
      #pragma unroll 1
      for (long j = lane; j < m; j += 32) s = fma(Ys[YI(j, p)], Ys[YI(j, q)], s);
      s = warp_sum(s);
      if (lane == 0) gy[e] = s;
    }
    __syncthreads();
    STAMP(33);
    double badA = 1.0 / 0.0;
    #pragma unroll 1
    for (int rr = tid; rr < nr; rr += PT) {
      const long i = r0 + rr;
      double x[K], L[K][K], b[K], hv[K], gv[K];
#pragma unroll
      for (int p = 0; p < K; ++p) x[p] = xs[rr * K + p];
#pragma unroll
      for (int p = 0; p < K; ++p)
#pragma unroll
        for (int c = 0; c < K; ++c) L[p][c] = (c <= p) ? gy[p * K + c] : 0.0;
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const double ix = 1.0 / x[p];
        L[p][p] += a.rho + rs[rr * K + p] * ix;
        b[p] = mux * ix - gxs[rr * K + p];
      }
      double rd[K];
      if (!reg_chol<K>(L, rd)) badA = fmin(badA, (double)i);
#pragma unroll
      for (int p = 0; p < K; ++p) {
        double s = b[p];
#pragma unroll
        for (int q = 0; q < p; ++q) s -= L[p][q] * hv[q];
        hv[p] = s * rd[p];
      }
#pragma unroll
      for (int p = K - 1; p >= 0; --p) {
        double s = hv[p];
#pragma unroll
        for (int q = p + 1; q < K; ++q) s -= L[q][p] * gv[q];
        gv[p] = s * rd[p];
      }
      double Li[K][K];
      reg_inv_lower<K>(L, rd, Li);
#pragma unroll
      for (int p = 0; p < K; ++p) {
        rds[rr * K + p] = rd[p];
        hs[rr * K + p] = hv[p];
        gs[rr * K + p] = gv[p];
#pragma unroll
        for (int c = 0; c < K; ++c) Ls[(rr * K + p) * K + c] = (c <= p) ? L[p][c] : 0.0;
#pragma unroll
        for (int c = p; c < K; ++c) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < K; ++q)
            if (q >= c) s = fma(Li[q][p], Li[q][c], s);
          As[rr * KK + (p * K - p * (p - 1) / 2 + (c - p))] = s;
        }
      }
    }
    STAMP(31);
    {
      double v[1] = {badA};
      block_reduce_all<1, 1, 0>(v, red, rph);
      badA = v[0];
    }
    STAMP(32);
    #pragma unroll 1
    for (int e = tid; e < SA; e += PT) {
      double s = 0.0;
      if (e < KK * KK) {
        const int ab = e / KK, pq = e % KK;
        const int p = ia[pq], q = ic[pq];
        #pragma unroll 1
        for (int rr = 0; rr < nr; ++rr) s = fma(As[rr * KK + ab], xs[rr * K + p] * xs[rr * K + q], s);
      } else if (e < KK * KK + K * K) {
        const int qq = e - KK * KK, p = qq / K, c = qq % K;
        #pragma unroll 1
        for (int rr = 0; rr < nr; ++rr) s = fma(xs[rr * K + p], gs[rr * K + c], s);
      } else if (e < KK * KK + 2 * K * K) {
        const int qq = e - KK * KK - K * K, p = qq / K, c = qq % K;
        #pragma unroll 1
        for (int rr = 0; rr < nr; ++rr) s = fma(xs[rr * K + p], xs[rr * K + c], s);
      } else {
        s = badA;
      }
      __stcg(PA + (long)e * G + cta, s);
    }
    STAMP(1);
    grid_barrier(a.bar, epoch);
    STAMP(2);

    // ======== phase B: decision, Y side, row directions, quartic partials ========
    {
      constexpr int NGY = (2048 + PT - 1) / PT;
      double gyv[NGY];
      if (it > 0) {
#pragma unroll
        for (int q = 0; q < NGY; ++q) {
          const long e = tid + (long)q * PT;
          gyv[q] = e < N ? ldcg(a.gY + e) : 0.0;
        }
      }
      constexpr int EBA = (SA + NW - 1) / NW < 8 ? (SA + NW - 1) / NW : 8;
      reduce_mixed<EBA>(PA, G, 0, SA, ZHX, [&](long e) { return e == SA - 1 ? 1 : 0; });
      if (it > 0) {
#pragma unroll
        for (int q = 0; q < NGY; ++q) {
          const long e = tid + (long)q * PT;
          if (e < N) gYs[YI(e / K, e % K)] = gyv[q];
        }
      }
    }
    __syncthreads();
    STAMP(16);
    if (it > 0) {
      // KKT sums at the current point: X part from phase E, Y part replicated
      double v[6] = {0.0, 0.0, 0.0, 0.0, -1.0 / 0.0, -1.0 / 0.0};
      #pragma unroll 1
      for (long e = tid; e < N; e += PT) {
        const double y = Ys[e], s = Ss[e], g = gYs[e];
        const double ys = y * s;
        v[0] = fma(g - s, g - s, v[0]);
        v[1] = fma(ys - muy, ys - muy, v[1]);
        v[2] = fma(ys, ys, v[2]);
        v[3] += ys;
        v[4] = fmax(v[4], fabs(g));
        v[5] = fmax(v[5], y);
      }
      STAMP(17);
      block_reduce_all<6, 0, 0x30>(v, red, rph);
      const double st = sqrt(fmax(kx[1] + v[0], 0.0));
      const double e_mu = fmax(st, sqrt(fmax(kx[2] + v[1], 0.0)));
      const double e_0 = fmax(st, sqrt(fmax(kx[3] + v[2], 0.0)));
      if (cta == 0 && tid == 0) {
        double* rec = a.logv + (long)(it - 1) * LOGW;
        rec[3] = kx[0];
        rec[4] = e_mu;
        rec[5] = e_0;
        a.sc[0] = kx[0];
        a.sc[16] = kx[1];
        a.sc[17] = kx[2];
        a.sc[18] = kx[3];
        a.sc[19] = kx[4];
        a.sc[20] = v[0];
        a.sc[21] = v[1];
        a.sc[22] = v[2];
        a.sc[23] = v[3];
        a.sc[24] = kx[5];
        a.sc[25] = v[4];
        a.sc[26] = kx[6];
        a.sc[27] = v[5];
      }
      if (!(e_mu > a.eps_mu) || !(e_0 > a.tol0) || it >= a.max_iters) {
        status = 0;
        fact_it = it - 1;  // the factorization of the last step taken
        break;
      }
    }
    if (ZHX[SA - 1] < 1.0 / 0.0) {
      if (cta == 0 && tid == 0) a.fcodes[0] = (int)ZHX[SA - 1];
      status = 1;
      fact_it = it - 1;
      break;
    }
    // the factorization point's Y for the predictor (replicated: CTA 0 writes it; the
    // row-side snapshots are double-buffered in shared memory and written at exit)
    if (cta == 0)
      #pragma unroll 1
      for (long e = tid; e < N; e += PT) a.Ytf[e] = Ys[YI(e / K, e % K)];

    STAMP(3);
    // ---- Y side (replicated): rhs, D_j, t_j = D_j^{-1} rhs_j, D_j^{-1} packed
    int badD = 0x7F7F7F7F;
    #pragma unroll 1
    for (long j = tid; j < m; j += PT) {
      double y[K], L[K][K], rhs[K], tv[K], iy[K];
#pragma unroll
      for (int p = 0; p < K; ++p) y[p] = Ys[YI(j, p)];
#pragma unroll
      for (int p = 0; p < K; ++p) {
        double ra = 0.0;
#pragma unroll
        for (int c = 0; c < K; ++c) ra = fma(Hs[p * K + c], y[c], ra);
        iy[p] = 1.0 / y[p];
        rhs[p] = (muy * iy[p] - gYs[YI(j, p)]) - ra;
      }
#pragma unroll
      for (int p = 0; p < K; ++p)
#pragma unroll
        for (int c = 0; c < K; ++c) L[p][c] = (c <= p) ? XtXs[p * K + c] : 0.0;
#pragma unroll
      for (int p = 0; p < K; ++p) L[p][p] += a.rho + Ss[YI(j, p)] * iy[p];
      double rd[K];
      if (!reg_chol<K>(L, rd)) badD = min(badD, (int)j);
      double Li[K][K];
      reg_inv_lower<K>(L, rd, Li);
#pragma unroll
      for (int p = 0; p < K; ++p) {
        if (cta == 0) {
#pragma unroll
          for (int c = 0; c < K; ++c) a.LD[(j * K + p) * K + c] = (c <= p) ? L[p][c] : 0.0;
        }
#pragma unroll
        for (int c = p; c < K; ++c) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < K; ++q)
            if (q >= c) s = fma(Li[q][p], Li[q][c], s);
          dinv[DI(j, (p * K - p * (p - 1) / 2 + (c - p)))] = s;
        }
      }
      reg_solve<K>(L, rd, rhs, tv);
#pragma unroll
      for (int p = 0; p < K; ++p) Ts[YI(j, p)] = tv[p];
    }
    {
      double v[1] = {(double)badD};
      block_reduce_all<1, 1, 0>(v, red, rph);
      badD = (int)v[0];
    }
    STAMP(4);
    // G = sum_j (y_j y_j^T) (x) D_j^{-1} (packed), u = U^T t.  G is an outer product per
    // column: warp w < GW owns two rows ab of G and forms all KK columns pq from one
    // load of D_j^{-1} (KK words) and two y_j y_j^T products, so a column costs KK + 4
    // shared-memory loads for 2 KK FMAs (one entry per warp and lane-strided columns
    // cost three loads per FMA and made this pass shared-memory bound at m = 500);
    // the other warps form u.
    {
      constexpr int GW = (KK + 1) / 2;
      static_assert(GW < NW, "G rows need fewer warps than the CTA has");
      if (wid < GW) {
        const int ab0 = 2 * wid, ab1 = (2 * wid + 1 < KK) ? 2 * wid + 1 : 2 * wid;
        const int a0 = ia[ab0], b0 = ic[ab0], a1 = ia[ab1], b1 = ic[ab1];
        double acc[2 * KK];
#pragma unroll
        for (int q = 0; q < 2 * KK; ++q) acc[q] = 0.0;
        #pragma unroll 1
        for (long j = lane; j < m; j += 32) {
          const double yy0 = Ys[YI(j, a0)] * Ys[YI(j, b0)];
          const double yy1 = Ys[YI(j, a1)] * Ys[YI(j, b1)];
#pragma unroll
          for (int pq = 0; pq < KK; ++pq) {
            const double dv = dinv[DI(j, pq)];
            acc[pq] = fma(yy0, dv, acc[pq]);
            acc[KK + pq] = fma(yy1, dv, acc[KK + pq]);
          }
        }
        using WH = WarpHalve<2 * KK, 0, 0>;
        const double tot = WH::run(acc);
        constexpr int SH = 5 - WH::LG;
        const int q = lane >> SH;
        if ((lane & ((1 << SH) - 1)) == 0 && q < 2 * KK) {
          const int ab = q < KK ? ab0 : ab1;
          if (q < KK || 2 * wid + 1 < KK) T1[ab * KK + (q % KK)] = tot;
        }
      } else {
        constexpr int NUW = NW - GW, EPU = (Q + NUW - 1) / NUW;
        double sacc[EPU];
        int o1[EPU], o2[EPU];
#pragma unroll
        for (int i2 = 0; i2 < EPU; ++i2) {
          const int e = (wid - GW) + NUW * i2;
          sacc[i2] = 0.0;
          o1[i2] = (e < Q ? e : 0) / K;
          o2[i2] = (e < Q ? e : 0) % K;
        }
        #pragma unroll 1
        for (long j = lane; j < m; j += 32) {
#pragma unroll
          for (int i2 = 0; i2 < EPU; ++i2)
            sacc[i2] = fma(Ys[YI(j, o1[i2])], Ts[YI(j, o2[i2])], sacc[i2]);
        }
        warp_reduce_multi<EPU, 0, 0>(sacc);
        if (lane == 0) {
#pragma unroll
          for (int i2 = 0; i2 < EPU; ++i2) {
            const int e = (wid - GW) + NUW * i2;
            if (e < Q) u[e] = sacc[i2];
          }
        }
      }
    }
    __syncthreads();
    STAMP(18);
    #pragma unroll 1
    for (int e = tid; e < Q * Q; e += PT) {
      const int r = e / Q, c = e % Q;
      const int p = r / K, q = r % K, b = c / K, d = c % K;
      const int pb_ = pk(p, b, K), qd = pk(q, d, K);
      Gm[e] = T1[pb_ * KK + qd];
      Zbm[e] = Zs[pb_ * KK + qd];
    }
    __syncthreads();
    if (tid < 32) {
      STAMP(24);
      const int f = warp_chol<Q>(Gm, dGi);
      STAMP(25);
      if (tid == 0) s_fail = f;
    }
    __syncthreads();
    STAMP(19);
    #pragma unroll 1
    for (int e = tid; e < Q * Q; e += PT) {
      const int r = e / Q, c = e % Q;
      double s = 0.0;
      for (int q = c; q < Q; ++q) s = fma(Zbm[r * Q + q], Gm[q * Q + c], s);
      T1[e] = s;
    }
    __syncthreads();
    STAMP(20);
    #pragma unroll 1
    for (int e = tid; e < Q * Q; e += PT) {
      const int r = e / Q, c = e % Q;
      double s = 0.0;
      for (int q = r; q < Q; ++q) s = fma(Gm[q * Q + r], T1[q * Q + c], s);
      Hm[e] = (r == c ? 1.0 : 0.0) - s;
    }
    __syncthreads();
    STAMP(21);
    if (tid < 32) {
      STAMP(26);
      const int f = warp_chol<Q>(Hm, dHi);
      STAMP(27);
      if (tid == 0 && s_fail < 0) s_fail = f;
    }
    __syncthreads();
    STAMP(22);
    if (cta == 0)
      #pragma unroll 1
      for (int e = tid; e < Q * Q; e += PT) {
        a.LG[e] = Gm[e];
        a.LH[e] = Hm[e];
        a.Zb[e] = Zbm[e];
      }
    if (s_fail >= 0 || badD != 0x7F7F7F7F) {
      if (cta == 0 && tid == 0) {
        a.fcodes[1] = s_fail;
        a.fcodes[2] = badD;
      }
      status = 1;
      fact_it = it;
      break;
    }
    STAMP(23);
    // w = LG^{-T} LH^{-T} LH^{-1} LG^T Zb u: warp 0, lane = row; the triangular
    // solves go column by column (one division + one shuffle per step)
    if (tid < 32) {
      const int r = tid;
      __syncwarp();
      double v = 0.0;
      if (r < Q)
        for (int c = 0; c < Q; ++c) v = fma(Zbm[r * Q + c], u[c], v);
      if (r < Q) w[r] = v;
      __syncwarp();
      double acc = 0.0;
      if (r < Q)
        for (int q = r; q < Q; ++q) acc = fma(Gm[q * Q + r], w[q], acc);
      __syncwarp();
      double z = 0.0;
      const double hdi = (r < Q) ? dHi[r] : 0.0, gdi = (r < Q) ? dGi[r] : 0.0;
#pragma unroll 1
      for (int j = 0; j < Q; ++j) {  // LH z = LG^T Zb u
        const double zj = __shfl_sync(0xffffffffu, acc * hdi, j);
        const double hij = (r < Q) ? Hm[r * Q + j] : 0.0;
        const double nacc = acc - hij * zj;
        z = (r == j) ? zj : z;
        acc = (r > j && r < Q) ? nacc : acc;
      }
      STAMP(28);
      acc = z;
#pragma unroll 1
      for (int j = Q - 1; j >= 0; --j) {  // LH^T z2 = z
        const double zj = __shfl_sync(0xffffffffu, acc * hdi, j);
        const double hji = (r < Q) ? Hm[j * Q + r] : 0.0;
        const double nacc = acc - hji * zj;
        z = (r == j) ? zj : z;
        acc = (r < j) ? nacc : acc;
      }
      acc = z;
#pragma unroll 1
      for (int j = Q - 1; j >= 0; --j) {  // LG^T w = z2
        const double zj = __shfl_sync(0xffffffffu, acc * gdi, j);
        const double gji = (r < Q) ? Gm[j * Q + r] : 0.0;
        const double nacc = acc - gji * zj;
        z = (r == j) ? zj : z;
        acc = (r < j) ? nacc : acc;
      }
      __syncwarp();
      if (r < Q) w[r] = z;
    }
    __syncthreads();
    STAMP(5);
    // dY_j = t_j + D_j^{-1}(W^T y_j); Y-side scalars
    {
      double v[3] = {0.0, 1.0 / 0.0, 1.0 / 0.0};
      #pragma unroll 1
      for (long j = tid; j < m; j += PT) {
        double rv[K], out[K], y[K];
#pragma unroll
        for (int p = 0; p < K; ++p) y[p] = Ys[YI(j, p)];
#pragma unroll
        for (int p = 0; p < K; ++p) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < K; ++c) s = fma(y[c], w[c * K + p], s);
          rv[p] = s;
        }
#pragma unroll
        for (int p = 0; p < K; ++p) {  // D_j^{-1} (W^T y_j) with the packed inverse
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < K; ++c) s = fma(dinv[DI(j, pk(p, c, K))], rv[c], s);
          out[p] = s;
        }
#pragma unroll
        for (int p = 0; p < K; ++p) {
          const double d = Ts[YI(j, p)] + out[p];
          Ts[YI(j, p)] = d;
          const double s = Ss[YI(j, p)];
          const double ds = muy / y[p] - s - (s / y[p]) * d;
          v[0] = fma(d, gYs[YI(j, p)] - muy / y[p], v[0]);
          if (d < 0.0) v[1] = fmin(v[1], -a.tau * y[p] / d);
          if (ds < 0.0) v[2] = fmin(v[2], -a.tau * s / ds);
        }
      }
      block_reduce_all<3, 0x6, 0>(v, red, rph);
      if (tid == 0) {
        scal[0] = v[0];
        scal[1] = v[1];
        scal[2] = v[2];
      }
    }
    #pragma unroll 1
    for (int e = wid; e < K * K; e += NW) {  // Gdy = sum_j y_j dy_j^T
      const int p = e / K, c = e % K;
      double s = 0.0;
      #pragma unroll 1
      for (long j = lane; j < m; j += 32) s = fma(Ys[YI(j, p)], Ts[YI(j, c)], s);
      s = warp_sum(s);
      if (lane == 0) Gdy[e] = s;
    }
    __syncthreads();
    STAMP(6);
    // ---- rows: dX, dR (back substitution), X-side scalars
    double pb[9] = {0.0, 1.0 / 0.0, 1.0 / 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    #pragma unroll 1
    for (int rr = tid; rr < nr; rr += PT) {
      double L[K][K], v[K], q[K], t[K], dx[K], x[K], rd[K];
#pragma unroll
      for (int p = 0; p < K; ++p) {
        x[p] = xs[rr * K + p];
        rd[p] = rds[rr * K + p];
#pragma unroll
        for (int c = 0; c < K; ++c) L[p][c] = Ls[(rr * K + p) * K + c];
      }
#pragma unroll
      for (int p = 0; p < K; ++p) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < K; ++b) s = fma(Gdy[p * K + b], x[b], s);
        v[p] = s;
      }
#pragma unroll
      for (int p = 0; p < K; ++p) {
        double s = v[p];
#pragma unroll
        for (int c = 0; c < p; ++c) s -= L[p][c] * q[c];
        q[p] = s * rd[p];
      }
#pragma unroll
      for (int p = 0; p < K; ++p) t[p] = hs[rr * K + p] - q[p];
#pragma unroll
      for (int p = K - 1; p >= 0; --p) {
        double s = t[p];
#pragma unroll
        for (int c = p + 1; c < K; ++c) s -= L[c][p] * dx[c];
        dx[p] = s * rd[p];
      }
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const double r = rs[rr * K + p], d = dx[p];
        const double dr = mux / x[p] - r - (r / x[p]) * d;
        dxs[rr * K + p] = d;
        drs[rr * K + p] = dr;
        pb[0] = fma(d, gxs[rr * K + p] - mux / x[p], pb[0]);
        if (d < 0.0) pb[1] = fmin(pb[1], -a.tau * x[p] / d);
        if (dr < 0.0) pb[2] = fmin(pb[2], -a.tau * r / dr);
      }
    }
    __syncthreads();
    STAMP(7);
    // ---- quartic partials over own rows x all columns (F recomputed from M)
    // thread = one column j (its y_j, dy_j in registers) x every RS-th own row: the
    // row operands are warp broadcasts and M's row segment is contiguous, so the
    // pass reads shared memory once per element (the element-major loop re-read
    // y_j and dy_j per element and was bound by shared-memory wavefronts)
    if (q_roff < q_rs) {
      #pragma unroll 1
      for (long j = q_j0; j < m; j += PT) {
        double y[K], dy[K];
#pragma unroll
        for (int p = 0; p < K; ++p) {
          y[p] = Ys[YI(j, p)];
          dy[p] = Ts[YI(j, p)];
        }
        #pragma unroll 2
        for (int rr = q_roff; rr < nr; rr += q_rs) {
          double fv = -Mp[(long)rr * m + j];
#pragma unroll
          for (int p = 0; p < K; ++p) fv = fma(xs[rr * K + p], y[p], fv);
          double bv = 0.0, cv = 0.0;
#pragma unroll
          for (int p = 0; p < K; ++p) {
            const double x = xs[rr * K + p], dx = dxs[rr * K + p];
            bv = fma(dx, y[p], fma(x, dy[p], bv));
            cv = fma(dx, dy[p], cv);
          }
          pb[3] = fma(fv, fv, pb[3]);
          pb[4] = fma(fv, bv, pb[4]);
          pb[5] = fma(bv, bv, pb[5]);
          pb[6] = fma(fv, cv, pb[6]);
          pb[7] = fma(bv, cv, pb[7]);
          pb[8] = fma(cv, cv, pb[8]);
        }
      }
    }
    STAMP(34);
    // Speculative first trial batch: a1max = min(1, y ratio, x ratio) where only the
    // x ratio still needs the grid; with a1s = min(1, y ratio) (replicated) the
    // partial barrier sums of trials 0..TB-1 ride along with this barrier.  After it,
    // a1max == a1s (the x rows did not bind, the common case) makes them exact and
    // phase C skips one grid barrier and one L2 round trip; otherwise phase C
    // recomputes the batch with the true a1max.
    {
      const double a1s = fmin(1.0, scal[1]);
      double ax, ay;
      trial_sums(wid, a1s, ax, ay);
      if (lane == 0) {
        __stcg(PB + (long)(9 + 2 * wid) * G + cta, ax);
        __stcg(PB + (long)(10 + 2 * wid) * G + cta, ay);
      }
    }
    {
      block_reduce_all<9, 0x6, 0>(pb, red, rph);
#pragma unroll
      for (int q = 0; q < 9; ++q)
        if (tid == q) __stcg(PB + (long)q * G + cta, pb[q]);
    }
    STAMP(8);
    grid_barrier(a.bar, epoch);
    STAMP(9);

    // ======== phase C: Armijo (quartic + barrier trials in batches) ========
    // [3] gtp_x [4] a1x [5] a2x [6..11] quartic
    reduce_mixed<4>(PB, G, 0, 9 + 2 * TB, pbv, [](long e) { return (e == 1 || e == 2) ? 1 : 0; });
    __syncthreads();
    const double gtp = pbv[0] + scal[0];
    const double a1s = fmin(1.0, scal[1]);
    const double a1max = fmin(fmin(1.0, pbv[1]), scal[1]);
    const double a2max = fmin(fmin(1.0, pbv[2]), scal[2]);
    const double ab = pbv[4], bb = pbv[5], ac = pbv[6], bc = pbv[7], cc = pbv[8];
    const bool spec_ok = (a1max == a1s);
    int tsel = -1;
    for (int batch = 0;; ++batch) {
      const int t0 = batch * TB;
      const double* bsum = pbv + 9;
      if (batch > 0 || !spec_ok) {
        // warp q = trial t0 + q
        double ax, ay;
        trial_sums(t0 + wid, a1max, ax, ay);
        double* pc = PC + (long)(batch & 1) * G * 2 * TB;
        if (lane == 0) {
          __stcg(pc + (long)(2 * wid) * G + cta, ax);
          __stcg(pc + (long)(2 * wid + 1) * G + cta, ay);
        }
        STAMP(10);
        grid_barrier(a.bar, epoch);
        reduce_entries<2, 0>(pc, G, 0, 2 * TB, bars);
        __syncthreads();
        bsum = bars;
      } else {
        STAMP(10);
      }
      if (tid < 32) {
        // lane q evaluates trial t0 + q with the arithmetic of armijo_pick (csrc/small.cu)
        // and of the host loop; the first lane that accepts (or passes max_bt) decides
        const double c2 = __dadd_rn(__dmul_rn(0.5, bb), ac);
        const int t = t0 + lane;
        bool acc = false, stall = false;
        if (lane < TB) {
          if (t > a.max_bt) {
            stall = true;
          } else {
            const double a1 = ldexp(a1max, -t);  // == a1max / 2^t exactly
            const double q2 = __dmul_rn(a1, a1), q3 = __dmul_rn(q2, a1), q4 = __dmul_rn(q3, a1);
            double quad = __dadd_rn(__dmul_rn(a1, ab), __dmul_rn(q2, c2));
            quad = __dadd_rn(quad, __dmul_rn(q3, bc));
            quad = __dadd_rn(quad, __dmul_rn(__dmul_rn(0.5, q4), cc));
            const double bar = __dadd_rn(__dmul_rn(a.wx, bsum[2 * lane]),
                                         __dmul_rn(a.wy, bsum[2 * lane + 1]));
            const double dphi = __dsub_rn(quad, __dmul_rn(a.mu, bar));
            acc = dphi <= __dmul_rn(__dmul_rn(a.eta, a1), gtp);
          }
        }
        const unsigned hit = __ballot_sync(0xffffffffu, acc || stall);
        if (lane == 0) {
          if (hit == 0u) {
            s_t = -1;
          } else {
            const int q = __ffs(hit) - 1;
            const bool st_q = (t0 + q) > a.max_bt;
            s_t = st_q ? -3 : t0 + q;
          }
        }
      }
      __syncthreads();
      tsel = s_t;
      if (tsel != -1) break;
    }
    if (tsel == -3) {
      if (cta == 0 && tid == 0) {
        double* rec = a.logv + (long)it * LOGW;
        rec[0] = (double)(a.max_bt + 1);
        rec[1] = 0.0;
        rec[2] = 0.0;
      }
      status = 2;
      fact_it = it;
      break;
    }
    STAMP(11);
    const double a1 = ldexp(a1max, -tsel);
    const double a2 = a2max;

    // ======== phase D: update, residual, graX, graY / KKT / ||F||^2 partials ====
    #pragma unroll 1
    for (long e = tid; e < N; e += PT) {
      const double y = Ys[e], s = Ss[e], d = Ts[e];
      const double ds = muy / y - s - (s / y) * d;
      Ys[e] = nudge(y, d, a1, a.tau);
      Ss[e] = nudge(s, ds, a2, a.tau);
    }
    #pragma unroll 1
    for (long e = tid; e < (long)nr * K; e += PT) {
      xs[e] = nudge(xs[e], dxs[e], a1, a.tau);
      rs[e] = nudge(rs[e], drs[e], a2, a.tau);
    }
    __syncthreads();
    STAMP(29);
    double kv[7] = {0.0, 0.0, 0.0, 0.0, 0.0, -1.0 / 0.0, -1.0 / 0.0};  // fsq, k0..k3, kg, kx
    // warps [0, NW/2): rows, RPW per warp in flight (F, graX, ||F||^2, X-part KKT);
    // warps [NW/2, NW): graY partials, thread per column; the two run concurrently
    if (wid < NW / 2) {
      constexpr int HW = NW / 2;
      constexpr int RPW = K <= 2 ? 4 : 3;  // c2: 20-21 rows per CTA in two passes
#pragma unroll 1
      for (int rb = wid; rb < nr; rb += RPW * HW) {
        int rr2[RPW];
#pragma unroll
        for (int u = 0; u < RPW; ++u) rr2[u] = rb + u * HW;
        double x[RPW][K], g[RPW][K];
#pragma unroll
        for (int u = 0; u < RPW; ++u)
#pragma unroll
          for (int p = 0; p < K; ++p) {
            x[u][p] = rr2[u] < nr ? xs[rr2[u] * K + p] : 0.0;
            g[u][p] = 0.0;
          }
#pragma unroll 1
        for (long j = lane; j < m; j += 32) {
          double y[K];
#pragma unroll
          for (int p = 0; p < K; ++p) y[p] = Ys[YI(j, p)];
#pragma unroll
          for (int u = 0; u < RPW; ++u) {
            if (rr2[u] >= nr) continue;
            double fv = -Mp[(long)rr2[u] * m + j];
#pragma unroll
            for (int p = 0; p < K; ++p) fv = fma(x[u][p], y[p], fv);
            kv[0] = fma(fv, fv, kv[0]);
#pragma unroll
            for (int p = 0; p < K; ++p) g[u][p] = fma(fv, y[p], g[u][p]);
          }
        }
        {
          // recursive-halving warp sums of the 2K row gradients; the lane that ends
          // up holding entry (u, p) also does its KKT terms
          using WH = WarpHalve<RPW * K, 0, 0>;
          double gf[RPW * K];
#pragma unroll
          for (int q = 0; q < RPW * K; ++q) gf[q] = g[q / K][q % K];
          const double gq = WH::run(gf);
          constexpr int SH = 5 - WH::LG;
          const int q = lane >> SH;
          if ((lane & ((1 << SH) - 1)) == 0 && q < RPW * K) {
            const int u = q / K, p = q - u * K;
            const int rr = rb + u * HW;
            if (rr < nr) {
              gxs[rr * K + p] = gq;
              const double r = rs[rr * K + p], xv = xs[rr * K + p];
              const double xr = xv * r;
              kv[1] = fma(gq - r, gq - r, kv[1]);
              kv[2] = fma(xr - mux, xr - mux, kv[2]);
              kv[3] = fma(xr, xr, kv[3]);
              kv[4] += xr;
              kv[5] = fmax(kv[5], fabs(gq));
              kv[6] = fmax(kv[6], xv);
            }
          }
        }
      }
    } else {
#pragma unroll 1
      for (long j = tid - PT / 2; j < m; j += PT / 2) {
        double acc[K], yj[K];
#pragma unroll
        for (int p = 0; p < K; ++p) {
          acc[p] = 0.0;
          yj[p] = Ys[YI(j, p)];
        }
#pragma unroll 4
        for (int rr = 0; rr < nr; ++rr) {
          double fv = -Mp[(long)rr * m + j];
#pragma unroll
          for (int p = 0; p < K; ++p) fv = fma(xs[rr * K + p], yj[p], fv);
#pragma unroll
          for (int p = 0; p < K; ++p) acc[p] = fma(fv, xs[rr * K + p], acc[p]);
        }
#pragma unroll
        for (int p = 0; p < K; ++p) __stcg(PG + (j * K + p) * G + cta, acc[p]);
      }
    }
    STAMP(30);
    {
      block_reduce_all<7, 0, 0x60>(kv, red, rph);
#pragma unroll
      for (int q = 0; q < 7; ++q)
        if (tid == q) __stcg(PD + (long)q * G + cta, kv[q]);
    }
    if (cta == 0 && tid == 0) {
      double* rec = a.logv + (long)it * LOGW;
      unsigned long long tns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
      rec[0] = (double)tsel;
      rec[1] = a1;
      rec[2] = a2;
      rec[6] = (double)tns;
    }
    STAMP(12);
    grid_barrier(a.bar, epoch);
    STAMP(13);

    // ======== phase E: graY slice totals; X-part KKT sums and ||F||^2 ========
    {
      const long e0 = y0, e1 = y1;
      // the slice of graY on warps 0..3 and the KKT / ||F||^2 partials on warps 4..7
      auto sum_kind = [](long) { return 0; };
      reduce_mixed<2, decltype(sum_kind), true>(PG, G, e0, e1, a.gY + e0, sum_kind, 0, NW / 2);
      reduce_mixed<1>(PD, G, 0, 7, kx, [](long e) { return e >= 5 ? 2 : 0; }, NW / 2, NW / 2);
    }
    STAMP(14);
    ++it;
    // the barrier after the next phase A publishes graY
  }

  // ---- write the state back ----------------------------------------------------
  __syncthreads();
  if (fact_it >= 0) {  // the predictor reuses the last step's factorization
    const double* Lc = Lsb + (long)(fact_it & 1) * nrm * K * K;
    const double* xsn = xsnap + (long)(fact_it & 1) * nrm * K;
    #pragma unroll 1
    for (long e = tid; e < (long)nr * K * K; e += PT) a.L[r0 * K * K + e] = Lc[e];
    #pragma unroll 1
    for (long e = tid; e < (long)nr * K; e += PT) a.Xf[r0 * K + e] = xsn[e];
  }
  if (it > 0) {
    // F = X Y - M at the final point, with phase D's expression (phase D no longer
    // stores F every iteration: only the last one is consumed by the host)
    #pragma unroll 1
    for (int rr = q_roff; rr < nr && q_roff < q_rs; rr += q_rs) {
      #pragma unroll 1
      for (long j = q_j0; j < m; j += PT) {
        double fv = -Mp[(long)rr * m + j];
#pragma unroll
        for (int p = 0; p < K; ++p) fv = fma(xs[rr * K + p], Ys[YI(j, p)], fv);
        a.Fout[(r0 + rr) * m + j] = fv;
      }
    }
  }
  #pragma unroll 1
  for (long e = tid; e < (long)nr * K; e += PT) {
    a.X[r0 * K + e] = xs[e];
    a.R[r0 * K + e] = rs[e];
    a.gX[r0 * K + e] = gxs[e];
  }
  if (cta == 0) {
    #pragma unroll 1
    for (long e = tid; e < N; e += PT) {
      a.Yt[e] = Ys[YI(e / K, e % K)];
      a.S[e] = Ss[YI(e / K, e % K)];
    }
    if (tid == 0) {
      a.status[0] = it;
      a.status[1] = status;
    }
  }
}
#undef YI
#undef DI

template <int K>
long p_smem_bytes(long n, long m, int G, bool with_m) {
  const long nrm = (n + G - 1) / G;
  return smem_doubles<K>(nrm, m, with_m) * (long)sizeof(double);
}

constexpr long SMEM_CAP = 210 * 1024;  // dynamic part; static <= 15 KB, 227 KB per CTA in all

constexpr int P_MAX_GRID = 160;  // 5 lanes x 32 CTAs in reduce_entries, pbar length

// one CTA per SM (the cooperative launch needs every CTA resident)
int p_max_grid() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1)
      sms = 1;
  }
  return sms < P_MAX_GRID ? sms : P_MAX_GRID;
}

int p_grid(long n) {
  long g = (n + 15) / 16;
  const int cap = p_max_grid();
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

#define NMFB_PK(k, MACRO)               \
  switch (k) {                          \
    MACRO(1) MACRO(2) MACRO(3) MACRO(4) \
    default: return 0;                  \
  }

extern "C" int nmfb_persist_supported(long n, long m, long k, int grid, int m_is_f32) {
  if (k < 1 || k > 4 || m < 1 || n < 1 || m * k > 2048) return 0;
  // the fixed-order partial reductions sum at most P_MAX_GRID CTAs and every CTA must
  // be co-resident (one per SM)
  if (grid < 0 || grid > p_max_grid()) return 0;
  const int G = grid > 0 ? grid : p_grid(n);
  if ((n + G - 1) / G > 4096) return 0;
  // fp32 M is only read from shared memory (no fp32 global path): it must fit
#define CASE(KK_) \
  case KK_: return p_smem_bytes<KK_>(n, m, G, m_is_f32 != 0) <= SMEM_CAP ? 1 : 0;
  NMFB_PK(k, CASE)
#undef CASE
}

extern "C" long nmfb_persist_work_len(long n, long m, long k, int grid) {
  const int G = grid > 0 ? grid : p_grid(n);
  return wlayout(G, m, (int)k).total;
}

// One cooperative launch = the Gauss-Newton inner loop (see the file header).
// log: max_iters x 8 doubles [t, alpha1, alpha2, ||F||^2, E_mu, E_0, globaltimer ns, -];
// status (device int[2]): [iterations done, exit code].
extern "C" int nmfb_ipm_persist(const void* M, int m_is_f32, long n, long m, long k, double* X,
                                double* R, double* gX, double* Yt, double* S, double* gY,
                                double* Fout, double* L, double* Xf, double* Ytf, double* LD,
                                double* LG, double* LH, double* Zb, double mu, double wx,
                                double wy, double rho, double tau, double eta, double eps_mu,
                                double tol0, int max_bt, int ntrials, int max_iters, double* sc, int* fcodes,
                                double* logv, int* status, double* work, unsigned int* bar,
                                int grid, long long* prof, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!nmfb_persist_supported(n, m, k, grid, m_is_f32)) return NMFB_EUNSUPPORTED;
  if (max_iters < 1) return NMFB_EINVAL;
  const int G = grid > 0 ? grid : p_grid(n);
  PArgs a;
  a.M = M;
  a.n = n;
  a.m = m;
  a.X = X;
  a.R = R;
  a.gX = gX;
  a.Yt = Yt;
  a.S = S;
  a.gY = gY;
  a.Fout = Fout;
  a.L = L;
  a.Xf = Xf;
  a.Ytf = Ytf;
  a.LD = LD;
  a.LG = LG;
  a.LH = LH;
  a.Zb = Zb;
  a.sc = sc;
  a.logv = logv;
  a.work = work;
  a.fcodes = fcodes;
  a.status = status;
  a.bar = bar;
  a.mu = mu;
  a.wx = wx;
  a.wy = wy;
  a.rho = rho;
  a.tau = tau;
  a.eta = eta;
  a.eps_mu = eps_mu;
  a.tol0 = tol0;
  a.max_bt = max_bt;
  a.ntrials = ntrials;
  a.max_iters = max_iters;
  a.prof = prof;
  cudaMemsetAsync(bar, 0, (size_t)G * sizeof(unsigned int), st);
  void* args[] = {&a};
  cudaError_t err = cudaSuccess;
#define LAUNCH(KK_, T_)                                                                        \
  {                                                                                            \
    const bool wm = p_smem_bytes<KK_>(n, m, G, true) <= SMEM_CAP;                             \
    if (!wm && m_is_f32) return NMFB_EUNSUPPORTED;                                            \
    a.m_in_smem = wm ? 1 : 0;                                                                  \
    const long bytes = p_smem_bytes<KK_>(n, m, G, wm);                                        \
    nmfb_smem_attr(k_ipm_persist<KK_, T_>, \
                         (int)bytes);                                                          \
    ++g_nmfb_launches;                                                                         \
    err = cudaLaunchCooperativeKernel((const void*)k_ipm_persist<KK_, T_>, dim3(G), dim3(PT), \
                                      args, (size_t)bytes, st);                                \
  }
#define CASE(KK_)            \
  case KK_:                  \
    if (m_is_f32)            \
      LAUNCH(KK_, float)     \
    else                     \
      LAUNCH(KK_, double)    \
    break;
  switch (k) {
    CASE(1) CASE(2) CASE(3) CASE(4)
    default: return NMFB_EUNSUPPORTED;
  }
#undef CASE
#undef LAUNCH
  if (err != cudaSuccess) return NMFB_ELAUNCH;
  NMFB_CHECK_LAUNCH();
  return NMFB_OK;
}
