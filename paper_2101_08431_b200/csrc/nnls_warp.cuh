// Warp-cooperative, bit-exact active-set NNLS (the reference's nnls_batch,
// _kernels_numba.py:277-477, restated in csrc/surface.cu's k_nnls).  Shared by
// csrc/surface.cu (the batched entry) and csrc/stage1_persist.cu.  Include only
// from files compiled with -fmad=false: every scalar follows the reference's
// operation sequence, so the results are the reference's bits.
#pragma once
#include <stdint.h>

namespace {

#define FULLM 0xffffffffu
// --------------------------------------------------------------------------
// nnls_batch, warp per right-hand side (production path, same bits as k_nnls):
// lane j owns index j (d_j, x_j, w_j, z_j, row j of the passive Cholesky factor
// and row j of ctc).  Every scalar goes through the reference's operation
// sequence: column-oriented sweeps subtract terms in the reference's index
// order, the backward solve gathers its terms in ascending order with
// shuffles, argmax keeps the first maximum (ballot), and the file is compiled
// with -fmad=false.  The passive set is a lane mask, uniform across the warp.
// --------------------------------------------------------------------------
// Several right-hand sides share a warp when k is small: segment width W (a power
// of two >= k) carries one rhs; segments diverge freely (per-segment masks and
// width-W shuffles), which interleaves independent dependency chains.
template <int K, int W>
struct WNnls {
  double Lr[K];  // row `sl` of L (global column index)
  double C[K];   // row `sl` of ctc
  int sl;        // lane within the segment
  unsigned sm;   // segment mask (lanes of this rhs)
  // optional factor table (csrc/surface.cu k_factor_table): T[(pm K + i) K + j] is the
  // passive factor of subset pm in global indices, okf[pm] its PD flag.  The same
  // operation sequence computed once per subset instead of once per rhs and trip
  // (the reference's factor cache keyed by the passive signature,
  // _kernels_numba.py:296-298, 334-349).
  const double* T = nullptr;
  const double* okf = nullptr;

  __device__ __forceinline__ double sh(double v, int src) const { return __shfl_sync(sm, v, src, W); }

  __device__ __forceinline__ bool factor(unsigned pm) {
    if (T != nullptr) {
      const double* row = T + ((long)pm * K + (sl < K ? sl : 0)) * K;
#pragma unroll
      for (int c = 0; c < K; ++c) Lr[c] = sl < K ? __ldg(row + c) : 0.0;
      return __ldg(okf + pm) != 0.0;
    }
#pragma unroll
    for (int c = 0; c < K; ++c) Lr[c] = 0.0;
    bool ok = true;
#pragma unroll
    for (int gj = 0; gj < K; ++gj) {
      if (!ok || !((pm >> gj) & 1u)) continue;
      double acc = C[gj];  // lane gj: ctc[gj][gj]; lane gi: ctc[gi][gj]
#pragma unroll
      for (int gp = 0; gp < gj; ++gp) {
        if (!((pm >> gp) & 1u)) continue;
        const double ljp = sh(Lr[gp], gj);
        acc = acc - Lr[gp] * ljp;
      }
      const double accj = sh(acc, gj);
      if (accj <= 0.0) {
        ok = false;
        continue;
      }
      const double ljj = sqrt(accj);
      const bool below = sl > gj && sl < K && ((pm >> sl) & 1u);
      const double lij = acc / ljj;
      Lr[gj] = (sl == gj) ? ljj : (below ? lij : Lr[gj]);
    }
    return ok;
  }

  // z <- (L L^T)^{-1} b on the passive lanes (chol_solve_small order)
  __device__ __forceinline__ double solve(unsigned pm, double b) const {
    double acc = b, zf = 0.0;
#pragma unroll
    for (int gi = 0; gi < K; ++gi) {
      if (!((pm >> gi) & 1u)) continue;
      const double zi = sh(acc / Lr[gi], gi);
      zf = (sl == gi) ? zi : zf;
      const double nacc = acc - Lr[gi] * zi;
      acc = (sl > gi && sl < K && ((pm >> sl) & 1u)) ? nacc : acc;
    }
    double zb = 0.0;
#pragma unroll
    for (int gi = K - 1; gi >= 0; --gi) {
      if (!((pm >> gi) & 1u)) continue;
      double a = zf;
#pragma unroll
      for (int gp = gi + 1; gp < K; ++gp) {
        if (!((pm >> gp) & 1u)) continue;
        a = a - sh(Lr[gi] * zb, gp);  // L[gp][gi] z[gp], gp ascending
      }
      const double zi = a / Lr[gi];
      zb = (sl == gi) ? zi : zb;
    }
    return zb;
  }

  // _passive_solve_refined: z = solve(d); r = d - C_PP z; z += solve(r)
  __device__ __forceinline__ double solve_refined(unsigned pm, double d) const {
    const double z = solve(pm, d);
    double acc = d;
#pragma unroll
    for (int gp = 0; gp < K; ++gp) {
      if (!((pm >> gp) & 1u)) continue;
      acc = acc - C[gp] * sh(z, gp);
    }
    const double dz = solve(pm, acc);
    return z + dz;
  }

  // w_j = d_j - sum_p ctc[j][p] x_p (p ascending, all p)
  __device__ __forceinline__ double grad(double d, double x) const {
    double acc = d;
#pragma unroll
    for (int p = 0; p < K; ++p) acc = acc - C[p] * sh(x, p);
    return acc;
  }
};


// One bit-exact NNLS solve per warp segment (nnls_batch semantics for one rhs).
// Inputs per lane: d (ctb entry of this lane's index; 0 beyond k); C rows of ctc
// already in s.C.  seed_passive: this lane's seed bit (used when use_seed).
// Outputs: x (this lane), pm (passive mask), nch, r2 (valid in every lane), st.
template <int K, int W>
__device__ __forceinline__ void nnls_seg_solve(WNnls<K, W>& s, double d, double btb, double tol_t,
                                               bool use_seed, bool seed_passive, long max_changes,
                                               double& x_out, unsigned& pm_out, long& nch_out,
                                               double& r2_out, int& st_out) {
  const int sl = s.sl;
  const unsigned sm = s.sm;
  const int shift = (W == 32) ? 0 : (int)(__ffs(sm) - 1);
  const bool own = sl < K;
  double x = 0.0, w = 0.0;
  unsigned pm = 0u;
  bool solved = false;
  long nch = 0;
  if (use_seed) {
    const bool spas = own && seed_passive;
    pm = (__ballot_sync(sm, spas) >> shift) & ((W == 32) ? 0xffffffffu : ((1u << W) - 1u));
    if (pm == 0u) {
      if (!__any_sync(sm, own && d > tol_t)) {
        x = 0.0;
        solved = true;
      }
    } else if (s.factor(pm)) {
      const double z = s.solve_refined(pm, d);
      const bool passive = own && ((pm >> sl) & 1u);
      if (!__any_sync(sm, passive && z < 0.0)) {
        x = passive ? z : 0.0;
        const double wj = s.grad(d, x);
        const bool bad = own && (passive ? (fabs(wj) > tol_t) : (wj > tol_t));
        w = wj;
        solved = !__any_sync(sm, bad);
      }
    }
  }
  int st = 0;
  if (!solved) {
    pm = 0u;
    x = 0.0;
    w = d;
    for (;;) {
      const bool cand = own && !((pm >> sl) & 1u) && w > tol_t;
      double v = cand ? w : -1.0 / 0.0;
#pragma unroll
      for (int o = W / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(sm, v, o, W));
      const unsigned hit = (__ballot_sync(sm, cand && w == v) >> shift);
      const unsigned hits = (W == 32) ? hit : (hit & ((1u << W) - 1u));
      if (hits == 0u) break;
      const int jmax = __ffs(hits) - 1;  // first maximum, as the sequential scan
      pm |= 1u << jmax;
      nch += 1;
      if (nch > max_changes) {
        st = 1;
        break;
      }
      for (;;) {
        if (pm == 0u) break;
        if (!s.factor(pm)) {
          st = 2;
          break;
        }
        const double z = s.solve_refined(pm, d);
        const bool passive = own && ((pm >> sl) & 1u);
        if (!__any_sync(sm, passive && z <= 0.0)) {
          x = passive ? z : 0.0;
          break;
        }
        const bool neg = passive && z <= 0.0;
        const double ratio = neg ? x / (x - z) : 1.0 / 0.0;
        double alpha = ratio;
#pragma unroll
        for (int o = W / 2; o > 0; o >>= 1) alpha = fmin(alpha, __shfl_xor_sync(sm, alpha, o, W));
        alpha = alpha < 1.0 ? alpha : 1.0;
        const double newx = x + alpha * (z - x);
        const bool drop = neg && ratio <= alpha;
        if (passive) x = drop ? 0.0 : (newx > 0.0 ? newx : 0.0);
        const unsigned dmw = __ballot_sync(sm, drop) >> shift;
        const unsigned dm = (W == 32) ? dmw : (dmw & ((1u << W) - 1u));
        pm &= ~dm;
        nch += __popc(dm);
        if (nch > max_changes) {
          st = 1;
          break;
        }
      }
      if (st != 0) break;
      w = s.grad(d, x);
    }
  }
  // r2 = btb - sum_j (2 x_j) d_j + sum_j x_j (ctc x)_j, j ascending
  double acc2 = 0.0;
#pragma unroll
  for (int p = 0; p < K; ++p) acc2 = acc2 + s.C[p] * s.sh(x, p);
  const double t1 = 2.0 * x * d, t2 = x * acc2;
  double r2 = btb;
#pragma unroll
  for (int j = 0; j < K; ++j) r2 = r2 - s.sh(t1, j);
#pragma unroll
  for (int j = 0; j < K; ++j) r2 = r2 + s.sh(t2, j);
  x_out = x;
  pm_out = pm;
  nch_out = nch;
  r2_out = r2 > 0.0 ? r2 : 0.0;
  st_out = st;
}


// --------------------------------------------------------------------------
// nnls_batch, one THREAD per right-hand side with every per-rhs vector in
// registers (exact K, fully unrolled) and the passive factors read from a table of
// all 2^K subsets (built by the same column-oriented factor as WNnls, so the bits
// match).  The passive set is a bit mask; loops run over all K indices in
// ascending order and skip non-passive terms with selects (acc stays bit-identical
// to the reference's loop over passive positions), so a warp stays converged
// inside a Lawson-Hanson trip.
//   STAGED = true : T is the global table; the current subset's factor is staged
//                   into this thread's shared-memory slot (packed, stride TabT<K>) by
//                   cp.async once per trip (csrc/surface.cu k_nnls_tab)
//   STAGED = false: T is a (small) table in shared memory, read in place
//                   (csrc/stage1_persist.cu)
// --------------------------------------------------------------------------
// threads per block of k_nnls_tab (= the stride of the per-thread factor slots): 64, or 32
// above k = 12 so the K(K+1)/2-entry slots stay within the 48 KB of static shared memory
template <int K>
struct TabT {
  static constexpr int v = K > 12 ? 32 : 64;
};

template <int K, bool STAGED>
struct TNnls {
  static constexpr int KT = K * (K + 1) / 2;
  const double* C;     // ctc (K x K, shared memory: broadcast reads)
  static constexpr int TS = TabT<K>::v;
  double* sL;          // STAGED: this thread's slot, packed entry e at sL[e * TS]
  const double* Lt;    // !STAGED: the current subset's K x K factor (shared memory)
  double d[K];

  __device__ __forceinline__ static bool bit(unsigned pm, int i) { return (pm >> i) & 1u; }
  __device__ __forceinline__ static constexpr int tri(int i, int j) { return i * (i + 1) / 2 + j; }
  __device__ __forceinline__ double l(int i, int j) const {
    return STAGED ? sL[tri(i, j) * TS] : Lt[i * K + j];
  }

  __device__ __forceinline__ void stage(const double* __restrict__ T, unsigned pm) {
    if (!STAGED) {
      Lt = T + (long)pm * K * K;
      return;
    }
    // every entry an asynchronous global -> shared copy, all in flight together
    const double* Lg = T + (long)pm * K * K;
    const unsigned base = (unsigned)__cvta_generic_to_shared(sL);
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                         base + (unsigned)(tri(i, j) * TS * sizeof(double))),
                     "l"(Lg + i * K + j)
                     : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  // the staged factor is complete (no-op for the in-place table)
  __device__ __forceinline__ void stage_wait() const {
    if (STAGED) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }

  // RN(a / b) from the correctly rounded reciprocal r = RN(1 / b) (Markstein): q0 = RN(a r),
  // the exact residual a - b q0 by FMA, one correction -- three dependent operations on the
  // substitution's critical chain instead of the division sequence; bit-identical to a / b
  __device__ __forceinline__ static double mdiv(double a, double b, double r) {
    const double q0 = a * r;
    const double e = fma(-b, q0, a);
    return fma(e, r, q0);
  }

  // _chol_solve_small (:247-258) on the passive indices; ri[i] = RN(1 / l(i, i))
  __device__ __forceinline__ void solve(unsigned pm, const double (&b)[K], double (&z)[K],
                                        const double (&ri)[K]) const {
    // A non-passive index p contributes l * z[p] = (+0) * (+0): the subset table holds
    // exact zeros off the passive rows / columns (WNnls::factor starts from Lr = 0) and
    // z[p] is +0, and acc - (+0) == acc bit for bit -- so the reference's skip of
    // non-passive positions needs no select on the dependent chain.
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double acc = b[i];
#pragma unroll
      for (int p = 0; p < i; ++p) acc = acc - l(i, p) * z[p];
      z[i] = bit(pm, i) ? mdiv(acc, l(i, i), ri[i]) : 0.0;
    }
    asm volatile("" ::: "memory");
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
      double acc = z[i];
#pragma unroll
      for (int p = i + 1; p < K; ++p) acc = acc - l(p, i) * z[p];
      z[i] = bit(pm, i) ? mdiv(acc, l(i, i), ri[i]) : 0.0;
    }
  }

  // _passive_solve_refined (:261-274): z = solve(d); r = d - C_PP z; z += solve(r)
  // staged == true: the caller already issued stage(T, pm) (beside its own loads)
  __device__ __forceinline__ void solve_refined(const double* __restrict__ T, unsigned pm,
                                                double (&z)[K], bool staged = false) {
    if (!staged) stage(T, pm);
    stage_wait();
    // compiler memory barriers: the two solves re-read the factor instead of keeping
    // all K(K+1)/2 entries live in registers between them
    asm volatile("" ::: "memory");
    // the K reciprocal pivots of this subset's factor, independent of one another (their
    // latencies overlap), shared by the four substitutions of the refined solve
    double ri[K];
#pragma unroll
    for (int i = 0; i < K; ++i) ri[i] = bit(pm, i) ? __drcp_rn(l(i, i)) : 0.0;
    solve(pm, d, z, ri);
    asm volatile("" ::: "memory");
    double r[K], dz[K];
#pragma unroll
    for (int a = 0; a < K; ++a) {
      double acc = d[a];
#pragma unroll
      for (int b = 0; b < K; ++b) acc = acc - C[a * K + b] * z[b];  // z[b] = +0 off the passive set
      r[a] = acc;
    }
    solve(pm, r, dz, ri);
#pragma unroll
    for (int a = 0; a < K; ++a) z[a] = bit(pm, a) ? z[a] + dz[a] : 0.0;
  }

  // w_j = d_j - sum_p ctc[j][p] x_p over ALL p (the reference's dual loop)
  __device__ __forceinline__ void grad(const double (&x)[K], double (&w)[K]) const {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double acc = d[j];
#pragma unroll
      for (int p = 0; p < K; ++p) acc -= C[j * K + p] * x[p];
      w[j] = acc;
    }
  }
};

// One bit-exact nnls_batch solve (warm try :306-375, cold Lawson-Hanson :377-461,
// residual :468-476) for the rhs in s.d.  okf[pm] != 0: subset pm's factor is PD.
template <int K, bool STAGED>
__device__ __forceinline__ void tnnls_solve(TNnls<K, STAGED>& s, const double* __restrict__ T,
                                            const double* __restrict__ okf, double btb,
                                            double tol_t, bool use_seed, unsigned seed_pm,
                                            long max_changes, double (&x)[K], unsigned& pm_out,
                                            long& nch_out, double& r2_out, int& st_out) {
  using TN = TNnls<K, STAGED>;
  double z[K], w[K];
  unsigned pm = 0u;
  long nch = 0;
  bool solved = false;
  if (use_seed) {
    pm = seed_pm;
    if (pm == 0u) {
      bool ok = true;
#pragma unroll
      for (int j = 0; j < K; ++j) ok = ok && !(s.d[j] > tol_t);
      if (ok) {
#pragma unroll
        for (int j = 0; j < K; ++j) x[j] = 0.0;
        solved = true;
      }
    } else if (s.stage(T, pm), okf[pm] == 0.0) {  // factor copy and the PD word in flight together
      s.stage_wait();  // not PD: drain the copy before the cold start restages the slot
    } else {
      s.solve_refined(T, pm, z, true);
      bool feas = true;
#pragma unroll
      for (int a = 0; a < K; ++a) feas = feas && !(TN::bit(pm, a) && z[a] < 0.0);
      if (feas) {
#pragma unroll
        for (int j = 0; j < K; ++j) x[j] = TN::bit(pm, j) ? z[j] : 0.0;
        s.grad(x, w);
        bool dual_ok = true;
#pragma unroll
        for (int j = 0; j < K; ++j)
          dual_ok = dual_ok && !(TN::bit(pm, j) ? (fabs(w[j]) > tol_t) : (w[j] > tol_t));
        solved = dual_ok;
      }
    }
  }
  int st = 0;
  if (!solved) {
    pm = 0u;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      x[j] = 0.0;
      w[j] = s.d[j];
    }
    for (;;) {
      int jmax = -1;
      double wmax = tol_t;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const bool c = !TN::bit(pm, j) && w[j] > wmax;
        wmax = c ? w[j] : wmax;
        jmax = c ? j : jmax;
      }
      if (jmax < 0) break;
      pm |= 1u << jmax;
      nch += 1;
      if (nch > max_changes) {
        st = 1;
        break;
      }
      for (;;) {
        if (pm == 0u) break;
        s.stage(T, pm);  // the subset's factor on its way while its PD word is read
        if (okf[pm] == 0.0) {
          s.stage_wait();
          st = 2;
          break;
        }
        s.solve_refined(T, pm, z, true);
        bool all_pos = true;
#pragma unroll
        for (int a = 0; a < K; ++a) all_pos = all_pos && !(TN::bit(pm, a) && z[a] <= 0.0);
        if (all_pos) {
#pragma unroll
          for (int j = 0; j < K; ++j) x[j] = TN::bit(pm, j) ? z[j] : 0.0;
          break;
        }
        double alpha = 1.0;
#pragma unroll
        for (int a = 0; a < K; ++a) {
          if (TN::bit(pm, a) && z[a] <= 0.0) {
            const double ratio = x[a] / (x[a] - z[a]);
            alpha = ratio < alpha ? ratio : alpha;
          }
        }
        unsigned drop = 0u;
#pragma unroll
        for (int a = 0; a < K; ++a) {
          if (!TN::bit(pm, a)) continue;
          const double xa = x[a];
          const double newx = xa + alpha * (z[a] - xa);
          if (z[a] <= 0.0 && xa / (xa - z[a]) <= alpha) {
            x[a] = 0.0;
            drop |= 1u << a;
          } else {
            x[a] = newx > 0.0 ? newx : 0.0;
          }
        }
        pm &= ~drop;
        nch += __popc(drop);
        if (nch > max_changes) {
          st = 1;
          break;
        }
      }
      if (st != 0) break;
      s.grad(x, w);
    }
  }
  // resid2 = btb - sum_j (2 x_j) d_j + sum_j x_j (ctc x)_j, j ascending (:468-476)
  double r2 = btb;
#pragma unroll
  for (int j = 0; j < K; ++j) r2 -= 2.0 * x[j] * s.d[j];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double acc = 0.0;
#pragma unroll
    for (int p = 0; p < K; ++p) acc += s.C[j * K + p] * x[p];
    r2 += x[j] * acc;
  }
  pm_out = pm;
  nch_out = nch;
  r2_out = r2 > 0.0 ? r2 : 0.0;
  st_out = st;
}

#undef FULLM

}  // namespace
