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

#undef FULLM

}  // namespace
