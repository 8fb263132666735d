/*
 * nmfb200.h -- C ABI of libnmfb200.so, the B200 (sm_100a) implementation of
 * the two-stage NMF hot path of arXiv 2101.08431 (reference: nmfstream).
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer owned by the caller (torch / cudaMalloc);
 *    `stream` is a cudaStream_t passed as void*.  Calls are asynchronous on
 *    that stream unless stated.
 *  - Arrays are C-contiguous; float64 unless stated; bool arrays are uint8.
 *    Layouts follow the reference kernels (_kernels_numba.py): x_rows (n,k) =
 *    X, y_cols (m,k) = Y^T, l (n,k,k) lower factors, S (mk,mk), r_acc (m,k).
 *  - Return value: 0 ok, <0 argument (-1) / launch (-2) / memory (-3) /
 *    unsupported (-4) error.  Per-item failures are reported through device
 *    status buffers with the reference's codes; nothing throws across the ABI.
 *  - k <= 16 (NMFB_MAX_K).
 *
 * The "surface" entries replace, one for one, the seven functions of the
 * reference's kernel module, selected by the reference's (missing) backend
 * switch (/root/reference/pkg/src/nmfstream/_kernels_numba.py:3-4,
 * _kernels_numpy.py:3-5).  They are bit-identical to the reference kernels.
 */
#ifndef NMFB200_H
#define NMFB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- reference-surface kernels (bit-identical) -------------------------- */

/* replaces nnls_batch(ctc, ctb, btb, warm_passive, warm_mode, tol, max_changes)
 * -> (x, passive, changes, resid2, status)   _kernels_numba.py:277-477
 * seed_scratch (nrhs*k bytes) and flag_scratch (1 int) are required for
 * warm_mode 1 only (the chain fixed point synchronises the stream). */
int nmfb_surface_nnls_batch(const double *ctc, const double *ctb, const double *btb,
                            const uint8_t *warm_passive, int warm_mode, const double *tol,
                            long max_changes, long nrhs, long k, double *x, uint8_t *passive,
                            long long *changes, double *resid2, int8_t *status,
                            uint8_t *seed_scratch, int *flag_scratch, void *stream);

/* replaces block_cholesky(blocks) -> (L, bad)   _kernels_numba.py:12-29
 * *bad receives INT_MAX when every block is positive definite (maps to -1). */
int nmfb_surface_block_cholesky(const double *blocks, long nb, long k, double *out, int *bad,
                                void *stream);

/* replaces block_solve_lower / block_solve_lower_t(l, b)   _kernels_numba.py:32-57
 * b, z: (nb, k, r) */
int nmfb_surface_block_solve_lower(const double *l, const double *b, long nb, long k, long r,
                                   int transposed, double *z, void *stream);

/* replaces schur_reduce(x_rows, y_cols, l, h, resid, full) -> (S, r_acc)
 * _kernels_numba.py:72-143.  resid (n,m) is read only when full != 0. */
int nmfb_surface_schur_reduce(const double *x_rows, const double *y_cols, const double *l,
                              const double *h, const double *resid, long n, long m, long k,
                              int full, double *s_acc, double *r_acc, void *stream);

/* replaces rhs_reduce(x_rows, y_cols, l, h, resid, full) -> r_acc
 * _kernels_numba.py:146-178 */
int nmfb_surface_rhs_reduce(const double *x_rows, const double *y_cols, const double *l,
                            const double *h, const double *resid, long n, long m, long k,
                            int full, double *r_acc, void *stream);

/* replaces back_substitute(x_rows, y_cols, l, h, dy_rows, resid, full) -> dx
 * _kernels_numba.py:181-224 */
int nmfb_surface_back_substitute(const double *x_rows, const double *y_cols, const double *l,
                                 const double *h, const double *dy_rows, const double *resid,
                                 long n, long m, long k, int full, double *dx, void *stream);


/* ---- production entries (device-resident two-stage solver) ---------------
 * Products over M (n x m, fp64 or fp32 when *_is_f32 != 0); reductions use a
 * fixed decomposition (bit-reproducible).  `work` buffers are caller-owned
 * scratch of at least the stated length (doubles). */

/* nnls_batch (same arguments, results and codes as nmfb_surface_nnls_batch) with a
 * caller workspace `ftab` of nmfb_nnls_ftab_len(k) doubles (0 when k > 12: the table
 * is then not used).  The passive Cholesky factor of every subset of {0..k-1} is
 * computed once per call in the reference's operation order and shared by all
 * right-hand sides and Lawson-Hanson trips -- the reference's factor cache keyed by
 * the passive signature (_kernels_numba.py:296-298, 334-349) -- so the bits match. */
long nmfb_nnls_ftab_len(long k);
/* Build the subset factor table of ctc into ftab (for a later nmfb_nnls_batch_ws call with
 * ftab_len negated = "table already built"), e.g. on a second stream concurrently with the
 * product that computes ctb. */
int nmfb_nnls_ftab_build(const double *ctc, long k, double *ftab, long ftab_len, void *stream);
int nmfb_nnls_batch_ws(const double *ctc, const double *ctb, const double *btb,
                       const uint8_t *warm_passive, int warm_mode, const double *tol,
                       long max_changes, long nrhs, long k, double *x, uint8_t *passive,
                       long long *changes, double *resid2, int8_t *status,
                       uint8_t *seed_scratch, int *flag_scratch, double *ftab, long ftab_len,
                       void *stream);

/* out (rows, k) = scale * A B, A (rows, cols), B (cols, k); tol[i] =
 * 1e-12 max(1, ||out_i||_inf) when tol != NULL; work >= nmfb_rowprod_work_len.
 * Replaces the driver products M Y^T (update_X) and F Y^T. */
long nmfb_rowprod_work_len(long rows, long cols, long k, int a_is_f32);
int nmfb_rowprod(const void *A, int a_is_f32, long rows, long cols, const double *B, long k,
                 double *out, double *tol, double scale, double *work, long work_len,
                 void *stream);

/* out (cols, k) = scale * A^T B, A (rows, cols), B (rows, k): X^T M (update_Y,
 * SPEC.md:200), the Grams X^T X / Y Y^T, F^T X (graY).  work >= nmfb_colprod_work_len. */
long nmfb_colprod_work_len(long rows, long cols, long k);
int nmfb_colprod(const void *A, int a_is_f32, long rows, long cols, const double *B, long k,
                 double *out, double *tol, double scale, double *work, long work_len,
                 void *stream);

/* Both streaming products of one pass over A (rows, cols), cols even: outR (rows, k) =
 * A B1 with B1 (cols, k), and outC (cols, k) = A^T B2 with B2 (rows, k).  The stage-2
 * Armijo pass M dY^T / M^T dX (residual-free mode; the refresh then updates M Y^T and
 * M^T X incrementally).  Deterministic.  work >= nmfb_dualprod_work_len. */
long nmfb_dualprod_work_len(long rows, long cols, long k);
int nmfb_dualprod(const void *A, int a_is_f32, long rows, long cols, const double *B1,
                  const double *B2, long k, double *outR, double *outC, double *work,
                  long work_len, void *stream);

/* btb of both half-sweeps: squared row and column norms of M. */
int nmfb_sqnorms(const void *A, int a_is_f32, long rows, long cols, double *row_out,
                 double *col_out, double *work, long work_len, void *stream);

/* stats = [||Xn-X||^2 + ||Yn-Y||^2, ||X||^2 + ||Y||^2, sum r2] */
int nmfb_stage1_stats(const double *Xo, const double *Xn, long nx, const double *Yo,
                      const double *Yn, long ny, const double *r2, long nr, double *stats,
                      double *work, long work_len, void *stream);

/* tol[r] = 1e-12 max(1, ||c_r||_inf) for a product already reduced across ranks */
int nmfb_row_tol(const double *c, long rows, long k, double *tol, void *stream);

/* *acc = min(*acc, (tag << 40) | (i << 8) | st[i]) over the i with st[i] != 0 (acc
 * initialised to all ones by the caller): the first failing rhs of the earliest tagged
 * batch and its status code; tag < 2^24, len < 2^32. */
int nmfb_first_failure_i8(const int8_t *st, long len, long tag, unsigned long long *acc,
                          void *stream);
/* *out = first index with st != 0, 0x7F7F7F7F when none (nnls status scan) */
int nmfb_first_nonzero_i8(const int8_t *st, long len, int *out, void *stream);

/* number of partial blocks used by the IPM reductions (work sizing) */
int nmfb_ipm_reduce_blocks(void);

/* F = X Y - M, graX = F Y^T, out[0] = ||F||^2 (SPEC.md:265 assemble_gradients) */
int nmfb_residual(const void *M, int m_is_f32, long n, long m, long k, const double *X,
                  const double *Yt, double *F, double *gX, double *out, double *work,
                  void *stream);

/* R1 blocks + block Cholesky + h = L^{-1}(mux/x - graX), g = L^{-T} h,
 * Apk = packed R1^{-1}, XXpk = packed x x^T; *bad = first failing row (0x7F7F7F7F: none) */
int nmfb_r1_factor(const double *GY, const double *X, const double *R, const double *gX,
                   double mux, double rho, long n, long k, double *L, double *h, double *g,
                   double *Apk, double *XXpk, int *bad, void *stream);

/* h = L^{-1}(scale b1), g = L^{-T} h (predictor right-hand side with reused factors) */
int nmfb_hg(const double *L, const double *b1, double b1_scale, long n, long k, double *h,
            double *g, void *stream);

/* out (ca, cb) = A^T B for A (rows, ca), B (rows, cb); work >= nmfb_atb_work_len */
long nmfb_atb_work_len(long rows, long ca, long cb);
int nmfb_atb(const double *A, long rows, long ca, const double *B, long cb, double *out,
             double *work, long work_len, void *stream);

/* P[i][(p,q,a)] = x_ip Rinv_i[q,a]  (full-Hessian coupling, n x k^3) */
int nmfb_make_p(const double *X, const double *Apk, long n, long k, double *P, void *stream);

/* A (mk, mk) lower block triangle = blockdiag(X^T X + rho I + Diag(s/y)) - S
 * (S = schur_reduce's s_acc, _kernels_numba.py:72; W != NULL adds the full-C
 * cross terms) */
int nmfb_schur_assemble(const double *Yt, const double *S, long m, long k, const double *Zpk,
                        const double *XtX, double rho, const double *W, double *A,
                        void *stream);

/* full-C residual term: A -= sum_i f_ij f_il Rinv_i (lower block triangle) */
long nmfb_term4_work_len(long n, long m, long k);
int nmfb_schur_term4(const double *F, long n, long m, long k, const double *Apk, double *A,
                     double *work, long work_len, void *stream);

/* rhs = muy/y - graY - r_acc, r_acc_j = H y_j (+ (F^T g)_j when FtG != NULL)
 * (rhs_reduce, _kernels_numba.py:146) */
int nmfb_schur_rhs(const double *Yt, const double *gY, const double *H, const double *FtG,
                   double muy, long m, long k, double *rhs, void *stream);

/* back_substitute (_kernels_numba.py:181) + dr, ds + reductions:
 * out = [(dx,dy).grad phi, alpha1_max, alpha2_max, row part of the first, column part]
 * */
int nmfb_direction(const double *L, const double *Xf, const double *h, const double *Gdy,
                   const double *FdY, const double *X, const double *R, const double *gX,
                   double mux, const double *Yt, const double *S, const double *gY,
                   const double *dY, double muy, double tau, long n, long m, long k, double *dX,
                   double *dR, double *dS, double *out, double *work, long work_len,
                   void *stream);

/* Armijo in one pass over M: out = [AA, AB, BB, AC, BC, CC] for A = F,
 * B = dX Y + X dY, C = dX dY (SPEC.md:319 armijo_search) */
int nmfb_quartic(const double *F, long n, long m, long k, const double *X, const double *dX,
                 const double *Yt, const double *dYt, double *out, double *work, void *stream);

/* out[2t + {0,1}] = sum log1p(a_t dv/v) over X / Y, a_t = (*alpha_max) 2^-t */
int nmfb_barrier_trials(const double *X, const double *dX, long nx, const double *Yt,
                        const double *dYt, long ny, const double *alpha_max, int ntrials,
                        double *out, double *work, long work_len, void *stream);

/* Armijo acceptance on the device: reads the scalar block written by
 * nmfb_direction / nmfb_quartic / nmfb_barrier_trials (gtp, alpha maxima, quartic
 * coefficients, barrier sums) and writes alpha1, t, alpha2 (graph-capturable). */
int nmfb_armijo_select(double *sc, double mu, double wx, double wy, double eta,
                       int max_backtracks, const int *fcodes, void *stream);
/* graph capture helper: while mu_dev != NULL, r1_factor / schur_rhs / direction /
 * kkt_sums / armijo_select / armijo_lazy read [mu, wx mu, wy mu] from mu_dev at run
 * time instead of their scalar arguments (a captured iteration then replays for any
 * mu); pass NULL after the capture. */
int nmfb_set_mu_source(const double *mu_dev);

/* nmfb_barrier_trials + nmfb_armijo_select with lazy trial batches: trials 0..7, a
 * device pre-check, the remaining trials only when it did not decide (their launches
 * return at once otherwise), then the full search -- the same accepted t.  Uses
 * sc[31] as the decided flag; graph-capturable; single rank (the X-side trial sums
 * are not all-reduced). */
int nmfb_armijo_lazy(const double *X, const double *dX, long nx, const double *Yt,
                     const double *dYt, long ny, double *sc, int ntrials, double mu, double wx,
                     double wy, double eta, int max_backtracks, const int *fcodes, double *work,
                     long work_len, void *stream);
/* nmfb_step_nudge that ORs 1 into *flag when an entry was nudged; alpha from alpha_dev
 * when it is not NULL */
int nmfb_step_nudge_flag(double *v, const double *dv, long len, const double *alpha_dev,
                         double alpha, double tau, int *flag, void *stream);
/* residual-free refresh after a clean step (*flag == 0): MY += a MdY (nlen entries),
 * MX += a MtdX (mlen entries), a = *alpha_dev or alpha; nothing when *flag != 0 */
int nmfb_ffree_advance(double *MY, const double *MdY, long nlen, double *MX, const double *MtdX,
                       long mlen, const double *alpha_dev, double alpha, const int *flag,
                       void *stream);
/* The whole update of SPEC.md:359 in one launch: x, y += a1 (dx, dy) with the nudge rule (a
 * nudged entry ORs 1 into *flag when flag != NULL), r, s += a2 (dr, ds), and, when MY / MX are
 * given (residual-free dual mode), M Y^T += a1 M dY^T and M^T X += a1 M^T dX (the caller
 * recomputes both after a nudged step).  a1 / a2 from device memory when the pointer is
 * not NULL. */
int nmfb_step_all(double *X, const double *dX, long nk, double *Y, const double *dY, long mk,
                  double *R, const double *dR, double *S, const double *dS, double *MY,
                  const double *MdY, double *MX, const double *MtdX, const double *a1_dev,
                  double a1, const double *a2_dev, double a2, double tau, int *flag,
                  void *stream);
/* as nmfb_step_nudge with alpha read from device memory */
int nmfb_step_nudge_dev(double *v, const double *dv, long len, const double *alpha, double tau,
                        void *stream);

/* v += alpha dv with the (1 - tau) nudge */
int nmfb_step_nudge(double *v, const double *dv, long len, double alpha, double tau,
                    void *stream);

/* E (PAPER Eq. 9) ingredients, out[12]; R == NULL scores primal-only duals
 * (SPEC.md:420 kkt_error_primal_only) */
int nmfb_kkt_sums(const double *X, const double *R, const double *gX, long nx, const double *Yt,
                  const double *S, const double *gY, long ny, double mux, double muy,
                  double *out, double *work, void *stream);

/* mu_aff numerator (PAPER Eq. 7) */
int nmfb_affine_mu(const double *X, const double *dX, const double *R, const double *dR, long nx,
                   const double *Yt, const double *dY, const double *S, const double *dS, long ny,
                   double a1, double a2, double *out, double *work, void *stream);

int nmfb_clamp_min(double *v, long len, double lo, void *stream);
int nmfb_fill(double *v, long len, double c, void *stream);

/* spd_solve: in-place lower Cholesky of A (N x N); *info = first
 * non-positive pivot column or -1.  Then (L L^T) x = b in place on b. */
int nmfb_dense_cholesky(double *A, long N, int *info, void *stream);
int nmfb_dense_solve(const double *L, long N, double *b, void *stream);
/* Factor and forward-substitute in one launch (b <- L^{-1} b rides along as one more tile
 * row of the dataflow Cholesky, csrc/dense_flow.cuh), then nmfb_dense_solve_back finishes
 * b <- L^{-T} b: the spd_solve of SPEC.md:68 for the full-coupling directions, whose
 * right-hand side is known before the factorization.  nmfb_dense_solve_mode: 1 forward,
 * 2 backward, 3 both, with an existing factor (the predictor's reuse).
 * The dense factor / solve entries keep their scratch in device globals: call them from one
 * stream at a time per process. */
int nmfb_dense_cholesky_rhs(double *A, long N, double *b, int *info, void *stream);
int nmfb_dense_solve_back(const double *L, long N, double *b, void *stream);
int nmfb_dense_solve_mode(const double *L, long N, double *b, int mode, void *stream);
/* profiling aid: buf (device, 8 int64 per tile, global tile order) receives globaltimer
 * stamps of the dataflow factorization's phases; NULL switches it off */
int nmfb_flow_profile(long long *buf);

/* Exact low-rank Gauss-Newton reduced-system solve (replaces the dense mk x mk
 * spd_solve when the coupling is C-bar, PAPER Eq. 12): S = U Zb U^T with
 * U = Y^T (x) I_k has rank <= k^2.
 *   nmfb_d_factor:       D_j = X^T X + rho I + Diag(s_j/y_j) = LD_j LD_j^T, packed D_j^{-1}, y_j y_j^T
 *   nmfb_lowrank_factor: LG = chol(G), G = U^T D^{-1} U; LH = chol(I - LG^T Zb LG); *info = -1 iff
 *                        the reduced matrix is positive definite.  work >= 2 k^4 doubles (Zb kept
 *                        in work[0, k^4) for the solves)
 *   nmfb_lowrank_solve:  dy = (D - U Zb U^T)^{-1} rhs */
int nmfb_d_factor(const double *XtX, const double *Yt, const double *S, double rho, long m,
                  long k, double *LD, double *Dinvpk, double *YYpk, int *bad, void *stream);
int nmfb_lowrank_factor(const double *Zpk, const double *Gpk, long k, double *LG, double *LH,
                        double *work, int *info, void *stream);
int nmfb_lowrank_solve(const double *LD, const double *Yt, const double *LG, const double *LH,
                       const double *Zb, long m, long k, const double *rhs, double *dy, double *u,
                       double *w, double *cwork, long cwork_len, void *stream);

/* Fused small-problem Gauss-Newton iteration (k <= 4, m k <= 2048; configs c1-c3):
 * the same mathematics as the general entries in 3 + 3 kernels with deterministic
 * last-CTA reductions.  tickets: 4 zero-initialised uint32 counters (self-resetting). */
int nmfb_small_supported(long n, long m, long k);
long nmfb_small_work_len(long n, long m, long k);
int nmfb_small_direction(const double *X, const double *R, const double *gX, const double *Yt,
                         const double *S, const double *gY, long n, long m, long k, double mux,
                         double muy, double rho, double tau, double *L, double *h, double *LD,
                         double *LG, double *LH, double *Zb, double *Z, double *H, double *XtX,
                         double *dX, double *dR, double *dY, double *dS, double *Gdy, double *sc,
                         int *iscal, double *work, unsigned int *tickets, void *stream);
int nmfb_small_step_refresh(const void *M, int m_is_f32, long n, long m, long k, double *X,
                            double *R, double *Yt, double *S, const double *dX, const double *dR,
                            const double *dY, const double *dS, double *Xf, double *Ytf,
                            double *Fold, double *Fnew, double *gX, double *gY, double mu,
                            double wx, double wy, double eta, int max_bt, double tau, int ntrials,
                            double *sc, const int *fcodes, double *work, unsigned int *tickets,
                            void *stream);

/* Residual-free IPM pieces for large M (no n x m workspace; csrc/ipm.cu):
 *   grad[r] = V[r] G - MV[r], part[b] = partial <V, MV>   (graX = X YY^T - M Y^T and
 *   graY = Y^T XX - (X^T M)^T);  sc[0] = ||M||^2 - 2<X, M Y^T> + <XX, YY>;
 *   sc[10..15] = quartic Armijo coefficients from k x k Grams and traces. */
int nmfb_ffree_grad_rows(const double *V, const double *G, const double *MV, long rows, long k,
                         double *grad, double *part, void *stream);
int nmfb_ffree_fsq(const double *part, double mnorm2, const double *XX, const double *YY, long k,
                   double *sc, double *xm_out, void *stream);
int nmfb_ffree_quartic(const double *A1, const double *A2, const double *XX, const double *B1,
                       const double *B2, const double *YY, const double *Dgx, const double *Dgy,
                       const double *Dmd, long k, double *sc, void *stream);

/* number of kernel launches issued by this library so far (host counter) */
unsigned long long nmfb_launch_count(void);
/* Select the TMA-fed fp64 streaming products (1, default) or the register-direct DMMA
 * kernels (0) for nmfb_rowprod / nmfb_colprod; -1 only queries.  Returns the previous
 * setting.  (Both are deterministic; the row products are bit-identical.) */
int nmfb_tma_products(int on);
/* Select the tcgen05 (tf32 x 3 split, fp32 accumulate per 512-column chunk, fp64 partials)
 * products for an fp32 M (1, default) or the FP64 DMMA kernels (0); -1 only queries. */
int nmfb_tc_products(int on);
/* Name of the last CUDA error behind an NMFB_ELAUNCH return ("no error" if none). */
const char *nmfb_last_cuda_error(void);


/* Persistent Gauss-Newton inner loop for small problems (csrc/persist.cu): one
 * cooperative launch runs PAPER Alg. 2's inner iterations while
 * E(.;mu) > eps_mu and E(.;0) > tol0, up to max_iters.  log: max_iters x 8 doubles per iteration
 * [t, alpha1, alpha2, ||F||^2, E_mu, E_0, globaltimer ns, -]; status (device
 * int[2]) = [iterations done, exit code 0 done / 1 factorization failure (no step)
 * / 2 Armijo stall].  fcodes = [R1 failing row, capacitance info, D failing col]
 * (host initialises 0x7F7F7F7F, -1, 0x7F7F7F7F).  grid = 0: automatic.  prof
 * (optional, may be NULL): 16 clock64 stamps per iteration from CTA 0 (phase timing). */
int nmfb_persist_supported(long n, long m, long k, int grid, int m_is_f32);
long nmfb_persist_work_len(long n, long m, long k, int grid);
int nmfb_ipm_persist(const void *M, int m_is_f32, long n, long m, long k, double *X, double *R,
                     double *gX, double *Yt, double *S, double *gY, double *Fout, double *L,
                     double *Xf, double *Ytf, double *LD, double *LG, double *LH, double *Zb,
                     double mu, double wx, double wy, double rho, double tau, double eta,
                     double eps_mu, double tol0, int max_bt, int ntrials, int max_iters, double *sc,
                     int *fcodes, double *logv, int *status, double *work, unsigned int *bar,
                     int grid, long long *prof, void *stream);


/* Up to four k x k Grams out_q = A_q^T B_q over the same rows (row-major fp64 inputs,
 * unused slots NULL); deterministic.  work >= nmfb_grams_work_len(rows, k, count). */
/* creates the per-device cuBLAS handle used by nmfb_atb for large A^T B (plain
 * DGEMM); call once outside CUDA-graph capture (later calls are capturable). */
int nmfb_blas_init(void *stream);
long nmfb_grams_work_len(long rows, long k, long count);
int nmfb_grams(int count, const double *A0, const double *B0, double *O0, const double *A1,
               const double *B1, double *O1, const double *A2, const double *B2, double *O2,
               const double *A3, const double *B3, double *O3, long rows, long k, double *work,
               long work_len, void *stream);


/* Persistent stage 1 for small problems (csrc/stage1_persist.cu, k <= 8): every ANLS
 * sweep of run_stage1 in one cooperative launch, the same
 * bit-exact NNLS as nmfb_surface_nnls_batch.  X (n x k), Yt (m x k), pX, pY are
 * updated in place; Xn is unused scratch; Yn (m x k) is scratch; stX / stY receive
 * the per-rhs NNLS status of the last sweep.  tol_fixed < 0: per-rhs tolerance
 * 1e-12 max(1, ||ctb||_inf).  first_mode: 0 cold, 2 seeded from pX / pY.  fixed: run
 * exactly max_sweeps.  logv: per sweep [0.5 sum r2, step, norm, -]; status (device
 * int[3]) = [sweeps, converged, failed]. */
int nmfb_stage1_persist_supported(long n, long m, long k, int m_is_f32);
/* profiling hook: per-sweep phase clocks of CTA 0 (prof[sweep * 16 + i]); NULL disables */
int nmfb_stage1_set_prof(long long *prof);
long nmfb_stage1_persist_work_len(long n, long m, long k);
int nmfb_stage1_persist(const void *M, int m_is_f32, long n, long m, long k, double *X, double *Yt,
                        double *Xn, double *Yn, uint8_t *pX, uint8_t *pY, const double *row_n2,
                        const double *col_n2, int8_t *stX, int8_t *stY, double tol_fixed,
                        int first_mode, int max_sweeps, int fixed, double eps_stol, double *logv,
                        int *status, double *work, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* NMFB200_H */
