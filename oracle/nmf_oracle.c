/*
 * oracle/nmf_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the seven hot kernels of the reference `nmfstream`
 * package (/root/reference/pkg/src/nmfstream/_kernels_numba.py).  Each
 * function states the reference lines it follows.  The arithmetic is
 * written in the same operation order as the numba loops and is compiled
 * with -ffp-contract=off (numba emits no FMA), so the
 * results are bit-identical to the reference kernels; tests/golden pins
 * that against vectors produced by the reference itself.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference arm may load this library.  It is the checker, never
 * the product: the product path is paper_2101_08431_b200/csrc (CUDA).
 *
 * Layouts: all arrays C-contiguous float64 unless stated; bool arrays are
 * uint8 (numpy bool_ is one byte).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define IDX2(a, b, nb) ((size_t)(a) * (size_t)(nb) + (size_t)(b))
#define IDX3(a, b, c, nb, nc) (((size_t)(a) * (size_t)(nb) + (size_t)(b)) * (size_t)(nc) + (size_t)(c))

/* block_cholesky  -- _kernels_numba.py:12-29.
 * blocks (nb,k,k) -> out (nb,k,k) zero-initialised by the caller.
 * Returns the first non-PD block index or -1.  Blocks after the failing one
 * are left zero, the failing block is partially filled (numba returns early). */
long orc_block_cholesky(const double *blocks, long nb, long k, double *out)
{
    for (long b = 0; b < nb; ++b) {
        const double *A = blocks + (size_t)b * k * k;
        double *L = out + (size_t)b * k * k;
        for (long j = 0; j < k; ++j) {
            double s = A[IDX2(j, j, k)];
            for (long p = 0; p < j; ++p) s -= L[IDX2(j, p, k)] * L[IDX2(j, p, k)];
            if (s <= 0.0) return b;
            L[IDX2(j, j, k)] = sqrt(s);
            for (long i = j + 1; i < k; ++i) {
                double t = A[IDX2(i, j, k)];
                for (long p = 0; p < j; ++p) t -= L[IDX2(i, p, k)] * L[IDX2(j, p, k)];
                L[IDX2(i, j, k)] = t / L[IDX2(j, j, k)];
            }
        }
    }
    return -1;
}

/* block_solve_lower -- _kernels_numba.py:32-43.  l (nb,k,k), b (nb,k,r) -> z */
void orc_block_solve_lower(const double *l, const double *b, long nb, long k, long r, double *z)
{
    for (long t = 0; t < nb; ++t) {
        const double *L = l + (size_t)t * k * k;
        for (long c = 0; c < r; ++c)
            for (long i = 0; i < k; ++i) {
                double s = b[IDX3(t, i, c, k, r)];
                for (long p = 0; p < i; ++p) s -= L[IDX2(i, p, k)] * z[IDX3(t, p, c, k, r)];
                z[IDX3(t, i, c, k, r)] = s / L[IDX2(i, i, k)];
            }
    }
}

/* block_solve_lower_t -- _kernels_numba.py:46-57 (solves L^T z = b). */
void orc_block_solve_lower_t(const double *l, const double *b, long nb, long k, long r, double *z)
{
    for (long t = 0; t < nb; ++t) {
        const double *L = l + (size_t)t * k * k;
        for (long c = 0; c < r; ++c)
            for (long i = k - 1; i >= 0; --i) {
                double s = b[IDX3(t, i, c, k, r)];
                for (long p = i + 1; p < k; ++p) s -= L[IDX2(p, i, k)] * z[IDX3(t, p, c, k, r)];
                z[IDX3(t, i, c, k, r)] = s / L[IDX2(i, i, k)];
            }
    }
}

/* _solve_lower_cols -- _kernels_numba.py:60-69: out(k,m) <- L^{-1} rhs(k,m) */
static void solve_lower_cols(const double *L, const double *rhs, long k, long m, double *out)
{
    for (long c = 0; c < m; ++c)
        for (long i = 0; i < k; ++i) {
            double s = rhs[IDX2(i, c, m)];
            for (long p = 0; p < i; ++p) s -= L[IDX2(i, p, k)] * out[IDX2(p, c, m)];
            out[IDX2(i, c, m)] = s / L[IDX2(i, i, k)];
        }
}

/* schur_reduce -- _kernels_numba.py:72-143.
 * x_rows (n,k), y_cols (m,k), l (n,k,k), h (n,k), resid (n,m) (read only when
 * full), s_acc (mk,mk) and r_acc (m,k) zero-initialised by the caller. */
int orc_schur_reduce(const double *x_rows, const double *y_cols, const double *l,
                     const double *h, const double *resid, long n, long m, long k,
                     int full, double *s_acc, double *r_acc)
{
    const long mk = m * k;
    double *yt = (double *)malloc(sizeof(double) * k * m);
    double *w = (double *)malloc(sizeof(double) * k * m);
    if (!yt || !w) { free(yt); free(w); return -1; }
    for (long j = 0; j < m; ++j)
        for (long p = 0; p < k; ++p) yt[IDX2(p, j, m)] = y_cols[IDX2(j, p, k)];
    if (!full) {
        double *tj = (double *)malloc(sizeof(double) * m);
        if (!tj) { free(yt); free(w); return -1; }
        for (long i = 0; i < n; ++i) {
            solve_lower_cols(l + (size_t)i * k * k, yt, k, m, w);
            const double *u = x_rows + (size_t)i * k;
            const double *hi = h + (size_t)i * k;
            for (long j = 0; j < m; ++j) {
                double s = 0.0;
                for (long p = 0; p < k; ++p) s += w[IDX2(p, j, m)] * hi[p];
                tj[j] = s;
            }
            for (long j = 0; j < m; ++j)
                for (long p = 0; p < k; ++p) r_acc[IDX2(j, p, k)] += tj[j] * u[p];
            for (long j = 0; j < m; ++j)
                for (long lc = 0; lc < m; ++lc) {
                    double dot = 0.0;
                    for (long p = 0; p < k; ++p) dot += w[IDX2(p, j, m)] * w[IDX2(p, lc, m)];
                    for (long p = 0; p < k; ++p) {
                        long base_j = j * k + p;
                        double up = dot * u[p];
                        for (long q = 0; q < k; ++q) s_acc[IDX2(base_j, lc * k + q, mk)] += up * u[q];
                    }
                }
        }
        free(tj);
    } else {
        double *pinv = (double *)malloc(sizeof(double) * k * k);
        double *g = (double *)malloc(sizeof(double) * m * k * k);
        if (!pinv || !g) { free(pinv); free(g); free(yt); free(w); return -1; }
        for (long i = 0; i < n; ++i) {
            const double *li = l + (size_t)i * k * k;
            solve_lower_cols(li, yt, k, m, w);
            for (long c = 0; c < k; ++c)
                for (long row = k - 1; row >= 0; --row) {
                    double s = (row == c) ? 1.0 : 0.0;
                    for (long p = row + 1; p < k; ++p) s -= li[IDX2(p, row, k)] * pinv[IDX2(p, c, k)];
                    pinv[IDX2(row, c, k)] = s / li[IDX2(row, row, k)];
                }
            const double *u = x_rows + (size_t)i * k;
            const double *hi = h + (size_t)i * k;
            for (long j = 0; j < m; ++j) {
                double f = resid[IDX2(i, j, m)];
                for (long p = 0; p < k; ++p)
                    for (long q = 0; q < k; ++q)
                        g[IDX3(j, p, q, k, k)] = u[p] * w[IDX2(q, j, m)] + f * pinv[IDX2(p, q, k)];
            }
            for (long j = 0; j < m; ++j)
                for (long p = 0; p < k; ++p) {
                    double s = 0.0;
                    for (long q = 0; q < k; ++q) s += g[IDX3(j, p, q, k, k)] * hi[q];
                    r_acc[IDX2(j, p, k)] += s;
                }
            for (long j = 0; j < m; ++j)
                for (long lc = 0; lc < m; ++lc)
                    for (long p = 0; p < k; ++p) {
                        long base_j = j * k + p;
                        for (long q = 0; q < k; ++q) {
                            double dot = 0.0;
                            for (long c = 0; c < k; ++c)
                                dot += g[IDX3(j, p, c, k, k)] * g[IDX3(lc, q, c, k, k)];
                            s_acc[IDX2(base_j, lc * k + q, mk)] += dot;
                        }
                    }
        }
        free(pinv);
        free(g);
    }
    free(yt);
    free(w);
    return 0;
}

/* rhs_reduce -- _kernels_numba.py:146-178.  r_acc (m,k) zero-initialised. */
int orc_rhs_reduce(const double *x_rows, const double *y_cols, const double *l,
                   const double *h, const double *resid, long n, long m, long k,
                   int full, double *r_acc)
{
    double *yt = (double *)malloc(sizeof(double) * k * m);
    double *w = (double *)malloc(sizeof(double) * k * m);
    double *g = (double *)malloc(sizeof(double) * k);
    if (!yt || !w || !g) { free(yt); free(w); free(g); return -1; }
    for (long j = 0; j < m; ++j)
        for (long p = 0; p < k; ++p) yt[IDX2(p, j, m)] = y_cols[IDX2(j, p, k)];
    for (long i = 0; i < n; ++i) {
        const double *li = l + (size_t)i * k * k;
        solve_lower_cols(li, yt, k, m, w);
        const double *u = x_rows + (size_t)i * k;
        const double *hi = h + (size_t)i * k;
        for (long j = 0; j < m; ++j) {
            double s = 0.0;
            for (long p = 0; p < k; ++p) s += w[IDX2(p, j, m)] * hi[p];
            for (long p = 0; p < k; ++p) r_acc[IDX2(j, p, k)] += s * u[p];
        }
        if (full) {
            for (long row = k - 1; row >= 0; --row) {
                double s = hi[row];
                for (long p = row + 1; p < k; ++p) s -= li[IDX2(p, row, k)] * g[p];
                g[row] = s / li[IDX2(row, row, k)];
            }
            for (long j = 0; j < m; ++j) {
                double f = resid[IDX2(i, j, m)];
                for (long p = 0; p < k; ++p) r_acc[IDX2(j, p, k)] += f * g[p];
            }
        }
    }
    free(yt);
    free(w);
    free(g);
    return 0;
}

/* back_substitute -- _kernels_numba.py:181-224.  dx (n,k). */
int orc_back_substitute(const double *x_rows, const double *y_cols, const double *l,
                        const double *h, const double *dy_rows, const double *resid,
                        long n, long m, long k, int full, double *dx)
{
    double *yt = (double *)malloc(sizeof(double) * k * m);
    double *w = (double *)malloc(sizeof(double) * k * m);
    double *q = (double *)malloc(sizeof(double) * k);
    double *extra = (double *)malloc(sizeof(double) * k);
    double *fdy = (double *)malloc(sizeof(double) * k);
    if (!yt || !w || !q || !extra || !fdy) {
        free(yt); free(w); free(q); free(extra); free(fdy);
        return -1;
    }
    for (long j = 0; j < m; ++j)
        for (long p = 0; p < k; ++p) yt[IDX2(p, j, m)] = y_cols[IDX2(j, p, k)];
    for (long i = 0; i < n; ++i) {
        const double *li = l + (size_t)i * k * k;
        solve_lower_cols(li, yt, k, m, w);
        const double *u = x_rows + (size_t)i * k;
        for (long p = 0; p < k; ++p) q[p] = 0.0;
        for (long j = 0; j < m; ++j) {
            double t = 0.0;
            for (long p = 0; p < k; ++p) t += u[p] * dy_rows[IDX2(j, p, k)];
            for (long p = 0; p < k; ++p) q[p] += w[IDX2(p, j, m)] * t;
        }
        if (full) {
            for (long p = 0; p < k; ++p) {
                double s = 0.0;
                for (long j = 0; j < m; ++j) s += resid[IDX2(i, j, m)] * dy_rows[IDX2(j, p, k)];
                fdy[p] = s;
            }
            for (long row = 0; row < k; ++row) {
                double s = fdy[row];
                for (long p = 0; p < row; ++p) s -= li[IDX2(row, p, k)] * extra[p];
                extra[row] = s / li[IDX2(row, row, k)];
            }
            for (long p = 0; p < k; ++p) q[p] += extra[p];
        }
        for (long row = k - 1; row >= 0; --row) {
            double s = h[IDX2(i, row, k)] - q[row];
            for (long p = row + 1; p < k; ++p) s -= li[IDX2(p, row, k)] * dx[IDX2(i, p, k)];
            dx[IDX2(i, row, k)] = s / li[IDX2(row, row, k)];
        }
    }
    free(yt); free(w); free(q); free(extra); free(fdy);
    return 0;
}

/* ---------------- nnls_batch and helpers: _kernels_numba.py:227-477 ------ */

/* _passive_factor -- :227-244.  a_buf, l_buf are (k,k) scratch. */
static int passive_factor(const double *ctc, long k, const long *pidx, long np_,
                          double *a_buf, double *l_buf)
{
    for (long a = 0; a < np_; ++a)
        for (long b = 0; b < np_; ++b) a_buf[IDX2(a, b, k)] = ctc[IDX2(pidx[a], pidx[b], k)];
    for (long j = 0; j < np_; ++j) {
        double s = a_buf[IDX2(j, j, k)];
        for (long p = 0; p < j; ++p) s -= l_buf[IDX2(j, p, k)] * l_buf[IDX2(j, p, k)];
        if (s <= 0.0) return 0;
        l_buf[IDX2(j, j, k)] = sqrt(s);
        for (long i = j + 1; i < np_; ++i) {
            double t = a_buf[IDX2(i, j, k)];
            for (long p = 0; p < j; ++p) t -= l_buf[IDX2(i, p, k)] * l_buf[IDX2(j, p, k)];
            l_buf[IDX2(i, j, k)] = t / l_buf[IDX2(j, j, k)];
        }
    }
    return 1;
}

/* _chol_solve_small -- :247-258 */
static void chol_solve_small(const double *l_buf, long k, const double *b, long np_, double *z)
{
    for (long i = 0; i < np_; ++i) {
        double s = b[i];
        for (long p = 0; p < i; ++p) s -= l_buf[IDX2(i, p, k)] * z[p];
        z[i] = s / l_buf[IDX2(i, i, k)];
    }
    for (long i = np_ - 1; i >= 0; --i) {
        double s = z[i];
        for (long p = i + 1; p < np_; ++p) s -= l_buf[IDX2(p, i, k)] * z[p];
        z[i] = s / l_buf[IDX2(i, i, k)];
    }
}

/* _passive_solve_refined -- :261-274 (one iterative-refinement pass) */
static void passive_solve_refined(const double *d, long k, const long *pidx, long np_,
                                  const double *a_buf, const double *l_buf,
                                  double *z, double *rbuf, double *dz)
{
    for (long a = 0; a < np_; ++a) rbuf[a] = d[pidx[a]];
    chol_solve_small(l_buf, k, rbuf, np_, z);
    for (long a = 0; a < np_; ++a) {
        double s = d[pidx[a]];
        for (long b = 0; b < np_; ++b) s -= a_buf[IDX2(a, b, k)] * z[b];
        rbuf[a] = s;
    }
    chol_solve_small(l_buf, k, rbuf, np_, dz);
    for (long a = 0; a < np_; ++a) z[a] += dz[a];
}

/* nnls_batch -- :277-477.  Outputs zero-initialised by the caller:
 * x_out (nrhs,k) f64, p_out (nrhs,k) u8, changes_out (nrhs) i64,
 * resid2 (nrhs) f64, status (nrhs) i8.  The reference's passive-signature
 * factor cache (:296-298, :334-349) only skips recomputing an identical
 * factor; it is kept here so the operation sequence matches exactly. */
int orc_nnls_batch(const double *ctc, const double *ctb, const double *btb,
                   const uint8_t *warm_passive, long warm_mode, const double *tol,
                   long max_changes, long nrhs, long k,
                   double *x_out, uint8_t *p_out, int64_t *changes_out,
                   double *resid2, int8_t *status)
{
    uint8_t *passive = (uint8_t *)calloc(k, 1);
    uint8_t *prev_passive = (uint8_t *)calloc(k, 1);
    uint8_t *cache_sig = (uint8_t *)calloc(k, 1);
    double *x = (double *)calloc(k, sizeof(double));
    double *w = (double *)calloc(k, sizeof(double));
    double *z = (double *)calloc(k, sizeof(double));
    double *rbuf = (double *)calloc(k, sizeof(double));
    double *dz = (double *)calloc(k, sizeof(double));
    long *pidx = (long *)calloc(k, sizeof(long));
    double *a_buf = (double *)calloc(k * k, sizeof(double));
    double *l_buf = (double *)calloc(k * k, sizeof(double));
    int rc = 0;
    if (!passive || !prev_passive || !cache_sig || !x || !w || !z || !rbuf || !dz || !pidx ||
        !a_buf || !l_buf) {
        rc = -1;
        goto done;
    }
    int cache_valid = 0;
    for (long t = 0; t < nrhs; ++t) {
        const double *d = ctb + (size_t)t * k;
        const double tol_t = tol[t];
        int solved = 0;
        long nch = 0;
        int use_seed = 0;
        if (warm_mode == 2) {
            for (long j = 0; j < k; ++j) passive[j] = warm_passive[IDX2(t, j, k)] ? 1 : 0;
            use_seed = 1;
        } else if (warm_mode == 1 && t > 0) {
            for (long j = 0; j < k; ++j) passive[j] = prev_passive[j];
            use_seed = 1;
        }
        if (use_seed) {
            long np_ = 0;
            for (long j = 0; j < k; ++j)
                if (passive[j]) pidx[np_++] = j;
            if (np_ == 0) {
                int ok = 1;
                for (long j = 0; j < k; ++j)
                    if (d[j] > tol_t) { ok = 0; break; }
                if (ok) {
                    for (long j = 0; j < k; ++j) x[j] = 0.0;
                    solved = 1;
                }
            } else {
                int same = cache_valid;
                if (same)
                    for (long j = 0; j < k; ++j)
                        if (cache_sig[j] != passive[j]) { same = 0; break; }
                int ok = 1;
                if (!same) {
                    ok = passive_factor(ctc, k, pidx, np_, a_buf, l_buf);
                    if (ok) {
                        for (long j = 0; j < k; ++j) cache_sig[j] = passive[j];
                        cache_valid = 1;
                    } else {
                        cache_valid = 0;
                    }
                }
                if (ok) {
                    passive_solve_refined(d, k, pidx, np_, a_buf, l_buf, z, rbuf, dz);
                    int feas = 1;
                    for (long a = 0; a < np_; ++a)
                        if (z[a] < 0.0) { feas = 0; break; }
                    if (feas) {
                        for (long j = 0; j < k; ++j) x[j] = 0.0;
                        for (long a = 0; a < np_; ++a) x[pidx[a]] = z[a];
                        int dual_ok = 1;
                        for (long j = 0; j < k; ++j) {
                            double s = d[j];
                            for (long p = 0; p < k; ++p) s -= ctc[IDX2(j, p, k)] * x[p];
                            w[j] = s;
                            if (passive[j]) {
                                if (fabs(s) > tol_t) { dual_ok = 0; break; }
                            } else if (s > tol_t) {
                                dual_ok = 0;
                                break;
                            }
                        }
                        solved = dual_ok;
                    }
                }
            }
        }
        if (!solved) {
            for (long j = 0; j < k; ++j) {
                passive[j] = 0;
                x[j] = 0.0;
                w[j] = d[j];
            }
            int st = 0;
            for (;;) {
                long jmax = -1;
                double wmax = tol_t;
                for (long j = 0; j < k; ++j)
                    if (!passive[j] && w[j] > wmax) {
                        wmax = w[j];
                        jmax = j;
                    }
                if (jmax < 0) break;
                passive[jmax] = 1;
                nch += 1;
                if (nch > max_changes) { st = 1; break; }
                for (;;) {
                    long np_ = 0;
                    for (long j = 0; j < k; ++j)
                        if (passive[j]) pidx[np_++] = j;
                    if (np_ == 0) break;
                    int ok = passive_factor(ctc, k, pidx, np_, a_buf, l_buf);
                    if (!ok) {
                        cache_valid = 0;
                        st = 2;
                        break;
                    }
                    for (long j = 0; j < k; ++j) cache_sig[j] = passive[j];
                    cache_valid = 1;
                    passive_solve_refined(d, k, pidx, np_, a_buf, l_buf, z, rbuf, dz);
                    int all_pos = 1;
                    for (long a = 0; a < np_; ++a)
                        if (z[a] <= 0.0) { all_pos = 0; break; }
                    if (all_pos) {
                        for (long j = 0; j < k; ++j) x[j] = 0.0;
                        for (long a = 0; a < np_; ++a) x[pidx[a]] = z[a];
                        break;
                    }
                    double alpha = 1.0;
                    for (long a = 0; a < np_; ++a)
                        if (z[a] <= 0.0) {
                            double xa = x[pidx[a]];
                            double ratio = xa / (xa - z[a]);
                            if (ratio < alpha) alpha = ratio;
                        }
                    long ndrop = 0;
                    for (long a = 0; a < np_; ++a) {
                        long j = pidx[a];
                        double xa = x[j];
                        double newx = xa + alpha * (z[a] - xa);
                        if (z[a] <= 0.0 && xa / (xa - z[a]) <= alpha) {
                            x[j] = 0.0;
                            passive[j] = 0;
                            ndrop += 1;
                        } else {
                            x[j] = newx > 0.0 ? newx : 0.0;
                        }
                    }
                    nch += ndrop;
                    if (nch > max_changes) { st = 1; break; }
                }
                if (st != 0) break;
                for (long j = 0; j < k; ++j) {
                    double s = d[j];
                    for (long p = 0; p < k; ++p) s -= ctc[IDX2(j, p, k)] * x[p];
                    w[j] = s;
                }
            }
            status[t] = (int8_t)st;
        }
        for (long j = 0; j < k; ++j) {
            x_out[IDX2(t, j, k)] = x[j];
            p_out[IDX2(t, j, k)] = passive[j];
            prev_passive[j] = passive[j];
        }
        changes_out[t] = nch;
        double r2 = btb[t];
        for (long j = 0; j < k; ++j) r2 -= 2.0 * x[j] * d[j];
        for (long j = 0; j < k; ++j) {
            double s = 0.0;
            for (long p = 0; p < k; ++p) s += ctc[IDX2(j, p, k)] * x[p];
            r2 += x[j] * s;
        }
        resid2[t] = r2 > 0.0 ? r2 : 0.0;
    }
done:
    free(passive); free(prev_passive); free(cache_sig); free(x); free(w); free(z);
    free(rbuf); free(dz); free(pidx); free(a_buf); free(l_buf);
    return rc;
}
