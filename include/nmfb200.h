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

#ifdef __cplusplus
}
#endif

#endif /* NMFB200_H */
