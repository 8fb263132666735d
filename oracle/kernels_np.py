"""oracle.kernels_np -- TEST INFRASTRUCTURE ONLY (CPU baseline speed path).

Vectorised NumPy/BLAS restatement of the reference's Schur-side kernels in
the formulation of the reference's NumPy backend
(/root/reference/pkg/src/nmfstream/_kernels_numpy.py:50-131: chunked batched
solves + BLAS contractions, O(n m^2 k^2) GN / O(n m^2 k^3) full).  The
reference survey measured this backend much faster than the numba one at
large m, so the CPU baseline uses it; results agree
with the bit-exact C oracle to rounding (tests/test_oracle_golden.py).
"""
from __future__ import annotations

import numpy as np

_BUDGET = 4_000_000  # doubles per chunk temporary


def _chunks(n, per_row):
    step = max(1, min(n, _BUDGET // max(1, per_row)))
    for i0 in range(0, n, step):
        yield slice(i0, min(n, i0 + step))


def _w(l, yt, sl):
    """W_i = L_i^{-1} Y^T for the rows of one chunk -> (B, k, m)."""
    b = sl.stop - sl.start
    return np.linalg.solve(l[sl], np.broadcast_to(yt, (b,) + yt.shape))


def schur_reduce(x_rows, y_cols, l, h, resid, full):
    n, k = x_rows.shape
    m = y_cols.shape[0]
    yt = np.ascontiguousarray(y_cols.T)
    S = np.zeros((m * k, m * k))
    racc = np.zeros((m, k))
    if not full:
        for sl in _chunks(n, m * m + 2 * k * m):
            W = _w(l, yt, sl)
            T = np.matmul(W.transpose(0, 2, 1), W)                     # (B, m, m)
            XX = x_rows[sl, :, None] * x_rows[sl, None, :]               # (B, k, k)
            B = T.shape[0]
            S4 = (T.reshape(B, m * m).T @ XX.reshape(B, k * k)).reshape(m, m, k, k)
            S += S4.transpose(0, 2, 1, 3).reshape(m * k, m * k)
            wh = np.einsum("bpj,bp->bj", W, h[sl])
            racc += wh.T @ x_rows[sl]
    else:
        eye = np.eye(k)
        for sl in _chunks(n, 2 * m * k * k):
            B = sl.stop - sl.start
            linv = np.linalg.solve(l[sl], np.broadcast_to(eye, (B, k, k)))
            W = linv @ yt                                                # (B, k, m)
            pinv = linv.transpose(0, 2, 1)
            G = (x_rows[sl, None, :, None] * W.transpose(0, 2, 1)[:, :, None, :]
                 + resid[sl, :, None, None] * pinv[:, None, :, :])      # (B, m, k, k)
            G2 = G.transpose(1, 2, 0, 3).reshape(m * k, B * k)
            S += G2 @ G2.T
            racc += np.einsum("bjpq,bq->jp", G, h[sl])
    return S, racc


def rhs_reduce(x_rows, y_cols, l, h, resid, full):
    n, k = x_rows.shape
    m = y_cols.shape[0]
    yt = np.ascontiguousarray(y_cols.T)
    racc = np.zeros((m, k))
    for sl in _chunks(n, 2 * k * m):
        W = _w(l, yt, sl)
        racc += np.einsum("bpj,bp->bj", W, h[sl]).T @ x_rows[sl]
        if full:
            g = np.linalg.solve(l[sl].transpose(0, 2, 1), h[sl][:, :, None])[:, :, 0]
            racc += resid[sl].T @ g
    return racc


def back_substitute(x_rows, y_cols, l, h, dy_rows, resid, full):
    n, k = x_rows.shape
    yt = np.ascontiguousarray(y_cols.T)
    t = x_rows @ dy_rows.T                                               # (n, m)
    q = np.empty((n, k))
    for sl in _chunks(n, 2 * k * yt.shape[1]):
        W = _w(l, yt, sl)
        q[sl] = np.einsum("bpj,bj->bp", W, t[sl])
    if full:
        q += np.linalg.solve(l, (resid @ dy_rows)[:, :, None])[:, :, 0]
    return np.linalg.solve(l.transpose(0, 2, 1), (h - q)[:, :, None])[:, :, 0]
