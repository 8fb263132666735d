"""oracle.lowrank -- TEST INFRASTRUCTURE ONLY (the checker / CPU baseline, never the product).

The stage-2 algebra of ``oracle.driver`` (PAPER Algorithm 2) for
instances whose dense mk x mk Schur matrix cannot be formed on a host (BASELINE c4:
mk = 50 000 -> 20 GB and ~15 h per iteration through the reference's
``schur_reduce`` + LAPACK Cholesky).  Same Newton system, solved
exactly with two algebraic identities instead of the dense matrix:

* residual-free products: graX = X (Y Y^T) - M Y^T, graY = (X^T X) Y - X^T M,
  ||F||^2 = ||M||^2 - 2 <X, M Y^T> + <X^T X, Y Y^T>, and the Armijo quartic's inner
  products from k x k Grams plus one product M dY^T (three passes over M per iteration);
* the Gauss-Newton Schur correction of ``schur_reduce`` (_kernels_numba.py:83-106) is
  S = U Zb U^T with U = Y^T (x) I_k and Zb[(a,p),(b,q)] = sum_i R1_i^{-1}[a,b] x_ip x_iq
  (rank <= k^2), so (D - S) dy = rhs is solved by the push-through identity
  (I - Zb G) w = Zb U^T D^{-1} rhs, G = U^T D^{-1} U, dy = D^{-1}(rhs + U w), symmetrised
  as H = I - L_G^T Zb L_G with G = L_G L_G^T (A is PD <=> H is PD);
* back substitution dx_i = R1_i^{-1}(b1_i - P x_i), P = sum_j y_j dy_j^T
  (_kernels_numba.py:181-205 with the Gauss-Newton coupling).

This is the CPU restatement of csrc/lowrank.cu + the residual-free mode of
paper_2101_08431_b200/solver.py, vectorised with NumPy/BLAS (all host cores).  It is
checked against the dense oracle (which calls the reference-pinned kernels) on small
instances in tests/test_oracle_lowrank.py.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class NotPD(RuntimeError):
    pass


def _chol(A):
    try:
        return np.linalg.cholesky(A)
    except np.linalg.LinAlgError as e:
        raise NotPD(str(e)) from None


def gradients_free(X, Yt, M, Mn2, red=lambda a: a):
    """(||F||^2, graX (n,k), graY (m,k)) without forming F = X Y - M."""
    MY = M @ Yt  # (n,k): one pass over M
    MtX = red(M.T @ X)  # (m,k): one pass over M
    XtX = red(X.T @ X)
    YY = Yt.T @ Yt
    gX = X @ YY - MY
    gY = Yt @ XtX - MtX
    fsq = Mn2 - 2.0 * red(float(np.vdot(X, MY))) + float(np.vdot(XtX, YY))
    return fsq, gX, gY


def quartic_free(X, Yt, dX, dYt, gX, gY, M, red=lambda a: a):
    """Inner products (aa, ab, bb, ac, bc, cc) of A = F, B = dX Y + X dY, C = dX dY."""
    MdY = M @ dYt  # (n,k): the third pass over M
    XtX, YY = red(X.T @ X), Yt.T @ Yt
    A1, A2 = red(dX.T @ dX), red(dX.T @ X)  # dX^T dX, dX^T X
    B1, B2 = dYt.T @ dYt, Yt.T @ dYt  # dY dY^T, Y dY^T
    ab = red(float(np.vdot(dX, gX))) + float(np.vdot(dYt, gY))
    bb = float(np.vdot(A1, YY)) + 2.0 * float(np.vdot(A2.T, B2.T)) + float(np.vdot(XtX, B1))
    ac = float(np.vdot(A2, B2.T)) - red(float(np.vdot(dX, MdY)))
    bc = float(np.vdot(A1, B2)) + float(np.vdot(A2.T, B1))
    cc = float(np.vdot(A1, B1))
    return (np.nan, ab, bb, ac, bc, cc)


@dataclass
class LowrankFactor:
    Xf: np.ndarray
    Ytf: np.ndarray
    R1inv: np.ndarray  # (n,k,k)
    Dinv: np.ndarray  # (m,k,k)
    Zb: np.ndarray  # (k^2,k^2), index (a,p)
    LG: np.ndarray
    LH: np.ndarray


def factor(X, Yt, R, S, rho, red=lambda a: a):
    """R1 / D blocks, Zb, G and the capacitance factor at the current point."""
    n, k = X.shape
    m = Yt.shape[0]
    I = np.eye(k)
    R1 = (Yt.T @ Yt)[None] + rho * I[None] + (R / X)[:, :, None] * I[None]
    _chol(R1)  # the reference's block_cholesky PD test (_kernels_numba.py:21-22)
    R1inv = np.linalg.inv(R1)
    R1inv = 0.5 * (R1inv + R1inv.transpose(0, 2, 1))
    xx = (X[:, :, None] * X[:, None, :]).reshape(n, k * k)
    Z = red(R1inv.reshape(n, k * k).T @ xx)  # [(a,b),(p,q)]
    Zb = Z.reshape(k, k, k, k).transpose(0, 2, 1, 3).reshape(k * k, k * k)
    XtX = red(X.T @ X)
    D = XtX[None] + rho * I[None] + (S / Yt)[:, :, None] * I[None]
    _chol(D)
    Dinv = np.linalg.inv(D)
    Dinv = 0.5 * (Dinv + Dinv.transpose(0, 2, 1))
    yy = (Yt[:, :, None] * Yt[:, None, :]).reshape(m, k * k)
    G = (yy.T @ Dinv.reshape(m, k * k)).reshape(k, k, k, k).transpose(0, 2, 1, 3).reshape(k * k, k * k)
    G = 0.5 * (G + G.T)
    LG = _chol(G)
    H = np.eye(k * k) - LG.T @ Zb @ LG
    LH = _chol(0.5 * (H + H.T))
    return LowrankFactor(X.copy(), Yt.copy(), R1inv, Dinv, Zb, LG, LH)


def _solve_reduced(fac: LowrankFactor, rhs):
    """(D - U Zb U^T) dy = rhs (rhs, dy as (m,k))."""
    from scipy.linalg import solve_triangular

    k = rhs.shape[1]
    Dr = np.einsum("jpq,jq->jp", fac.Dinv, rhs)
    u = (fac.Ytf.T @ Dr).reshape(k * k)  # U^T D^{-1} rhs, index (a,p)
    z = fac.LG.T @ (fac.Zb @ u)
    v = solve_triangular(fac.LH, z, lower=True, check_finite=False)
    v = solve_triangular(fac.LH.T, v, lower=False, check_finite=False)
    w = solve_triangular(fac.LG.T, v, lower=False, check_finite=False).reshape(k, k)
    return np.einsum("jpq,jq->jp", fac.Dinv, rhs + fac.Ytf @ w)


def solve(fac: LowrankFactor, X, Yt, R, S, gX, gY, mux, muy, red=lambda a: a):
    """Newton direction at (X, Yt, R, S) with the factorization ``fac``
    (reduced solve, back substitution, dr/ds)."""
    b1 = mux / X - gX
    g = np.einsum("iab,ib->ia", fac.R1inv, b1)  # R1^{-1} b1
    racc = fac.Ytf @ red(g.T @ fac.Xf)  # r_acc[j,p] = sum_a y_ja sum_i g_ia x_ip
    b2 = muy / Yt - gY
    dy = _solve_reduced(fac, b2 - racc)
    Pm = fac.Ytf.T @ dy  # sum_j y_j dy_j^T
    dx = np.einsum("iab,ib->ia", fac.R1inv, b1 - fac.Xf @ Pm.T)
    dr = mux / X - R - (R / X) * dx
    ds = muy / Yt - S - (S / Yt) * dy
    gtp = red(float(np.vdot(dx, gX - mux / X))) + float(np.vdot(dy, gY - muy / Yt))
    return dx, dy, dr, ds, gtp
