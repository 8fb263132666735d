"""oracle.driver -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

CPU restatement of the reference's stage drivers.  The reference ships the
kernels but not the drivers, so this module restates
them from the reference's normative text and calls the bit-exact C kernels
of ``oracle.kernels`` for every kernel-level operation:

* anls-stage      SPEC.md:165-242, PAPER.md:93-128 (Algorithm 1)
* ipm-stage       SPEC.md:244-374, PAPER.md:136-366 (Algorithm 2, Eqs. 3-11)
* Schur solve     SPEC.md:68-76, PAPER.md:464-530 (Eqs. 12-13)
* two-stage       SPEC.md:376-451, PAPER.md:532-619 (Algorithm 3, Eqs. 14-18)

Frozen open semantics (DESIGN.md "Frozen semantics" lists the same items):

1. Warm mode: sweep 0 cold (mode 0), later sweeps mode 2 seeded with the
   previous sweep's passive sets.
2. Stage-1 stop: ||(x,y)_{k+1}-(x,y)_k|| <= eps_stol (1 + ||(x,y)_k||) checked
   after every full sweep, or the sweep cap.
3. Armijo uses the exact quartic expansion of the residual along the step
   (phi is evaluated as phi(0) + dphi(alpha) with log1p barrier increments),
   the same function as SPEC.md:310-327 evaluated without cancellation.
4. Predictor reuses the last Newton solve's factors with the
   right-hand side evaluated at the current point; it is skipped once
   E(.;0) <= tol (it could only change mu, not the iterate).
5. Relative KKT tolerance: eps_abs = tol_rel * max(1, E_primal(X0, Y0)).
6. E uses Diag(y) for "s^T Diag(Y)".
7. Nudge: an updated entry that is not strictly positive becomes
   (1 - tau) times its previous value.
8. Termination: run_ipm stops as soon as E(.;0) <= tol ("terminates when
   E(.;0) <= eps_TOL"), checked after every inner iteration; the inner loop's own
   test E(.;mu) <= mu can be unreachable once mu ~ 1e-15.
9. Barrier weights: default "balanced" (n w_x = m w_y, = the single mu when n = m);
   "paper" is the literal single-mu reading (see barrier_weights).
10. Hessian switch: default "inertia".  Algorithm 3 sets flag = (sigma <= sigma_c) after
   every outer iteration; with the flag set the direction uses the full coupling C
   (PAPER.md:564-590).  "paper": a full-C direction that is not positive definite or not
   a descent direction clears the flag and the iteration uses C-bar (Alg. 3 literally).
   "inertia": such a direction is recomputed with both diagonal blocks shifted,
   rho -> rho + delta, delta = 0, then delta_last / 3 (or rho when there is no previous
   shift), growing 4x until the Schur matrix factors and the direction is descent
   (INERTIA_MAX_TRIES attempts, then the C-bar fallback of "paper").  The literal rule
   stalls on the BASELINE peak instances: along the rotational ambiguity of the
   factorisation the residual coupling dominates the curvature, the Gauss-Newton
   direction overshoots (Armijo t = 6-7 for hundreds of iterations) and the full C is
   indefinite there ("Reaching the tolerance").
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import solve_triangular

from oracle import kernels as _KC
from oracle import kernels_np as _KN
from oracle import lowrank as _LR


class _Kernels:
    """Kernel table used by the driver: the bit-exact C port by default;
    ``set_schur_backend("numpy")`` swaps the Schur-side kernels for the
    vectorised NumPy-backend formulation (CPU-baseline speed path)."""

    def __init__(self):
        self.set("c")

    def set(self, which):
        self.block_cholesky = _KC.block_cholesky
        self.block_solve_lower = _KC.block_solve_lower
        self.block_solve_lower_t = _KC.block_solve_lower_t
        self.nnls_batch = _KC.nnls_batch
        src = _KN if which == "numpy" else _KC
        self.schur_reduce = src.schur_reduce
        self.rhs_reduce = src.rhs_reduce
        self.back_substitute = src.back_substitute
        self.which = which


K = _Kernels()


def set_schur_backend(which: str) -> None:
    """"c" (bit-exact port of _kernels_numba) or "numpy" (_kernels_numpy formulation)."""
    K.set(which)


# ----------------------------------------------------------------------------
# configuration
# ----------------------------------------------------------------------------
@dataclass
class Stage1Config:
    eps_stol: float = 1e-3
    max_sweeps: int = 200
    tol_kkt: float | None = None  # None -> 1e-12 * max(1, ||C^T d||_inf) per rhs
    fixed_sweeps: int = 0  # >0: exactly this many sweeps, no step test


@dataclass
class IpmParams:
    tau: float = 0.9
    eta: float = 0.5
    sigma_cap: float = 0.99
    sigma_c: float = 0.01
    eps_tol: float = 1e-6
    max_iter: int = 500
    max_backtracks: int = 60
    fixed_iters: int = 0  # >0: run exactly this many inner iterations
    barrier: str = "balanced"  # default; "paper": one mu (PAPER Eq. 4, literal); see barrier_weights
    hessian: str = "inertia"  # "inertia" (default) | "paper" (frozen semantics 10)
    schur_solver: str = "dense"  # "dense" mk x mk Cholesky | "lowrank" (oracle.lowrank, GN only)
    residual: str = "dense"  # "dense" (form F) | "free" (oracle.lowrank products; GN only)


@dataclass
class TransitionParams:
    rho0_scale: float = 1e-6


class OracleError(RuntimeError):
    def __init__(self, kind, index=-1):
        super().__init__(f"{kind} (index {index})")
        self.kind, self.index = kind, index


# ----------------------------------------------------------------------------
# row sharding (paper_2101_08431_b200.dist): rows of M / X / R are local, Y / S
# replicated; contractions over rows are summed across ranks (gloo on CPU).
# ----------------------------------------------------------------------------
def _red(comm, a, op="sum"):
    """All-reduce a numpy array / float across ranks (identity without comm)."""
    if comm is None or not comm.active:
        return a
    import torch

    scalar = np.isscalar(a) or np.ndim(a) == 0
    t = torch.as_tensor(np.array(a, dtype=np.float64, ndmin=1)).clone()
    {"sum": comm.sum_, "max": comm.max_, "min": comm.min_}[op](t)
    out = t.numpy()
    return float(out[0]) if scalar else out.reshape(np.shape(a))


# ----------------------------------------------------------------------------
# products (numpy/OpenBLAS, as in the reference's missing drivers)
# ----------------------------------------------------------------------------
def objective(X, Yt, M):
    """1/2 ||X Y - M||_F^2 (Yt = Y^T, (m,k))."""
    F = X @ Yt.T - M
    return 0.5 * float(np.vdot(F, F))


def gradients(X, Yt, M, comm=None):
    """graX = vec(Y F^T) -> (n,k) = F Y^T; graY = vec(X^T F) -> (m,k)."""
    F = X @ Yt.T - M
    return F, F @ Yt, _red(comm, F.T @ X)


_gradients = gradients


def kkt_error(X, Yt, R, S, graX, graY, mu, wx=1.0, wy=1.0, comm=None):
    """SPEC.md:274 / PAPER Eq. 9 (Diag(y) reading)."""
    xs = _red(comm, np.array([np.sum((graX - R) ** 2), np.sum((X * R - wx * mu) ** 2)]))
    st = math.sqrt(float(xs[0] + np.sum((graY - S) ** 2)))
    cp = math.sqrt(float(xs[1] + np.sum((Yt * S - wy * mu) ** 2)))
    return max(st, cp)


def kkt_error_primal_only(X, Yt, M, comm=None):
    """SPEC.md:420 / PAPER.md:633-639: E(x,y,max(graX,0),max(graY,0);0)."""
    _, gX, gY = gradients(X, Yt, M, comm)
    return kkt_error(X, Yt, np.maximum(gX, 0.0), np.maximum(gY, 0.0), gX, gY, 0.0, comm=comm)


def _nnls_tol(ctb, tol_kkt):
    if tol_kkt is not None:
        return np.full(ctb.shape[0], float(tol_kkt))
    if ctb.shape[0] == 0:
        return np.zeros(0)
    return 1e-12 * np.maximum(1.0, np.abs(ctb).max(axis=1))


def _raise_status(status, what, comm=None):
    bad = np.flatnonzero(status)
    if comm is not None and comm.active:  # every rank raises together
        anybad = _red(comm, float(bad.size > 0), "max")
        if anybad and not bad.size:
            raise OracleError(f"status failure on another rank in {what}")
    if bad.size:
        i = int(bad[0])
        kind = "MaxIterationsExceeded" if status[i] == 1 else "RankDeficientPassiveSet"
        raise OracleError(f"{kind} in {what}", i)


# ----------------------------------------------------------------------------
# stage 1: ANLS (Algorithm 1)
# ----------------------------------------------------------------------------
def update_X(X, Yt, M, pX, mode, cfg, row_norm2, comm=None):
    """rows of X <- NNLS(C = Y^T, d = M_i,:) (rows are rank-local)."""
    ctc = Yt.T @ Yt
    ctb = M @ Yt
    tol = _nnls_tol(ctb, cfg.tol_kkt)
    k = X.shape[1]
    x, p, ch, r2, st = K.nnls_batch(ctc, ctb, row_norm2, pX, mode, tol, 3 * k)
    _raise_status(st, "update_X", comm)
    return x, p, ch, r2


def update_Y(X, Yt, M, pY, mode, cfg, col_norm2, comm=None):
    """columns of Y <- NNLS(C = X, d = M_:,j) (Grams summed over ranks).

    With ``comm``: every rank solves its column range (dist.row_range over m) and the
    columns are all-gathered, as the device solver does (paper_2101_08431_b200/dist.py)."""
    ctc = _red(comm, X.T @ X)
    ctb = _red(comm, M.T @ X)
    tol = _nnls_tol(ctb, cfg.tol_kkt)
    k = X.shape[1]
    if comm is None or not comm.active:
        y, p, ch, r2, st = K.nnls_batch(ctc, ctb, col_norm2, pY, mode, tol, 3 * k)
        _raise_status(st, "update_Y")
        return y, p, ch, r2
    import torch

    from paper_2101_08431_b200.dist import row_range

    m = ctb.shape[0]
    a, b = row_range(m, comm.world, comm.rank)
    ys, ps, chs, r2s, sts = K.nnls_batch(ctc, ctb[a:b].copy(), col_norm2[a:b].copy(),
                                         pY[a:b].copy(), mode, tol[a:b].copy(), 3 * k)
    out = []
    for loc, shape, dt in ((ys, (m, k), torch.float64), (ps, (m, k), torch.uint8),
                           (chs, (m,), torch.int64), (r2s, (m,), torch.float64),
                           (sts, (m,), torch.int8)):
        t = torch.zeros(shape, dtype=dt)
        t[a:b] = torch.as_tensor(np.asarray(loc)).to(dt).reshape((b - a,) + shape[1:])
        out.append(comm.allgather_rows(t).numpy())
    y, p, ch, r2, st = out
    _raise_status(st, "update_Y")
    return y, p.astype(bool), ch, r2


@dataclass
class Stage1Result:
    X: np.ndarray
    Yt: np.ndarray
    pX: np.ndarray
    pY: np.ndarray
    sweeps: int
    converged: bool
    trace: list = field(default_factory=list)
    changes_X: list = field(default_factory=list)
    changes_Y: list = field(default_factory=list)
    seconds: float = 0.0


def run_stage1(M, X, Yt, cfg=None, pX=None, pY=None, comm=None):
    """SPEC.md:209 run_stage1.  X (n,k), Yt = Y^T (m,k).  Carries optional.

    With ``comm``: M, X, pX are this rank's row block; Yt, pY replicated."""
    cfg = cfg or Stage1Config()
    t0 = time.perf_counter()
    X = np.array(X, dtype=np.float64)
    Yt = np.array(Yt, dtype=np.float64)
    n, k = X.shape
    m = Yt.shape[0]
    have_carry = pX is not None
    pX = np.zeros((n, k), bool) if pX is None else pX.copy()
    pY = np.zeros((m, k), bool) if pY is None else pY.copy()
    row_n2 = np.einsum("ij,ij->i", M, M)
    col_n2 = _red(comm, np.einsum("ij,ij->j", M, M))
    res = Stage1Result(X, Yt, pX, pY, 0, False)
    nsweeps = cfg.fixed_sweeps if cfg.fixed_sweeps > 0 else cfg.max_sweeps
    for sweep in range(nsweeps):
        mode = 2 if (sweep > 0 or have_carry) else 0
        Xn, pX, chX, _ = update_X(X, Yt, M, pX, mode, cfg, row_n2, comm)
        Yn, pY, chY, r2Y = update_Y(Xn, Yt, M, pY, mode, cfg, col_n2, comm)
        xs = _red(comm, np.array([np.sum((Xn - X) ** 2), np.sum(X ** 2)]))
        step = math.sqrt(float(xs[0] + np.sum((Yn - Yt) ** 2)))
        nrm = math.sqrt(float(xs[1] + np.sum(Yt ** 2)))
        X, Yt = Xn, Yn
        res.sweeps = sweep + 1
        res.trace.append((time.perf_counter() - t0, 0.5 * float(np.sum(r2Y)), step))
        res.changes_X.append(int(chX.sum()))
        res.changes_Y.append(int(chY.sum()))
        if cfg.fixed_sweeps <= 0 and step <= cfg.eps_stol * (1.0 + nrm):
            res.converged = True
            break
    res.X, res.Yt, res.pX, res.pY = X, Yt, pX, pY
    res.seconds = time.perf_counter() - t0
    return res


# ----------------------------------------------------------------------------
# stage 2: interior point (Algorithm 2) with the Hessian switch (Algorithm 3)
# ----------------------------------------------------------------------------
@dataclass
class IpmState:
    X: np.ndarray
    Yt: np.ndarray
    R: np.ndarray
    S: np.ndarray
    mu: float
    rho: float
    flag: bool = False


def transition(X, Yt, M, eps_tol, tp=None, comm=None):
    """SPEC.md:393 / PAPER Eqs. 14-18."""
    tp = tp or TransitionParams()
    big = max(_red(comm, float(X.max(initial=0.0)), "max"), float(Yt.max(initial=0.0)))
    if big <= 0.0:
        raise OracleError("DegenerateFactor")
    rho0 = tp.rho0_scale * big
    X = np.maximum(X, rho0)
    Yt = np.maximum(Yt, rho0)
    _, gX, gY = gradients(X, Yt, M, comm)
    R = np.full_like(X, _red(comm, float(np.abs(gX).max(initial=0.0)), "max"))
    S = np.full_like(Yt, np.abs(gY).max())
    n, k = X.shape
    m = Yt.shape[0]
    n = int(_red(comm, float(n)))
    mu = (_red(comm, float(np.vdot(X, R))) + float(np.vdot(Yt, S))) / (n * k + m * k)
    return IpmState(X, Yt, R, S, mu, eps_tol, False)


def fraction_to_boundary(v, dv, tau):
    """SPEC.md:301 / PAPER Eq. 6 for one stacked vector: min(1, min -tau v/dv)."""
    neg = dv < 0.0
    if not np.any(neg):
        return 1.0
    return float(min(1.0, np.min(-tau * v[neg] / dv[neg])))


def _ftb2(a, da, b, db, tau, comm=None):
    return min(_red(comm, fraction_to_boundary(a.ravel(), da.ravel(), tau), "min"),
               fraction_to_boundary(b.ravel(), db.ravel(), tau))


@dataclass
class Factorization:
    X: np.ndarray
    Yt: np.ndarray
    F: np.ndarray
    L: np.ndarray
    Ls: np.ndarray  # lower Cholesky factor of the mk x mk Schur matrix
    full: bool


def schur_matrix(XtX, rho, S_over_Y, Sacc):
    """blockdiag(X^T X + rho I + Diag(s_j/y_j)) - S."""
    m, k = S_over_Y.shape
    A = -Sacc
    base = XtX + rho * np.eye(k)
    for j in range(m):
        sl = slice(j * k, (j + 1) * k)
        A[sl, sl] += base + np.diag(S_over_Y[j])
    return A


def spd_factor(A):
    """lower Cholesky; None when not positive definite."""
    try:
        return np.linalg.cholesky(A)
    except np.linalg.LinAlgError:
        return None


def spd_solve_factored(Ls, b):
    z = solve_triangular(Ls, b, lower=True, check_finite=False)
    return solve_triangular(Ls.T, z, lower=False, check_finite=False)


def barrier_weights(n, m, barrier):
    """Per-block barrier weights (wx, wy): mu_X = wx*mu, mu_Y = wy*mu.

    "paper": wx = wy = 1 (PAPER Eqs. 4, 9 and the merit function).
    "balanced": n*wx = m*wy, (n*wx + m*wy)/(n+m) = 1.  With one mu and n != m
    the perturbed KKT system has no solution: summing x_ip*graX_ip - y_pj*graY_pj
    over one component gives 0 for any (X, Y) (scale invariance of XY), which
    forces mu*(n - m) = 0 at a central point; the balanced weights restore it.
    """
    if barrier == "paper":
        return 1.0, 1.0
    if barrier == "balanced":
        return (n + m) / (2.0 * n), (n + m) / (2.0 * m)
    raise ValueError(barrier)


def newton_direction(M, st: IpmState, F, gX, gY, full, wx=1.0, wy=1.0, comm=None):
    """R1 blocks, Schur reduction, mk x mk solve, back-sub.

    Returns (dx, dy, dr, ds, gtp, fact) or None when the Schur matrix is not
    positive definite (SchurNotPositiveDefinite; only expected with full C).
    """
    X, Yt, R, S, mu, rho = st.X, st.Yt, st.R, st.S, st.mu, st.rho
    n, k = X.shape
    YYt = Yt.T @ Yt
    R1 = YYt[None] + rho * np.eye(k)[None] + np.einsum("ip,pq->ipq", R / X, np.eye(k))
    L, bad = K.block_cholesky(R1)
    if _red(comm, float(bad >= 0), "max"):
        raise OracleError("NotPositiveDefinite", bad)
    mux, muy = wx * mu, wy * mu
    b1 = mux / X - gX
    h = K.block_solve_lower(L, b1[:, :, None])[:, :, 0]
    Sacc, racc = K.schur_reduce(X, Yt, L, h, F, full)
    Sacc, racc = _red(comm, Sacc), _red(comm, racc)
    A = schur_matrix(_red(comm, X.T @ X), rho, S / Yt, Sacc)
    Ls = spd_factor(A)
    if Ls is None:
        if full:
            return None
        raise OracleError("NotPositiveDefinite (Schur, Gauss-Newton)")
    b2 = muy / Yt - gY
    dy = spd_solve_factored(Ls, (b2 - racc).ravel()).reshape(Yt.shape)
    dx = K.back_substitute(X, Yt, L, h, dy, F, full)
    dr = mux / X - R - (R / X) * dx
    ds = muy / Yt - S - (S / Yt) * dy
    gtp = _red(comm, float(np.vdot(dx, gX - mux / X))) + float(np.vdot(dy, gY - muy / Yt))
    return dx, dy, dr, ds, gtp, Factorization(X, Yt, F, L, Ls, full)


def quartic_coeffs(X, Yt, dX, dYt, M, comm=None):
    """Inner products of A = XY-M, B = dX Y + X dY, C = dX dY (one pass over M)."""
    A = X @ Yt.T - M
    B = dX @ Yt.T + X @ dYt.T
    C = dX @ dYt.T
    v = np.array([np.vdot(A, A), np.vdot(A, B), np.vdot(B, B), np.vdot(A, C), np.vdot(B, C),
                  np.vdot(C, C)])
    return tuple(float(x) for x in _red(comm, v))


def merit_delta(coef, alpha, X, dX, Yt, dYt, mu, wx=1.0, wy=1.0, comm=None):
    """phi(x + a dx, y + a dy) - phi(x, y), evaluated without cancellation."""
    _, ab, bb, ac, bc, cc = coef
    a2, a3 = alpha * alpha, alpha * alpha * alpha
    quad = alpha * ab + a2 * (0.5 * bb + ac) + a3 * bc + 0.5 * (a3 * alpha) * cc
    bx = _red(comm, float(np.sum(np.log1p(alpha * dX / X))))
    by = float(np.sum(np.log1p(alpha * dYt / Yt)))
    return quad - mu * (wx * bx + wy * by)  # same evaluation order as the device selector


def merit_phi(X, Yt, M, mu):
    """SPEC.md:310."""
    if np.any(X <= 0) or np.any(Yt <= 0):
        raise OracleError("NonPositiveInput")
    return objective(X, Yt, M) - mu * (float(np.sum(np.log(X))) + float(np.sum(np.log(Yt))))


def _nudge(new, old, tau):
    bad = ~(new > 0.0)
    if np.any(bad):
        new = np.where(bad, (1.0 - tau) * old, new)
    return new


INERTIA_GROW = 4.0
INERTIA_SHRINK = 3.0
INERTIA_MAX_TRIES = 40


def full_direction(M, st: IpmState, F, gX, gY, wx, wy, p: IpmParams, delta_last, comm=None):
    """Full-coupling direction under frozen semantics 10.

    Returns (out, delta): out is newton_direction's tuple, or None when the full
    coupling is rejected ("paper": first failure; "inertia": every shift failed)."""
    rho0 = st.rho
    delta = 0.0
    tries = 1 if p.hessian == "paper" else INERTIA_MAX_TRIES
    try:
        for _ in range(tries):
            st.rho = rho0 + delta
            out = newton_direction(M, st, F, gX, gY, True, wx, wy, comm)
            if out is not None and out[4] < 0.0:
                return out, delta
            if delta > 0.0:
                delta *= INERTIA_GROW
            else:
                delta = delta_last / INERTIA_SHRINK if delta_last > 0.0 else rho0
    finally:
        st.rho = rho0
    return None, delta_last


@dataclass
class IpmResult:
    state: IpmState
    iters: int
    outer: int
    converged: bool
    E0: float
    trace: list = field(default_factory=list)
    armijo_t: list = field(default_factory=list)
    flags: list = field(default_factory=list)
    deltas: list = field(default_factory=list)  # inertia shift of each full-coupling iteration
    seconds: float = 0.0


def predictor_sigma(st: IpmState, gX, gY, fact: Factorization, p: IpmParams, comm=None):
    """SPEC.md:328 / PAPER Eqs. 7-8, reusing the last Newton factorization."""
    X, Yt, R, S = st.X, st.Yt, st.R, st.S
    n, k = X.shape
    m = Yt.shape[0]
    b1 = -gX
    h = K.block_solve_lower(fact.L, b1[:, :, None])[:, :, 0]
    racc = _red(comm, K.rhs_reduce(fact.X, fact.Yt, fact.L, h, fact.F, fact.full))
    dy = spd_solve_factored(fact.Ls, (-gY - racc).ravel()).reshape(Yt.shape)
    dx = K.back_substitute(fact.X, fact.Yt, fact.L, h, dy, fact.F, fact.full)
    dr = -R - (R / X) * dx
    ds = -S - (S / Yt) * dy
    a1 = _ftb2(X, dx, Yt, dy, 1.0, comm)
    a2 = _ftb2(R, dr, S, ds, 1.0, comm)
    nk = int(_red(comm, float(n))) * k + m * k
    xs = _red(comm, np.array([np.vdot(X + a1 * dx, R + a2 * dr), np.vdot(X, R)]))
    mu_aff = (float(xs[0]) + float(np.vdot(Yt + a1 * dy, S + a2 * ds))) / nk
    mu_bar = (float(xs[1]) + float(np.vdot(Yt, S))) / nk
    return min((mu_aff / mu_bar) ** 3, p.sigma_cap)


def predictor_sigma_lowrank(st: IpmState, gX, gY, fac, p: IpmParams, comm=None):
    """predictor_sigma with the rank-k^2 factorization (same Eqs. 7-8)."""
    X, Yt, R, S = st.X, st.Yt, st.R, st.S
    n, k = X.shape
    m = Yt.shape[0]
    dx, dy, dr, ds, _ = _LR.solve(fac, X, Yt, R, S, gX, gY, 0.0, 0.0, lambda a: _red(comm, a))
    a1 = _ftb2(X, dx, Yt, dy, 1.0, comm)
    a2 = _ftb2(R, dr, S, ds, 1.0, comm)
    nk = int(_red(comm, float(n))) * k + m * k
    xs = _red(comm, np.array([np.vdot(X + a1 * dx, R + a2 * dr), np.vdot(X, R)]))
    mu_aff = (float(xs[0]) + float(np.vdot(Yt + a1 * dy, S + a2 * ds))) / nk
    mu_bar = (float(xs[1]) + float(np.vdot(Yt, S))) / nk
    return min((mu_aff / mu_bar) ** 3, p.sigma_cap)


def _gn_direction(M, st, F, gX, gY, wx, wy, p, comm):
    """Gauss-Newton direction: dense Schur system, or the rank-k^2 identity."""
    if p.schur_solver != "lowrank":
        return newton_direction(M, st, F, gX, gY, False, wx, wy, comm)
    red = lambda a: _red(comm, a)  # noqa: E731
    try:
        fac = _LR.factor(st.X, st.Yt, st.R, st.S, st.rho, red)
    except _LR.NotPD as e:
        raise OracleError(f"NotPositiveDefinite (low-rank Gauss-Newton system: {e})") from None
    dx, dy, dr, ds, gtp = _LR.solve(fac, st.X, st.Yt, st.R, st.S, gX, gY, wx * st.mu,
                                    wy * st.mu, red)
    return dx, dy, dr, ds, gtp, fac


def run_ipm(M, st: IpmState, p: IpmParams = None, comm=None):
    """SPEC.md:337 run_ipm: Algorithm 2 nested loops + Algorithm 3 switch.

    ``p.residual == "free"`` / ``p.schur_solver == "lowrank"``: the same iteration with
    the residual-free products and the rank-k^2 Schur identity of ``oracle.lowrank``
    (instances whose F or dense Schur matrix does not fit; Gauss-Newton coupling only,
    as on the device)."""
    p = p or IpmParams()
    t0 = time.perf_counter()
    free = p.residual == "free"
    red = lambda a: _red(comm, a)  # noqa: E731
    Mn2 = red(float(np.vdot(M, M))) if free else 0.0

    def gradients(X, Yt, M, comm):  # noqa: F811  (residual-free or dense)
        if free:
            fsq, gX_, gY_ = _LR.gradients_free(X, Yt, M, Mn2, red)
            return fsq, gX_, gY_
        return _gradients(X, Yt, M, comm)

    def fnorm2(F):
        return F if free else red(float(np.vdot(F, F)))

    def quartic(X, Yt, dX, dYt, gX, gY):
        if free:
            return _LR.quartic_free(X, Yt, dX, dYt, gX, gY, M, red)
        return quartic_coeffs(X, Yt, dX, dYt, M, comm)

    F, gX, gY = gradients(st.X, st.Yt, M, comm)
    E0 = kkt_error(st.X, st.Yt, st.R, st.S, gX, gY, 0.0, comm=comm)
    res = IpmResult(st, 0, 0, False, E0)
    cap = p.fixed_iters if p.fixed_iters > 0 else p.max_iter
    tol = 0.0 if p.fixed_iters > 0 else p.eps_tol
    fact = None
    e_zero = E0
    delta_last = 0.0
    wx, wy = barrier_weights(int(_red(comm, float(st.X.shape[0]))), st.Yt.shape[0], p.barrier)
    while e_zero > tol and res.iters < cap:
        eps_mu = st.mu
        # frozen semantics 8: run_ipm terminates as soon as E(.;0) <= tol (checked after
        # every inner iteration, not only when the inner loop reaches eps_mu)
        while (kkt_error(st.X, st.Yt, st.R, st.S, gX, gY, st.mu, wx, wy, comm) > eps_mu
               and e_zero > tol and res.iters < cap):
            out = None
            used_full = False
            if st.flag and not free:
                out, delta = full_direction(M, st, F, gX, gY, wx, wy, p, delta_last, comm)
                if out is None:
                    st.flag = False
                else:
                    used_full = True
                    delta_last = delta
                    res.deltas.append(delta)
            if out is None:
                out = _gn_direction(M, st, F, gX, gY, wx, wy, p, comm)
            dx, dy, dr, ds, gtp, fact = out
            a1max = _ftb2(st.X, dx, st.Yt, dy, p.tau, comm)
            a2max = _ftb2(st.R, dr, st.S, ds, p.tau, comm)
            coef = quartic(st.X, st.Yt, dx, dy, gX, gY)
            t = 0
            while True:
                a1 = a1max / (2.0 ** t)
                if merit_delta(coef, a1, st.X, dx, st.Yt, dy, st.mu, wx, wy, comm) <= p.eta * a1 * gtp:
                    break
                t += 1
                if t > p.max_backtracks:
                    raise OracleError("LineSearchStall", res.iters)
            st.X = _nudge(st.X + a1 * dx, st.X, p.tau)
            st.Yt = _nudge(st.Yt + a1 * dy, st.Yt, p.tau)
            st.R = _nudge(st.R + a2max * dr, st.R, p.tau)
            st.S = _nudge(st.S + a2max * ds, st.S, p.tau)
            res.iters += 1
            res.armijo_t.append(t)
            res.flags.append(used_full)
            F, gX, gY = gradients(st.X, st.Yt, M, comm)
            e_zero = kkt_error(st.X, st.Yt, st.R, st.S, gX, gY, 0.0, comm=comm)
            res.trace.append((time.perf_counter() - t0, 0.5 * fnorm2(F), e_zero, st.mu, a1,
                              a2max, t))
        res.outer += 1
        e_zero = kkt_error(st.X, st.Yt, st.R, st.S, gX, gY, 0.0, comm=comm)
        if e_zero <= tol or res.iters >= cap:
            break
        if fact is None:  # no Newton solve yet: factor at the current point
            fact = _gn_direction(M, st, F, gX, gY, wx, wy, p, comm)[5]
        if isinstance(fact, _LR.LowrankFactor):
            sigma = predictor_sigma_lowrank(st, gX, gY, fact, p, comm)
        else:
            sigma = predictor_sigma(st, gX, gY, fact, p, comm)
        st.mu = sigma * st.mu
        st.flag = sigma <= p.sigma_c and not free
    res.converged = e_zero <= tol
    res.state = st
    res.seconds = time.perf_counter() - t0
    return res


# ----------------------------------------------------------------------------
# two-stage orchestrator (Algorithm 3)
# ----------------------------------------------------------------------------
@dataclass
class SolveReport:
    X: np.ndarray
    Yt: np.ndarray
    objective: float
    kkt: float
    eps_abs: float
    stage1: Stage1Result
    ipm: IpmResult | None
    converged: bool
    stage1_time: float
    stage2_time: float


def run_two_stage(M, X0, Y0, tol_rel=1e-10, s1=None, ipm=None, tp=None, stage="two_stage",
                  pX=None, pY=None, e_scale=None, comm=None):
    """SPEC.md:411 run_two_stage.  X0 (n,k), Y0 (k,m).  With ``comm`` M / X0 / pX
    are this rank's row block (paper_2101_08431_b200.dist)."""
    M = np.asarray(M, dtype=np.float64)
    X0 = np.asarray(X0, dtype=np.float64)
    Yt0 = np.ascontiguousarray(np.asarray(Y0, dtype=np.float64).T)
    if e_scale is None:
        e_scale = max(1.0, kkt_error_primal_only(X0, Yt0, M, comm))
    eps_abs = tol_rel * e_scale
    p = ipm or IpmParams()
    p.eps_tol = eps_abs
    s1 = s1 or Stage1Config()
    if stage == "ipm_only":
        r1 = Stage1Result(X0.copy(), Yt0.copy(), np.zeros(X0.shape, bool),
                          np.zeros(Yt0.shape, bool), 0, False)
    else:
        r1 = run_stage1(M, X0, Yt0, s1, pX, pY, comm)
    if stage == "anls_only":
        X, Yt = r1.X, r1.Yt
        e = kkt_error_primal_only(X, Yt, M, comm)
        return SolveReport(X, Yt, _red(comm, objective(X, Yt, M)), e, eps_abs,
                           r1, None, e <= eps_abs, r1.seconds, 0.0)
    st = transition(r1.X, r1.Yt, M, eps_abs, tp, comm)
    r2 = run_ipm(M, st, p, comm)
    X, Yt = r2.state.X, r2.state.Yt
    F, gX, gY = gradients(X, Yt, M, comm)
    kkt = kkt_error(X, Yt, r2.state.R, r2.state.S, gX, gY, 0.0, comm=comm)
    return SolveReport(X, Yt, _red(comm, objective(X, Yt, M)), kkt, eps_abs, r1, r2, r2.converged,
                       r1.seconds, r2.seconds)
