"""oracle/lowrank.py (residual-free products + rank-k^2 Schur identity: the CPU baseline's
and the c4 parity tests' stage 2) against the dense oracle over the reference-pinned kernels."""
import numpy as np

from oracle import driver as D
from oracle import lowrank as LR


def test_direction_and_quartic_match_dense():
    rng = np.random.default_rng(7)
    for n, m, k in [(40, 12, 3), (60, 9, 4), (30, 20, 10)]:
        M = rng.uniform(0, 1, (n, m))
        X, Yt = rng.uniform(0.1, 1, (n, k)), rng.uniform(0.1, 1, (m, k))
        R, S = rng.uniform(0.01, 0.1, (n, k)), rng.uniform(0.01, 0.1, (m, k))
        st = D.IpmState(X, Yt, R, S, 1e-3, 1e-6)
        F, gX, gY = D.gradients(X, Yt, M)
        fsq, gX2, gY2 = LR.gradients_free(X, Yt, M, float(np.vdot(M, M)))
        assert np.allclose(gX, gX2, rtol=0, atol=1e-12) and np.allclose(gY, gY2, rtol=0, atol=1e-12)
        assert abs(fsq - np.vdot(F, F)) <= 1e-12 * max(1.0, fsq)
        dx, dy, dr, ds, gtp, _ = D.newton_direction(M, st, F, gX, gY, False, 1.0, 1.0)
        fac = LR.factor(X, Yt, R, S, st.rho)
        got = LR.solve(fac, X, Yt, R, S, gX, gY, 1e-3, 1e-3)
        for a, b in zip(got[:4], (dx, dy, dr, ds)):
            assert np.abs(a - b).max() <= 1e-9 * max(1.0, np.abs(b).max())
        assert abs(got[4] - gtp) <= 1e-9 * abs(gtp)
        c1 = D.quartic_coeffs(X, Yt, dx, dy, M)
        c2 = LR.quartic_free(X, Yt, dx, dy, gX, gY, M)
        for a, b in zip(c1[1:], c2[1:]):
            assert abs(a - b) <= 1e-9 * max(1.0, abs(a))


def test_lowrank_ipm_follows_dense_oracle():
    """The same IPM iterations (identical Armijo decisions) through the rank-k^2 solve."""
    from paper_2101_08431_b200 import data

    M, X0, Y0 = data.dense(300, 30, 6, 104)[:3]
    s1 = D.run_stage1(M, X0, Y0.T.copy(), D.Stage1Config(fixed_sweeps=5))
    runs = []
    for solver, resid in (("dense", "dense"), ("lowrank", "free")):
        st = D.transition(s1.X, s1.Yt, M, 1e-7)
        runs.append(D.run_ipm(M, st, D.IpmParams(fixed_iters=12, schur_solver=solver,
                                                 residual=resid, hessian="paper")))
    a, b = runs
    n = min(len(a.flags), a.flags.index(True) if True in a.flags else len(a.flags))
    assert n >= 8
    assert a.armijo_t[:n] == b.armijo_t[:n]
    for i in range(n):
        assert abs(a.trace[i][1] - b.trace[i][1]) <= 1e-9 * a.trace[i][1]
