"""SPEC.md known-answer examples and acceptance criteria on the CPU oracle.

These pin the oracle driver (the reference ships no driver, so its behaviour is
anchored on SPEC's examples and properties).
"""
import itertools
import math

import numpy as np
import pytest

from oracle import driver as D
from oracle import kernels as K


def test_objective_kat():
    assert D.objective(np.array([[2.0]]), np.array([[3.0]]), np.array([[5.0]])) == 0.5


def test_kkt_error_kat():  # max{0, ||(2,1)||} = sqrt(5)
    e = D.kkt_error(np.array([[2.0]]), np.array([[1.0]]), np.array([[1.0]]), np.array([[1.0]]),
                    np.array([[1.0]]), np.array([[1.0]]), 0.0)
    assert e == pytest.approx(math.sqrt(5.0), abs=1e-15)


def test_fraction_to_boundary_kats():
    assert D.fraction_to_boundary(np.array([1.0]), np.array([-1.0]), 0.9) == pytest.approx(0.9)
    assert D.fraction_to_boundary(np.array([1.0, 2.0]), np.array([-2.0, -1.0]), 0.9) == pytest.approx(0.45)
    assert D.fraction_to_boundary(np.array([1.0]), np.array([3.0]), 0.9) == 1.0


def test_merit_kat():
    one = np.array([[1.0]])
    assert D.merit_phi(one, one, one, 1.0) == 0.0


def test_transition_kats():
    X = np.array([[2.0, 0.0]])
    Yt = np.array([[1.0, 0.5]])
    st = D.transition(X, Yt, np.array([[1.0]]), 1e-6)
    assert st.X[0, 1] == pytest.approx(2e-6)
    _, gX, gY = D.gradients(st.X, st.Yt, np.array([[1.0]]))
    assert np.all(st.R == np.abs(gX).max()) and np.all(st.S == np.abs(gY).max())
    nk = 2 * 1 + 2 * 1
    assert st.mu == pytest.approx((np.vdot(st.X, st.R) + np.vdot(st.Yt, st.S)) / nk)
    assert st.rho == 1e-6


def _brute_nnls(C, d):
    k = C.shape[1]
    best, bx = np.inf, None
    for r in range(k + 1):
        for S in itertools.combinations(range(k), r):
            x = np.zeros(k)
            if S:
                sol, *_ = np.linalg.lstsq(C[:, S], d, rcond=None)
                if np.any(sol < -1e-12):
                    continue
                x[list(S)] = np.maximum(sol, 0)
            f = 0.5 * np.sum((C @ x - d) ** 2)
            if f < best:
                best, bx = f, x
    return best, bx


def test_acceptance1_nnls_vs_bruteforce():
    rng = np.random.default_rng(1)
    for _ in range(200):
        rows, k = rng.integers(3, 11), rng.integers(1, 9)
        rows = max(rows, k)
        C = rng.standard_normal((rows, k))
        d = rng.standard_normal(rows)
        ctb = (C.T @ d)[None]
        tol = 1e-12 * max(1.0, np.abs(ctb).max())
        x, p, ch, r2, st = K.nnls_batch(C.T @ C, ctb, np.array([d @ d]), np.zeros((1, k), bool), 0,
                                        np.array([tol]), 3 * k)
        assert st[0] == 0
        f = 0.5 * np.sum((C @ x[0] - d) ** 2)
        fb, _ = _brute_nnls(C, d)
        assert abs(f - fb) <= 1e-10
        w = C.T @ (d - C @ x[0])
        assert np.all(np.abs(x[0] * w) <= 1e-8)


def _dense_kkt(st, M, full):
    X, Yt, R, S, mu, rho = st.X, st.Yt, st.R, st.S, st.mu, st.rho
    n, k = X.shape
    m = Yt.shape[0]
    F = X @ Yt.T - M
    gX, gY = F @ Yt, F.T @ X
    nk, mk = n * k, m * k
    C = np.zeros((mk, nk))
    for j in range(m):
        for i in range(n):
            blk = np.outer(X[i], Yt[j])
            if full:
                blk = blk + F[i, j] * np.eye(k)
            C[j * k:(j + 1) * k, i * k:(i + 1) * k] = blk
    x, y, r, s = X.ravel(), Yt.ravel(), R.ravel(), S.ravel()
    N = 2 * (nk + mk)
    A = np.zeros((N, N))
    A[:nk, :nk] = np.kron(np.eye(n), Yt.T @ Yt) + rho * np.eye(nk)
    A[:nk, nk:nk + mk] = C.T
    A[:nk, nk + mk:2 * nk + mk] = -np.eye(nk)
    A[nk:nk + mk, :nk] = C
    A[nk:nk + mk, nk:nk + mk] = np.kron(np.eye(m), X.T @ X) + rho * np.eye(mk)
    A[nk:nk + mk, 2 * nk + mk:] = -np.eye(mk)
    A[nk + mk:2 * nk + mk, :nk] = np.diag(r)
    A[nk + mk:2 * nk + mk, nk + mk:2 * nk + mk] = np.diag(x)
    A[2 * nk + mk:, nk:nk + mk] = np.diag(s)
    A[2 * nk + mk:, 2 * nk + mk:] = np.diag(y)
    b = np.concatenate([r - gX.ravel(), s - gY.ravel(), mu - r * x, mu - s * y])
    sol = np.linalg.solve(A, b)
    return (sol[:nk].reshape(n, k), sol[nk:nk + mk].reshape(m, k),
            sol[nk + mk:2 * nk + mk].reshape(n, k), sol[2 * nk + mk:].reshape(m, k))


@pytest.mark.parametrize("backend", ["c", "numpy"])
def test_acceptance2_newton_vs_dense_kkt(backend):
    rng = np.random.default_rng(2)
    D.set_schur_backend(backend)
    try:
        done = 0
        for trial in range(50):
            n, m, k = [(8, 4, 2), (12, 5, 2), (10, 6, 3)][trial % 3]
            X = rng.uniform(0.1, 1, (n, k))
            Yt = rng.uniform(0.1, 1, (m, k))
            M = rng.uniform(0, 1, (n, m))
            st = D.IpmState(X, Yt, rng.uniform(0.1, 1, (n, k)), rng.uniform(0.1, 1, (m, k)),
                            float(rng.uniform(0.01, 0.5)), 1e-3)
            F, gX, gY = D.gradients(X, Yt, M)
            for full in (False, True):
                out = D.newton_direction(M, st, F, gX, gY, full)
                if out is None:
                    assert full
                    continue
                ref = _dense_kkt(st, M, full)
                for a, b in zip(out[:4], ref):
                    assert np.abs(a - b).max() <= 1e-8 * max(1.0, np.abs(b).max())
                done += 1
        assert done >= 50
    finally:
        D.set_schur_backend("c")


def test_acceptance3_gradients_fd():
    rng = np.random.default_rng(3)
    for _ in range(20):
        n, m, k = 6, 5, 2
        X, Yt, M = rng.uniform(0, 1, (n, k)), rng.uniform(0, 1, (m, k)), rng.uniform(0, 1, (n, m))
        _, gX, gY = D.gradients(X, Yt, M)
        h = 1e-6
        for (A, G) in ((X, gX), (Yt, gY)):
            for idx in np.ndindex(A.shape):
                A[idx] += h
                fp = D.objective(X, Yt, M)
                A[idx] -= 2 * h
                fm = D.objective(X, Yt, M)
                A[idx] += h
                fd = (fp - fm) / (2 * h)
                assert abs(fd - G[idx]) <= 1e-5 * max(1.0, abs(G[idx]))


def test_acceptance4_anls_monotone():
    rng = np.random.default_rng(4)
    n, m, k = 200, 20, 3
    M = np.maximum(rng.uniform(0, 1, (n, k)) @ rng.uniform(0, 1, (k, m)) + rng.normal(0, 0.1, (n, m)), 0)
    X, Yt = rng.uniform(0, 1, (n, k)), rng.uniform(0, 1, (m, k))
    pX, pY = np.zeros((n, k), bool), np.zeros((m, k), bool)
    rn, cn = np.einsum("ij,ij->i", M, M), np.einsum("ij,ij->j", M, M)
    f = D.objective(X, Yt, M)
    cfg = D.Stage1Config()
    for sweep in range(50):
        mode = 0 if sweep == 0 else 2
        X, pX, _, _ = D.update_X(X, Yt, M, pX, mode, cfg, rn)
        f1 = D.objective(X, Yt, M)
        assert f1 <= f * (1 + 1e-12)
        Yt, pY, _, _ = D.update_Y(X, Yt, M, pY, mode, cfg, cn)
        f2 = D.objective(X, Yt, M)
        assert f2 <= f1 * (1 + 1e-12)
        f = f2
        assert np.all(X >= 0) and np.all(Yt >= 0)


def test_acceptance5_ipm_invariants_balanced():  # SPEC.md:596 (invariants on a run)
    rng = np.random.default_rng(5)
    n, m, k = 120, 15, 3
    M = np.maximum(rng.uniform(0, 1, (n, k)) @ rng.uniform(0, 1, (k, m)) + rng.normal(0, 0.1, (n, m)), 0)
    X0, Y0 = rng.uniform(0, 1, (n, k)), rng.uniform(0, 1, (k, m))
    rep = D.run_two_stage(M, X0, Y0, tol_rel=1e-6, e_scale=1.0,
                          ipm=D.IpmParams(barrier="balanced", max_iter=200))
    st = rep.ipm.state
    assert np.all(st.X > 0) and np.all(st.Yt > 0) and np.all(st.R > 0) and np.all(st.S > 0)
    assert rep.converged and rep.kkt <= 1e-6
    assert rep.objective <= D.objective(rep.stage1.X, rep.stage1.Yt, M) * (1 + 1e-6)


def test_hessian_switch_kat():
    assert 0.005 <= D.IpmParams().sigma_c and not (0.5 <= D.IpmParams().sigma_c)


def test_predictor_sigma_arith():
    cap = D.IpmParams().sigma_cap
    assert min(0.5 ** 3, cap) == 0.125 and min(1.0 ** 3, cap) == 0.99 and min(0.0, cap) == 0.0
