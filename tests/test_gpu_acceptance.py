"""SPEC.md acceptance criteria 5-7 (PRIMARY) run through the device solver.

5: interior-point invariants on a full run at (500, 30, 3): strict positivity, Armijo
   at every accepted step, mu strictly decreasing across outer iterations, E(.;0) <= 1e-6.
6: two_stage reaches E <= 1e-6 on >= 8 of 10 seeds at (2000, 50, 3) while anls_only does
   not, and two_stage f <= anls_only f on every seed.
7: spread of the two_stage objective across the 10 seeds <= 1e-4 relative.
The synthetic family is the paper's section 5.4 one (io.generate_synthetic, noise 0.1).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_acceptance5_full_run_invariants():
    import torch

    from paper_2101_08431_b200 import data, io, solver
    from paper_2101_08431_b200.config import IpmParams, Stage1Config

    M, _, _ = io.generate_synthetic(500, 30, 3, 0.1, seed=5)
    X0, Y0 = data.init_factors(500, 30, 3, 5)
    P = solver.Problem(M, 3)
    X, Yt, _, _, _ = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T), Stage1Config())
    X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, 1e-6)
    eng, r = solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(eps_tol=1e-6))
    assert r.converged and r.trace[-1][2] <= 1e-6
    for t in (eng.X, eng.Yt, eng.R, eng.S):
        assert bool((t > 0).all())
    mus = [rec[3] for rec in r.trace]
    outer_mus = [mus[0]] + [b for a, b in zip(mus, mus[1:]) if b != a]
    assert all(b < a for a, b in zip(outer_mus, outer_mus[1:]))
    assert max(r.armijo_t) <= IpmParams().max_backtracks
    torch.cuda.synchronize()


def test_acceptance6_7_two_stage_vs_anls_only():
    import torch

    from paper_2101_08431_b200 import data, io, run_two_stage

    n, m, k = 2000, 50, 3
    M, _, _ = io.generate_synthetic(n, m, k, 0.1, seed=2021)
    Md = torch.as_tensor(M).cuda()
    two_E, two_f, anls_E, anls_f = [], [], [], []
    for seed in range(10):
        X0, Y0 = data.init_factors(n, m, k, seed)
        a = run_two_stage(Md, X0, Y0, tol_rel=1e-6, stage="two_stage", e_scale=1.0)
        b = run_two_stage(Md, X0, Y0, tol_rel=1e-6, stage="anls_only", e_scale=1.0)
        two_E.append(a.final_kkt_error)
        two_f.append(a.final_objective)
        anls_E.append(b.final_kkt_error)
        anls_f.append(b.final_objective)
    assert sum(e <= 1e-6 for e in two_E) >= 8
    assert sum(e > 1e-6 for e in anls_E) >= 8
    assert all(tf <= af for tf, af in zip(two_f, anls_f))
    f = np.asarray(two_f)
    assert (f.max() - f.min()) / f.mean() <= 1e-4
