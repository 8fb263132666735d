"""Device-vs-oracle deviation of the fixed-iteration IPM parity cases next to the spread
between the oracle's own two Schur backends (C loops vs NumPy): the measured conditioning
bound behind tests/test_gpu_solver.py::test_ipm_parity."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from oracle import driver as D  # noqa: E402
from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams  # noqa: E402

CASES = [("c1", "paper", 40, 1e-7, "lowrank", "auto"), ("c1", "balanced", 60, 1e-7, "lowrank", "auto"),
         ("c1", "balanced", 50, 1e-5, "lowrank", "auto"), ("c1", "balanced", 50, 1e-5, "dense", "auto"),
         ("c1", "paper", 40, 1e-7, "lowrank", "free"), ("c2", "balanced", 35, 1e-6, "lowrank", "auto"),
         ("c2", "paper", 30, 1e-6, "lowrank", "free")]


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


for name, barrier, iters, eps, solve, resid in CASES:
    M, X0, Y0, _, _ = data.make(data.CONFIGS[name])
    ro = D.run_stage1(M, X0, Y0.T.copy())
    P = solver.Problem(M, X0.shape[1])
    X, Yt, R, S, mu, rho = solver.transition(P, P.to_dev(ro.X), P.to_dev(ro.Yt), eps)
    eng, r = solver.run_ipm(P, X, Yt, R, S, mu, rho,
                            IpmParams(fixed_iters=iters, barrier=barrier, schur_solver=solve,
                                      residual=resid, hessian="paper"))
    outs, secs = {}, {}
    for be in ("numpy", "c"):
        D.set_schur_backend(be)
        st = D.transition(ro.X, ro.Yt, M, eps)
        t = time.perf_counter()
        outs[be] = D.run_ipm(M, st, D.IpmParams(fixed_iters=iters, barrier=barrier, hessian="paper"))
        secs[be] = time.perf_counter() - t
    D.set_schur_backend("c")
    a, b = outs["numpy"], outs["c"]
    dev = max(rel(eng.X.cpu().numpy(), a.state.X), rel(eng.Yt.cpu().numpy(), a.state.Yt))
    spr = max(rel(b.state.X, a.state.X), rel(b.state.Yt, a.state.Yt))
    print(f"{name} {barrier} {iters} {eps:g} {solve} {resid}: device-oracle {dev:.2e}  oracle[c]-oracle[numpy] "
          f"{spr:.2e}  decisions {r.armijo_t == a.armijo_t == b.armijo_t}  oracle s: numpy {secs['numpy']:.1f} c {secs['c']:.1f}",
          flush=True)
