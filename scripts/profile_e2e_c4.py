"""Host-side breakdown of the bench's e2e leg on c4 (public run_two_stage on pinned host M,
fixed 50 sweeps + 20 IPM iterations): where the time beyond the device step goes."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import data, run_two_stage, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

cfg = data.CONFIGS["c4"]
M, X0, Y0, _, _ = data.make(cfg)
Mh = torch.from_numpy(M).pin_memory()
T = {}


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + time.perf_counter() - t
        return r
    setattr(mod, name, g)


if len(sys.argv) > 1 and sys.argv[1] == "keep":  # as bench.py: a live device-resident problem
    P0 = solver.Problem(M, cfg.k)
    X, Yt, *_ = solver.run_stage1(P0, P0.to_dev(X0), P0.to_dev(Y0.T),
                                  Stage1Config(fixed_sweeps=cfg.fixed_sweeps))
    X, Yt, R, S, mu, rho = solver.transition(P0, X, Yt, 1e-7)
    solver.run_ipm(P0, X, Yt, R, S, mu, rho, IpmParams(fixed_iters=cfg.fixed_ipm))
    torch.cuda.synchronize()
for nm in ("Problem", "run_stage1", "transition", "run_ipm", "kkt_error_primal_only_dev"):
    wrap(solver, nm)
for rep in range(3):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = run_two_stage(Mh, X0, Y0, tol_rel=cfg.tol, s1=Stage1Config(fixed_sweeps=cfg.fixed_sweeps),
                      ipm=IpmParams(fixed_iters=cfg.fixed_ipm), e_scale=1.0)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print("total %.2f ms" % (1e3 * tot), {k: round(1e3 * v, 2) for k, v in T.items()},
          "other %.2f ms" % (1e3 * (tot - sum(T.values()))), flush=True)
