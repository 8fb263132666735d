"""Median per-iteration time of the persistent inner loop (c2 paper / c2 balanced / c3)."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402


def one(name, barrier, iters, m=None, persistent=True):
    cfg = data.CONFIGS[name]
    M, X0, Y0, _, _ = data.make(cfg)
    if m:
        M, Y0 = M[:, :m], Y0[:, :m]
    P = solver.Problem(M, cfg.k)
    X, Yt, pX, pY, r1 = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T), Stage1Config())
    X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, 1e-7)
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng, r2 = solver.run_ipm(P, X, Yt, R, S, mu, rho,
                             IpmParams(fixed_iters=iters, barrier=barrier, persistent=persistent))
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t) / r2.iters


for name, barrier, m in [("c2", "paper", None), ("c2", "balanced", None), ("c3", "balanced", 500)]:
    ts = [one(name, barrier, 300, m) for _ in range(7)]
    print(f"{name} {barrier} m={m}: median {statistics.median(ts[2:]):.4f} ms/it  "
          f"min {min(ts[2:]):.4f}", flush=True)
