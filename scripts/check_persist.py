"""Persistent inner loop vs the graph-replayed six-kernel iteration on c1/c2/c3 slices."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402


def run(name, persistent, iters, barrier="paper", m=None):
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
                             IpmParams(fixed_iters=iters, persistent=persistent, barrier=barrier))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    return r2, X.cpu().numpy(), Yt.cpu().numpy(), dt


for name, m, barrier in [("c1", None, "paper"), ("c2", None, "paper"), ("c2", None, "balanced"),
                         ("c3", 200, "balanced"), ("c3", 500, "balanced")]:
    for rep in range(2):
        ra, Xa, Ya, ta = run(name, False, 300, barrier, m)
        rb, Xb, Yb, tb = run(name, True, 300, barrier, m)
    same_t = ra.armijo_t == rb.armijo_t
    rel = max(np.abs(Xa - Xb).max() / np.abs(Xa).max(), np.abs(Ya - Yb).max() / np.abs(Ya).max())
    print(f"{name} m={m} {barrier}: iters {ra.iters}/{rb.iters} outer {ra.outer}/{rb.outer} "
          f"same_t {same_t} rel {rel:.2e} graph {1e3 * ta / ra.iters:.4f} ms/it "
          f"persist {1e3 * tb / rb.iters:.4f} ms/it", flush=True)
