"""Time-to-tolerance of the c1/c2 two-stage solves on the device (frozen semantics 10).

python scripts/converge.py c1 c2 [--hessian inertia|paper] [--cap 1000] [--oracle]
--oracle also runs oracle.driver on the same instance (CPU; minutes at c2) and prints
both trajectories' iteration counts, Armijo histograms and final objective / E.
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--hessian", default="inertia")
    ap.add_argument("--cap", type=int, default=1000)
    ap.add_argument("--oracle", action="store_true")
    a = ap.parse_args()
    for name in a.configs:
        cfg = data.CONFIGS[name]
        M, X0, Y0, _, _ = data.make(cfg)
        Md = torch.as_tensor(M).cuda()
        solver.run_two_stage(Md, X0, Y0, ipm=IpmParams(max_iter=5, hessian=a.hessian))  # warm-up
        torch.cuda.synchronize()
        t = time.perf_counter()
        rep = solver.run_two_stage(Md, X0, Y0, tol_rel=cfg.tol,
                                   ipm=IpmParams(max_iter=a.cap, hessian=a.hessian))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        r = rep.ipm
        out = {"config": name, "hessian": a.hessian, "seconds": dt, "status": rep.status,
               "sweeps": rep.stage1.sweeps, "ipm_iters": r.iters, "outer": r.outer,
               "full_iters": int(sum(r.flags)), "shifted": int(sum(d > 0 for d in r.deltas)),
               "E0": rep.final_kkt_error, "eps_abs": rep.eps_abs, "f": rep.final_objective,
               "armijo_hist": np.bincount(r.armijo_t).tolist() if r.armijo_t else []}
        if a.oracle:
            from oracle import driver as D

            D.set_schur_backend("numpy")
            t = time.perf_counter()
            o = D.run_two_stage(M, X0, Y0, tol_rel=cfg.tol,
                                ipm=D.IpmParams(max_iter=a.cap, hessian=a.hessian))
            out["oracle"] = {"seconds": time.perf_counter() - t, "converged": o.converged,
                             "ipm_iters": o.ipm.iters, "E0": o.kkt, "f": o.objective,
                             "armijo_hist": np.bincount(o.ipm.armijo_t).tolist(),
                             "same_t_prefix": next((i for i, (x, y) in enumerate(
                                 zip(r.armijo_t, o.ipm.armijo_t)) if x != y),
                                 min(len(r.armijo_t), len(o.ipm.armijo_t)))}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
