"""Run one BASELINE configuration end to end on the device and print a JSON summary.

python scripts/run_config.py c4 [--ipm N] [--sweeps N] [--barrier paper|balanced]
c5 generates its 32 GB fp32 M on the device (data.dense_device).
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--ipm", type=int, default=None)
    ap.add_argument("--sweeps", type=int, default=None)
    ap.add_argument("--barrier", default="balanced")
    a = ap.parse_args()
    cfg = data.CONFIGS[a.name]
    dev = torch.device("cuda", 0)
    t0 = time.perf_counter()
    if a.name == "c5":
        M, X0, Y0 = data.dense_device(cfg.n, cfg.m, cfg.k, cfg.seed, dev, torch.float32)
    else:
        M, X0, Y0, _, _ = data.make(cfg)
    tgen = time.perf_counter() - t0
    P = solver.Problem(M, cfg.k)
    del M
    X0d, Yt0d = P.to_dev(X0), P.to_dev(Y0.T)
    sweeps = a.sweeps if a.sweeps is not None else cfg.fixed_sweeps
    ipm = a.ipm if a.ipm is not None else cfg.fixed_ipm
    out = {"config": a.name, "n": cfg.n, "m": cfg.m, "k": cfg.k, "dtype": str(P.M.dtype),
           "gen_s": tgen}
    torch.cuda.synchronize()
    # warm-up sweep (module load, workspace)
    solver.run_stage1(P, X0d, Yt0d, Stage1Config(fixed_sweeps=1))
    torch.cuda.synchronize()
    t = time.perf_counter()
    X, Yt, pX, pY, r1 = solver.run_stage1(P, X0d, Yt0d, Stage1Config(fixed_sweeps=sweeps))
    torch.cuda.synchronize()
    ts = time.perf_counter() - t
    out.update(stage1_sweeps=r1.sweeps, stage1_s=ts, anls_sweeps_per_s=r1.sweeps / ts,
               objective_after_stage1=r1.trace[-1][1])
    if ipm > 0:
        t = time.perf_counter()
        Xc, Ytc, R, S, mu, rho = solver.transition(P, X, Yt, 1e-10)
        eng, r2 = solver.run_ipm(P, Xc, Ytc, R, S, mu, rho,
                                 IpmParams(fixed_iters=ipm, barrier=a.barrier))
        torch.cuda.synchronize()
        ti = time.perf_counter() - t
        out.update(ipm_iters=r2.iters, ipm_s=ti, ipm_iters_per_s=r2.iters / ti,
                   ipm_outer=r2.outer, armijo_t=r2.armijo_t, full_hessian=r2.flags,
                   ipm_ms_per_iter_steady=(1e3 * (r2.trace[-1][0] - r2.trace[1][0]) / (len(r2.trace) - 2)
                                           if len(r2.trace) > 2 else None),
                   kkt_E0=r2.trace[-1][2] if r2.trace else None,
                   objective_after_ipm=r2.trace[-1][1] if r2.trace else None,
                   small_path=bool(eng.small))
    out["peak_mem_gb"] = torch.cuda.max_memory_allocated() / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
