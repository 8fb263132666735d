"""One warmed-up bench.py c2 step (stage 1 + transition + IPM to tol/cap) inside
cudaProfilerStart/Stop, with a host-side time breakdown."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

cfg = data.CONFIGS["c2"]
M, X0, Y0, _, _ = data.peaks(cfg.n, cfg.m, cfg.k, cfg.seed)
P = solver.Problem(M, cfg.k)
X0d, Yt0d = P.to_dev(X0), P.to_dev(Y0.T)
e_scale = max(1.0, solver.kkt_error_primal_only_dev(P, X0d, Yt0d)[0])
eps_abs = cfg.tol * e_scale


def step(prof=False):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    X, Yt, pX, pY, r1 = solver.run_stage1(P, X0d, Yt0d, Stage1Config())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, eps_abs)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    p0 = P.persist_seconds
    eng, r2 = solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(eps_tol=eps_abs, max_iter=500))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    return (r1.sweeps, r2.iters, r2.outer, sum(r2.flags), 1e3 * (t1 - t0), 1e3 * (t2 - t1),
            1e3 * (t3 - t2), 1e3 * (P.persist_seconds - p0))


for _ in range(3):
    step()
torch.cuda.profiler.start()
r = step()
torch.cuda.profiler.stop()
print("sweeps %d ipm %d outer %d fullH %d | stage1 %.2f ms transition %.2f ms ipm %.2f ms "
      "(persistent launches %.2f ms)" % r)
