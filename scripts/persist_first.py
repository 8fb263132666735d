"""Time the first persistent launches in a fresh process (module load / setup costs)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

cfg = data.CONFIGS["c2"]
M, X0, Y0, _, _ = data.make(cfg)
for rep in range(3):
    P = solver.Problem(M, cfg.k)
    X, Yt, pX, pY, r1 = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T), Stage1Config())
    X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, 1e-7)
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng, r2 = solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(fixed_iters=int(sys.argv[1])))
    torch.cuda.synchronize()
    print(rep, "run_ipm", round(time.perf_counter() - t, 4), "persist_s", round(P.persist_seconds, 4),
          "iters", r2.iters, flush=True)
