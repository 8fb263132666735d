"""One c2 solve with the persistent inner loop (for ncu captures of k_ipm_persist)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = data.CONFIGS[name]
M, X0, Y0, _, _ = data.make(cfg)
P = solver.Problem(M, cfg.k)
X, Yt, pX, pY, r1 = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T), Stage1Config())
X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, 1e-7)
eng, r2 = solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(fixed_iters=iters))
torch.cuda.synchronize()
print("ipm iters", r2.iters, "persist", P.persist_iters, "s", P.persist_seconds)
