"""ncu launch list of dense-Schur IPM iterations at the last c3 chunk size (m = 500, k = 4).

Each dense fallback of the c3 streaming session runs this path (mk = 2000).
run under: ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ...
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

cfg = data.CONFIGS["c3"]
M, X0, Y0, _, _ = data.make(cfg)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 500
M, Y0 = M[:, :m], Y0[:, :m]
P = solver.Problem(M, cfg.k)
X, Yt, pX, pY, _ = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T), Stage1Config())
X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, 1e-7)
prm = dict(fixed_iters=2, schur_solver="dense", persistent=False, use_graphs=False)
solver.run_ipm(P, X.clone(), Yt.clone(), R.clone(), S.clone(), mu, rho, IpmParams(**prm))
torch.cuda.synchronize()
torch.cuda.profiler.start()
solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(**prm))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
