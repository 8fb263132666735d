"""ncu launch list of the c2 full-Hessian dense directions only (cudaProfilerStart/Stop
around IpmEngine.direction(full=True) calls of one warmed-up c2 solve)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

cfg = data.CONFIGS["c2"]
M, X0, Y0, _, _ = data.make(cfg)
P = solver.Problem(M, cfg.k)
X0d, Yt0d = P.to_dev(X0), P.to_dev(Y0.T)
eps = cfg.tol * max(1.0, solver.kkt_error_primal_only_dev(P, X0d, Yt0d)[0])
orig = solver.IpmEngine.direction
state = {"on": False}


def wrapped(self, full, force_dense=False):
    if state["on"] and full:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        r = orig(self, full, force_dense)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return r
    return orig(self, full, force_dense)


solver.IpmEngine.direction = wrapped
for rep in range(2):
    state["on"] = rep == 1
    X, Yt, pX, pY, _ = solver.run_stage1(P, X0d, Yt0d, Stage1Config())
    X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, eps)
    solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(eps_tol=eps, max_iter=500))
torch.cuda.synchronize()
print("done")
