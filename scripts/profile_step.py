"""One warmed-up c2 two-stage solve (for ncu launch lists / captures)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cfg = data.CONFIGS[name]
M, X0, Y0, _, _ = data.make(cfg)
P = solver.Problem(M, cfg.k)
X0d, Yt0d = P.to_dev(X0), P.to_dev(Y0.T)
for rep in range(2):
    X, Yt, pX, pY, r1 = solver.run_stage1(P, X0d, Yt0d, Stage1Config(fixed_sweeps=cfg.fixed_sweeps))
    X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, 1e-7)
    eng, r2 = solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(fixed_iters=iters))
    torch.cuda.synchronize()
    print("rep", rep, "launches", P.lib.nmfb_launch_count(), "sweeps", r1.sweeps, "ipm", r2.iters,
          "stage1_s %.5f ipm_s %.5f per_iter_ms %.4f" % (r1.seconds, r2.seconds,
                                                         1e3 * r2.seconds / max(1, r2.iters)))
