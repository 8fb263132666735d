"""Warm c4/c5-style IPM iterations for ncu launch lists (stage 1 then N IPM iterations)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = data.CONFIGS[name]
M, X0, Y0, _, _ = data.make(cfg)
P = solver.Problem(M, cfg.k)
X, Yt, _, _, _ = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T), Stage1Config(fixed_sweeps=5))
for rep in range(2):
    Xc, Ytc, R, S, mu, rho = solver.transition(P, X, Yt, 1e-10)
    eng, r2 = solver.run_ipm(P, Xc, Ytc, R, S, mu, rho, IpmParams(fixed_iters=iters))
    torch.cuda.synchronize()
    print("rep", rep, "launches", P.lib.nmfb_launch_count(), "ipm", r2.iters)
