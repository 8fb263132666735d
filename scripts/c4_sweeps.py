"""A few c4 ANLS sweeps (+ optional IPM iterations): the target of the ncu captures.

python scripts/c4_sweeps.py [sweeps] [ipm]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402


def main():
    sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    ipm = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    cfg = data.CONFIGS["c4"]
    M, X0, Y0, _, _ = data.make(cfg)
    P = solver.Problem(M, cfg.k)
    X, Yt, _, _, r1 = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T),
                                        Stage1Config(fixed_sweeps=sweeps))
    if ipm:
        X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, 1e-7)
        solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(fixed_iters=ipm))
    torch.cuda.synchronize()
    print("ok", r1.sweeps, r1.trace[-1][1])


if __name__ == "__main__":
    main()
