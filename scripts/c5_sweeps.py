"""A few c5 ANLS sweeps (+ optional IPM iterations) on the device-generated fp32 M
(200000 x 40000, k = 16): the target of launch lists / ncu captures.

python scripts/c5_sweeps.py [sweeps] [ipm] [rows]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402


def main():
    sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ipm = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    cfg = data.CONFIGS["c5"]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.n
    dev = torch.device("cuda", 0)
    M, X0, Y0 = data.dense_device(n, cfg.m, cfg.k, cfg.seed, dev, torch.float32, rows=(0, n))
    P = solver.Problem(M, cfg.k)
    del M
    X, Yt, _, _, r1 = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T),
                                        Stage1Config(fixed_sweeps=sweeps))
    if ipm:
        X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, 1e-10)
        solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(fixed_iters=ipm))
    torch.cuda.synchronize()
    print("ok", r1.sweeps, r1.trace[-1][1])


if __name__ == "__main__":
    main()
