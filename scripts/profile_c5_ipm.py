"""Launch list of steady c5 IPM iterations (fp32 M 200000 x 40000, k = 16).

ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file out.csv python scripts/profile_c5_ipm.py [ITERS]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = data.CONFIGS["c5"]
dev = torch.device("cuda", 0)
M, X0, Y0 = data.dense_device(cfg.n, cfg.m, cfg.k, cfg.seed, dev, torch.float32)
P = solver.Problem(M, cfg.k)
del M
X, Yt, _, _, _ = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T), Stage1Config(fixed_sweeps=3))
X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, 1e-10)
solver.run_ipm(P, X.clone(), Yt.clone(), R.clone(), S.clone(), mu, rho, IpmParams(fixed_iters=3))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.profiler.start()
e0.record()
solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(fixed_iters=iters))
e1.record()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{iters} iterations: {e0.elapsed_time(e1) / iters:.2f} ms per iteration")
