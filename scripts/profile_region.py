"""ncu launch list of one region only (cudaProfilerStart/Stop): stage-1 sweeps or IPM iterations.

python scripts/profile_region.py c4 ipm 3      # 3 IPM iterations after 3 sweeps + transition
python scripts/profile_region.py c4 anls 3     # 3 warm ANLS sweeps
run under: ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ...
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

name, what, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
cfg = data.CONFIGS[name]
if cfg.name == "c5":
    dev = torch.device("cuda", 0)
    M, X0, Y0 = data.dense_device(cfg.n, cfg.m, cfg.k, cfg.seed, dev, torch.float32)
else:
    M, X0, Y0, _, _ = data.make(cfg)
P = solver.Problem(M, cfg.k)
del M
X0d, Yt0d = P.to_dev(X0), P.to_dev(Y0.T)
X, Yt, pX, pY, _ = solver.run_stage1(P, X0d, Yt0d, Stage1Config(fixed_sweeps=3))
if what == "anls":
    solver.run_stage1(P, X, Yt, Stage1Config(fixed_sweeps=n), pX=pX, pY=pY)  # warm-up
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    solver.run_stage1(P, X, Yt, Stage1Config(fixed_sweeps=n), pX=pX, pY=pY)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
else:
    Xc, Ytc, R, S, mu, rho = solver.transition(P, X, Yt, 1e-10)
    solver.run_ipm(P, Xc.clone(), Ytc.clone(), R.clone(), S.clone(), mu, rho, IpmParams(fixed_iters=2))
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    eng, r2 = solver.run_ipm(P, Xc, Ytc, R, S, mu, rho, IpmParams(fixed_iters=n))
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print("done")
