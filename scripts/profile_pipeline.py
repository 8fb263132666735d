"""Wall time of each submit() / result() of the c4 SolvePipeline (bench e2e leg)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import SolvePipeline, data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

cfg = data.CONFIGS["c4"]
M, X0, Y0, _, _ = data.make(cfg)
Mh = torch.from_numpy(M).pin_memory()
P0 = solver.Problem(M, cfg.k)
e_scale = max(1.0, solver.kkt_error_primal_only_dev(P0, P0.to_dev(X0), P0.to_dev(Y0.T))[0])
del P0
pipe = SolvePipeline(cfg.n, cfg.m, cfg.k, tol_rel=cfg.tol, s1=Stage1Config(fixed_sweeps=cfg.fixed_sweeps),
                     ipm=IpmParams(fixed_iters=cfg.fixed_ipm), e_scale=e_scale)
for _ in range(2):
    pipe.submit(Mh, X0, Y0)
for _ in range(2):
    pipe.result()
torch.cuda.synchronize()
N = 8
t0 = time.perf_counter()
pipe.submit(Mh, X0, Y0)
ts = [time.perf_counter() - t0]
for i in range(N):
    a = time.perf_counter()
    if i + 1 < N:
        pipe.submit(Mh, X0, Y0)
    b = time.perf_counter()
    rep = pipe.result()
    c = time.perf_counter()
    ts.append((b - a, c - b, rep.stage1.seconds, rep.ipm.seconds))
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f"first submit {1e3 * ts[0]:.2f} ms; total {1e3 * tot:.1f} ms = {1e3 * tot / N:.2f} ms per step")
for i, (s, r, s1, s2) in enumerate(ts[1:]):
    print(f"step {i}: submit {1e3 * s:.2f} ms, result {1e3 * r:.2f} ms (stage1 {1e3 * s1:.2f}, ipm {1e3 * s2:.2f})")
# the same without the pipeline's copies: device-resident M
Md = torch.as_tensor(M).cuda()
Pd = solver.Problem(Md, cfg.k)
kw = dict(tol_rel=cfg.tol, s1=Stage1Config(fixed_sweeps=cfg.fixed_sweeps), ipm=IpmParams(fixed_iters=cfg.fixed_ipm),
          e_scale=e_scale, problem=Pd)
for _ in range(2):
    solver.run_two_stage(None, X0, Y0, **kw)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    rep = solver.run_two_stage(None, X0, Y0, **kw)
torch.cuda.synchronize()
print(f"run_two_stage on a resident M (no H2D of M): {1e3 * (time.perf_counter() - t0) / 5:.2f} ms per call "
      f"(stage1 {1e3 * rep.stage1.seconds:.2f}, ipm {1e3 * rep.ipm.seconds:.2f})")
