"""Wall-clock of run_ipm (fixed iterations) on c4 / c5, graphs on and off, twice each."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = data.CONFIGS[name]
if name == "c5":
    M, X0, Y0 = data.dense_device(cfg.n, cfg.m, cfg.k, cfg.seed, torch.device("cuda", 0), torch.float32)
else:
    M, X0, Y0, _, _ = data.make(cfg)
P = solver.Problem(M, cfg.k)
del M
X, Yt, _, _, _ = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T), Stage1Config(fixed_sweeps=3))
order = [g == "1" for g in sys.argv[2].split(",")] if len(sys.argv) > 2 else [True, False, True]
for graphs in order:
    Xc, Ytc, R, S, mu, rho = solver.transition(P, X, Yt, 1e-10)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng, r2 = solver.run_ipm(P, Xc, Ytc, R, S, mu, rho, IpmParams(fixed_iters=cfg.fixed_ipm or 10,
                                                                  use_graphs=graphs))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    tr = r2.trace
    steady = (tr[-1][0] - tr[2][0]) / (len(tr) - 3) if len(tr) > 3 else float("nan")
    print(f"{name} graphs={graphs}: {r2.iters} its {1e3 * dt / r2.iters:.3f} ms/it overall, "
          f"steady {1e3 * steady:.3f} ms/it; first its "
          f"{[round(1e3 * (tr[i][0] - (tr[i - 1][0] if i else 0.0)), 2) for i in range(min(4, len(tr)))]}",
          flush=True)
