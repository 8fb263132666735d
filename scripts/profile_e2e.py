"""Host-side breakdown of one public run_two_stage call on c2 (bench e2e leg)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver, run_two_stage  # noqa: E402
from paper_2101_08431_b200.config import IpmParams  # noqa: E402

cfg = data.CONFIGS["c2"]
M, X0, Y0, _, _ = data.peaks(cfg.n, cfg.m, cfg.k, cfg.seed)
Mh = torch.from_numpy(M).pin_memory()
T = {}
orig = {}


def wrap(mod, name):
    f = getattr(mod, name)
    orig[name] = f

    def g(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + time.perf_counter() - t
        return r
    setattr(mod, name, g)


for nm in ("Problem", "run_stage1", "transition", "run_ipm", "kkt_error_primal_only_dev"):
    wrap(solver, nm)
for rep in range(4):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep_ = run_two_stage(Mh, X0, Y0, tol_rel=cfg.tol, ipm=IpmParams(max_iter=500), e_scale=None)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
print("total %.2f ms" % (1e3 * tot), {k: round(1e3 * v, 2) for k, v in T.items()},
      "other %.2f ms" % (1e3 * (tot - sum(T.values()))))
