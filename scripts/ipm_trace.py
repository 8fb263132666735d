"""Print the stage-2 trajectory of one config (E(.;0), mu, alpha, Armijo t, Hessian flags)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2101_08431_b200 import data, run_two_stage  # noqa: E402
from paper_2101_08431_b200.config import IpmParams  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
barrier = sys.argv[2] if len(sys.argv) > 2 else "balanced"
cfg = data.CONFIGS[name]
M, X0, Y0, _, _ = data.make(cfg)
rep = run_two_stage(M, X0, Y0, tol_rel=cfg.tol, ipm=IpmParams(max_iter=500, barrier=barrier))
r = rep.ipm
print(name, barrier, "status", rep.status, "eps_abs", rep.eps_abs, "sweeps", rep.stage1.sweeps,
      "ipm", r.iters, "outer", r.outer, "full-H iters", sum(r.flags), "final E", rep.final_kkt_error)
print("t histogram", np.bincount(np.array(r.armijo_t)).tolist())
tr = r.trace
for i in list(range(0, len(tr), max(1, len(tr) // 25))) + [len(tr) - 1]:
    s, obj, e0, mu, a1, a2, t = tr[i]
    print(f"it {i:4d} f {obj:.10e} E0 {e0:.3e} mu {mu:.3e} a1 {a1:.3e} a2 {a2:.3e} t {t} "
          f"full {r.flags[i]}")
