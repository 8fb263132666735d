"""Convergence anatomy of a c3 column prefix solved cold by the two-stage method:
iterations, full-coupling / shifted counts, Armijo histogram, E(.;0) and mu along the run.

python scripts/c3_prefix.py M_PREFIX [cap] [hessian]
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams  # noqa: E402

mm = int(sys.argv[1])
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
hess = sys.argv[3] if len(sys.argv) > 3 else "inertia"
cfg = data.CONFIGS["c3"]
M, X0, Y0, _, _ = data.make(cfg)
M, Y0 = np.ascontiguousarray(M[:, :mm]), np.ascontiguousarray(Y0[:, :mm])
import time
t = time.perf_counter()
rep = solver.run_two_stage(torch.as_tensor(M).cuda(), X0, Y0, tol_rel=1e-10,
                           ipm=IpmParams(max_iter=cap, hessian=hess))
torch.cuda.synchronize()
dt = time.perf_counter() - t
r = rep.ipm
print(f"m={mm}: {dt:.2f} s, status {rep.status}, sweeps {rep.stage1.sweeps}, ipm {r.iters}, "
      f"outer {r.outer}, full {sum(r.flags)}, shifted {sum(d > 0 for d in r.deltas)}, "
      f"dense fallbacks {r.dense_fallbacks}, E0 {rep.final_kkt_error:.3e} eps {rep.eps_abs:.3e}")
print("armijo hist", np.bincount(r.armijo_t).tolist())
tr = r.trace
for i in list(range(0, len(tr), max(1, len(tr) // 12))) + [len(tr) - 1]:
    s, f, e0, mu = tr[i][:4]
    print(f"  it {i:4d} t={s:7.3f}s f={f:.6e} E0={e0:.3e} mu={mu:.3e} full={r.flags[i] if i < len(r.flags) else '-'}")
