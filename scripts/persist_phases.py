"""Per-phase clock breakdown of the persistent inner loop (CTA 0 stamps)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
grid = int(sys.argv[2]) if len(sys.argv) > 2 else 0
m = int(sys.argv[3]) if len(sys.argv) > 3 else 0
barrier = sys.argv[4] if len(sys.argv) > 4 else "paper"
cfg = data.CONFIGS[name]
M, X0, Y0, _, _ = data.make(cfg)
if m:
    M, Y0 = M[:, :m], Y0[:, :m]
names = ["A rows", "bar1", "reduce+decide", "Y factor", "G/capacitance", "dY", "rows dX",
         "quartic", "bar2", "trials", "bar3+select", "update+residual", "bar4", "phase E"]
for rep in range(2):
    P = solver.Problem(M, cfg.k)
    P.persist_prof = torch.zeros((4096, 40), dtype=torch.int64, device=P.dev)
    X, Yt, pX, pY, r1 = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T), Stage1Config())
    X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, 1e-7)
    eng, r2 = solver.run_ipm(P, X, Yt, R, S, mu, rho,
                             IpmParams(fixed_iters=200, persist_grid=grid, barrier=barrier))
    torch.cuda.synchronize()
pr = P.persist_prof.cpu().numpy()[20:180].astype(np.float64)
d = np.median(np.diff(pr[:, :15], axis=1), axis=0) / 1.965e3  # us at 1965 MHz
print(name, barrier, "grid", grid, "m", m, "per-iteration us:", round(float(d.sum()), 2),
      "wall ms/it", round(1e3 * P.persist_seconds / max(P.persist_iters, 1), 4))
for nm, v in zip(names, d):
    print(f"  {nm:16s} {v:8.2f}")
sub = {"B: reduce->gY sync": (2, 16), "B: KKT local": (16, 17), "B: KKT reduce+commit": (17, 3),
       "C: G accumulate": (4, 18), "C: unpack+chol G": (18, 19), "C: T1": (19, 20),
       "C: Hm": (20, 21), "C: chol H": (21, 22), "C: writes+check": (22, 23),
       "C: w solve": (23, 5), "chol G inside": (24, 25), "chol H inside": (26, 27),
       "w: matvec+fwd": (23, 28), "w: 2 back": (28, 5),
       "A: YY^T": (0, 33), "A: row factors": (33, 31), "A: badA reduce": (31, 32), "A: partials": (32, 1),
       "Q: pass": (7, 34), "Q: reduce+store": (34, 8),
       "D: nudge": (11, 29), "D: rows/graY": (29, 30), "D: reduce+store": (30, 12)}
for nm, (i, j) in sub.items():
    print(f"  {nm:22s} {float(np.median(pr[:, j] - pr[:, i])) / 1.965e3:8.2f}")
print("armijo t histogram:", np.bincount(np.array(r2.armijo_t)).tolist())

