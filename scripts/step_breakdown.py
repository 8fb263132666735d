"""Host-timed breakdown of one warmed-up c2 bench step (synchronize around each engine call).

python scripts/step_breakdown.py [c2]
"""
import collections
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = data.CONFIGS[name]
M, X0, Y0, _, _ = data.make(cfg)
if len(sys.argv) > 2:  # column prefix (c3 chunk sizes)
    mm = int(sys.argv[2])
    M, Y0 = M[:, :mm], Y0[:, :mm]
P = solver.Problem(M, cfg.k)
X0d, Yt0d = P.to_dev(X0), P.to_dev(Y0.T)
e_scale = max(1.0, solver.kkt_error_primal_only_dev(P, X0d, Yt0d)[0])
eps_abs = cfg.tol * e_scale
acc = collections.defaultdict(float)
cnt = collections.Counter()


def wrap(owner, attr, label):
    fn = getattr(owner, attr)

    def w(*a, **kw):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn(*a, **kw)
        torch.cuda.synchronize()
        acc[label] += time.perf_counter() - t
        cnt[label] += 1
        return r
    setattr(owner, attr, w)


for attr in ("direction", "persist_run", "predictor_sigma", "refresh", "armijo_launch",
             "remember_factorization"):
    wrap(solver.IpmEngine, attr, attr)


def step():
    X, Yt, pX, pY, r1 = solver.run_stage1(P, X0d, Yt0d, Stage1Config())
    X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, eps_abs)
    return solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(eps_tol=eps_abs, max_iter=1000))


for rep in range(3):
    acc.clear()
    cnt.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    X, Yt, pX, pY, r1 = solver.run_stage1(P, X0d, Yt0d, Stage1Config())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, eps_abs)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    eng, r2 = solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(eps_tol=eps_abs, max_iter=1000))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
print(f"total {1e3 * (t3 - t0):.3f} ms: stage1 {1e3 * (t1 - t0):.3f} transition {1e3 * (t2 - t1):.3f} "
      f"ipm {1e3 * (t3 - t2):.3f} (iters {r2.iters}, outer {r2.outer}, fullH {sum(r2.flags)}, "
      f"dense fallbacks {r2.dense_fallbacks}, persist iters {P.persist_iters})")
for k_, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"  {k_:24s} {cnt[k_]:4d} calls {1e3 * v:9.3f} ms")
