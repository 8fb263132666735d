"""Solver-level parity report: device solver vs the CPU oracle on one config.

python scripts/parity_solver.py c1 [ipm_iters] [barrier]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import driver as D  # noqa: E402  (checker)
from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / max(1e-300, np.abs(b).max()))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    barrier = sys.argv[3] if len(sys.argv) > 3 else "paper"
    cfg = data.CONFIGS[name]
    M, X0, Y0, _, _ = data.make(cfg)
    t = time.time()
    P = solver.Problem(M, cfg.k)
    import torch
    X = P.to_dev(X0)
    Yt = P.to_dev(Y0.T)
    Xg, Ytg, pX, pY, r1 = solver.run_stage1(P, X, Yt, Stage1Config())
    torch.cuda.synchronize()
    tg = time.time() - t
    t = time.time()
    ro = D.run_stage1(M, X0, Y0.T.copy())
    to = time.time() - t
    print(f"stage1 sweeps gpu={r1.sweeps} oracle={ro.sweeps}  time gpu={tg:.3f}s oracle={to:.3f}s")
    print(f"  rel X {rel(Xg.cpu().numpy(), ro.X):.2e}  rel Y {rel(Ytg.cpu().numpy(), ro.Yt):.2e}"
          f"  passive X equal {np.array_equal(pX.bool().cpu().numpy(), ro.pX)}"
          f"  passive Y equal {np.array_equal(pY.bool().cpu().numpy(), ro.pY)}")
    print(f"  obj gpu {r1.trace[-1][1]:.15e} oracle {ro.trace[-1][1]:.15e}")
    # transition + fixed ipm iterations, both from the ORACLE's stage-1 point
    eps = 1e-7
    st = D.transition(ro.X, ro.Yt, M, eps)
    Xd, Yd, Rd, Sd, mud, rhod = solver.transition(P, P.to_dev(ro.X), P.to_dev(ro.Yt), eps)
    print(f"transition mu gpu {mud:.15e} oracle {st.mu:.15e}  R {Rd[0,0].item():.15e} {st.R[0,0]:.15e}")
    p = IpmParams(fixed_iters=iters, barrier=barrier)
    t = time.time()
    eng, r2 = solver.run_ipm(P, Xd, Yd, Rd, Sd, mud, rhod, p)
    torch.cuda.synchronize()
    tg = time.time() - t
    p2 = D.IpmParams(fixed_iters=iters, barrier=barrier)
    t = time.time()
    r2o = D.run_ipm(M, st, p2)
    to = time.time() - t
    print(f"ipm iters gpu={r2.iters} oracle={r2o.iters} outer {r2.outer}/{r2o.outer} time gpu={tg:.3f}s oracle={to:.3f}s")
    print("  t gpu   ", r2.armijo_t)
    print("  t oracle", r2o.armijo_t)
    print("  flags equal", r2.flags == r2o.flags, "t equal", r2.armijo_t == r2o.armijo_t)
    print(f"  rel X {rel(eng.X.cpu().numpy(), r2o.state.X):.2e} rel Y {rel(eng.Yt.cpu().numpy(), r2o.state.Yt):.2e}"
          f" rel R {rel(eng.R.cpu().numpy(), r2o.state.R):.2e} rel S {rel(eng.S.cpu().numpy(), r2o.state.S):.2e}")
    print(f"  mu gpu {eng.mu:.6e} oracle {r2o.state.mu:.6e}")
    for a, b in list(zip(r2.trace, r2o.trace))[:: max(1, iters // 10)]:
        print(f"   f {a[1]:.12e} {b[1]:.12e}  E {a[2]:.6e} {b[2]:.6e}  a1 {a[4]:.3e} {b[4]:.3e}")


if __name__ == "__main__":
    main()
