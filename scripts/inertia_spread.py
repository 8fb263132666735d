"""Spread of the c1 60-iteration inertia-shifted trajectory between correct implementations:
device (dataflow dense kernels, or NMFB_DENSE_FLOW=0 for the panel kernels) vs the oracle
with its NumPy-backend Schur kernels, and the oracle's C backend vs its NumPy backend."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from oracle import driver as D  # noqa: E402
from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 60
M, X0, Y0, _, _ = data.make(data.CONFIGS["c1"])
ro = D.run_stage1(M, X0, Y0.T.copy())
P = solver.Problem(M, 3)
X, Yt, R, S, mu, rho = solver.transition(P, P.to_dev(ro.X), P.to_dev(ro.Yt), 1e-7)
eng, r = solver.run_ipm(P, X, Yt, R, S, mu, rho, IpmParams(fixed_iters=iters))
outs = {}
for be in ("numpy", "c"):
    D.set_schur_backend(be)
    st = D.transition(ro.X, ro.Yt, M, 1e-7)
    outs[be] = D.run_ipm(M, st, D.IpmParams(fixed_iters=iters))
D.set_schur_backend("c")


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


for be, o in outs.items():
    print(f"device vs oracle[{be}]: decisions equal {r.armijo_t == o.armijo_t and r.flags == o.flags} "
          f"X {rel(eng.X.cpu().numpy(), o.state.X):.3e} Y {rel(eng.Yt.cpu().numpy(), o.state.Yt):.3e}")
a, b = outs["numpy"], outs["c"]
print(f"oracle[c] vs oracle[numpy]: decisions equal {a.armijo_t == b.armijo_t and a.flags == b.flags} "
      f"X {rel(b.state.X, a.state.X):.3e} Y {rel(b.state.Yt, a.state.Yt):.3e}")
