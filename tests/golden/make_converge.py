"""Generate tests/golden/converge_c1c2.json: the oracle's two-stage solves of BASELINE c1 and
c2 to relative KKT 1e-10 under frozen semantics 10 (hessian="inertia", cap 1000).

TEST INFRASTRUCTURE: the oracle driver (oracle/driver.py over the reference-pinned C kernels
and the NumPy-backend Schur kernels) is run here once (c2 takes ~6 minutes of CPU); the GPU
test tests/test_gpu_converge.py checks the device solve against these numbers.

    python tests/golden/make_converge.py
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle import driver as D  # noqa: E402
from paper_2101_08431_b200 import data  # noqa: E402


def main():
    D.set_schur_backend("numpy")
    out = {}
    for name in ("c1", "c2"):
        cfg = data.CONFIGS[name]
        M, X0, Y0, _, _ = data.make(cfg)
        t = time.perf_counter()
        rep = D.run_two_stage(M, X0, Y0, tol_rel=cfg.tol, ipm=D.IpmParams(max_iter=1000))
        r = rep.ipm
        out[name] = {"seconds": time.perf_counter() - t, "converged": bool(rep.converged),
                     "sweeps": rep.stage1.sweeps, "ipm_iters": r.iters, "outer": r.outer,
                     "E0": rep.kkt, "eps_abs": rep.eps_abs, "objective": rep.objective,
                     "full_iters": int(sum(r.flags)),
                     "armijo_t": [int(t) for t in r.armijo_t], "flags": [bool(f) for f in r.flags],
                     "deltas": [float(d) for d in r.deltas],
                     "mu": [float(rec[3]) for rec in r.trace]}
        print(name, {k: v for k, v in out[name].items() if not isinstance(v, list)}, flush=True)
    with open(os.path.join(HERE, "converge_c1c2.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
