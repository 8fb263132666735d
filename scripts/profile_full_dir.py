"""Launch list of full-coupling (inertia-shifted) IPM iterations on a c3 column prefix or c2.

python scripts/profile_full_dir.py c3 M_PREFIX ITERS   |   c2 0 ITERS
Runs the cold two-stage solve for ITERS iterations twice; the second run is bracketed by
cudaProfilerStart/Stop (ncu --profile-from-start off).  Also prints the wall time per IPM
iteration of the flagged (full-coupling) iterations.
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams  # noqa: E402

name, mm, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = data.CONFIGS[name]
M, X0, Y0, _, _ = data.make(cfg)
if mm:
    M, Y0 = np.ascontiguousarray(M[:, :mm]), np.ascontiguousarray(Y0[:, :mm])
Md = torch.as_tensor(M).cuda()
for rep_i in range(2):
    torch.cuda.synchronize()
    if rep_i:
        torch.cuda.profiler.start()
    t0 = time.perf_counter()
    rep = solver.run_two_stage(Md, X0, Y0, tol_rel=1e-10, ipm=IpmParams(max_iter=iters))
    torch.cuda.synchronize()
    if rep_i:
        torch.cuda.profiler.stop()
    r = rep.ipm
    tr = [t[0] for t in r.trace]
    dts = np.diff(np.array([0.0] + tr))
    fl = np.array(r.flags[:len(dts)], bool)
    print(f"{name} m={M.shape[1]}: {time.perf_counter() - t0:.3f} s, ipm {r.iters}, full {int(fl.sum())} "
          f"(tries beyond the first: {sum(d > 0 for d in r.deltas)} shifted), "
          f"ms per full iteration {1e3 * dts[fl].mean() if fl.any() else float('nan'):.3f}, "
          f"ms per GN iteration {1e3 * dts[~fl].mean() if (~fl).any() else float('nan'):.4f}")
