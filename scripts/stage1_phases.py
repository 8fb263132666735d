"""Per-phase clock breakdown of the persistent stage 1 (CTA 0 stamps), config c2."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import Stage1Config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = data.CONFIGS[name]
M, X0, Y0, _, _ = data.make(cfg)
names = ["YY^T + ctb", "tol + X NNLS", "X partials", "gsync1", "reduce X^T X, ctb_Y",
         "Y NNLS + stats partials", "gsync2", "stats reduce", "step test + reload Y"]
for rep in range(2):
    P = solver.Problem(M, cfg.k)
    prof = torch.zeros((512, 16), dtype=torch.int64, device=P.dev)
    P.lib.nmfb_stage1_set_prof(prof.data_ptr())
    X, Yt, pX, pY, r = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T), Stage1Config())
    torch.cuda.synchronize()
    P.lib.nmfb_stage1_set_prof(None)
pr = prof.cpu().numpy()[2:r.sweeps - 1, :10].astype(np.float64)
d = np.median(np.diff(pr, axis=1), axis=0) / 1.965e3
print(name, "sweeps", r.sweeps, "per-sweep us", round(float(d.sum()), 2))
for nm, v in zip(names, d):
    print(f"  {nm:28s} {v:8.2f}")
