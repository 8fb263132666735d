"""Full per-iteration IPM trace of a c3 column prefix (cold two-stage solve) or of chosen
chunks of the streaming session, written as text for offline reading.

python scripts/c3_trace.py prefix M_PREFIX CAP OUT
python scripts/c3_trace.py stream CAP OUT M_A M_B ...   (chunks whose width is listed)
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams  # noqa: E402
from paper_2101_08431_b200.stream import StreamSession  # noqa: E402


def dump(fh, tag, rep):
    r = rep.ipm
    fh.write(f"# {tag}: status {rep.status} sweeps {rep.stage1.sweeps} ipm {r.iters} outer {r.outer} "
             f"full {sum(r.flags)} shifted {sum(d > 0 for d in r.deltas)} dense_fb {r.dense_fallbacks} "
             f"E0 {rep.final_kkt_error:.3e} eps {rep.eps_abs:.3e} f {rep.final_objective:.9e}\n")
    di = 0
    for i, tr in enumerate(r.trace):
        s, f, e0, mu, a1, a2, t = tr[:7]
        fl = r.flags[i] if i < len(r.flags) else False
        d = 0.0
        if fl and di < len(r.deltas):
            d = r.deltas[di]
            di += 1
        fh.write(f"{i:5d} f={f:.10e} E0={e0:.3e} mu={mu:.3e} a1={a1:.3e} a2={a2:.3e} t={t} full={int(fl)} "
                 f"delta={d:.2e}\n")


cfg = data.CONFIGS["c3"]
M, X0, Y0, _, _ = data.make(cfg)
mode = sys.argv[1]
if mode == "prefix":
    mm, cap, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    Mp, Y0p = np.ascontiguousarray(M[:, :mm]), np.ascontiguousarray(Y0[:, :mm])
    rep = solver.run_two_stage(torch.as_tensor(Mp).cuda(), X0, Y0p, tol_rel=1e-10,
                               ipm=IpmParams(max_iter=cap))
    with open(out, "w") as fh:
        dump(fh, f"prefix m={mm}", rep)
else:
    cap, out = int(sys.argv[2]), sys.argv[3]
    want = {int(v) for v in sys.argv[4:]}
    mk = lambda: IpmParams(max_iter=cap)  # noqa: E731
    s = StreamSession(M[:, :cfg.m_start], X0, Y0[:, :cfg.m_start], ipm_factory=mk, m_max=cfg.m)
    with open(out, "w") as fh:
        if s.m in want:
            dump(fh, f"chunk m={s.m}", s.chunks[-1][2])
        for m0 in range(cfg.m_start, cfg.m, cfg.m_step):
            rep = s.append(M[:, m0:m0 + cfg.m_step])
            fh.write(f"## m={s.m} {rep.status} ipm {rep.ipm.iters} E {rep.final_kkt_error:.3e}\n")
            if s.m in want:
                dump(fh, f"chunk m={s.m}", rep)
            if s.m >= max(want):
                break
