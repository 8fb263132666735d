import sys
sys.path.insert(0, ".")
import torch
from paper_2101_08431_b200 import data
from paper_2101_08431_b200.config import IpmParams
from paper_2101_08431_b200.stream import StreamSession
cfg = data.CONFIGS["c3"]
M, X0, Y0, _, _ = data.make(cfg)
s = StreamSession(M[:, :20], X0, Y0[:, :20], ipm_factory=lambda: IpmParams(max_iter=100), m_max=500)
for m0 in range(20, 80, 10):
    s.append(M[:, m0:m0 + 10])
for c in s.chunks:
    r = c[2]
    print(c[0], "eps_abs %.3e" % r.eps_abs, "E %.3e" % r.final_kkt_error, r.status, r.ipm.iters if r.ipm else 0)
