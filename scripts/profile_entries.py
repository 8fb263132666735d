"""Per-C-ABI-entry device time (CUDA events around every eager library call) of a
two-stage solve: where the time of a converging c2 (or c1/c3-prefix) solve goes.

python scripts/profile_entries.py [c2] [--cap 1000]
Graph-replayed / persistent launches are attributed to the entry that launched them.
"""
import argparse
import collections
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c2")
ap.add_argument("--cap", type=int, default=1000)
a = ap.parse_args()
cfg = data.CONFIGS[a.config]
M, X0, Y0, _, _ = data.make(cfg)
Md = torch.as_tensor(M).cuda()
solver.run_two_stage(Md, X0, Y0, ipm=IpmParams(max_iter=5))  # warm-up (builds, captures)
log = []
orig = solver.Problem._call


def timed(self, name, *args, tag=None):
    if torch.cuda.is_current_stream_capturing():
        return orig(self, name, *args, tag=tag)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = orig(self, name, *args, tag=tag)
    e1.record()
    log.append((name, e0, e1))
    return r


solver.Problem._call = timed
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
rep = solver.run_two_stage(Md, X0, Y0, tol_rel=cfg.tol, ipm=IpmParams(max_iter=a.cap))
ev[1].record()
torch.cuda.synchronize()
tot = ev[0].elapsed_time(ev[1])
acc, cnt = collections.defaultdict(float), collections.Counter()
for name, e0, e1 in log:
    acc[name] += e0.elapsed_time(e1)
    cnt[name] += 1
print(f"{a.config}: total {tot:.2f} ms (converged {rep.converged}, ipm iters {rep.ipm.iters}, "
      f"full {sum(rep.ipm.flags)}); instrumented entries {sum(acc.values()):.2f} ms")
for k, v in sorted(acc.items(), key=lambda x: -x[1])[:30]:
    print(f"  {k:28s} {cnt[k]:6d} calls {v:9.2f} ms  {1e3 * v / cnt[k]:8.1f} us/call")
