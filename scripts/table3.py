"""Multi-seed benchmark table in the paper's Table III layout (SPEC.md:545-566 cmd_bench).

python scripts/table3.py [--sizes 2000x50x3,...] [--seeds 10] [--variants two_stage,anls_only,ipm_only]
                         [--tol 1e-6] [--out DIR]

Each cell: the paper's synthetic family (PAPER section 5.4, noise 0.1), seeded U(0,1) initial
points, one solve per seed on the GPU; reports wall time of the solve phase, final E(.;0)
and f = 0.5 ||XY - M||^2 as avrg(min,max), as CSV and aligned text.  Per-solve JSON
reports and CSV traces go to DIR/cells/.
"""
import argparse
import csv
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import data, io, report, run_two_stage  # noqa: E402
from paper_2101_08431_b200.config import IpmParams  # noqa: E402


def triplet(v):
    v = np.asarray(v, dtype=np.float64)
    return f"{v.mean():.6g}({v.min():.6g},{v.max():.6g})"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="2000x50x3")
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--variants", default="two_stage,anls_only,ipm_only")
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--barrier", default="paper")
    ap.add_argument("--max-ipm", type=int, default=500)
    ap.add_argument("--out", default="gpurun_out/table3")
    a = ap.parse_args()
    sizes = [tuple(int(x) for x in s.split("x")) for s in a.sizes.split(",")]
    variants = a.variants.split(",")
    rows = []
    for (n, m, k) in sizes:
        M, _, _ = io.generate_synthetic(n, m, k, 0.1, seed=2021)
        Md = torch.as_tensor(M).cuda()
        for var in variants:
            secs, errs, objs, stats = [], [], [], []
            for seed in range(a.seeds):
                X0, Y0 = data.init_factors(n, m, k, seed)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                try:
                    rep = run_two_stage(Md, X0, Y0, tol_rel=a.tol, stage=var,
                                        ipm=IpmParams(max_iter=a.max_ipm, barrier=a.barrier))
                    torch.cuda.synchronize()
                    dt = time.perf_counter() - t0
                    secs.append(rep.stage1_time + rep.stage2_time if rep.stage2_time else dt)
                    errs.append(rep.final_kkt_error)
                    objs.append(rep.final_objective)
                    stats.append(rep.status)
                    report.write_report(rep, os.path.join(a.out, "cells"), f"{n}x{m}x{k}_{var}_s{seed}")
                except Exception as exc:  # per-cell failure is recorded, the run continues
                    stats.append(f"Error:{type(exc).__name__}")
            rows.append({"size": f"({n},{m},{k})", "variant": var,
                         "cpu_s": triplet(secs) if secs else "-", "E": triplet(errs) if errs else "-",
                         "f": triplet(objs) if objs else "-",
                         "status": ",".join(sorted(set(stats)))})
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, "table3.csv"), "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)
    widths = {c: max(len(c), *(len(r[c]) for r in rows)) for c in rows[0]}
    lines = ["  ".join(c.ljust(widths[c]) for c in rows[0])]
    lines += ["  ".join(r[c].ljust(widths[c]) for c in r) for r in rows]
    text = "\n".join(lines)
    open(os.path.join(a.out, "table3.txt"), "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
