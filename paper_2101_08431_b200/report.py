"""SolveReport / trace emission.

``trace_records`` merges the stage-1 sweep trace and the stage-2 iteration trace
into the reference's ordered records (wall_time_s, stage, objective, kkt_error,
mu, flag) with strictly increasing wall time; ``write_report`` writes the JSON
report (SolveReport fields) and the plot-ready CSV trace for one solve.
"""
from __future__ import annotations

import csv
import json
import math
import os

from .config import SolveReport

CSV_COLUMNS = ("wall_time_s", "stage", "objective", "kkt_error", "mu", "flag")


def trace_records(rep: SolveReport):
    recs = []
    last = -math.inf
    for (secs, obj, *_rest) in rep.stage1.trace:
        t = max(float(secs), math.nextafter(last, math.inf))
        recs.append((t, "anls", float(obj), math.nan, math.nan, False))
        last = t
    if rep.ipm is not None:
        base = rep.stage1_time
        flags = list(rep.ipm.flags) + [False] * max(0, len(rep.ipm.trace) - len(rep.ipm.flags))
        for (secs, obj, e0, mu, *_rest), fl in zip(rep.ipm.trace, flags):
            t = max(base + float(secs), math.nextafter(last, math.inf))
            recs.append((t, "ipm", float(obj), float(e0), float(mu), bool(fl)))
            last = t
    return recs


def report_dict(rep: SolveReport) -> dict:
    d = {"status": rep.status, "final_objective": rep.final_objective,
         "final_kkt_error": rep.final_kkt_error, "eps_abs": rep.eps_abs,
         "stage1_time": rep.stage1_time, "stage2_time": rep.stage2_time,
         "anls_sweeps": rep.stage1.sweeps, "ipm_iterations": rep.ipm.iters if rep.ipm else 0,
         "ipm_outer": rep.ipm.outer if rep.ipm else 0,
         "full_hessian_iterations": int(sum(rep.ipm.flags)) if rep.ipm else 0,
         "n": int(rep.X.shape[0]), "m": int(rep.Yt.shape[0]), "k": int(rep.X.shape[1]),
         "error": rep.error}
    return d


def write_report(rep: SolveReport, out_dir: str, name: str = "solve") -> tuple[str, str]:
    os.makedirs(out_dir, exist_ok=True)
    jpath = os.path.join(out_dir, f"{name}.json")
    cpath = os.path.join(out_dir, f"{name}_trace.csv")
    with open(jpath, "w") as fh:
        json.dump(report_dict(rep), fh, indent=1, sort_keys=True)
    with open(cpath, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_COLUMNS)
        for r in trace_records(rep):
            w.writerow([f"{r[0]:.9f}", r[1], repr(r[2]), repr(r[3]), repr(r[4]), int(r[5])])
    return jpath, cpath


__all__ = ["trace_records", "report_dict", "write_report", "CSV_COLUMNS"]
