#!/usr/bin/env python
"""Benchmark of the B200 two-stage NMF hot path (one JSON line on rank 0).

Workload (BASELINE.json configs[1], "c2"): fp64 n=3000, m=100, k=3 peak/logistic
instance; one STEP = one complete two-stage solve (stage-1 ANLS to eps_STOL,
transition, stage-2 IPM to relative KKT 1e-10 or the 500-iteration cap) from
the seeded initial factors, inputs resident in HBM.  value = solver iterations
(ANLS sweeps + IPM iterations) per second, summed over ranks (weak scaling:
every rank solves its own seeded replica).  Auxiliary: c4 (20000 x 5000 x 10)
ANLS sweeps/s with the HBM roofline of its product kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOAD = "c2"
IPM_CAP = 500
# DRAM bytes per IPM iteration of the roofline entry from one `ncu --set full` capture
# (cold-cache, serialised replay), scaled to the live launch's iteration count.
NCU_TRAFFIC = {
    "nmfb_ipm_persist": {"dram_bytes_per_iteration": (2809344 + 137472) / 200,
                         "source": "profiles/r01_ncu_persist_c2.txt (200-iteration launch)"},
}
CPU_IPM_SAMPLE = 20  # bounded CPU sample: full stage 1 + this many IPM iterations


def _metric():
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:  # pragma: no cover
        return "ANLS sweeps/s + IPM iters/s, time-to-tolerance, % HBM roofline at 1/2/4/8 GPU"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.gpu = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------
# reference arm: the CPU oracle port (numpy-backend Schur kernels)
# ----------------------------------------------------------------------------
def cpu_sample(M, X0, Y0, tol_rel, e_scale, ipm_iters=IPM_CAP):
    """Bounded CPU sample of the same workload.

    Runs the full stage 1 and the first CPU_IPM_SAMPLE IPM iterations, then
    extrapolates the IPM part to ``ipm_iters`` iterations (the per-iteration
    cost is flat: same matrix sizes every iteration) so the CPU number has the
    same sweep/iteration mix as the GPU step.  -> (units, seconds, cores)
    """
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
    from oracle import driver as D  # checker/baseline only

    D.set_schur_backend("numpy")
    t0 = time.perf_counter()
    r1 = D.run_stage1(M, X0, Y0.T.copy())
    t1 = time.perf_counter()
    st = D.transition(r1.X, r1.Yt, M, tol_rel * e_scale)
    r2 = D.run_ipm(M, st, D.IpmParams(fixed_iters=CPU_IPM_SAMPLE, eps_tol=tol_rel * e_scale))
    t2 = time.perf_counter()
    per_it = (t2 - t1) / max(1, r2.iters)
    return r1.sweeps + ipm_iters, (t1 - t0) + per_it * ipm_iters, os.cpu_count()


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from oracle import driver as D
    from paper_2101_08431_b200 import data

    cfg = data.CONFIGS[WORKLOAD]
    M, X0, Y0, _, _ = data.make(cfg)
    e_scale = max(1.0, D.kkt_error_primal_only(X0, Y0.T.copy(), M))
    for _ in range(args.warmup):
        cpu_sample(M, X0, Y0, cfg.tol, e_scale)
    its, secs = 0, 0.0
    for _ in range(args.steps):
        i, s, cores = cpu_sample(M, X0, Y0, cfg.tol, e_scale)
        its, secs = its + i, secs + s
    value = its / secs
    sample = (f"{WORKLOAD}: full stage 1 + first {CPU_IPM_SAMPLE} IPM iterations per step, "
              f"IPM part extrapolated to {IPM_CAP} iterations (oracle port, numpy-backend Schur)")
    line = {"impl": "reference", "metric": _metric(), "value": value,
            "unit": "solver iterations/s (ANLS sweeps + IPM iterations)", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": _workload_desc(cfg)},
            "cpu_baseline": {"value": value, "unit": "solver iterations/s", "cores": cores,
                             "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "solver iterations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def _workload_desc(cfg):
    from paper_2101_08431_b200.config import IpmParams

    return (f"{cfg.name}: two-stage NMF solve, fp64 n={cfg.n} m={cfg.m} k={cfg.k} peak/logistic "
            f"generator, stage 1 to eps_STOL=1e-3 then IPM to relative KKT {cfg.tol:g} "
            f"(cap {IPM_CAP} IPM iterations, barrier={IpmParams().barrier})")


# ----------------------------------------------------------------------------
# B200 arm
# ----------------------------------------------------------------------------
def run_b200(args):
    import torch

    from paper_2101_08431_b200 import data, solver
    from paper_2101_08431_b200.config import IpmParams, Stage1Config

    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    cfg = data.CONFIGS[WORKLOAD]
    seed = cfg.seed + 1000 * rank  # weak scaling: one seeded replica per rank
    M, X0, Y0, _, _ = data.peaks(cfg.n, cfg.m, cfg.k, seed)
    P = solver.Problem(M, cfg.k)
    X0d, Yt0d = P.to_dev(X0), P.to_dev(Y0.T)
    e_scale = max(1.0, solver.kkt_error_primal_only_dev(P, X0d, Yt0d)[0])
    eps_abs = cfg.tol * e_scale
    timed_entry = args.roofline_entry
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2

    def step(use_graphs=True):
        X, Yt, pX, pY, r1 = solver.run_stage1(P, X0d, Yt0d, Stage1Config())
        X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, eps_abs)
        eng, r2 = solver.run_ipm(P, X, Yt, R, S, mu, rho,
                                 IpmParams(eps_tol=eps_abs, max_iter=IPM_CAP,
                                           use_graphs=use_graphs))
        return r1.sweeps, r2.iters, r2.converged, r2.trace[-1][2] if r2.trace else float("nan")

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    # instrument the dominant entry with CUDA events on the launching stream
    P.instrument = {timed_entry}
    P.event_log = []
    P.event_times = []
    if ws > 1:
        torch.distributed.barrier()
    clocks = Clocks(local)
    clocks.start()
    torch.cuda.synchronize()
    launches0 = P.lib.nmfb_launch_count() + P.graph_kernel_launches
    piters0 = P.persist_iters
    total_ms, sweeps, iters, conv, kkt = 0.0, 0, 0, True, 0.0
    stream = torch.cuda.current_stream()
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s, i, c, e = step()
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
        sweeps, iters, conv, kkt = sweeps + s, iters + i, conv and c, e
    torch.cuda.synchronize()
    launches = P.lib.nmfb_launch_count() + P.graph_kernel_launches - launches0
    piters = P.persist_iters - piters0
    clk = clocks.stop()
    if ws > 1:
        import torch.distributed as dist

        tt = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
        units = torch.tensor([sweeps + iters, sweeps, iters], device=dev, dtype=torch.float64)
        dist.all_reduce(units)
        tot_units, tot_sw, tot_it = (float(v) for v in units.tolist())
    else:
        tot_units, tot_sw, tot_it = float(sweeps + iters), float(sweeps), float(iters)
    kt = [a.elapsed_time(b) for a, b in P.event_log] + list(P.event_times)
    kt_note = "CUDA events around every launch of the entry inside the timed steps"
    if P.graph_timing_failed or not kt:
        # events inside replayed graphs were not timeable: re-run ONE step with graphs
        # off right after the timed region and time the entry's launches there
        P.event_log, P.event_times = [], []
        step(use_graphs=False)
        torch.cuda.synchronize()
        kt = [a.elapsed_time(b) for a, b in P.event_log]
        kt_note = ("CUDA events around the entry's launches in one extra step with graphs "
                   "disabled, right after the timed region (events inside replayed graphs "
                   "are not timeable)")
    P.instrument = set()
    value = tot_units / (total_ms / 1e3)
    # e2e through the public API with host inputs (H2D of M/X0/Y0, D2H of X, Y, R, S)
    from paper_2101_08431_b200 import run_two_stage

    Mh = torch.from_numpy(M).pin_memory()
    e2e_ms, e2e_units = 0.0, 0
    ne2e = max(1, min(args.steps, 3))
    # one untimed call first: the public API builds a fresh Problem per call, and the
    # first one after the timed region pays the caching allocator's cudaMalloc
    run_two_stage(Mh, X0, Y0, tol_rel=cfg.tol, ipm=IpmParams(max_iter=IPM_CAP), e_scale=e_scale)
    for _ in range(ne2e):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = run_two_stage(Mh, X0, Y0, tol_rel=cfg.tol, ipm=IpmParams(max_iter=IPM_CAP),
                            e_scale=e_scale)
        torch.cuda.synchronize()
        e2e_ms += 1e3 * (time.perf_counter() - t0)
        e2e_units += rep.stage1.sweeps + rep.ipm.iters
    aux5 = None
    if args.aux:
        try:  # the auxiliary configs never cost the headline line
            aux5 = aux_c5(dev, None, ws, rank)
        except Exception as exc:  # noqa: BLE001
            aux5 = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    h2d = M.nbytes + X0.nbytes + Y0.nbytes
    d2h = 2 * (cfg.n * cfg.k + cfg.m * cfg.k) * 8 + (cfg.n * cfg.k + cfg.m * cfg.k) * 8
    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0
    peaks, peak_src = _peaks()
    fp64_peak = measure_fp64_peak(dev)
    avg_ms = float(np.mean(kt)) if kt else float("nan")
    # nmfb_ipm_persist = one cooperative launch per inner loop (csrc/persist.cu); per
    # IPM iteration it touches M three times (quartic coefficients, residual/graX,
    # graY) plus O((n+m)k) vectors: algorithmic bytes per launch = that x iterations
    # per launch.  M stays in shared memory across the launch, so the DRAM traffic
    # (ncu) is ~one read of M per launch.
    per_it = 3 * cfg.n * cfg.m * 8 + 12 * (cfg.n + cfg.m) * cfg.k * 8
    it_per_launch = piters / max(len(kt), 1) if timed_entry == "nmfb_ipm_persist" else 1.0
    nbytes = per_it * it_per_launch
    achieved = nbytes / (avg_ms * 1e-3) / 1e9 if kt else None
    ncu = NCU_TRAFFIC.get(timed_entry)
    traffic = ncu["dram_bytes_per_iteration"] * it_per_launch if ncu else None
    line = {
        "metric": _metric(), "value": value,
        "unit": "solver iterations/s (ANLS sweeps + IPM iterations)",
        "n_gpus": ws, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (peak/logistic generator, PCG64 seed per rank)",
        "config": {"workload": _workload_desc(cfg), "parallelism": f"replicas x{ws}",
                   "l2": "M is L2-resident (2.4 MB); a 256 MB buffer is written between timed steps"},
        "anls_sweeps_per_s": tot_sw / (total_ms / 1e3),
        "ipm_iters_per_s": tot_it / (total_ms / 1e3),
        "time_to_tol_s": total_ms / 1e3 / args.steps,
        "converged": bool(conv), "final_kkt": kkt,
        "roofline": {"bound": "hbm",
                     "kernel": f"{timed_entry} (k_ipm_persist: the whole Gauss-Newton inner "
                               "loop in one cooperative launch)",
                     "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": (achieved / peaks["hbm_gbs"]) if achieved else None,
                     "traffic": traffic, "launches": len(kt), "avg_ms": avg_ms,
                     "iterations_per_launch": it_per_launch, "timing": kt_note,
                     "algorithmic_bytes": nbytes, "peak_source": peak_src,
                     "traffic_source": ncu["source"] if ncu else None,
                     "note": "latency-bound: c2's M (2.4 MB) is held in shared memory for the "
                             "whole launch, each iteration is a chain of 3 grid barriers (a 4th "
                             "only when Armijo backtracks past 7 halvings) and k^2-sized serial "
                             "solves; aux reports the HBM-bound c4 products"},
        "fp64_dgemm_tflops_measured": fp64_peak,
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": {"value": e2e_units / (e2e_ms / 1e3), "unit": "solver iterations/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_ms / ne2e},
    }
    if args.aux:
        try:
            line["aux"] = aux_c4(dev, peaks, peak_src)
        except Exception as exc:  # noqa: BLE001
            line["aux"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        line["aux_c5"] = aux5
    if ws == 1 and not args.no_cpu:
        try:
            gpu_ipm = int(round(tot_it / args.steps))
            its, secs, cores = cpu_sample(M, X0, Y0, cfg.tol, e_scale, ipm_iters=gpu_ipm)
            line["cpu_baseline"] = {"value": its / secs, "unit": "solver iterations/s",
                                    "cores": cores, "kind": "port",
                                    "sample": f"{WORKLOAD}: full stage 1 + first {CPU_IPM_SAMPLE} "
                                              f"IPM iterations, IPM part extrapolated to {gpu_ipm} "
                                              "(oracle port, numpy-backend Schur)"}
        except Exception as exc:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": f"{type(exc).__name__}: {exc}"[:300]}
    print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def measure_fp64_peak(dev):
    import torch

    a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    b = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2 * 8192 ** 3 / (best * 1e-3) / 1e12


def aux_c4(dev, peaks, peak_src):
    """c4 (dense 20000 x 5000, k=10) fixed ANLS sweeps: sweeps/s + product-kernel HBM roofline."""
    import torch

    from paper_2101_08431_b200 import data, solver
    from paper_2101_08431_b200.config import Stage1Config

    cfg = data.CONFIGS["c4"]
    M, X0, Y0, _, _ = data.dense(cfg.n, cfg.m, cfg.k, cfg.seed)
    P = solver.Problem(M, cfg.k)
    X0d, Yt0d = P.to_dev(X0), P.to_dev(Y0.T)
    solver.run_stage1(P, X0d, Yt0d, Stage1Config(fixed_sweeps=3))
    P.instrument = {"nmfb_rowprod"}
    P.event_log = []
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nsw = cfg.fixed_sweeps
    solver.run_stage1(P, X0d, Yt0d, Stage1Config(fixed_sweeps=nsw))
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    kt = [a.elapsed_time(b) for a, b in P.event_log]
    P.instrument = set()
    # rowprod over M (n x m) for ctb = M Y^T: algorithmic bytes = M + Y + out + tol
    big = [t for t in kt]
    avg = float(np.mean(big))
    nbytes = cfg.n * cfg.m * 8 + cfg.m * cfg.k * 8 + cfg.n * cfg.k * 8 + cfg.n * 8
    gbs = nbytes / (avg * 1e-3) / 1e9
    # stage 2 on the same instance: transition + the fixed 20 IPM iterations
    from paper_2101_08431_b200.config import IpmParams

    X, Yt, _, _, _ = solver.run_stage1(P, X0d, Yt0d, Stage1Config(fixed_sweeps=nsw))
    ipm_ms = []
    for _ in range(2):  # run 0 is the warm-up (first graph capture, engine buffers)
        Xc, Ytc, R, S, mu, rho = solver.transition(P, X, Yt, 1e-10)
        torch.cuda.synchronize()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record()
        eng, r2 = solver.run_ipm(P, Xc, Ytc, R, S, mu, rho, IpmParams(fixed_iters=cfg.fixed_ipm))
        e3.record()
        e3.synchronize()
        ipm_ms.append(e2.elapsed_time(e3))
    cold_ms, ipm_ms = ipm_ms
    # steady state: iterations 3.. of the measured run from the per-iteration wall times
    # (the first iterations of a run include the CUDA-graph captures, 1-2 per F buffer)
    tr = [t[0] for t in r2.trace]
    steady_ms = (1e3 * (tr[-1] - tr[2]) / (len(tr) - 3)) if len(tr) > 4 else None
    return {"workload": f"c4: {nsw} ANLS sweeps + {cfg.fixed_ipm} IPM iterations, dense fp64 "
                        f"n={cfg.n} m={cfg.m} k={cfg.k} (CPU reference: IPM infeasible, "
                        "~15 h/iteration per SURVEY.md section 6)",
            "anls_sweeps_per_s": nsw / (ms / 1e3), "ms_per_sweep": ms / nsw,
            "ipm_iters_per_s": r2.iters / (ipm_ms / 1e3), "ms_per_ipm_iter": ipm_ms / r2.iters,
            "ms_per_ipm_iter_first_run": cold_ms / r2.iters,
            "ms_per_ipm_iter_steady": steady_ms,
            "roofline": {"bound": "hbm", "kernel": "nmfb_rowprod (ctb = M Y^T, X-update)",
                         "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / peaks["hbm_gbs"], "traffic": None,
                         "algorithmic_bytes": nbytes, "avg_ms": avg, "peak_source": peak_src}}


def aux_c5(dev, peaks, ws, rank):
    """c5 (200000 x 40000 fp32 M, k=16): 30 ANLS sweeps, rows sharded over the ranks."""
    import torch

    from paper_2101_08431_b200 import data, solver
    from paper_2101_08431_b200.config import Stage1Config
    from paper_2101_08431_b200.dist import Comm, row_range

    cfg = data.CONFIGS["c5"]
    comm = Comm.from_env()
    a, b = row_range(cfg.n, ws, rank)
    M, X0, Y0 = data.dense_device(cfg.n, cfg.m, cfg.k, cfg.seed, dev, torch.float32, rows=(a, b))
    P = solver.Problem(M, cfg.k, comm=comm)
    del M
    X0d, Yt0d = P.to_dev(X0), P.to_dev(Y0.T)
    solver.run_stage1(P, X0d, Yt0d, Stage1Config(fixed_sweeps=1))
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, _, _, _, r1 = solver.run_stage1(P, X0d, Yt0d, Stage1Config(fixed_sweeps=cfg.fixed_sweeps))
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    per_sweep_bytes = 2 * cfg.n * cfg.m * 4  # two passes over fp32 M per sweep
    gbs = per_sweep_bytes * cfg.fixed_sweeps / (ms * 1e-3) / 1e9
    out = {"workload": f"c5 ANLS: {cfg.fixed_sweeps} sweeps, fp32 M {cfg.n} x {cfg.m}, k={cfg.k}, "
                       f"rows sharded over {ws} GPU(s) (strong scaling)",
           "anls_sweeps_per_s": cfg.fixed_sweeps / (ms / 1e3), "ms_per_sweep": ms / cfg.fixed_sweeps,
           "stream_gbs_whole_job": gbs, "objective": r1.trace[-1][1]}
    del P
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--roofline-entry", default="nmfb_ipm_persist")
    ap.add_argument("--no-aux", dest="aux", action="store_false")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
