"""Config c3 end to end: streaming column append (chunks of 10 from m=20 to 500).

python scripts/run_stream.py [--ipm N] [--barrier paper|balanced] [--oracle-chunks C]
Prints per-chunk times and the total; --oracle-chunks times the CPU oracle session on
the first C chunks for comparison.
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data  # noqa: E402
from paper_2101_08431_b200.config import IpmParams  # noqa: E402
from paper_2101_08431_b200.stream import StreamSession  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ipm", type=int, default=0, help="fixed IPM iterations per chunk (0: to tol/cap)")
    ap.add_argument("--barrier", default="balanced")
    ap.add_argument("--cap", type=int, default=500, help="IPM iteration cap per chunk")
    ap.add_argument("--hessian", default="inertia")
    ap.add_argument("--oracle-chunks", type=int, default=0)
    a = ap.parse_args()
    cfg = data.CONFIGS["c3"]
    M, X0, Y0, _, _ = data.make(cfg)
    mk = (lambda: IpmParams(fixed_iters=a.ipm, barrier=a.barrier, hessian=a.hessian)) if a.ipm else \
        (lambda: IpmParams(barrier=a.barrier, max_iter=a.cap, hessian=a.hessian))
    # warm-up (module load, graph capture paths)
    StreamSession(M[:, :cfg.m_start], X0, Y0[:, :cfg.m_start], ipm_factory=mk)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = StreamSession(M[:, :cfg.m_start], X0, Y0[:, :cfg.m_start], ipm_factory=mk)
    err = None
    for m0 in range(cfg.m_start, cfg.m, cfg.m_step):
        try:
            s.append(M[:, m0:m0 + cfg.m_step])
        except Exception as e:  # record where the session stopped
            err = f"m={m0 + cfg.m_step}: {type(e).__name__}: {e}"
            break
    torch.cuda.synchronize()
    total = time.perf_counter() - t0
    chunks = [{"m": c[0], "s": round(c[1], 5), "sweeps": c[2].stage1.sweeps,
               "ipm": c[2].ipm.iters if c[2].ipm else 0, "E": c[2].final_kkt_error,
               "status": c[2].status,
               "dense_fallbacks": c[2].ipm.dense_fallbacks if c[2].ipm else 0} for c in s.chunks]
    out = {"config": "c3", "chunks": len(chunks), "total_s": total,
           "mean_chunk_ms": 1e3 * total / len(chunks), "error": err,
           "per_chunk": chunks}
    if a.oracle_chunks:
        from oracle import driver as D
        from oracle import stream as OS

        D.set_schur_backend("numpy")
        mko = (lambda: D.IpmParams(fixed_iters=a.ipm, barrier=a.barrier)) if a.ipm else \
            (lambda: D.IpmParams(barrier=a.barrier))
        t0 = time.perf_counter()
        so = OS.OracleStream(M[:, :cfg.m_start], X0, Y0[:, :cfg.m_start], ipm_factory=mko)
        for c in range(a.oracle_chunks - 1):
            m0 = cfg.m_start + c * cfg.m_step
            so.append(M[:, m0:m0 + cfg.m_step])
        out["oracle_first_chunks"] = a.oracle_chunks
        out["oracle_s"] = time.perf_counter() - t0
        out["gpu_first_chunks_s"] = sum(c[1] for c in s.chunks[:a.oracle_chunks])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
