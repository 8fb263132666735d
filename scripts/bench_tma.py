"""TMA-fed fp64 products (csrc/tma_prod.cu) vs the register-direct DMMA kernels:
correctness (row product bit-identical, column product vs torch fp64) and CUDA-event
timings with the HBM fraction.

python scripts/bench_tma.py
"""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import solver  # noqa: E402

PEAK = (json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
        if os.path.exists("MEASURED_PEAKS.json") else 6549.4)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    shapes = ((20000, 5000, 10), (20000, 5000, 16), (20000, 5000, 8), (4100, 2050, 7),
              (8000, 3000, 5), (40000, 10000, 10))
    if len(sys.argv) > 1:  # "c4": only the c4 shape (ncu captures)
        shapes = shapes[:1]
    for n, m, k in shapes:
        M = torch.rand((n, m), generator=g, device=dev, dtype=torch.float64)
        P = solver.Problem(M, k)
        X = torch.rand((n, k), generator=g, device=dev, dtype=torch.float64)
        Yt = torch.rand((m, k), generator=g, device=dev, dtype=torch.float64)
        res = {"shape": [n, m, k]}
        outs = {}
        for on in (1, 0):
            P.lib.nmfb_tma_products(on)
            r, c = P.buf(n, k), P.buf(m, k)
            P.rowprod(P.M, n, m, Yt, k, r, None, 0)
            P.colprod(P.M, n, m, X, k, c, None, 0)
            torch.cuda.synchronize()
            outs[on] = (r.clone(), c.clone())
            b = n * m * 8 + (n + m) * k * 8
            tr = timeit(lambda: P.rowprod(P.M, n, m, Yt, k, r, None, 0))
            tc = timeit(lambda: P.colprod(P.M, n, m, X, k, c, None, 0))
            dw = torch.empty(P.lib.nmfb_dualprod_work_len(n, m, k), dtype=torch.float64,
                             device=dev)
            dr, dc = P.buf(n, k), P.buf(m, k)
            P.dualprod(Yt, X, dr, dc, dw)
            torch.cuda.synchronize()
            outs[("dual", on)] = (dr.clone(), dc.clone())
            td = timeit(lambda: P.dualprod(Yt, X, dr, dc, dw))
            res["tma" if on else "old"] = {"row_ms": tr, "row_frac": b / tr / 1e6 / PEAK,
                                           "col_ms": tc, "col_frac": b / tc / 1e6 / PEAK,
                                           "dual_ms": td, "dual_frac": b / td / 1e6 / PEAK}
        P.lib.nmfb_tma_products(1)
        rr, cr = M @ Yt, M.t() @ X
        res["row_bit_identical"] = bool(torch.equal(outs[1][0], outs[0][0]))
        res["row_relerr"] = float(((outs[1][0] - rr).abs().max() / rr.abs().max()).item())
        res["col_relerr"] = float(((outs[1][1] - cr).abs().max() / cr.abs().max()).item())
        for on in (1, 0):
            dr, dc = outs[("dual", on)]
            res[f"dual_relerr_{on}"] = max(float(((dr - rr).abs().max() / rr.abs().max()).item()),
                                           float(((dc - cr).abs().max() / cr.abs().max()).item()))
        res["col_relerr_old"] = float(((outs[0][1] - cr).abs().max() / cr.abs().max()).item())
        print(json.dumps(res), flush=True)
        del M, P


if __name__ == "__main__":
    main()
