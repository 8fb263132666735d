"""tcgen05 tf32x3 products for an fp32 M (csrc/tc_prod.cu) vs the FP64 DMMA kernels:
accuracy against fp64 torch and CUDA-event timings with the HBM fraction.

python scripts/bench_tc.py [small]
"""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import solver  # noqa: E402

PEAK = (json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
        if os.path.exists("MEASURED_PEAKS.json") else 6549.4)


def timeit(fn, reps=10):
    for _ in range(2):
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
    shapes = [(4100, 2052, 10), (20000, 5000, 16), (8192, 4096, 5), (50000, 40000, 16)]
    if len(sys.argv) > 1 and sys.argv[1] == "small":
        shapes = shapes[:3]
    if len(sys.argv) > 1 and sys.argv[1] == "c5":
        shapes = [(200000, 40000, 16)]
    for n, m, k in shapes:
        M = torch.rand((n, m), generator=g, device=dev, dtype=torch.float32)
        P = solver.Problem(M, k)
        Yt = torch.rand((m, k), generator=g, device=dev, dtype=torch.float64)
        X = torch.rand((n, k), generator=g, device=dev, dtype=torch.float64)
        res = {"shape": [n, m, k]}
        outs = {}
        for on in (1, 0):
            P.lib.nmfb_tc_products(on)
            r, c = P.buf(n, k), P.buf(m, k)
            P.rowprod(P.M, n, m, Yt, k, r, None, 1)
            P.colprod(P.M, n, m, X, k, c, None, 1)
            torch.cuda.synchronize()
            outs[on] = (r.clone(), c.clone())
            b = n * m * 4 + (n + m) * k * 8
            tr = timeit(lambda: P.rowprod(P.M, n, m, Yt, k, r, None, 1))
            tc = timeit(lambda: P.colprod(P.M, n, m, X, k, c, None, 1))
            res["tc" if on else "dmma"] = {"row_ms": tr, "row_frac": b / tr / 1e6 / PEAK,
                                           "col_ms": tc, "col_frac": b / tc / 1e6 / PEAK}
        P.lib.nmfb_tc_products(1)
        if n * m <= 4e8:
            Md = M.double()
            rr, cr = Md @ Yt, Md.t() @ X
            for on in (1, 0):
                r, c = outs[on]
                res[f"row_relerr_{on}"] = float(((r - rr).abs().max() / rr.abs().max()).item())
                res[f"col_relerr_{on}"] = float(((c - cr).abs().max() / cr.abs().max()).item())
        else:
            r1, r0 = outs[1][0], outs[0][0]
            res["row_rel_vs_dmma"] = float(((r1 - r0).abs().max() / r0.abs().max()).item())
        print(json.dumps(res), flush=True)
        del M, P
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
