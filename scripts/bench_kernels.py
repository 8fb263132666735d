"""Isolated timings (CUDA events) of the stage-1 kernels at c4 / c5 shapes.

python scripts/bench_kernels.py [c4|c5]
"""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import solver  # noqa: E402

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6449.1


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


def main(name):
    n, m, k, dt = {"c4": (20000, 5000, 10, torch.float64), "c5": (200000, 40000, 16, torch.float32),
                   "c5h": (50000, 40000, 16, torch.float32)}[name]
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    M = torch.rand((n, m), generator=g, device=dev, dtype=dt)
    P = solver.Problem(M, k)
    s = M.element_size()
    X = torch.rand((n, k), generator=g, device=dev, dtype=torch.float64)
    Yt = torch.rand((m, k), generator=g, device=dev, dtype=torch.float64)
    ctbX, tolX = P.buf(n, k), P.buf(n)
    ctbY, tolY = P.buf(m, k), P.buf(m)
    out = {}
    t = timeit(lambda: P.rowprod(P.M, n, m, Yt, k, ctbX, tolX, P.f32))
    b = n * m * s + (n + m) * k * 8 + n * 8
    out["rowprod"] = dict(ms=t, GBs=b / t / 1e6, frac=b / t / 1e6 / PEAK)
    t = timeit(lambda: P.colprod(P.M, n, m, X, k, ctbY, tolY, P.f32))
    out["colprod"] = dict(ms=t, GBs=b / t / 1e6, frac=b / t / 1e6 / PEAK)
    # NNLS (mode 2 with all-passive seeds, the steady state on dense data)
    GY, GX = P.buf(k, k), P.buf(k, k)
    P.colprod(Yt, m, k, Yt, k, GY)
    P.colprod(X, n, k, X, k, GX)
    seeds = torch.ones((n, k), dtype=torch.uint8, device=dev)
    x, p = P.buf(n, k), P.buf(n, k, dtype=torch.uint8)
    ch, r2, st = P.buf(n, dtype=torch.int64), P.buf(n), P.buf(n, dtype=torch.int8)
    _p = solver._p

    def nnls(mode):
        P._call("nmfb_surface_nnls_batch", _p(GY), _p(ctbX), _p(P.row_n2), _p(seeds), mode, _p(tolX),
                3 * k, n, k, _p(x), _p(p), _p(ch), _p(r2), _p(st), None, None, P.stream)
    out["nnls_warm_rows"] = dict(ms=timeit(lambda: nnls(2)), rhs=n)
    out["nnls_cold_rows"] = dict(ms=timeit(lambda: nnls(0), reps=3), rhs=n)
    print(json.dumps({"config": name, "n": n, "m": m, "k": k, "dtype": str(dt), **out}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c4")
