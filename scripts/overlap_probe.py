"""Does the batched NNLS (k_nnls_tab, latency-bound) overlap with a TMA streaming product
on a second stream?  c4 shapes: rowprod / colprod of the 800 MB M and an NNLS batch of
20000 (X side) or 5000 (Y side) right-hand sides, alone and concurrently.

python scripts/overlap_probe.py
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402

_p = solver._p


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfg = data.CONFIGS["c4"]
    M, X0, Y0, _, _ = data.make(cfg)
    P = solver.Problem(M, cfg.k)
    n, m, k = P.n, P.m, P.k
    X, Yt, pX, pY, r1 = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T),
                                          solver.Stage1Config(fixed_sweeps=5))
    GY = P.buf(k, k)
    P.colprod(Yt, m, k, Yt, k, GY)
    ctb, tol = P.buf(n, k), P.buf(n)
    P.rowprod(P.M, n, m, Yt, k, ctb, tol, 0)
    Xn, pXn = P.buf(n, k), torch.empty_like(pX)
    ch, r2 = P.buf(n, dtype=torch.int64), P.buf(n)
    st = P.buf(n, dtype=torch.int8)
    out, tol2 = P.buf(n, k), P.buf(n)
    side = torch.cuda.Stream()

    def prod():
        P.rowprod(P.M, n, m, Yt, k, out, tol2, 0)

    def nnls():
        P._call("nnls" and "nmfb_nnls_batch_ws", _p(GY), _p(ctb), _p(P.row_n2), _p(pX), 2,
                _p(tol), 3 * k, n, k, _p(Xn), _p(pXn), _p(ch), _p(r2), _p(st), None, None,
                _p(P.ftab), P.ftab_len, P.stream)

    def both():
        ev = torch.cuda.Event()
        ev.record()
        side.wait_event(ev)
        with torch.cuda.stream(side):
            nnls()
        prod()
        ev2 = torch.cuda.Event()
        ev2.record(side)
        torch.cuda.current_stream().wait_event(ev2)

    for name, fn in (("rowprod", prod), ("nnls_x", nnls), ("concurrent", both)):
        print(f"{name:12s} {1e3 * timed(fn):8.1f} us", flush=True)


if __name__ == "__main__":
    main()
