"""Histogram of active-set changes per right-hand side in the c4 stage-1 NNLS batches
(X side 20000 rows, Y side 5000 columns) at a few sweeps, and the time of each batch:
is the batch time set by a few long Lawson-Hanson chains?

python scripts/nnls_changes.py
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402

_p = solver._p


def main():
    cfg = data.CONFIGS["c4"]
    M, X0, Y0, _, _ = data.make(cfg)
    P = solver.Problem(M, cfg.k)
    n, m, k = P.n, P.m, P.k
    for sweeps in (1, 2, 5, 20, 49):
        X, Yt, pX, pY, _ = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T),
                                             solver.Stage1Config(fixed_sweeps=sweeps))
        for side, (A_rows, C, B, btb, seeds, cnt) in {
                "X": (n, Yt, None, P.row_n2, pX, n), "Y": (m, X, None, P.col_n2, pY, m)}.items():
            G = P.buf(k, k)
            P.colprod(C, C.shape[0], k, C, k, G)
            ctb, tol = P.buf(cnt, k), P.buf(cnt)
            if side == "X":
                P.rowprod(P.M, n, m, Yt, k, ctb, tol, 0)
            else:
                P.colprod(P.M, n, m, X, k, ctb, tol, 0)
            x, pn = P.buf(cnt, k), torch.empty_like(seeds)
            ch, r2 = P.buf(cnt, dtype=torch.int64), P.buf(cnt)
            st = P.buf(cnt, dtype=torch.int8)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for rep in range(2):
                e0.record()
                P._call("nmfb_nnls_batch_ws", _p(G), _p(ctb), _p(btb), _p(seeds), 2, _p(tol),
                        3 * k, cnt, k, _p(x), _p(pn), _p(ch), _p(r2), _p(st), None, None,
                        _p(P.ftab), P.ftab_len, P.stream)
                e1.record()
            torch.cuda.synchronize()
            c = ch.cpu().numpy()
            h = np.bincount(c)
            print(f"sweep {sweeps:2d} {side}: {e0.elapsed_time(e1) * 1e3:7.1f} us  changes: "
                  f"max {c.max()} mean {c.mean():.3f} hist {h.tolist()[:16]}", flush=True)


if __name__ == "__main__":
    main()
