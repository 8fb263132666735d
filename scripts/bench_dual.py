"""Time the one-pass dual product against rowprod + colprod (c4 / c5 shapes), CUDA events.

python scripts/bench_dual.py [n m k dtype]
"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import solver  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    n, m, k = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (20000, 5000, 10)
    dt = torch.float32 if len(sys.argv) > 4 and sys.argv[4] == "f32" else torch.float64
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    M = torch.rand((n, m), generator=g, device="cuda", dtype=torch.float64).to(dt)
    P = solver.Problem(M, k)
    B1 = torch.rand((m, k), generator=g, device="cuda", dtype=torch.float64)
    B2 = torch.rand((n, k), generator=g, device="cuda", dtype=torch.float64)
    oR, oC = P.buf(n, k), P.buf(m, k)
    work = P.buf(P.lib.nmfb_dualprod_work_len(n, m, k))
    us_dual = timeit(lambda: P.dualprod(B1, B2, oR, oC, work))
    us_row = timeit(lambda: P.rowprod(P.M, n, m, B1, k, oR, None, P.f32))
    us_col = timeit(lambda: P.colprod(P.M, n, m, B2, k, oC, None, P.f32))
    gb = n * m * M.element_size() / 1e9
    print(f"{n}x{m} k={k} {dt}: dual {us_dual:.1f} us ({gb / us_dual * 1e6:.0f} GB/s), "
          f"rowprod {us_row:.1f} + colprod {us_col:.1f} = {us_row + us_col:.1f} us "
          f"[variant {os.environ.get('NMFB_DUAL_VARIANT', '1')}]", flush=True)


if __name__ == "__main__":
    main()
