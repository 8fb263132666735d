"""One launch of each tcgen05 fp32 product at 50000 x 40000 x 16 (ncu target).

python scripts/tc_one.py [n m k]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import solver  # noqa: E402


def main():
    n, m, k = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (50000, 40000, 16)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    M = torch.rand((n, m), generator=g, device=dev, dtype=torch.float32)
    P = solver.Problem(M, k)
    Yt = torch.rand((m, k), generator=g, device=dev, dtype=torch.float64)
    X = torch.rand((n, k), generator=g, device=dev, dtype=torch.float64)
    r, c = P.buf(n, k), P.buf(m, k)
    P.rowprod(P.M, n, m, Yt, k, r, None, 1)
    P.colprod(P.M, n, m, X, k, c, None, 1)
    torch.cuda.synchronize()
    print("ok", float(r.sum()), float(c.sum()))


if __name__ == "__main__":
    main()
