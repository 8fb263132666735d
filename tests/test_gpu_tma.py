"""TMA-fed fp64 streaming products (csrc/tma_prod.cu) through the C-ABI.

M Y^T (row product) and M^T X (column product) against torch fp64 at ragged shapes
(rows not a multiple of the 128-row band / 32-row box, columns not a multiple of the
512-column chunk or the 16-column box), every k the TMA path takes (5..16, with the
DFMA tail for k = 9..12); for k outside 9..12 the row product is bit-identical to the
register-direct DMMA kernel (same accumulation order).  Also the regression for
kernels launched at two shared-memory sizes in one process (nmfb_smem_attr).
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(4100, 2050, k) for k in (5, 7, 8, 9, 10, 11, 12, 13, 16)] + [
    (20000, 5000, 10), (6000, 4096, 16), (4097, 3333 + 1, 10)]


@pytest.mark.parametrize("n,m,k", SHAPES)
def test_tma_products_match_fp64(n, m, k):
    from paper_2101_08431_b200 import solver

    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(n + m + k)
    M = torch.rand((n, m), generator=g, device=dev, dtype=torch.float64)
    P = solver.Problem(M, k)
    X = torch.rand((n, k), generator=g, device=dev, dtype=torch.float64)
    Yt = torch.rand((m, k), generator=g, device=dev, dtype=torch.float64)
    res = {}
    for on in (1, 0):
        prev = P.lib.nmfb_tma_products(on)
        r, c, tol = P.buf(n, k), P.buf(m, k), P.buf(n)
        P.rowprod(P.M, n, m, Yt, k, r, tol, 0)
        P.colprod(P.M, n, m, X, k, c, None, 0)
        torch.cuda.synchronize()
        res[on] = (r, c, tol)
        P.lib.nmfb_tma_products(prev)
    rr, cr = M @ Yt, M.t() @ X
    for on in (1, 0):
        r, c, tol = res[on]
        assert ((r - rr).abs().max() / rr.abs().max()).item() < 1e-13
        assert ((c - cr).abs().max() / cr.abs().max()).item() < 1e-13
        # per-row tolerance 1e-12 max(1, ||ctb_i||_inf), fused in the sum
        assert torch.allclose(tol, 1e-12 * torch.clamp(r.abs().max(1).values, min=1.0),
                              rtol=1e-15, atol=0)
    if not 9 <= k <= 12:
        assert torch.equal(res[1][0], res[0][0]), "TMA row product not bit-identical"
    # one-pass dual product (IPM: M dY^T and M^T dX together)
    dw = torch.empty(P.lib.nmfb_dualprod_work_len(n, m, k), dtype=torch.float64, device=dev)
    dr, dc = P.buf(n, k), P.buf(m, k)
    P.dualprod(Yt, X, dr, dc, dw)
    torch.cuda.synchronize()
    assert ((dr - rr).abs().max() / rr.abs().max()).item() < 1e-13
    assert ((dc - cr).abs().max() / cr.abs().max()).item() < 1e-13


def test_smem_attribute_across_problem_sizes():
    """A kernel first launched with a small dynamic shared-memory size, then with a larger
    one (k = 3 then k = 16 low-rank solves): the second launch must not fail (the attribute
    is a per-kernel cap)."""
    from paper_2101_08431_b200 import data, solver
    from paper_2101_08431_b200.config import IpmParams

    for n, m, k in ((400, 40, 3), (900, 60, 16)):
        M, X0, Y0 = data.dense(n, m, k, 7)[:3]
        P = solver.Problem(M, k)
        X, Yt, *_ = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T))
        X, Yt, R, S, mu, rho = solver.transition(P, X, Yt, 1e-9)
        _, r = solver.run_ipm(P, X, Yt, R, S, mu, rho,
                              IpmParams(fixed_iters=3, schur_solver="lowrank", persistent=False,
                                        fused_small=False))
        assert r.iters == 3


@pytest.mark.parametrize("n,m,k", [(4100, 2052, 10), (8192, 4096, 16), (5000, 3000, 5)])
def test_tcgen05_products_fp32(n, m, k):
    """fp32 M (config c5 storage): the tcgen05 tf32 x 3 row product (csrc/tc_prod.cu) against
    fp64 torch -- relative error ~2e-6 (tf32 split ~2^-21 per term, fp32 tensor-core
    accumulation flushed to fp64 every 128 columns); bound 1e-5."""
    from paper_2101_08431_b200 import solver

    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(n * k)
    M = torch.rand((n, m), generator=g, device=dev, dtype=torch.float32)
    P = solver.Problem(M, k)
    Yt = torch.rand((m, k), generator=g, device=dev, dtype=torch.float64)
    X = torch.rand((n, k), generator=g, device=dev, dtype=torch.float64)
    assert P.lib.nmfb_tc_products(-1) == 1
    r, c = P.buf(n, k), P.buf(m, k)
    P.rowprod(P.M, n, m, Yt, k, r, None, 1)
    P.colprod(P.M, n, m, X, k, c, None, 1)  # k_colprod_tc (A = Mh / Ml from tensor memory)
    torch.cuda.synchronize()
    rr, cr = M.double() @ Yt, M.double().t() @ X
    assert ((r - rr).abs().max() / rr.abs().max()).item() < 1e-5
    assert ((c - cr).abs().max() / cr.abs().max()).item() < 1e-5
