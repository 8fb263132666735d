"""Dense Schur-system kernels (full-Hessian coupling and the rank-k^2 fallback):
nmfb_dense_cholesky (single-CTA blocked N <= 128, cooperative above) and
nmfb_dense_solve (single-CTA N <= 640, cooperative above) against NumPy on SPD
matrices of the Schur sizes c1-c3 produce (mk = 150 ... 2000), plus the
failing-pivot report on an indefinite matrix."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2101_08431_b200 import _lib

    return _lib.load()


@pytest.mark.parametrize("N", [100, 130, 150, 300, 352, 641, 1000, 1760, 2000, 4096])
def test_dense_cholesky_and_solve(lib, N):
    import torch

    rng = np.random.default_rng(N)
    B = rng.standard_normal((N, N))
    A = B @ B.T / N + np.eye(N)
    d = torch.as_tensor(A).cuda()
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert lib.nmfb_dense_cholesky(d.data_ptr(), N, info.data_ptr(), s) == 0
    L = d.cpu().numpy()
    assert int(info.item()) == -1
    assert np.abs(np.triu(L, 1)).max() == 0.0
    assert np.abs(L @ L.T - A).max() / np.abs(A).max() < 1e-14
    rhs = rng.standard_normal(N)
    x = torch.as_tensor(rhs).cuda()
    assert lib.nmfb_dense_solve(d.data_ptr(), N, x.data_ptr(), s) == 0
    xr = np.linalg.solve(A, rhs)
    assert np.abs(x.cpu().numpy() - xr).max() / np.abs(xr).max() < 1e-12


@pytest.mark.parametrize("N", [130, 300, 999, 1760, 2000])
def test_dense_cholesky_rhs_and_modes(lib, N):
    """The factorization with the right-hand side riding along (b <- L^{-1} b in the same
    launch, csrc/dense_flow.cuh; odd N takes the fallback), the backward half, and the
    three modes of the solve with an existing factor, against NumPy; run twice (the flags
    and solution buffers are re-armed per launch) and bit-reproducible."""
    import scipy.linalg as sla
    import torch

    rng = np.random.default_rng(N + 1)
    B = rng.standard_normal((N, N))
    A = B @ B.T / N + np.eye(N)
    rhs = rng.standard_normal(N)
    Lr = np.linalg.cholesky(A)
    zr = sla.solve_triangular(Lr, rhs, lower=True)
    xr = sla.solve_triangular(Lr.T, zr, lower=False)
    s = torch.cuda.current_stream().cuda_stream
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    outs = []
    for _ in range(2):
        d = torch.as_tensor(A).cuda()
        b = torch.as_tensor(rhs).cuda()
        assert lib.nmfb_dense_cholesky_rhs(d.data_ptr(), N, b.data_ptr(), info.data_ptr(), s) == 0
        z = b.cpu().numpy().copy()
        assert int(info.item()) == -1
        L = d.cpu().numpy()
        assert np.abs(np.triu(L, 1)).max() == 0.0
        assert np.abs(L - Lr).max() / np.abs(Lr).max() < 1e-13
        assert np.abs(z - zr).max() / np.abs(zr).max() < 1e-12
        assert lib.nmfb_dense_solve_back(d.data_ptr(), N, b.data_ptr(), s) == 0
        x = b.cpu().numpy().copy()
        assert np.abs(x - xr).max() / np.abs(xr).max() < 1e-12
        outs.append((L, z, x))
    for a, c in zip(outs[0], outs[1]):
        assert np.array_equal(a, c)
    for mode, want in ((1, zr), (3, xr)):
        b = torch.as_tensor(rhs).cuda()
        assert lib.nmfb_dense_solve_mode(d.data_ptr(), N, b.data_ptr(), mode, s) == 0
        assert np.abs(b.cpu().numpy() - want).max() / np.abs(want).max() < 1e-12
    b = torch.as_tensor(zr).cuda()
    assert lib.nmfb_dense_solve_mode(d.data_ptr(), N, b.data_ptr(), 2, s) == 0
    assert np.abs(b.cpu().numpy() - xr).max() / np.abs(xr).max() < 1e-12


@pytest.mark.parametrize("N", [120, 700, 1760])
def test_dense_cholesky_reports_failing_pivot(lib, N):
    import torch

    rng = np.random.default_rng(7)
    B = rng.standard_normal((N, N))
    A = B @ B.T / N + np.eye(N)
    A[N // 2, N // 2] = -5.0  # not positive definite from this pivot on
    d = torch.as_tensor(A).cuda()
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert lib.nmfb_dense_cholesky(d.data_ptr(), N, info.data_ptr(), s) == 0
    torch.cuda.synchronize()
    assert 0 <= int(info.item()) <= N // 2
    # and the same through the fused entry (the solve still terminates on the failed factor)
    d = torch.as_tensor(A).cuda()
    b = torch.ones(N, dtype=torch.float64, device="cuda")
    assert lib.nmfb_dense_cholesky_rhs(d.data_ptr(), N, b.data_ptr(), info.data_ptr(), s) == 0
    assert lib.nmfb_dense_solve_back(d.data_ptr(), N, b.data_ptr(), s) == 0
    torch.cuda.synchronize()
    assert 0 <= int(info.item()) <= N // 2


def test_first_failure_word(lib):
    """nmfb_first_failure_i8 keeps the earliest (tag, index) failure and its status code
    across several batches (the fixed-sweep stage-1 failure report)."""
    import torch

    s = torch.cuda.current_stream().cuda_stream
    acc = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    st = torch.zeros(5000, dtype=torch.int8, device="cuda")
    assert lib.nmfb_first_failure_i8(st.data_ptr(), 5000, 0, acc.data_ptr(), s) == 0
    assert int(acc.item()) == -1  # nothing failed
    st[4000] = 2
    st[1234] = 1
    assert lib.nmfb_first_failure_i8(st.data_ptr(), 5000, 7, acc.data_ptr(), s) == 0
    st2 = torch.zeros(300, dtype=torch.int8, device="cuda")
    st2[299] = 2
    assert lib.nmfb_first_failure_i8(st2.data_ptr(), 300, 9, acc.data_ptr(), s) == 0
    w = int(acc.item()) & ((1 << 64) - 1)
    assert (w >> 40, (w >> 8) & 0xFFFFFFFF, w & 0xFF) == (7, 1234, 1)
    st3 = torch.zeros(10, dtype=torch.int8, device="cuda")
    st3[3] = 2
    assert lib.nmfb_first_failure_i8(st3.data_ptr(), 10, 2, acc.data_ptr(), s) == 0
    w = int(acc.item()) & ((1 << 64) - 1)
    assert (w >> 40, (w >> 8) & 0xFFFFFFFF, w & 0xFF) == (2, 3, 2)
