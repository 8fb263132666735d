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


@pytest.mark.parametrize("N", [100, 150, 300, 641, 1000, 2000])
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


@pytest.mark.parametrize("N", [120, 700])
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
