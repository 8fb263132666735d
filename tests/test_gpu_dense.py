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
