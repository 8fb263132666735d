"""Time and check nmfb_dense_cholesky on random SPD matrices of the Schur sizes."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import _lib  # noqa: E402

lib = _lib.load()
for N in (100, 160, 256, 300, 352, 800, 2000):
    rng = np.random.default_rng(N)
    B = rng.standard_normal((N, N))
    A = B @ B.T / N + np.eye(N)
    d = torch.as_tensor(A).cuda()
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ts = []
    for rep in range(5):
        w = d.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = lib.nmfb_dense_cholesky(w.data_ptr(), N, info.data_ptr(), s)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    L = w.cpu().numpy()
    err = np.abs(L @ L.T - A).max() / np.abs(A).max()
    upper = np.abs(np.triu(L, 1)).max()
    rhs = torch.as_tensor(rng.standard_normal(N)).cuda()
    tss = []
    for rep in range(5):
        x = rhs.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.nmfb_dense_solve(w.data_ptr(), N, x.data_ptr(), s)
        e1.record()
        e1.synchronize()
        tss.append(e0.elapsed_time(e1) * 1e3)
    xs = np.linalg.solve(A, rhs.cpu().numpy())
    serr = np.abs(x.cpu().numpy() - xs).max() / np.abs(xs).max()
    print(f"N={N:5d}: chol {min(ts):8.1f} us  rc={rc} info={int(info.item())} relerr {err:.2e} "
          f"upper {upper:.1e} | solve (fwd+back) {min(tss):8.1f} us relerr {serr:.2e}", flush=True)
