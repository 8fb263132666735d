"""Time and check nmfb_lowrank_factor (unpack, chol(G), T1 = Zb LG, H = I - LG^T T1, chol(H))."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import _lib  # noqa: E402


def packed_index(k):
    idx = {}
    e = 0
    for a in range(k):
        for b in range(a, k):
            idx[(a, b)] = idx[(b, a)] = e
            e += 1
    return idx


def run(k, reps=20):
    rng = np.random.default_rng(k)
    KK, Q = k * (k + 1) // 2, k * k
    pk = packed_index(k)
    # G = sum_j (y y^T) (x) Dinv_j  (SPD), Z small symmetric -> H = I - LG^T Zb LG PD
    m = 4 * Q
    Gf = np.zeros((Q, Q))
    for _ in range(m):
        y = rng.uniform(0.1, 1, k)
        B = rng.standard_normal((k, k))
        D = B @ B.T + k * np.eye(k)
        Gf += np.kron(np.outer(y, y), np.linalg.inv(D))
    Zf = rng.standard_normal((Q, Q)) * 1e-3
    Zf = Zf @ Zf.T
    # packed storage [ab * KK + pq] for the (a,p),(b,q) entry
    Gpk = np.zeros(KK * KK)
    Zpk = np.zeros(KK * KK)
    for r in range(Q):
        for c in range(Q):
            a, p, b, q = r // k, r % k, c // k, c % k
            Gpk[pk[(a, b)] * KK + pk[(p, q)]] = Gf[r, c]
            Zpk[pk[(a, b)] * KK + pk[(p, q)]] = Zf[r, c]
    # re-symmetrise from packed (the packing only holds the symmetric parts)
    for r in range(Q):
        for c in range(Q):
            a, p, b, q = r // k, r % k, c // k, c % k
            Gf[r, c] = Gpk[pk[(a, b)] * KK + pk[(p, q)]]
            Zf[r, c] = Zpk[pk[(a, b)] * KK + pk[(p, q)]]
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    t = lambda a: torch.as_tensor(a).to(dev)  # noqa: E731
    Zd, Gd = t(Zpk), t(Gpk)
    LG, LH = torch.zeros(Q, Q, dtype=torch.float64, device=dev), torch.zeros(Q, Q, dtype=torch.float64, device=dev)
    work = torch.zeros(2 * Q * Q, dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: lib.nmfb_lowrank_factor(Zd.data_ptr(), Gd.data_ptr(), k, LG.data_ptr(), LH.data_ptr(),  # noqa: E731
                                        work.data_ptr(), info.data_ptr(), s)
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    e1.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / reps
    L = LG.cpu().numpy()
    errG = np.abs(L @ L.T - Gf).max() / np.abs(Gf).max()
    H = np.eye(Q) - L.T @ Zf @ L
    Lh = LH.cpu().numpy()
    errH = np.abs(Lh @ Lh.T - H).max() / np.abs(H).max()
    print(f"k={k} Q={Q}: {us:8.1f} us per factor  info={int(info.item())}  relerr G {errG:.2e} H {errH:.2e}",
          flush=True)


for k in (3, 4, 10, 16):
    run(k)
