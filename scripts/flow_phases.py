"""Phase anatomy of the dataflow Cholesky (csrc/dense_flow.cuh) along its critical path:
for each column j the diagonal tile (j, j) and the sub-diagonal tile (j+1, j).

python scripts/flow_phases.py N
stamps: 0 start, 1 accumulate done, 2 A_ij subtracted, 3 L_jj seen, 4 L_jj loaded,
5 factor / row sweeps done, 6 written, 7 published
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_08431_b200 import _lib  # noqa: E402

lib = _lib.load()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
rng = np.random.default_rng(N)
B = rng.standard_normal((N, N))
A = B @ B.T / N + np.eye(N)
T = (N + 31) // 32
ntiles = T * (T + 1) // 2
s = torch.cuda.current_stream().cuda_stream
info = torch.zeros(1, dtype=torch.int32, device="cuda")
for rep in range(3):
    d = torch.as_tensor(A).cuda()
    buf = torch.zeros(ntiles * 8, dtype=torch.int64, device="cuda")
    lib.nmfb_flow_profile(buf.data_ptr() if rep == 2 else None)
    lib.nmfb_dense_cholesky(d.data_ptr(), N, info.data_ptr(), s)
    torch.cuda.synchronize()
lib.nmfb_flow_profile(None)
st = buf.cpu().numpy().reshape(ntiles, 8).astype(np.float64)
t0 = st[:, 0][st[:, 0] > 0].min()
base = [j * T - j * (j - 1) // 2 for j in range(T)]
print(f"N={N} T={T}: total {(st[:, 7].max() - t0) / 1e3:.1f} us")
print("col |  diag: start  acc   sub   factor write publish | sub-diag: start acc  sub  Ljj-seen loaded sweeps write publish  (us from the previous diagonal publish)")
prev = t0
for j in range(T):
    dg = st[base[j]]
    line = f"{j:3d} | " + " ".join(f"{(dg[k] - prev) / 1e3:6.2f}" for k in (0, 1, 2, 5, 6, 7))
    if j + 1 < T:
        sd = st[base[j] + 1]
        line += " | " + " ".join(f"{(sd[k] - prev) / 1e3:6.2f}" for k in range(8))
    if j < 6 or j % 8 == 0 or j > T - 4:
        print(line)
    prev = dg[7]
