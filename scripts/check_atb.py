"""nmfb_atb (split-K DMMA A^T B with the fixed-order finish) against torch fp64 at the packed
capacitance shapes (ca = cb = k(k+1)/2) and a ragged general one; prints time and max error."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_08431_b200 import _lib  # noqa: E402

lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream
for n, ca, cb in ((20000, 55, 55), (5000, 55, 55), (20011, 55, 55), (200000, 136, 136), (3000, 10, 10),
                  (7777, 36, 55), (4097, 100, 27)):
    g = torch.Generator(device="cuda")
    g.manual_seed(n + ca)
    A = torch.rand(n, ca, dtype=torch.float64, device="cuda", generator=g) - 0.3
    B = torch.rand(n, cb, dtype=torch.float64, device="cuda", generator=g) - 0.3
    out = torch.empty(ca, cb, dtype=torch.float64, device="cuda")
    wl = lib.nmfb_atb_work_len(n, ca, cb)
    work = torch.empty(wl, dtype=torch.float64, device="cuda")
    for _ in range(3):
        rc = lib.nmfb_atb(A.data_ptr(), n, ca, B.data_ptr(), cb, out.data_ptr(), work.data_ptr(), wl, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        lib.nmfb_atb(A.data_ptr(), n, ca, B.data_ptr(), cb, out.data_ptr(), work.data_ptr(), wl, s)
    e1.record()
    e1.synchronize()
    ref = A.T @ B
    err = float((out - ref).abs().max() / ref.abs().max())
    print(f"{n} x {ca} x {cb}: rc {rc}, {e0.elapsed_time(e1) / 20 * 1e3:.1f} us, rel err {err:.2e}")
    assert rc == 0 and err < 1e-13
