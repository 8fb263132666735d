"""Drop-in kernel module: the seven reference kernels on the B200.

Same names, signatures, argument meanings, return tuples and failure codes as
the reference's kernel modules (/root/reference/pkg/src/nmfstream/
_kernels_numba.py and _kernels_numpy.py), so the reference's (missing)
``backend`` selector can hand this module to its drivers unchanged.  Each
call runs the bit-identical CUDA kernel of ``csrc/surface.cu`` through the
C-ABI of ``include/nmfb200.h``.

Inputs may be NumPy arrays (host: copied to the device and results copied
back, as the reference returns fresh NumPy arrays) or CUDA torch tensors
(device-resident: results stay on the device).  Like the reference, the
kernels never raise for numerical failures; they return codes.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib

__all__ = ["block_cholesky", "block_solve_lower", "block_solve_lower_t", "schur_reduce",
           "rhs_reduce", "back_substitute", "nnls_batch"]

_INT_MAX = 2**31 - 1


def _device():
    if not torch.cuda.is_available():
        from .errors import NativeLibraryError

        raise NativeLibraryError("no CUDA device: the B200 kernels have no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


class _Args:
    """Moves reference-style arguments to the device and results back."""

    def __init__(self, *arrays):
        self.host = not any(isinstance(a, torch.Tensor) for a in arrays if a is not None)
        self.dev = _device()

    def f64(self, a):
        if isinstance(a, torch.Tensor):
            return a.to(device=self.dev, dtype=torch.float64).contiguous()
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.dev)

    def u8(self, a):
        if isinstance(a, torch.Tensor):
            return a.to(device=self.dev, dtype=torch.uint8).contiguous()
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.bool_).view(np.uint8)).to(self.dev)

    def out(self, t, kind=None):
        if not self.host:
            return t.bool() if kind == "bool" else t
        a = t.cpu().numpy()
        return a.view(np.bool_) if kind == "bool" else a


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _ptr(t):
    return t.data_ptr() if t is not None and t.numel() > 0 else None


def block_cholesky(blocks):
    """_kernels_numba.py:12-29 -> (L, bad); bad = first non-PD block or -1."""
    a = _Args(blocks)
    b = a.f64(blocks)
    nb, k, _ = b.shape
    out = torch.empty_like(b)
    bad = torch.empty(1, dtype=torch.int32, device=a.dev)
    _lib.call("nmfb_surface_block_cholesky", _ptr(b), nb, k, _ptr(out), _ptr(bad), _stream())
    badv = int(bad.item())
    return a.out(out), (-1 if badv == _INT_MAX else badv)


def _trsm(l, b, transposed):
    a = _Args(l, b)
    L, B = a.f64(l), a.f64(b)
    nb, k, r = B.shape
    z = torch.empty_like(B)
    _lib.call("nmfb_surface_block_solve_lower", _ptr(L), _ptr(B), nb, k, r, int(transposed),
              _ptr(z), _stream())
    return a.out(z)


def block_solve_lower(l, b):
    """_kernels_numba.py:32-43: solve L[i] Z[i] = B[i]."""
    return _trsm(l, b, False)


def block_solve_lower_t(l, b):
    """_kernels_numba.py:46-57: solve L[i]^T Z[i] = B[i]."""
    return _trsm(l, b, True)


def _resid(a, resid, full):
    if full or resid is not None:
        return a.f64(resid)
    return None


def schur_reduce(x_rows, y_cols, l, h, resid, full):
    """_kernels_numba.py:72-143 -> (S (mk,mk), r_acc (m,k))."""
    a = _Args(x_rows, y_cols, l, h, resid)
    X, Yc, L, H = a.f64(x_rows), a.f64(y_cols), a.f64(l), a.f64(h)
    R = _resid(a, resid, full)
    n, k = X.shape
    m = Yc.shape[0]
    S = torch.empty((m * k, m * k), dtype=torch.float64, device=a.dev)
    racc = torch.empty((m, k), dtype=torch.float64, device=a.dev)
    _lib.call("nmfb_surface_schur_reduce", _ptr(X), _ptr(Yc), _ptr(L), _ptr(H), _ptr(R), n, m, k,
              int(bool(full)), _ptr(S), _ptr(racc), _stream())
    return a.out(S), a.out(racc)


def rhs_reduce(x_rows, y_cols, l, h, resid, full):
    """_kernels_numba.py:146-178 -> r_acc (m,k)."""
    a = _Args(x_rows, y_cols, l, h, resid)
    X, Yc, L, H = a.f64(x_rows), a.f64(y_cols), a.f64(l), a.f64(h)
    R = _resid(a, resid, full)
    n, k = X.shape
    m = Yc.shape[0]
    racc = torch.empty((m, k), dtype=torch.float64, device=a.dev)
    _lib.call("nmfb_surface_rhs_reduce", _ptr(X), _ptr(Yc), _ptr(L), _ptr(H), _ptr(R), n, m, k,
              int(bool(full)), _ptr(racc), _stream())
    return a.out(racc)


def back_substitute(x_rows, y_cols, l, h, dy_rows, resid, full):
    """_kernels_numba.py:181-224 -> dx (n,k)."""
    a = _Args(x_rows, y_cols, l, h, dy_rows, resid)
    X, Yc, L, H, DY = a.f64(x_rows), a.f64(y_cols), a.f64(l), a.f64(h), a.f64(dy_rows)
    R = _resid(a, resid, full)
    n, k = X.shape
    m = Yc.shape[0]
    dx = torch.empty((n, k), dtype=torch.float64, device=a.dev)
    _lib.call("nmfb_surface_back_substitute", _ptr(X), _ptr(Yc), _ptr(L), _ptr(H), _ptr(DY),
              _ptr(R), n, m, k, int(bool(full)), _ptr(dx), _stream())
    return a.out(dx)


def nnls_batch(ctc, ctb, btb, warm_passive, warm_mode, tol, max_changes, *, table=True):
    """_kernels_numba.py:277-477 -> (x, passive, changes, resid2, status).

    status per rhs: 0 solved, 1 change cap exceeded, 2 rank-deficient passive set.
    table (keyword-only extension): for k <= 16 factor every passive subset once per
    call (nmfb_nnls_batch_ws, the reference's factor cache); False runs the
    per-rhs factorizing kernels of nmfb_surface_nnls_batch.  Same bits either way.
    """
    a = _Args(ctc, ctb, btb, warm_passive, tol)
    C, B, BB, T = a.f64(ctc), a.f64(ctb), a.f64(btb), a.f64(tol)
    W = a.u8(warm_passive)
    nrhs, k = B.shape
    dev = a.dev
    x = torch.empty((nrhs, k), dtype=torch.float64, device=dev)
    p = torch.empty((nrhs, k), dtype=torch.uint8, device=dev)
    ch = torch.empty(nrhs, dtype=torch.int64, device=dev)
    r2 = torch.empty(nrhs, dtype=torch.float64, device=dev)
    st = torch.empty(nrhs, dtype=torch.int8, device=dev)
    seed = flag = None
    if int(warm_mode) == 1:
        seed = torch.empty((nrhs, k), dtype=torch.uint8, device=dev)
        flag = torch.empty(1, dtype=torch.int32, device=dev)
    flen = int(_lib.load().nmfb_nnls_ftab_len(k)) if table else 0
    if flen > 0:
        ftab = torch.empty(flen, dtype=torch.float64, device=dev)
        _lib.call("nmfb_nnls_batch_ws", _ptr(C), _ptr(B), _ptr(BB), _ptr(W), int(warm_mode),
                  _ptr(T), int(max_changes), nrhs, k, _ptr(x), _ptr(p), _ptr(ch), _ptr(r2),
                  _ptr(st), _ptr(seed), _ptr(flag), _ptr(ftab), flen, _stream())
    else:
        _lib.call("nmfb_surface_nnls_batch", _ptr(C), _ptr(B), _ptr(BB), _ptr(W),
                  int(warm_mode), _ptr(T), int(max_changes), nrhs, k, _ptr(x), _ptr(p), _ptr(ch),
                  _ptr(r2), _ptr(st), _ptr(seed), _ptr(flag), _stream())
    return a.out(x), a.out(p, "bool"), a.out(ch), a.out(r2), a.out(st)
