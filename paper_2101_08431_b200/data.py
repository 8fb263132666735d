"""Seeded synthetic problem instances (data-io).

The reference ships no generator for the benchmark configurations, so the
five BASELINE.json configurations are defined here once and shared by the
oracle tests, the GPU parity tests and bench.py.  The RNG is numpy PCG64
with a fixed draw order:

    X_true, Y_true, noise, X0, Y0

Peak generator (configs c1-c3): each true X column is a sum of 8 Gaussian
peaks on r = linspace(0, 30, n) (centre U(1,29), width U(0.1,0.5), height
U(0.2,1)); true Y rows are the softmax over the k components of logistic
curves 1/(1+exp(-s(t-t0))) on t = linspace(0,1,m) with t0 ~ U(.2,.8),
s ~ U(5,20), so every column of Y sums to 1; M = max(XY + N(0, (1e-3 max XY)^2), 0).

Dense generator (c4/c5): X_true, Y_true ~ U(0,1), M = XY + |N(0, 1e-2^2)|.
c5 (fp32 M, 32 GB) is generated on the device in row blocks (see
``dense_device``); X0/Y0 still come from the host PCG64 stream.

Initial factors: X0 (n,k), Y0 (k,m) ~ U(0,1).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    m: int
    k: int
    kind: str  # "peaks" | "dense"
    seed: int
    dtype: str = "f64"  # storage dtype of M
    tol: float = 1e-10  # relative KKT tolerance (two-stage to tolerance)
    fixed_sweeps: int = 0  # >0: run exactly this many ANLS sweeps
    fixed_ipm: int = 0  # >0: run exactly this many IPM iterations
    m_start: int = 0  # streaming: first chunk width
    m_step: int = 0  # streaming: chunk width


CONFIGS = {
    "c1": Config("c1", 300, 50, 3, "peaks", 101),
    "c2": Config("c2", 3000, 100, 3, "peaks", 102),
    "c3": Config("c3", 3000, 500, 4, "peaks", 103, m_start=20, m_step=10),
    "c4": Config("c4", 20000, 5000, 10, "dense", 104, fixed_sweeps=50, fixed_ipm=20),
    "c5": Config("c5", 200000, 40000, 16, "dense", 105, dtype="f32", fixed_sweeps=30,
                 fixed_ipm=10),
}


def _peaks_truth(rng, n, m, k):
    r = np.linspace(0.0, 30.0, n)
    centres = rng.uniform(1.0, 29.0, (k, 8))
    widths = rng.uniform(0.1, 0.5, (k, 8))
    heights = rng.uniform(0.2, 1.0, (k, 8))
    X = np.zeros((n, k))
    for p in range(k):
        for q in range(8):
            X[:, p] += heights[p, q] * np.exp(-((r - centres[p, q]) ** 2) / (2.0 * widths[p, q] ** 2))
    t = np.linspace(0.0, 1.0, m)
    t0 = rng.uniform(0.2, 0.8, k)
    slope = rng.uniform(5.0, 20.0, k)
    logit = 1.0 / (1.0 + np.exp(-slope[:, None] * (t[None, :] - t0[:, None])))
    e = np.exp(logit - logit.max(axis=0, keepdims=True))
    Y = e / e.sum(axis=0, keepdims=True)
    return X, Y


def peaks(n, m, k, seed):
    """Peak/logistic streaming-like instance -> (M, X0, Y0, X_true, Y_true)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    Xt, Yt = _peaks_truth(rng, n, m, k)
    clean = Xt @ Yt
    noise = rng.standard_normal((n, m)) * (1e-3 * clean.max())
    M = np.maximum(clean + noise, 0.0)
    X0 = rng.uniform(0.0, 1.0, (n, k))
    Y0 = rng.uniform(0.0, 1.0, (k, m))
    return M, X0, Y0, Xt, Yt


def dense(n, m, k, seed, dtype=np.float64):
    """Dense random instance (host) -> (M, X0, Y0, X_true, Y_true)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    Xt = rng.uniform(0.0, 1.0, (n, k))
    Yt = rng.uniform(0.0, 1.0, (k, m))
    M = Xt @ Yt
    M += np.abs(rng.standard_normal((n, m)) * 1e-2)
    X0 = rng.uniform(0.0, 1.0, (n, k))
    Y0 = rng.uniform(0.0, 1.0, (k, m))
    return M.astype(dtype, copy=False), X0, Y0, Xt, Yt


def make(cfg: Config):
    """Host instance for a named config (c1-c4; c5 is device-generated)."""
    if cfg.kind == "peaks":
        return peaks(cfg.n, cfg.m, cfg.k, cfg.seed)
    if cfg.name == "c5":
        raise ValueError("c5 (32 GB fp32 M) is generated on the device: use dense_device()")
    return dense(cfg.n, cfg.m, cfg.k, cfg.seed)


def init_factors(n, m, k, seed):
    """init_factors: X (n,k), Y (k,m) ~ U(0,1) from a PCG64 stream."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(0.0, 1.0, (n, k)), rng.uniform(0.0, 1.0, (k, m))


def dense_device(n, m, k, seed, device, dtype, row_block=8192, rows=None):
    """Device-side dense generator for c5-sized M (torch Philox, row blocks).

    Returns (M_dev, X0, Y0): M_dev holds rows [a, b) of M (all rows when
    ``rows`` is None) in the requested dtype; X0 (rows, k) and Y0 (k, m) are
    float64 host arrays from PCG64(seed).  The truth factors come from a
    device generator seeded with ``seed``; the |N(0, 1e-2)| noise of row block
    r comes from its own generator seeded (seed, r), so any row range (a rank's
    shard) is generated independently and identically to the full matrix.
    """
    import torch

    a, b = (0, n) if rows is None else rows
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    Xt = torch.rand((n, k), generator=g, device=device, dtype=torch.float64)
    Yt = torch.rand((k, m), generator=g, device=device, dtype=torch.float64)
    M = torch.empty((b - a, m), device=device, dtype=dtype)
    gb = torch.Generator(device=device)
    for r in range(a // row_block, (b + row_block - 1) // row_block):
        i0, i1 = r * row_block, min(n, (r + 1) * row_block)
        gb.manual_seed(int(seed) * 1000003 + r)
        blk = Xt[i0:i1] @ Yt
        blk += torch.randn((i1 - i0, m), generator=gb, device=device, dtype=torch.float64).abs_() * 1e-2
        lo, hi = max(i0, a), min(i1, b)
        M[lo - a:hi - a] = blk[lo - i0:hi - i0].to(dtype)
        del blk
    rng = np.random.Generator(np.random.PCG64(seed))
    X0 = rng.uniform(0.0, 1.0, (n, k))[a:b]
    Y0 = rng.uniform(0.0, 1.0, (k, m))
    return M, X0, Y0
