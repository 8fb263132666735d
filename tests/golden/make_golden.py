"""Generate the golden kernel vectors from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference kernels
(/root/reference/pkg/src/nmfstream/_kernels_numba.py and _kernels_numpy.py)
as a namespace package, feeds them seeded inputs, and writes
tests/golden/kernels_golden.npz.  The reference cannot travel to the GPU
box, so the fixtures are committed; tests/test_oracle_golden.py pins the
C oracle against them bit-for-bit and the GPU parity tests reuse them.
Numba's on-disk cache is redirected to a temp dir so nothing is written into
/root/reference.
"""
from __future__ import annotations

import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="nmf_numba_cache_"))
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "kernels_golden.npz")


def _load_reference():
    sys.path.insert(0, REF_SRC)
    from nmfstream import _kernels_numba as kn  # noqa: WPS433
    from nmfstream import _kernels_numpy as kp  # noqa: WPS433
    return kn, kp


def _spd_blocks(rng, nb, k, rho=1e-3):
    a = rng.standard_normal((nb, k + 2, k))
    return np.einsum("bik,bil->bkl", a, a) + rho * np.eye(k)


def main():
    kn, kp = _load_reference()
    rng = np.random.default_rng(20210121)
    g = {}

    # --- block_cholesky / block_solve_lower(_t) -------------------------------
    for k in (1, 2, 3, 4, 10, 16):
        blocks = _spd_blocks(rng, 7, k)
        g[f"chol_k{k}_in"] = blocks
        L, bad = kn.block_cholesky(blocks)
        g[f"chol_k{k}_L"], g[f"chol_k{k}_bad"] = L, np.int64(bad)
        for r in (1, 3):
            b = rng.standard_normal((7, k, r))
            g[f"tri_k{k}_r{r}_b"] = b
            g[f"tri_k{k}_r{r}_z"] = kn.block_solve_lower(L, b)
            g[f"tri_k{k}_r{r}_zt"] = kn.block_solve_lower_t(L, b)
    # a non-PD block in the middle: index 3 must be reported, later blocks zero
    blocks = _spd_blocks(rng, 6, 4)
    blocks[3] = -np.eye(4) + 0.1
    blocks[5] = -np.eye(4)
    g["cholbad_in"] = blocks
    L, bad = kn.block_cholesky(blocks)
    g["cholbad_L"], g["cholbad_bad"] = L, np.int64(bad)

    # --- schur_reduce / rhs_reduce / back_substitute --------------------------
    for (n, m, k) in ((8, 4, 2), (12, 5, 2), (10, 6, 3), (20, 7, 4), (33, 9, 3), (16, 5, 10)):
        tag = f"s_{n}_{m}_{k}"
        x = rng.uniform(0.05, 1.0, (n, k))
        yc = rng.uniform(0.05, 1.0, (m, k))
        r = rng.uniform(0.01, 2.0, (n, k))
        blocks = (yc.T @ yc)[None] + 1e-6 * np.eye(k)[None] + np.einsum("ip,pq->ipq", r / x, np.eye(k))
        L, bad = kn.block_cholesky(blocks)
        assert bad == -1
        h = rng.standard_normal((n, k))
        resid = rng.standard_normal((n, m)) * 0.3
        dy = rng.standard_normal((m, k))
        g[tag + "_x"], g[tag + "_y"], g[tag + "_l"], g[tag + "_h"] = x, yc, L, h
        g[tag + "_f"], g[tag + "_dy"] = resid, dy
        for full in (False, True):
            S, racc = kn.schur_reduce(x, yc, L, h, resid, full)
            g[f"{tag}_S{int(full)}"], g[f"{tag}_racc{int(full)}"] = S, racc
            g[f"{tag}_rr{int(full)}"] = kn.rhs_reduce(x, yc, L, h, resid, full)
            g[f"{tag}_dx{int(full)}"] = kn.back_substitute(x, yc, L, h, dy, resid, full)
            # numpy backend (secondary reference) for the tolerance-level check
            Sn, raccn = kp.schur_reduce(x, yc, L, h, resid, full)
            g[f"{tag}_S{int(full)}_np"], g[f"{tag}_racc{int(full)}_np"] = Sn, raccn

    # --- nnls_batch -----------------------------------------------------------
    cases = []
    for k in (1, 2, 3, 4, 8, 10, 16):
        for mode in (0, 1, 2):
            cases.append((k, mode, "gauss"))
            cases.append((k, mode, "nmf"))
    ci = 0
    for (k, mode, kind) in cases:
        nrhs = 64
        if kind == "gauss":
            C = rng.standard_normal((k + 3, k))
            D = rng.standard_normal((nrhs, k + 3))
        else:  # NMF-like: nonnegative C, smoothly varying nonnegative d (streaming)
            C = rng.uniform(0, 1, (3 * k + 5, k))
            base = rng.uniform(0, 1, (k,))
            D = np.empty((nrhs, 3 * k + 5))
            for t in range(nrhs):
                coef = np.clip(base + 0.3 * np.sin(0.2 * t + np.arange(k)), -0.2, None)
                D[t] = C @ coef + 0.05 * rng.standard_normal(3 * k + 5)
        ctc = C.T @ C
        ctb = D @ C
        btb = np.einsum("ij,ij->i", D, D)
        tol = 1e-12 * np.maximum(1.0, np.abs(ctb).max(axis=1))
        # seeds: a previous solve on a perturbed problem (mode 2), garbage otherwise
        prev = kn.nnls_batch(ctc, ctb * (1 + 0.05 * rng.standard_normal(ctb.shape)), btb,
                             np.zeros((nrhs, k), np.bool_), 0, tol, 3 * k)
        seeds = prev[1].copy()
        seeds[::7] = rng.uniform(size=(seeds[::7].shape)) < 0.5  # some random seeds
        seeds[::11] = False  # some empty seeds
        out = kn.nnls_batch(ctc, ctb, btb, seeds, mode, tol, 3 * k)
        outp = kp.nnls_batch(ctc, ctb, btb, seeds, mode, tol, 3 * k)
        pre = f"nnls{ci}_"
        g[pre + "meta"] = np.array([k, mode, 3 * k], np.int64)
        g[pre + "ctc"], g[pre + "ctb"], g[pre + "btb"], g[pre + "tol"] = ctc, ctb, btb, tol
        g[pre + "seed"] = seeds
        for name, v in zip(("x", "p", "ch", "r2", "st"), out):
            g[pre + name] = v
        g[pre + "x_np"] = outp[0]
        ci += 1

    # status 1 (change cap) and status 2 (rank-deficient passive set)
    k = 6
    # singular Gram whose Cholesky pivot is exactly 0 on the passive set {4, 5}
    ctc = np.eye(k)
    ctc[4, 5] = ctc[5, 4] = -1.0  # [[1,-1],[-1,1]] block: second pivot is exactly 0
    ctb = rng.standard_normal((40, k))
    btb = np.einsum("ij,ij->i", ctb, ctb) + 1.0
    tol = 1e-12 * np.maximum(1.0, np.abs(ctb).max(axis=1))
    for mc in (1, 2, 18):
        out = kn.nnls_batch(ctc, ctb, btb, np.zeros((40, k), np.bool_), 0, tol, mc)
        pre = f"nnls{ci}_"
        g[pre + "meta"] = np.array([k, 0, mc], np.int64)
        g[pre + "ctc"], g[pre + "ctb"], g[pre + "btb"], g[pre + "tol"] = ctc, ctb, btb, tol
        g[pre + "seed"] = np.zeros((40, k), np.bool_)
        for name, v in zip(("x", "p", "ch", "r2", "st"), out):
            g[pre + name] = v
        g[pre + "x_np"] = out[0]
        ci += 1
    # empty batch
    pre = f"nnls{ci}_"
    k = 3
    g[pre + "meta"] = np.array([k, 2, 9], np.int64)
    g[pre + "ctc"], g[pre + "ctb"] = np.eye(k), np.zeros((0, k))
    g[pre + "btb"], g[pre + "tol"] = np.zeros(0), np.zeros(0)
    g[pre + "seed"] = np.zeros((0, k), np.bool_)
    out = kn.nnls_batch(g[pre + "ctc"], g[pre + "ctb"], g[pre + "btb"], g[pre + "seed"], 2,
                        g[pre + "tol"], 9)
    for name, v in zip(("x", "p", "ch", "r2", "st"), out):
        g[pre + name] = v
    g[pre + "x_np"] = out[0]
    ci += 1
    g["nnls_count"] = np.int64(ci)

    # SPEC.md:127 known answer: C = I, d = (3, -2) -> x = (3, 0)
    out = kn.nnls_batch(np.eye(2), np.array([[3.0, -2.0]]), np.array([13.0]),
                        np.zeros((1, 2), np.bool_), 0, np.array([1e-12 * 3]), 6)
    g["kat_nnls_x"] = out[0]

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
