"""GPU parity of the seven reference-surface kernels: BIT-IDENTICAL to the reference.

Golden vectors were produced by the unmodified reference (tests/golden/make_golden.py);
larger random cases are checked against the C oracle, itself pinned bit-for-bit.
"""
import numpy as np
import pytest

from oracle import kernels as ok

pytestmark = pytest.mark.gpu

KS = (1, 2, 3, 4, 10, 16)


@pytest.fixture(scope="module")
def K():
    from paper_2101_08431_b200 import kernels

    return kernels


@pytest.mark.parametrize("k", KS)
def test_block_cholesky(golden, K, k):
    L, bad = K.block_cholesky(golden[f"chol_k{k}_in"])
    assert bad == int(golden[f"chol_k{k}_bad"]) == -1
    assert np.array_equal(L, golden[f"chol_k{k}_L"])


def test_block_cholesky_failure(golden, K):
    L, bad = K.block_cholesky(golden["cholbad_in"])
    assert bad == 3
    assert np.array_equal(L, golden["cholbad_L"])


@pytest.mark.parametrize("k", KS)
@pytest.mark.parametrize("r", (1, 3))
def test_triangular(golden, K, k, r):
    L, b = golden[f"chol_k{k}_L"], golden[f"tri_k{k}_r{r}_b"]
    assert np.array_equal(K.block_solve_lower(L, b), golden[f"tri_k{k}_r{r}_z"])
    assert np.array_equal(K.block_solve_lower_t(L, b), golden[f"tri_k{k}_r{r}_zt"])


SHAPES = ((8, 4, 2), (12, 5, 2), (10, 6, 3), (20, 7, 4), (33, 9, 3), (16, 5, 10))


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("full", (0, 1))
def test_schur_rhs_backsub(golden, K, shape, full):
    tag = "s_%d_%d_%d" % shape
    x, y, l, h = (golden[tag + s] for s in ("_x", "_y", "_l", "_h"))
    f, dy = golden[tag + "_f"], golden[tag + "_dy"]
    S, racc = K.schur_reduce(x, y, l, h, f, full)
    assert np.array_equal(S, golden[f"{tag}_S{full}"])
    assert np.array_equal(racc, golden[f"{tag}_racc{full}"])
    assert np.array_equal(K.rhs_reduce(x, y, l, h, f, full), golden[f"{tag}_rr{full}"])
    assert np.array_equal(K.back_substitute(x, y, l, h, dy, f, full), golden[f"{tag}_dx{full}"])


@pytest.mark.parametrize("table", (True, False))
def test_nnls_golden(golden, K, table):
    """Both device formulations against the reference's own outputs: the subset
    factor table + register thread kernel (k <= 12) and the per-rhs factorizing
    kernels of nmfb_surface_nnls_batch."""
    for c in range(int(golden["nnls_count"])):
        pre = f"nnls{c}_"
        k, mode, mc = (int(v) for v in golden[pre + "meta"])
        out = K.nnls_batch(golden[pre + "ctc"], golden[pre + "ctb"], golden[pre + "btb"],
                           golden[pre + "seed"], mode, golden[pre + "tol"], mc, table=table)
        for name, v in zip(("x", "p", "ch", "r2", "st"), out):
            ref = golden[pre + name]
            assert v.shape == ref.shape and v.dtype == ref.dtype, (c, name)
            assert np.array_equal(v, ref), (c, name, k, mode)


def _nmf_like(rng, nrhs, k, drift):
    C = rng.uniform(0, 1, (3 * k + 4, k))
    coef = np.cumsum(rng.standard_normal((nrhs, k)) * drift, axis=0) + rng.uniform(0, 1, k)
    D = coef @ C.T + 0.05 * rng.standard_normal((nrhs, 3 * k + 4))
    ctc, ctb = C.T @ C, D @ C
    return ctc, ctb, np.einsum("ij,ij->i", D, D), 1e-12 * np.maximum(1, np.abs(ctb).max(1))


@pytest.mark.parametrize("k,nrhs", [(3, 5000), (4, 5000), (10, 5000), (12, 4000), (13, 3000),
                                     (16, 5000), (4, 20000), (10, 12000), (16, 20000)])
@pytest.mark.parametrize("mode", (0, 1, 2))
@pytest.mark.parametrize("table", (True, False))
def test_nnls_large_vs_oracle(K, k, nrhs, mode, table):
    """Bit-identical to the reference on every device formulation: the subset
    factor table + register thread kernel (k <= 16; 2^16 subsets = 135 MB at k = 16),
    warp per rhs (small batches) and thread per rhs (no table, batches > 8192)."""
    rng = np.random.default_rng(1000 + 10 * k + mode)
    ctc, ctb, btb, tol = _nmf_like(rng, nrhs, k, 0.05)
    seed = ok.nnls_batch(ctc, ctb * 1.01, btb, np.zeros((nrhs, k), bool), 0, tol, 3 * k)[1]
    ref = ok.nnls_batch(ctc, ctb, btb, seed, mode, tol, 3 * k)
    out = K.nnls_batch(ctc, ctb, btb, seed, mode, tol, 3 * k, table=table)
    for name, a, b in zip(("x", "p", "ch", "r2", "st"), out, ref):
        assert np.array_equal(a, b), (name, k, mode)


@pytest.mark.parametrize("k", (2, 5, 10, 16))
def test_nnls_table_cold_and_rank_deficient(K, k):
    """Table path on cold starts with many Lawson-Hanson trips, the change cap
    (status 1) and a rank-deficient Gram (status 2: failing subsets in the table)."""
    rng = np.random.default_rng(77 + k)
    nrhs = 3000
    C = rng.uniform(0, 1, (3 * k + 4, k))
    C[:, -1] = C[:, 0]  # duplicated column: every subset holding both is not PD
    D = rng.standard_normal((nrhs, 3 * k + 4))
    ctc, ctb = C.T @ C, D @ C
    btb = np.einsum("ij,ij->i", D, D)
    tol = 1e-12 * np.maximum(1, np.abs(ctb).max(1))
    for mc in (3 * k, 2):
        ref = ok.nnls_batch(ctc, ctb, btb, np.zeros((nrhs, k), bool), 0, tol, mc)
        out = K.nnls_batch(ctc, ctb, btb, np.zeros((nrhs, k), bool), 0, tol, mc)
        for name, a, b in zip(("x", "p", "ch", "r2", "st"), out, ref):
            assert np.array_equal(a, b), (name, k, mc)


def test_nnls_chain_many_switches(K):
    """Mode 1 with frequent passive-set changes along the chain (fixed point iterates)."""
    rng = np.random.default_rng(7)
    k, nrhs = 4, 3000
    ctc, ctb, btb, tol = _nmf_like(rng, nrhs, k, 0.6)
    ref = ok.nnls_batch(ctc, ctb, btb, np.zeros((nrhs, k), bool), 1, tol, 3 * k)
    out = K.nnls_batch(ctc, ctb, btb, np.zeros((nrhs, k), bool), 1, tol, 3 * k)
    for name, a, b in zip(("x", "p", "ch", "r2", "st"), out, ref):
        assert np.array_equal(a, b), name


def test_surface_large_schur_backsub(K):
    rng = np.random.default_rng(3)
    n, m, k = 300, 40, 3
    x = rng.uniform(0.05, 1, (n, k))
    yc = rng.uniform(0.05, 1, (m, k))
    r = rng.uniform(0.01, 2, (n, k))
    blocks = (yc.T @ yc)[None] + 1e-6 * np.eye(k) + np.einsum("ip,pq->ipq", r / x, np.eye(k))
    L, bad = ok.block_cholesky(blocks)
    h = rng.standard_normal((n, k))
    f = 0.1 * rng.standard_normal((n, m))
    dy = rng.standard_normal((m, k))
    for full in (0, 1):
        S, ra = K.schur_reduce(x, yc, L, h, f, full)
        So, rao = ok.schur_reduce(x, yc, L, h, f, full)
        assert np.array_equal(S, So) and np.array_equal(ra, rao)
        assert np.array_equal(K.rhs_reduce(x, yc, L, h, f, full), ok.rhs_reduce(x, yc, L, h, f, full))
        assert np.array_equal(K.back_substitute(x, yc, L, h, dy, f, full),
                              ok.back_substitute(x, yc, L, h, dy, f, full))
