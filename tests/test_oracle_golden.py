"""The C oracle reproduces the reference kernels bit-for-bit.

Golden vectors come from the unmodified reference (tests/golden/make_golden.py);
this pins oracle/nmf_oracle.c before anything is checked against it.
"""
import numpy as np
import pytest

from oracle import kernels as ok

KS = (1, 2, 3, 4, 10, 16)


@pytest.mark.parametrize("k", KS)
def test_block_cholesky_bitexact(golden, k):
    L, bad = ok.block_cholesky(golden[f"chol_k{k}_in"])
    assert bad == int(golden[f"chol_k{k}_bad"])
    assert np.array_equal(L, golden[f"chol_k{k}_L"])


def test_block_cholesky_failure_index(golden):
    L, bad = ok.block_cholesky(golden["cholbad_in"])
    assert bad == int(golden["cholbad_bad"]) == 3
    assert np.array_equal(L, golden["cholbad_L"])


@pytest.mark.parametrize("k", KS)
@pytest.mark.parametrize("r", (1, 3))
def test_block_triangular_bitexact(golden, k, r):
    L = golden[f"chol_k{k}_L"]
    b = golden[f"tri_k{k}_r{r}_b"]
    assert np.array_equal(ok.block_solve_lower(L, b), golden[f"tri_k{k}_r{r}_z"])
    assert np.array_equal(ok.block_solve_lower_t(L, b), golden[f"tri_k{k}_r{r}_zt"])


SHAPES = ((8, 4, 2), (12, 5, 2), (10, 6, 3), (20, 7, 4), (33, 9, 3), (16, 5, 10))


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("full", (0, 1))
def test_schur_rhs_backsub_bitexact(golden, shape, full):
    tag = "s_%d_%d_%d" % shape
    x, y, l, h = (golden[tag + s] for s in ("_x", "_y", "_l", "_h"))
    f, dy = golden[tag + "_f"], golden[tag + "_dy"]
    S, racc = ok.schur_reduce(x, y, l, h, f, full)
    assert np.array_equal(S, golden[f"{tag}_S{full}"])
    assert np.array_equal(racc, golden[f"{tag}_racc{full}"])
    # the numpy backend agrees to rounding (secondary reference)
    np.testing.assert_allclose(S, golden[f"{tag}_S{full}_np"], rtol=1e-11, atol=1e-12)
    assert np.array_equal(ok.rhs_reduce(x, y, l, h, f, full), golden[f"{tag}_rr{full}"])
    assert np.array_equal(ok.back_substitute(x, y, l, h, dy, f, full), golden[f"{tag}_dx{full}"])


def test_nnls_batch_bitexact(golden):
    n = int(golden["nnls_count"])
    seen_status = set()
    for c in range(n):
        pre = f"nnls{c}_"
        k, mode, mc = (int(v) for v in golden[pre + "meta"])
        out = ok.nnls_batch(golden[pre + "ctc"], golden[pre + "ctb"], golden[pre + "btb"],
                            golden[pre + "seed"], mode, golden[pre + "tol"], mc)
        for name, v in zip(("x", "p", "ch", "r2", "st"), out):
            ref = golden[pre + name]
            assert v.dtype == ref.dtype, (c, name)
            assert np.array_equal(v, ref), (c, name, k, mode)
        seen_status.update(int(s) for s in out[4])
    assert seen_status == {0, 1, 2}


def test_nnls_kat_spec127(golden):
    # C = I, d = (3, -2) -> x = (3, 0)
    out = ok.nnls_batch(np.eye(2), np.array([[3.0, -2.0]]), np.array([13.0]),
                        np.zeros((1, 2), bool), 0, np.array([3e-12]), 6)
    assert np.array_equal(out[0], golden["kat_nnls_x"])
    assert np.array_equal(out[0], np.array([[3.0, 0.0]]))
