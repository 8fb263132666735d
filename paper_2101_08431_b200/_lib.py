"""ctypes binding of libnmfb200.so (include/nmfb200.h).

The product path has no CPU fallback: if the library is missing or fails to
load, every entry point raises ``NativeLibraryError``.
"""
from __future__ import annotations

import ctypes
import os

from .errors import NativeLibraryError

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("NMFB_SO") or os.path.join(_HERE, "libnmfb200.so")  # NMFB_SO: A/B builds

P = ctypes.c_void_p
L = ctypes.c_long
I = ctypes.c_int
D = ctypes.c_double

# name -> argtypes (all return int status)
SIGNATURES = {
    "nmfb_surface_nnls_batch": [P, P, P, P, I, P, L, L, L, P, P, P, P, P, P, P, P],
    "nmfb_surface_block_cholesky": [P, L, L, P, P, P],
    "nmfb_surface_block_solve_lower": [P, P, L, L, L, I, P, P],
    "nmfb_surface_schur_reduce": [P, P, P, P, P, L, L, L, I, P, P, P],
    "nmfb_surface_rhs_reduce": [P, P, P, P, P, L, L, L, I, P, P],
    "nmfb_surface_back_substitute": [P, P, P, P, P, P, L, L, L, I, P, P],
    # production entries
    "nmfb_nnls_ftab_len": [L],
    "nmfb_first_failure_i8": [P, L, L, P, P],
    "nmfb_stage1_set_prof": [P],
    "nmfb_blas_init": [P],
    "nmfb_set_mu_source": [P],
    "nmfb_nnls_batch_ws": [P, P, P, P, I, P, L, L, L, P, P, P, P, P, P, P, P, L, P],
    "nmfb_rowprod_work_len": [L, L, L, I],
    "nmfb_rowprod": [P, I, L, L, P, L, P, P, D, P, L, P],
    "nmfb_colprod_work_len": [L, L, L],
    "nmfb_colprod": [P, I, L, L, P, L, P, P, D, P, L, P],
    "nmfb_sqnorms": [P, I, L, L, P, P, P, L, P],
    "nmfb_stage1_stats": [P, P, L, P, P, L, P, L, P, P, L, P],
    "nmfb_first_nonzero_i8": [P, L, P, P],
    "nmfb_row_tol": [P, L, L, P, P],
    "nmfb_ipm_reduce_blocks": [],
    "nmfb_residual": [P, I, L, L, L, P, P, P, P, P, P, P],
    "nmfb_r1_factor": [P, P, P, P, D, D, L, L, P, P, P, P, P, P, P],
    "nmfb_hg": [P, P, D, L, L, P, P, P],
    "nmfb_atb_work_len": [L, L, L],
    "nmfb_atb": [P, L, L, P, L, P, P, L, P],
    "nmfb_make_p": [P, P, L, L, P, P],
    "nmfb_schur_assemble": [P, P, L, L, P, P, D, P, P, P],
    "nmfb_schur_term4": [P, L, L, L, P, P, P, L, P],
    "nmfb_term4_work_len": [L, L, L],
    "nmfb_schur_rhs": [P, P, P, P, D, L, L, P, P],
    "nmfb_direction": [P, P, P, P, P, P, P, P, D, P, P, P, P, D, D, L, L, L, P, P, P, P, P, L, P],
    "nmfb_quartic": [P, L, L, L, P, P, P, P, P, P, P],
    "nmfb_barrier_trials": [P, P, L, P, P, L, P, I, P, P, L, P],
    "nmfb_step_nudge": [P, P, L, D, D, P],
    "nmfb_armijo_select": [P, D, D, D, D, I, P, P],
    "nmfb_armijo_lazy": [P, P, L, P, P, L, P, I, D, D, D, D, I, P, P, L, P],
    "nmfb_step_nudge_dev": [P, P, L, P, D, P],
    "nmfb_step_nudge_flag": [P, P, L, P, D, D, P, P],
    "nmfb_ffree_advance": [P, P, L, P, P, L, P, D, P, P],
    "nmfb_step_all": [P, P, L, P, P, L, P, P, P, P, P, P, P, P, P, D, P, D, D, P, P],
    "nmfb_kkt_sums": [P, P, P, L, P, P, P, L, D, D, P, P, P],
    "nmfb_affine_mu": [P, P, P, P, L, P, P, P, P, L, D, D, P, P, P],
    "nmfb_clamp_min": [P, L, D, P],
    "nmfb_fill": [P, L, D, P],
    "nmfb_dense_cholesky": [P, L, P, P],
    "nmfb_dense_solve": [P, L, P, P],
    "nmfb_dense_cholesky_rhs": [P, L, P, P, P],
    "nmfb_dense_solve_back": [P, L, P, P],
    "nmfb_dense_solve_mode": [P, L, P, I, P],
    "nmfb_flow_profile": [P],
    "nmfb_launch_count": [],
    "nmfb_last_cuda_error": [],
    "nmfb_tma_products": [I],
    "nmfb_tc_products": [I],
    "nmfb_nnls_ftab_build": [P, L, P, L, P],
    "nmfb_d_factor": [P, P, P, D, L, L, P, P, P, P, P],
    "nmfb_ffree_grad_rows": [P, P, P, L, L, P, P, P],
    "nmfb_ffree_fsq": [P, D, P, P, L, P, P, P],
    "nmfb_ffree_quartic": [P, P, P, P, P, P, P, P, P, L, P, P],
    "nmfb_small_supported": [L, L, L],
    "nmfb_persist_supported": [L, L, L, I, I],
    "nmfb_dualprod_work_len": [L, L, L],
    "nmfb_dualprod": [P, I, L, L, P, P, L, P, P, P, L, P],
    "nmfb_grams_work_len": [L, L, L],
    "nmfb_stage1_persist_supported": [L, L, L, I],
    "nmfb_stage1_persist_work_len": [L, L, L],
    "nmfb_stage1_persist": [P, I, L, L, L] + [P] * 10 + [D, I, I, I, D, P, P, P, P],
    "nmfb_grams": [I] + [P] * 12 + [L, L, P, L, P],
    "nmfb_persist_work_len": [L, L, L, I],
    "nmfb_ipm_persist": [P, I, L, L, L] + [P] * 14 + [D] * 8 + [I, I, I] + [P] * 6 + [I, P, P],
    "nmfb_small_work_len": [L, L, L],
    "nmfb_small_direction": [P, P, P, P, P, P, L, L, L, D, D, D, D] + [P] * 19,
    "nmfb_small_step_refresh": [P, I, L, L, L] + [P] * 14 + [D, D, D, D, I, D, I, P, P, P, P, P],
    "nmfb_lowrank_factor": [P, P, L, P, P, P, P, P],
    "nmfb_lowrank_solve": [P, P, P, P, P, L, L, P, P, P, P, P, L, P],
}
RESTYPES = {"nmfb_dualprod_work_len": ctypes.c_long, "nmfb_nnls_ftab_len": ctypes.c_long, "nmfb_colprod_work_len": ctypes.c_long, "nmfb_rowprod_work_len": ctypes.c_long, "nmfb_atb_work_len": ctypes.c_long,
            "nmfb_launch_count": ctypes.c_ulonglong, "nmfb_last_cuda_error": ctypes.c_char_p, "nmfb_small_work_len": ctypes.c_long,
            "nmfb_persist_work_len": ctypes.c_long, "nmfb_grams_work_len": ctypes.c_long,
            "nmfb_term4_work_len": ctypes.c_long,
            "nmfb_stage1_persist_work_len": ctypes.c_long}

_lib = None


def header_symbols() -> list[str]:
    """Function names declared in include/nmfb200.h."""
    import re

    hdr = os.path.join(os.path.dirname(_HERE), "include", "nmfb200.h")
    with open(hdr) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(nmfb_[a-z0-9_]+)\s*\(", text)))


def load(path: str | None = None):
    """Load (once) and return the ctypes library object."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or SO_PATH
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} not found: build it with `python -m paper_2101_08431_b200._build` "
            "(there is no CPU fallback)")
    try:
        so = ctypes.CDLL(path)
    except OSError as exc:  # pragma: no cover - depends on the box
        raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
    for name, argt in SIGNATURES.items():
        fn = getattr(so, name)
        fn.argtypes = argt
        fn.restype = RESTYPES.get(name, ctypes.c_int)
    _lib = so
    return so


def call(name: str, *args) -> None:
    rc = getattr(load(), name)(*args)
    if rc != 0:
        raise NativeLibraryError(f"{name} returned {rc}")
