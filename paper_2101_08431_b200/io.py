"""Host-side data I/O of the solve path.

Matrices enter the device path as dense row-major arrays; this module reads and
writes the reference's documented text formats and applies its preprocessing.
Nothing here touches the GPU.

* ``load_matrix`` / ``save_matrix`` -- CSV or whitespace-delimited decimal text, one
  matrix row per line, optional header line; writes 17 significant digits so a
  save -> load round trip is exact.
* ``shift_nonnegative`` -- per-column or per-row shift by the opposite of a negative
  minimum (PAPER section 5.2).
* ``generate_synthetic`` -- the paper's synthetic family (PAPER section 5.4: X, Y ~
  U(0,1), M = max(XY + N(0, noise_std^2), 0)), PCG64, draw order X, Y, noise.
"""
from __future__ import annotations

import numpy as np

from .errors import ParseError, RaggedRows


def load_matrix(path, format: str = "csv", header: bool = False) -> np.ndarray:
    """SPEC.md:471 load_matrix(path, format in {csv, whitespace}) -> (n, m) float64."""
    if format not in ("csv", "whitespace"):
        raise ValueError(f"unknown format {format!r}")
    rows, width = [], None
    with open(path, "r") as fh:
        for ln, line in enumerate(fh, start=1):
            if header and ln == 1:
                continue
            text = line.strip()
            if not text:
                continue
            cells = [c.strip() for c in text.split(",")] if format == "csv" else text.split()
            vals = []
            for col, c in enumerate(cells, start=1):
                try:
                    vals.append(float(c))
                except ValueError:
                    raise ParseError(f"not a decimal real: {c!r} (line {ln}, column {col})", ln, col) from None
            if width is None:
                width = len(vals)
            elif len(vals) != width:
                raise RaggedRows(f"expected {width} values, found {len(vals)} (line {ln})", ln)
            rows.append(vals)
    if not rows:
        raise ParseError("empty matrix file", 1, 1)
    return np.asarray(rows, dtype=np.float64)


def save_matrix(path, M, format: str = "csv") -> None:
    """Write M with 17 significant digits (exact round trip through load_matrix)."""
    sep = "," if format == "csv" else " "
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2:
        raise ValueError("save_matrix expects a 2-D array")
    with open(path, "w") as fh:
        for row in M:
            fh.write(sep.join(format_real(v) for v in row))
            fh.write("\n")


def format_real(v: float) -> str:
    return f"{float(v):.17g}"


def shift_nonnegative(M, axis: str = "column") -> np.ndarray:
    """per slice along ``axis``, add -min when min < 0 (others unchanged)."""
    M = np.array(M, dtype=np.float64, copy=True)
    if axis not in ("column", "row"):
        raise ValueError(f"axis must be 'column' or 'row', got {axis!r}")
    ax = 0 if axis == "column" else 1
    lo = M.min(axis=ax, keepdims=True)
    M -= np.where(lo < 0.0, lo, 0.0)
    return M


def generate_synthetic(n: int, m: int, k_true: int, noise_std: float, seed: int):
    """SPEC.md:488 generate_synthetic -> (M, X_true, Y_true): the paper's section 5.4 family."""
    if min(n, m, k_true) < 1 or noise_std < 0:
        raise ValueError("n, m, k_true >= 1 and noise_std >= 0 required")
    rng = np.random.Generator(np.random.PCG64(seed))
    X = rng.uniform(0.0, 1.0, (n, k_true))
    Y = rng.uniform(0.0, 1.0, (k_true, m))
    M = X @ Y
    if noise_std > 0:
        M = M + rng.standard_normal((n, m)) * noise_std
    return np.maximum(M, 0.0), X, Y


__all__ = ["load_matrix", "save_matrix", "shift_nonnegative", "generate_synthetic",
           "format_real"]
