"""data-io and SolveReport emission: host-only checks."""
import json
import math

import numpy as np
import pytest

from paper_2101_08431_b200 import io
from paper_2101_08431_b200.errors import ParseError, RaggedRows


def test_load_matrix_examples(tmp_path):
    p = tmp_path / "a.csv"
    p.write_text("1,2\n3,4\n")
    assert np.array_equal(io.load_matrix(p, "csv"), [[1, 2], [3, 4]])
    q = tmp_path / "b.txt"
    q.write_text("1 2 3\n")
    assert io.load_matrix(q, "whitespace").shape == (1, 3)
    r = tmp_path / "c.csv"
    r.write_text("1,2\n3\n")
    with pytest.raises(RaggedRows) as ei:
        io.load_matrix(r, "csv")
    assert ei.value.line == 2
    s = tmp_path / "d.csv"
    s.write_text("1,x\n")
    with pytest.raises(ParseError) as ei:
        io.load_matrix(s, "csv")
    assert (ei.value.line, ei.value.column) == (1, 2)
    h = tmp_path / "e.csv"
    h.write_text("a,b\n5,6\n")
    assert np.array_equal(io.load_matrix(h, "csv", header=True), [[5, 6]])


def test_save_load_round_trip_exact(tmp_path):
    rng = np.random.default_rng(3)
    M = rng.standard_normal((7, 5)) * 10.0 ** rng.integers(-300, 300, (7, 5))
    for fmt in ("csv", "whitespace"):
        p = tmp_path / f"m.{fmt}"
        io.save_matrix(p, M, fmt)
        assert np.array_equal(io.load_matrix(p, fmt), M)


def test_shift_nonnegative_examples():
    assert np.array_equal(io.shift_nonnegative([[-0.5], [1.0]], "column"), [[0.0], [1.5]])
    A = np.array([[0.0, 2.0], [1.0, 3.0]])
    assert np.array_equal(io.shift_nonnegative(A, "column"), A)
    assert np.array_equal(io.shift_nonnegative([[-2.0], [-1.0]], "column"), [[0.0], [1.0]])
    assert np.array_equal(io.shift_nonnegative([[-2.0, -1.0]], "row"), [[0.0, 1.0]])


def test_generate_synthetic_examples():
    M, X, Y = io.generate_synthetic(10, 4, 2, 0.0, 7)
    assert np.array_equal(M, X @ Y) and (M >= 0).all()
    M2, _, _ = io.generate_synthetic(10, 4, 2, 0.0, 7)
    assert np.array_equal(M, M2)
    M3, _, _ = io.generate_synthetic(2000, 50, 3, 0.1, 11)
    assert (M3 >= 0).all() and abs(M3.mean() - 0.75) < 0.05


def test_trace_records_and_report(tmp_path):
    from paper_2101_08431_b200 import report
    from paper_2101_08431_b200.config import IpmResult, SolveReport, Stage1Result

    s1 = Stage1Result(np.ones((3, 2)), np.ones((4, 2)), None, None, 2, True,
                      [(0.1, 5.0, 1.0), (0.1, 4.0, 0.5)])
    ip = IpmResult(2, 1, True, 1e-9, 1e-3, False,
                   trace=[(0.0, 3.0, 1e-3, 1e-2, 1, 1, 0), (0.2, 2.0, 1e-9, 1e-3, 1, 1, 0)],
                   armijo_t=[0, 0], flags=[False, True])
    rep = SolveReport("Converged", np.ones((3, 2)), np.ones((4, 2)), None, None, 2.0, 1e-9, 1e-8,
                      s1, ip, 0.3, 0.2)
    recs = report.trace_records(rep)
    times = [r[0] for r in recs]
    assert all(b > a for a, b in zip(times, times[1:]))
    assert [r[1] for r in recs] == ["anls", "anls", "ipm", "ipm"]
    assert recs[-1][5] is True and math.isnan(recs[0][3])
    j, c = report.write_report(rep, str(tmp_path), "x")
    d = json.load(open(j))
    assert d["status"] == "Converged" and d["full_hessian_iterations"] == 1
    lines = open(c).read().strip().split("\n")
    assert lines[0] == ",".join(report.CSV_COLUMNS) and len(lines) == 5
