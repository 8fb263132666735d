"""Streaming column append (config c3 semantics) on the GPU vs the oracle session."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_stream_parity_small():
    from oracle import driver as D
    from oracle import stream as OS
    from paper_2101_08431_b200 import data
    from paper_2101_08431_b200.config import IpmParams
    from paper_2101_08431_b200.stream import StreamSession

    M, X0, Y0, _, _ = data.peaks(600, 60, 4, 103)
    D.set_schur_backend("numpy")
    try:
        so = OS.OracleStream(M[:, :20], X0, Y0[:, :20], ipm_factory=lambda: D.IpmParams(fixed_iters=6, hessian="paper"))
        sg = StreamSession(M[:, :20], X0, Y0[:, :20], ipm_factory=lambda: IpmParams(fixed_iters=6, hessian="paper"))
        for m0 in range(20, 60, 10):
            so.append(M[:, m0:m0 + 10])
            sg.append(M[:, m0:m0 + 10])
    finally:
        D.set_schur_backend("c")
    assert len(so.chunks) == len(sg.chunks) == 5
    for (mo, _, ro), (mg, _, rg) in zip(so.chunks, sg.chunks):
        assert mo == mg
        assert ro.stage1.sweeps == rg.stage1.sweeps
        assert np.array_equal(ro.stage1.pY, rg.stage1.pY)
        assert ro.ipm.armijo_t == rg.ipm.armijo_t
        rel = np.abs(rg.Yt - ro.Yt).max() / np.abs(ro.Yt).max()
        assert rel < 1e-7, (mo, rel)


def test_stream_c3_dense_fallback_parity():
    """c3's second chunk under the paper barrier drifts until the rank-k^2
    capacitance loses positive definiteness by rounding; the device re-solves those
    iterations with the dense Schur system and must still follow the oracle (which
    always factors the dense system) decision for decision."""
    from oracle import driver as D
    from oracle import stream as OS
    from paper_2101_08431_b200 import data
    from paper_2101_08431_b200.config import IpmParams
    from paper_2101_08431_b200.stream import StreamSession

    cfg = data.CONFIGS["c3"]
    M, X0, Y0, _, _ = data.make(cfg)
    D.set_schur_backend("numpy")
    try:
        so = OS.OracleStream(M[:, :20], X0, Y0[:, :20],
                             ipm_factory=lambda: D.IpmParams(barrier="paper", hessian="paper"))
        sg = StreamSession(M[:, :20], X0, Y0[:, :20], ipm_factory=lambda: IpmParams(barrier="paper", hessian="paper"))
        so.append(M[:, 20:30])
        sg.append(M[:, 20:30])
    finally:
        D.set_schur_backend("c")
    rg, ro = sg.chunks[1][2], so.chunks[1][2]
    assert rg.ipm.dense_fallbacks > 0
    assert ro.ipm.armijo_t == rg.ipm.armijo_t
    rel = abs(rg.final_objective - ro.objective) / abs(ro.objective)
    assert rel < 1e-6, rel


def test_stream_c3_first_ten_chunks():
    """BASELINE c3, first 10 chunks (m = 20 -> 120) under the default barrier and Hessian
    rule, 15 IPM iterations per chunk, chunks fed as fp32 arrays (session storage fp64):
    one device-resident session (pre-allocated M, one Problem) against the oracle session
    on the same fp32-rounded columns -- same stage-1 sweeps and passive sets, same Armijo
    decisions, factors to 1e-7 per chunk."""
    import torch

    from oracle import driver as D
    from oracle import stream as OS
    from paper_2101_08431_b200 import data
    from paper_2101_08431_b200.config import IpmParams
    from paper_2101_08431_b200.stream import StreamSession

    cfg = data.CONFIGS["c3"]
    M, X0, Y0, _, _ = data.make(cfg)
    M32 = M.astype(np.float32)
    M64 = M32.astype(np.float64)
    m0, step = cfg.m_start, cfg.m_step
    D.set_schur_backend("numpy")
    try:
        so = OS.OracleStream(M64[:, :m0], X0, Y0[:, :m0],
                             ipm_factory=lambda: D.IpmParams(fixed_iters=15))
        sg = StreamSession(M32[:, :m0], X0, Y0[:, :m0], m_max=cfg.m,
                           ipm_factory=lambda: IpmParams(fixed_iters=15))
        P0 = sg.P
        for c in range(9):
            a = m0 + c * step
            so.append(M64[:, a:a + step])
            sg.append(M32[:, a:a + step])
    finally:
        D.set_schur_backend("c")
    assert sg.P is P0, "the session must keep one Problem (pre-allocated capacity)"
    assert sg.m == m0 + 9 * step == so.M.shape[1]
    assert torch.equal(sg.Md.cpu(), torch.as_tensor(M64[:, :sg.m]))
    for (mo, _, ro), (mg, _, rg) in zip(so.chunks, sg.chunks):
        assert mo == mg
        assert ro.stage1.sweeps == rg.stage1.sweeps, mo
        assert np.array_equal(ro.stage1.pY, rg.stage1.pY), mo
        assert ro.ipm.armijo_t == rg.ipm.armijo_t, mo
        rel = np.abs(rg.Yt - ro.Yt).max() / np.abs(ro.Yt).max()
        assert rel < 1e-7, (mo, rel)
