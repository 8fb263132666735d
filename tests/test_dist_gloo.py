"""Row-sharded (multi-GPU) decomposition checked on CPU with gloo, world_size 2.

The sharded solve reduces exactly the row contractions listed in
paper_2101_08431_b200/dist.py; here the oracle driver runs that decomposition on
two gloo ranks and must reproduce the single-process solve (same sweeps, same
passive sets, same Armijo decisions, factors to rounding).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2101_08431_b200.dist import Comm, row_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, M, X0, Y0, iters, barrier, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import driver as D

        D.set_schur_backend("numpy")
        comm = Comm.from_env()
        a, b = row_range(M.shape[0], world, rank)
        rep = D.run_two_stage(M[a:b], X0[a:b], Y0, tol_rel=1e-10,
                              ipm=D.IpmParams(fixed_iters=iters, barrier=barrier, hessian="paper"), comm=comm)
        out_q.put((rank, a, b, rep.X, rep.Yt, rep.stage1.sweeps, rep.stage1.pX, rep.stage1.pY,
                   rep.ipm.armijo_t, rep.ipm.flags, rep.objective, rep.kkt))
    finally:
        dist.destroy_process_group()


def test_row_range_partition():
    for n in (1, 7, 300, 3001):
        for w in (1, 2, 3, 8):
            spans = [row_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


@pytest.mark.parametrize("barrier", ["paper", "balanced"])
def test_sharded_two_stage_matches_single(barrier):
    from oracle import driver as D
    from paper_2101_08431_b200 import data

    M, X0, Y0, _, _ = data.peaks(300, 40, 3, 77)
    iters = 12
    D.set_schur_backend("numpy")
    try:
        ref = D.run_two_stage(M, X0, Y0, tol_rel=1e-10,
                              ipm=D.IpmParams(fixed_iters=iters, barrier=barrier, hessian="paper"))
    finally:
        D.set_schur_backend("c")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, X0, Y0, iters, barrier, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X = np.vstack([r[3] for r in res])
    pX = np.vstack([r[6] for r in res])
    for r in res:
        assert r[5] == ref.stage1.sweeps
        assert np.array_equal(r[7], ref.stage1.pY)
        assert r[8] == ref.ipm.armijo_t and r[9] == ref.ipm.flags
        assert np.abs(r[4] - ref.Yt).max() <= 1e-8 * np.abs(ref.Yt).max()
        assert abs(r[10] - ref.objective) <= 1e-9 * ref.objective
    assert np.array_equal(pX, ref.stage1.pX)
    assert np.abs(X - ref.X).max() <= 1e-8 * np.abs(ref.X).max()


def test_comm_flags_without_a_process_group():
    """Comm.single() is inactive and graph-capturable; a forced one-rank communicator is
    active (every collective of the sharded path is issued) and splits rows trivially."""
    from paper_2101_08431_b200.dist import Comm, row_range

    c = Comm.single()
    assert not c.active and c.root and c.graph_ok
    f = Comm(None, 1, 0, force=True)
    assert f.active and f.root and f.world == 1
    assert row_range(10, 1, 0) == (0, 10)
    assert [row_range(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
