"""The row-sharded device solver (dist.Comm) on one GPU: two ranks, gloo transport.

NCCL cannot place two ranks on one GPU, so the collectives go through gloo
(host-staged, no device-side waiting between ranks); every kernel is the
production kernel.  The sharded solve must reproduce the single-GPU solve.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, X0, Y0, iters, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2101_08431_b200 import solver
        from paper_2101_08431_b200.config import IpmParams
        from paper_2101_08431_b200.dist import Comm, row_range

        comm = Comm.from_env()
        a, b = row_range(M.shape[0], world, rank)
        rep = solver.run_two_stage(M[a:b], X0[a:b], Y0, tol_rel=1e-10,
                                   ipm=IpmParams(fixed_iters=iters, hessian="paper"), comm=comm)
        q.put((rank, rep.X, rep.Yt, rep.stage1.sweeps, rep.ipm.armijo_t, rep.ipm.flags,
               rep.final_objective, rep.eps_abs))
    finally:
        dist.destroy_process_group()


def test_sharded_device_solver_matches_single():
    import torch.multiprocessing as mp

    from paper_2101_08431_b200 import data, solver
    from paper_2101_08431_b200.config import IpmParams

    M, X0, Y0, _, _ = data.peaks(600, 50, 3, 91)
    iters = 15
    ref = solver.run_two_stage(M, X0, Y0, tol_rel=1e-10, ipm=IpmParams(fixed_iters=iters, hessian="paper"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, X0, Y0, iters, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    X = np.vstack([r[1] for r in res])
    for r in res:
        assert r[3] == ref.stage1.sweeps
        assert r[4] == ref.ipm.armijo_t and r[5] == ref.ipm.flags
        assert abs(r[7] - ref.eps_abs) <= 1e-12 * ref.eps_abs
        assert np.abs(r[2] - ref.Yt).max() <= 1e-7 * np.abs(ref.Yt).max()
        assert abs(r[6] - ref.final_objective) <= 1e-7 * ref.final_objective
    assert np.abs(X - ref.X).max() <= 1e-7 * np.abs(ref.X).max()


def _nccl_worker(rank, world, port, M, X0, Y0, sweeps, iters, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        from paper_2101_08431_b200 import solver
        from paper_2101_08431_b200.config import IpmParams, Stage1Config
        from paper_2101_08431_b200.dist import Comm, row_range

        comm = Comm.from_env()
        a, b = row_range(M.shape[0], world, rank)
        rep = solver.run_two_stage(M[a:b], X0[a:b], Y0, tol_rel=1e-10,
                                   s1=Stage1Config(fixed_sweeps=sweeps),
                                   ipm=IpmParams(fixed_iters=iters), comm=comm)
        q.put((rank, rep.X, rep.Yt, rep.stage1.sweeps, rep.ipm.armijo_t, rep.ipm.flags,
               rep.final_objective, rep.stage1.pX, rep.stage1.pY))
    finally:
        dist.destroy_process_group()


def test_nccl_two_gpus_c4_slice_matches_single():
    """Row-sharded solve over NCCL on two GPUs (bench.py --gpus 2's path) on a c4-shaped
    slice that takes the TMA products and the residual-free IPM: same sweeps, passive sets
    and Armijo decisions as one GPU.  Skipped on single-GPU boxes."""
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (NCCL cannot place two ranks on one device)")
    from paper_2101_08431_b200 import data, solver
    from paper_2101_08431_b200.config import IpmParams, Stage1Config

    M, X0, Y0, _, _ = data.dense(8192, 4096, 10, 7)
    sweeps, iters = 8, 6
    ref = solver.run_two_stage(M, X0, Y0, tol_rel=1e-10, s1=Stage1Config(fixed_sweeps=sweeps),
                               ipm=IpmParams(fixed_iters=iters))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, M, X0, Y0, sweeps, iters, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=900) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(np.vstack([r[7] for r in res]), ref.stage1.pX)
    for r in res:
        assert r[3] == ref.stage1.sweeps
        assert np.array_equal(r[8], ref.stage1.pY)
        assert r[4] == ref.ipm.armijo_t and r[5] == ref.ipm.flags
        assert abs(r[6] - ref.final_objective) <= 1e-9 * ref.final_objective
    X = np.vstack([r[1] for r in res])
    assert np.abs(X - ref.X).max() <= 1e-8 * np.abs(ref.X).max()


def _nccl_one_rank_worker(port, M, X0, Y0, sweeps, iters, f32, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["NMFB_FORCE_COMM"] = "1"
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2101_08431_b200 import solver
        from paper_2101_08431_b200.config import IpmParams, Stage1Config
        from paper_2101_08431_b200.dist import Comm

        comm = Comm.from_env()
        assert comm.active and comm.world == 1
        Md = torch.as_tensor(M).cuda()
        if f32:
            Md = Md.float()
        P = solver.Problem(Md, X0.shape[1], comm=comm)
        rep = solver.run_two_stage(None, X0, Y0, tol_rel=1e-10,
                                   s1=Stage1Config(fixed_sweeps=sweeps),
                                   ipm=IpmParams(fixed_iters=iters), comm=comm, problem=P)
        # the Gauss-Newton iterations replay CUDA graphs with the NCCL collectives captured
        assert comm.graph_ok and P.graph_kernel_launches > 0
        q.put((rep.X, rep.Yt, rep.stage1.sweeps, rep.ipm.armijo_t, rep.ipm.flags,
               rep.final_objective, rep.stage1.pX, rep.stage1.pY))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape", [("c4", 8192, 4096, 10, False), ("c2", 1200, 80, 3, False),
                                   ("c5", 6000, 3000, 16, True)])
def test_nccl_one_rank_sharded_path_matches_single(shape):
    """Every collective of the row-sharded solve issued through NCCL on this GPU (a one-rank
    communicator with Comm.force): the sums, minima, maxima and the all-gather of the column-
    split Y-side NNLS run on the device stream exactly as bench.py --gpus N issues them, and
    the solve reproduces the unsharded one (same sweeps, passive sets, Armijo decisions)."""
    import torch
    import torch.multiprocessing as mp

    from paper_2101_08431_b200 import data, solver
    from paper_2101_08431_b200.config import IpmParams, Stage1Config

    name, n, m, k, f32 = shape
    M, X0, Y0, _, _ = (data.dense(n, m, k, 7) if name != "c2" else data.peaks(n, m, k, 92))
    sweeps, iters = 6, 6
    Md = torch.as_tensor(M).cuda()
    ref = solver.run_two_stage(Md.float() if f32 else Md, X0, Y0, tol_rel=1e-10,
                               s1=Stage1Config(fixed_sweeps=sweeps), ipm=IpmParams(fixed_iters=iters))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_one_rank_worker, args=(_port(), M, X0, Y0, sweeps, iters, f32, q))
    p.start()
    r = q.get(timeout=900)
    p.join(timeout=120)
    assert p.exitcode == 0
    tol = 1e-4 if f32 else 1e-8
    assert r[2] == ref.stage1.sweeps
    if not f32:
        assert np.array_equal(r[6], ref.stage1.pX) and np.array_equal(r[7], ref.stage1.pY)
        assert r[3] == ref.ipm.armijo_t and r[4] == ref.ipm.flags
    assert abs(r[5] - ref.final_objective) <= tol * ref.final_objective
    assert np.abs(r[0] - ref.X).max() <= tol * np.abs(ref.X).max()
    assert np.abs(r[1] - ref.Yt).max() <= tol * np.abs(ref.Yt).max()
