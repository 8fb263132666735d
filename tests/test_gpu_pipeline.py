"""SolvePipeline (two resident problem slots, next instance's H2D under the current solve):
the solves are run_two_stage on the slot, so every instance must reproduce its direct solve."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("f32", [False, True])
def test_pipeline_matches_direct_solves(f32):
    import torch

    from paper_2101_08431_b200 import SolvePipeline, data, solver
    from paper_2101_08431_b200.config import IpmParams, Stage1Config

    n, m, k = 4096, 2048, 10
    insts = [data.dense(n, m, k, 20 + s)[:3] for s in range(4)]
    dt = torch.float32 if f32 else torch.float64
    kw = dict(tol_rel=1e-10, s1=Stage1Config(fixed_sweeps=5), ipm=IpmParams(fixed_iters=4))
    ref = []
    for M, X0, Y0 in insts:
        Md = torch.as_tensor(M).to("cuda", dtype=dt)
        ref.append(solver.run_two_stage(Md, X0, Y0, tol_rel=1e-10, s1=Stage1Config(fixed_sweeps=5),
                                        ipm=IpmParams(fixed_iters=4)))
    pipe = SolvePipeline(n, m, k, dtype=dt, **kw)
    host = [torch.from_numpy(M).to(dt).pin_memory() for M, _, _ in insts]
    got = []
    pipe.submit(host[0], insts[0][1], insts[0][2])
    for i in range(len(insts)):
        if i + 1 < len(insts):
            pipe.submit(host[i + 1], insts[i + 1][1], insts[i + 1][2])
        got.append(pipe.result())
    assert pipe.h2d_bytes >= sum(h.numel() * h.element_size() for h in host)
    for a, b in zip(got, ref):
        assert a.stage1.sweeps == b.stage1.sweeps and a.ipm.armijo_t == b.ipm.armijo_t
        assert np.array_equal(a.stage1.pX, b.stage1.pX) and np.array_equal(a.stage1.pY, b.stage1.pY)
        assert np.array_equal(a.X, b.X) and np.array_equal(a.Yt, b.Yt)
        assert a.final_objective == b.final_objective


def test_pipeline_slot_accounting():
    import torch

    from paper_2101_08431_b200 import SolvePipeline, data
    from paper_2101_08431_b200.config import IpmParams, Stage1Config

    M, X0, Y0, _, _ = data.peaks(300, 40, 3, 5)
    pipe = SolvePipeline(300, 40, 3, s1=Stage1Config(fixed_sweeps=2), ipm=IpmParams(fixed_iters=2))
    with pytest.raises(RuntimeError):
        pipe.result()
    pipe.submit(M, X0, Y0)
    pipe.submit(M, X0, Y0)
    with pytest.raises(RuntimeError):
        pipe.submit(M, X0, Y0)
    with pytest.raises(ValueError):
        SolvePipeline(300, 40, 3).submit(M[:, :10], X0, Y0[:, :10])
    a, b = pipe.result(), pipe.result()
    assert np.array_equal(a.X, b.X)
    torch.cuda.synchronize()
