"""c4 IPM iteration under a (one-rank, forced) NCCL communicator: CUDA-graph replay with the
collectives captured vs the eager path (NMFB_COMM_GRAPHS=0).

python scripts/comm_graphs.py
"""
import os
import sys

sys.path.insert(0, ".")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
os.environ["NMFB_FORCE_COMM"] = "1"
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2101_08431_b200 import data, solver  # noqa: E402
from paper_2101_08431_b200.config import IpmParams, Stage1Config  # noqa: E402
from paper_2101_08431_b200.dist import Comm  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
cfg = data.CONFIGS["c4"]
M, X0, Y0, _, _ = data.make(cfg)
comm = Comm.from_env()
P = solver.Problem(M, cfg.k, comm=comm)
X, Yt, _, _, _ = solver.run_stage1(P, P.to_dev(X0), P.to_dev(Y0.T), Stage1Config(fixed_sweeps=5))
for rep in range(2):
    Xs, Yts, R, S, mu, rho = solver.transition(P, X.clone(), Yt.clone(), 1e-7)
    solver.run_ipm(P, Xs, Yts, R, S, mu, rho, IpmParams(fixed_iters=3))
    Xs, Yts, R, S, mu, rho = solver.transition(P, X.clone(), Yt.clone(), 1e-7)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, r = solver.run_ipm(P, Xs, Yts, R, S, mu, rho, IpmParams(fixed_iters=20))
    e1.record()
    torch.cuda.synchronize()
print(f"graphs {'on' if comm.graph_ok else 'off'}: {e0.elapsed_time(e1) / 20:.3f} ms per IPM iteration "
      f"(graph kernel launches {P.graph_kernel_launches}), objective {r.trace[-1][1]:.6e}")
dist.destroy_process_group()
