"""Row sharding of M across the GPUs of one node.

Rows of M (and of X, R, F, graX, the R1 factors) are partitioned in
contiguous blocks; Y, S, graY and every k- or k^2-sized quantity are
replicated.  The exchanges are exactly the contractions over rows:

  stage 1, per sweep   X^T X (k x k) and X^T M (m x k)            sum
                       step / norm statistics (X part)             sum
                       NNLS status scan                            min
  stage 2, per iter    ||F||^2, graY = F^T X, X^T X, H, Z          sum
                       [full Hessian] W = F^T P, term-4 of A       sum
                       KKT / Armijo / affine sums (X part)          sum
                       fraction-to-boundary minima                 min
                       maxima for the transition                   max

The Y-side NNLS of stage 1 is split by columns: every rank solves the columns
row_range(m, world, rank) of the all-reduced X^T M and the columns (with their
passive sets, residuals and statuses) are all-gathered (north_star: "each solves
m/p ... followed by an allgather").  The stage-2 reduced (k^2 capacitance or dense
mk) solve and the replicated updates run redundantly on every rank with identical
inputs, so their (deterministic) results are identical everywhere and need no
broadcast.  ``Comm`` wraps torch.distributed (NCCL on GPUs, gloo on CPU);
``Comm.single()`` is the no-op used on one GPU.
"""
from __future__ import annotations

import torch


def row_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of rows owned by ``rank`` (sizes differ by at most 1)."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


class Comm:
    def __init__(self, group=None, world: int = 1, rank: int = 0, force: bool = False):
        # force: treat a one-rank group as sharded, so that every collective of the sharded
        # path is issued (a one-GPU box exercising the NCCL path: tests/test_gpu_dist.py)
        self.group, self.world, self.rank, self.force = group, world, rank, bool(force)

    @classmethod
    def single(cls):
        return cls(None, 1, 0)

    @classmethod
    def from_env(cls):
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            import os

            return cls(None, dist.get_world_size(), dist.get_rank(),
                       force=os.environ.get("NMFB_FORCE_COMM", "0") == "1")
        return cls.single()

    @property
    def active(self):
        return self.world > 1 or self.force

    @property
    def root(self):
        return self.rank == 0

    @property
    def graph_ok(self):
        """Collectives of this communicator can be captured into a CUDA graph (NCCL: they are
        stream-ordered kernels; gloo stages through the host and cannot)."""
        if not self.active:
            return True
        import os

        import torch.distributed as dist

        if os.environ.get("NMFB_COMM_GRAPHS", "1") == "0":
            return False
        try:
            return dist.get_backend(self.group) == "nccl"
        except Exception:  # noqa: BLE001
            return False

    def _ar(self, t: torch.Tensor, op):
        if not self.active or t.numel() == 0:
            return t
        import torch.distributed as dist

        dist.all_reduce(t, op=op, group=self.group)
        return t

    def sum_(self, t):
        import torch.distributed as dist

        return self._ar(t, dist.ReduceOp.SUM) if self.active else t

    def max_(self, t):
        import torch.distributed as dist

        return self._ar(t, dist.ReduceOp.MAX) if self.active else t

    def min_(self, t):
        import torch.distributed as dist

        return self._ar(t, dist.ReduceOp.MIN) if self.active else t

    def allgather_rows(self, t: torch.Tensor) -> torch.Tensor:
        """t (rows, ...): every rank filled rows row_range(rows, world, rank); afterwards
        every rank holds all rows (padded equal-size all_gather; NCCL or gloo)."""
        if not self.active or t.shape[0] == 0:
            return t
        import torch.distributed as dist

        rows = t.shape[0]
        chunk = (rows + self.world - 1) // self.world
        a, b = row_range(rows, self.world, self.rank)
        send = torch.zeros((chunk,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        send[: b - a] = t[a:b]
        recv = [torch.empty_like(send) for _ in range(self.world)]
        dist.all_gather(recv, send, group=self.group)
        for r in range(self.world):
            ar, br = row_range(rows, self.world, r)
            if r != self.rank:
                t[ar:br] = recv[r][: br - ar]
        return t

    def sum_float(self, v: float, device=None) -> float:
        if not self.active:
            return float(v)
        t = torch.tensor([float(v)], dtype=torch.float64, device=device)
        return float(self.sum_(t).item())
