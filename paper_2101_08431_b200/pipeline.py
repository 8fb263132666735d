"""Back-to-back two-stage solves of same-shaped problems with the next problem's data on
its way to the GPU while the current one is being solved.

The reference solves one instance per call (SPEC.md:411 run_two_stage); a caller with a
queue of instances (the Table III harness, solves ten seeds per size)
pays one host-to-device copy of M per instance.  ``SolvePipeline`` keeps two resident
``Problem`` slots: ``submit`` starts the copy of an instance into the free slot on a copy
stream (pinned host memory -> HBM by the copy engine, no SM work), ``result`` solves the
oldest submitted instance on the compute stream once its copy has landed.  With one
instance submitted ahead, the copy of instance i+1 runs under the solve of instance i.

    pipe = SolvePipeline(n, m, k)
    pipe.submit(M0, X0, Y0)
    for M1, X1, Y1 in rest:
        pipe.submit(M1, X1, Y1)     # H2D of the next instance, asynchronous
        rep = pipe.result()         # solve of the previous one
    rep = pipe.result()

Every solve is ``solver.run_two_stage(problem=slot)``: the same kernels, the same results.
"""
from __future__ import annotations

import collections

import numpy as np
import torch

from . import solver
from .dist import Comm
from .errors import NativeLibraryError


class SolvePipeline:
    def __init__(self, n, m, k, dtype=torch.float64, comm: Comm | None = None, depth: int = 2,
                 **solve_kw):
        """``solve_kw``: keyword arguments of run_two_stage (tol_rel, s1, ipm, tp, e_scale...)."""
        if not torch.cuda.is_available():
            raise NativeLibraryError("no CUDA device: the B200 solver has no CPU fallback")
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.n, self.m, self.k = int(n), int(m), int(k)
        self.solve_kw = solve_kw
        self.copy_stream = torch.cuda.Stream(self.dev)
        zero = torch.zeros((self.n, self.m), dtype=dtype, device=self.dev)
        self.slots = [solver.Problem(zero if i == 0 else zero.clone(), k, comm=comm)
                      for i in range(max(2, int(depth)))]
        self.free = collections.deque(range(len(self.slots)))
        self.pending = collections.deque()  # (slot, copied event, X0, Y0, per-job kwargs)
        self.idle = [None] * len(self.slots)  # compute-stream event: the slot's last solve ended
        self.h2d_bytes = 0

    def submit(self, M, X0, Y0, **kw):
        """Start the host-to-device copy of M (pinned host tensor / array, or a device tensor)
        into a free slot; returns immediately."""
        if not self.free:
            raise RuntimeError("SolvePipeline: every slot holds an unsolved instance; call result()")
        if isinstance(M, np.ndarray):
            M = torch.from_numpy(np.ascontiguousarray(M))
        i = self.free.popleft()
        P = self.slots[i]
        if tuple(M.shape) != (P.n, P.m):
            self.free.appendleft(i)
            raise ValueError(f"submit: shape {tuple(M.shape)} != {(P.n, P.m)}")
        cs = self.copy_stream
        if self.idle[i] is not None:
            cs.wait_event(self.idle[i])  # never overwrite M under a running solve
        with torch.cuda.stream(cs):
            # row blocks of ~32 MB: small transfers of the running solve (scalars, factors)
            # interleave with the bulk copy instead of queueing behind all of it
            rows = max(1, (32 << 20) // max(1, M.shape[1] * M.element_size()))
            for r0 in range(0, P.n, rows):
                src = M[r0:r0 + rows]
                if src.dtype != P.M.dtype:
                    src = src.to(self.dev, non_blocking=True)
                P.M[r0:r0 + rows].copy_(src, non_blocking=True)
            X0 = self._stage(X0)
            Y0 = self._stage(Y0)
            done = torch.cuda.Event()
            done.record(cs)
        if not M.is_cuda:
            self.h2d_bytes += M.numel() * M.element_size()
        self.pending.append((i, done, X0, Y0, kw))

    def _stage(self, a):
        """Initial factors to the device on the copy stream (Y0 (k, m) is kept as passed)."""
        if isinstance(a, torch.Tensor):
            t = a if a.is_cuda else a.pin_memory()
        else:
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).pin_memory()
        if not t.is_cuda:
            self.h2d_bytes += t.numel() * t.element_size()
        return t.to(self.dev, dtype=torch.float64, non_blocking=True)

    def result(self):
        """Solve the oldest submitted instance (waits for its copy on the device, not the
        host) and return its SolveReport."""
        if not self.pending:
            raise RuntimeError("SolvePipeline: nothing submitted")
        i, done, X0, Y0, kw = self.pending.popleft()
        P = self.slots[i]
        st = torch.cuda.current_stream(self.dev)
        st.wait_event(done)
        P.refresh_norms()
        args = dict(self.solve_kw)
        args.update(kw)
        rep = solver.run_two_stage(None, X0, Y0, problem=P, **args)
        ev = torch.cuda.Event()
        ev.record(st)
        self.idle[i] = ev
        self.free.append(i)
        return rep


__all__ = ["SolvePipeline"]
