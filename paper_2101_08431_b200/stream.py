"""Streaming column-append session (BASELINE config c3) on the B200.

The reference has no append API; semantics are frozen in
DESIGN.md (item 8) and restated by oracle/stream.py for the parity tests:

  * the first chunk is a two-stage solve from (X0, Y0) with cold carries;
  * ``append(M_new)`` initialises the new Y columns with one batched NNLS
    (C = X, d = the new columns; warm mode 1, the reference's streaming chain,
    _kernels_numba.py:312-315), extends the passive-set carries and re-runs the
    two-stage solve warm from (X, Y) and the carries (stage-1 mode 2 from sweep 0).

Per-chunk wall times are recorded in ``chunks`` as (m, seconds, SolveReport).
"""
from __future__ import annotations

import time

import numpy as np
import torch

from . import _lib, solver
from .config import IpmParams, Stage1Config
from .errors import status_error


class StreamSession:
    def __init__(self, M0, X0, Y0, tol_rel=1e-10, cfg: Stage1Config | None = None,
                 ipm_factory=IpmParams):
        self.tol_rel = tol_rel
        self.cfg = cfg or Stage1Config()
        self.ipm_factory = ipm_factory
        dev = torch.device("cuda", torch.cuda.current_device())
        self.Md = torch.as_tensor(np.ascontiguousarray(M0, dtype=np.float64)).to(dev)
        self.n = self.Md.shape[0]
        self.k = np.asarray(X0).shape[1]
        self.chunks = []
        t0 = time.perf_counter()
        P = solver.Problem(self.Md, self.k)
        rep = solver.run_two_stage(self.Md, X0, Y0, tol_rel, self.cfg, self.ipm_factory(),
                                   problem=P)
        torch.cuda.synchronize()
        self._keep(rep, time.perf_counter() - t0)

    def _keep(self, rep, secs):
        self.X, self.Yt = rep.X, rep.Yt
        self.pX, self.pY = rep.stage1.pX, rep.stage1.pY
        self.chunks.append((self.Md.shape[1], secs, rep))

    @property
    def m(self):
        return self.Md.shape[1]

    def append(self, Mnew):
        """Add columns (n, c) and re-solve warm; returns the chunk's SolveReport."""
        t0 = time.perf_counter()
        dev = self.Md.device
        Mn = torch.as_tensor(np.ascontiguousarray(Mnew, dtype=np.float64)).to(dev)
        c, k = Mn.shape[1], self.k
        Pn = solver.Problem(Mn, k)  # btb = column norms of the new block
        X = Pn.to_dev(self.X)
        ctc, ctb, tol = Pn.buf(k, k), Pn.buf(c, k), Pn.buf(c)
        Pn.colprod(X, self.n, k, X, k, ctc)
        Pn.colprod(Mn, self.n, c, X, k, ctb, tol)
        y, p = Pn.buf(c, k), Pn.buf(c, k, dtype=torch.uint8)
        ch, r2 = Pn.buf(c, dtype=torch.int64), Pn.buf(c)
        st = Pn.buf(c, dtype=torch.int8)
        seed, flag = torch.zeros((c, k), dtype=torch.uint8, device=dev), Pn.buf(1, dtype=torch.int32)
        _p = solver._p
        Pn._call("nmfb_surface_nnls_batch", _p(ctc), _p(ctb), _p(Pn.col_n2), _p(seed), 1, _p(tol),
                 3 * k, c, k, _p(y), _p(p), _p(ch), _p(r2), _p(st), _p(seed), _p(flag), Pn.stream)
        bad = torch.nonzero(st).flatten()
        if bad.numel():
            i = int(bad[0])
            raise status_error(int(st[i]), i, "stream append")
        self.Md = torch.cat([self.Md, Mn], dim=1).contiguous()
        Yt = np.vstack([self.Yt, y.cpu().numpy()])
        pY = np.vstack([self.pY, p.bool().cpu().numpy()])
        P = solver.Problem(self.Md, k)
        rep = solver.run_two_stage(self.Md, self.X, Yt.T, self.tol_rel, self.cfg,
                                   self.ipm_factory(), pX=self.pX, pY=pY, problem=P)
        torch.cuda.synchronize()
        self._keep(rep, time.perf_counter() - t0)
        return rep


__all__ = ["StreamSession", "_lib"]
