"""Streaming column-append session (BASELINE config c3) on the B200.

The reference has no append API; semantics are frozen in
DESIGN.md (item 8) and restated by oracle/stream.py for the parity tests:

  * the first chunk is a two-stage solve from (X0, Y0) with cold carries;
  * ``append(M_new)`` initialises the new Y columns with one batched NNLS
    (C = X, d = the new columns; warm mode 1, the reference's streaming chain,
    _kernels_numba.py:312-315), extends the passive-set carries and re-runs the
    two-stage solve warm from (X, Y) and the carries (stage-1 mode 2 from sweep 0).

Device residency: one ``Problem`` for the whole session with room for ``m_max`` columns
(M in two pre-allocated n x m_max buffers, every scratch buffer sized for m_max; an
append moves M once into the other buffer behind which the new columns land, and
advances the row / column norms by the new block only); X, Y and the passive-set
carries stay on the device between chunks.  Chunks may be fp32 or fp64 (converted on
the device to the session's storage type).

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
                 ipm_factory=IpmParams, m_max: int | None = None, dtype=torch.float64):
        self.tol_rel = tol_rel
        self.cfg = cfg or Stage1Config()
        self.ipm_factory = ipm_factory
        dev = torch.device("cuda", torch.cuda.current_device())
        M0 = torch.as_tensor(np.ascontiguousarray(M0)) if isinstance(M0, np.ndarray) else M0
        M0 = M0.to(dev, dtype=dtype)
        self.n = M0.shape[0]
        self.k = np.asarray(X0).shape[1] if not isinstance(X0, torch.Tensor) else X0.shape[1]
        self.chunks = []
        t0 = time.perf_counter()
        cap = max(int(m_max or 0), 2 * M0.shape[1])
        self.P = solver.Problem(M0, self.k, m_capacity=cap)
        # one KKT scale for the session (frozen semantics 12, oracle/stream.py): the first
        # chunk's seeded start; a warm start's own E_primal < 1 would make tol_rel absolute
        Xd = self.P.to_dev(X0)
        Ytd = self.P.to_dev(Y0.T if not isinstance(Y0, torch.Tensor) else Y0.t())
        self.e_scale = max(1.0, solver.kkt_error_primal_only_dev(self.P, Xd, Ytd)[0])
        rep = solver.run_two_stage(None, X0, Y0, tol_rel, self.cfg, self.ipm_factory(),
                                   problem=self.P, e_scale=self.e_scale)
        torch.cuda.synchronize()
        self._keep(rep, time.perf_counter() - t0)

    def _keep(self, rep, secs):
        d = rep.dev_state
        self.X, self.Yt, self.pX, self.pY = d["X"], d["Yt"], d["pX"], d["pY"]
        self.chunks.append((self.P.m, secs, rep))

    @property
    def m(self):
        return self.P.m

    @property
    def Md(self):
        return self.P.M

    def _grow(self, extra):
        """Capacity exceeded: one new Problem with twice the room (rare)."""
        P = self.P
        self.P = solver.Problem(P.M, self.k, m_capacity=2 * (P.m + extra))

    def append(self, Mnew):
        """Add columns (n, c) -- host or device, fp32 or fp64 -- and re-solve warm;
        returns the chunk's SolveReport."""
        t0 = time.perf_counter()
        c = Mnew.shape[1]
        if self.P.m + c > self.P.m_cap:
            self._grow(c)
        P, k = self.P, self.k
        m0 = P.m
        Mn = P.append_columns(Mnew)  # (n, c) on the device in the storage type
        X = self.X
        ctc, ctb, tol = P.buf(k, k), P.buf(c, k), P.buf(c)
        P.colprod(X, self.n, k, X, k, ctc)
        P.colprod(Mn, self.n, c, X, k, ctb, tol, P.f32)
        y, p = P.buf(c, k), P.buf(c, k, dtype=torch.uint8)
        ch, r2 = P.buf(c, dtype=torch.int64), P.buf(c)
        st = P.buf(c, dtype=torch.int8)
        seed = torch.zeros((c, k), dtype=torch.uint8, device=P.dev)
        flag = P.buf(1, dtype=torch.int32)
        _p = solver._p
        P._call("nmfb_surface_nnls_batch", _p(ctc), _p(ctb), _p(P.col_n2[m0:]), _p(seed), 1,
                _p(tol), 3 * k, c, k, _p(y), _p(p), _p(ch), _p(r2), _p(st), _p(seed), _p(flag),
                P.stream)
        bad = torch.nonzero(st).flatten()
        if bad.numel():
            i = int(bad[0])
            raise status_error(int(st[i]), i, "stream append")
        Yt = torch.cat([self.Yt, y])
        pY = torch.cat([self.pY, p]) if self.pY is not None else None
        rep = solver.run_two_stage(None, X, Yt.t(), self.tol_rel, self.cfg, self.ipm_factory(),
                                   pX=self.pX, pY=pY, problem=P, e_scale=self.e_scale)
        torch.cuda.synchronize()
        self._keep(rep, time.perf_counter() - t0)
        return rep


__all__ = ["StreamSession", "_lib"]
