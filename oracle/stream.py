"""oracle.stream -- TEST INFRASTRUCTURE ONLY: CPU restatement of the streaming
column-append session (BASELINE config c3).  The reference has no append API
(SURVEY.md section 3.2); the semantics frozen in DESIGN.md section 2 (item 8) are:

  * first chunk: two-stage solve from the seeded (X0, Y0[:, :m0]), cold carries;
  * append(M_new): new Y columns = NNLS(C = X, d = new columns of M) with warm
    mode 1 (the reference's "streaming chain", _kernels_numba.py:312-315),
    carries extended with their passive sets, then the two-stage solve warm
    from (X, Y) and the carries (stage-1 mode 2 from its first sweep);
  * one KKT scale for the whole session (frozen semantics 12): eps_abs = tol_rel *
    max(1, E_primal(X0, Y0)) of the FIRST chunk's seeded start, kept for every chunk
    (a warm start's own E_primal is below 1, which would turn the relative tolerance
    into an absolute 1e-10).
"""
from __future__ import annotations

import time

import numpy as np

from oracle import driver as D


class OracleStream:
    def __init__(self, M0, X0, Y0, tol_rel=1e-10, s1=None, ipm_factory=None):
        self.M = np.array(M0, dtype=np.float64)  # fp32 chunks are widened exactly
        self.tol_rel = tol_rel
        self.s1 = s1 or D.Stage1Config()
        self.ipm_factory = ipm_factory or D.IpmParams
        self.chunks = []
        t0 = time.perf_counter()
        self.e_scale = max(1.0, D.kkt_error_primal_only(
            np.asarray(X0, dtype=np.float64), np.ascontiguousarray(np.asarray(Y0).T), self.M))
        rep = D.run_two_stage(self.M, X0, Y0, tol_rel, self.s1, self.ipm_factory(),
                              e_scale=self.e_scale)
        self._keep(rep, time.perf_counter() - t0)

    def _keep(self, rep, secs):
        self.X, self.Yt = rep.X, rep.Yt
        self.pX, self.pY = rep.stage1.pX, rep.stage1.pY
        self.chunks.append((self.M.shape[1], secs, rep))

    def append(self, Mnew):
        t0 = time.perf_counter()
        Mnew = np.asarray(Mnew, dtype=np.float64)
        k = self.X.shape[1]
        ctc = self.X.T @ self.X
        ctb = Mnew.T @ self.X
        btb = np.einsum("ij,ij->j", Mnew, Mnew)
        tol = 1e-12 * np.maximum(1.0, np.abs(ctb).max(axis=1))
        y, p, ch, r2, st = D.K.nnls_batch(ctc, ctb, btb, np.zeros((Mnew.shape[1], k), bool), 1,
                                          tol, 3 * k)
        D._raise_status(st, "stream append")
        self.M = np.hstack([self.M, Mnew])
        Yt = np.vstack([self.Yt, y])
        pY = np.vstack([self.pY, p])
        rep = D.run_two_stage(self.M, self.X, Yt.T, self.tol_rel, self.s1, self.ipm_factory(),
                              pX=self.pX, pY=pY, e_scale=self.e_scale)
        self._keep(rep, time.perf_counter() - t0)
        return rep
