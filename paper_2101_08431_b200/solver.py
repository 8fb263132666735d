"""Device-resident two-stage NMF solver (the B200 hot path).

Host control flow follows the reference specification's drivers one for one
(PAPER Algorithms 1-3) and the frozen semantics listed in
DESIGN.md; every numeric step runs in libnmfb200.so through the C-ABI of
include/nmfb200.h.  The host reads back a handful of scalars per ANLS sweep
and two small scalar blocks per IPM iteration (pinned memory) to drive the
loop decisions; all vectors and matrices stay in HBM.

There is no CPU fallback: a missing library or device raises
NativeLibraryError.
"""
from __future__ import annotations

import functools
import gc
import math
import os
import time

import numpy as np
import torch

from . import _lib
from .dist import Comm, row_range
from .config import (IpmParams, IpmResult, SolveReport, Stage1Config, Stage1Result,
                     TransitionParams)
from .errors import (DegenerateFactor, LineSearchStall, NativeLibraryError,
                     NotPositiveDefinite, status_error)

_NONE = 0x7F7F7F7F
NTRIALS = 61  # t = 0..60
# inertia shift of the full-coupling direction (frozen semantics 10, oracle/driver.py)
INERTIA_GROW = 4.0
INERTIA_SHRINK = 3.0
INERTIA_MAX_TRIES = 40


def _nvtx(name):
    """NVTX range around a solver phase (ncu --nvtx-include / nsys timelines)."""
    def deco(f):
        @functools.wraps(f)
        def wrapped(*a, **kw):
            torch.cuda.nvtx.range_push(name)
            try:
                return f(*a, **kw)
            finally:
                torch.cuda.nvtx.range_pop()
        return wrapped
    return deco


def _p(t):
    return None if t is None else t.data_ptr()


def barrier_weights(n, m, barrier):
    """Per-block barrier weights (wx, wy): mu_X = wx mu, mu_Y = wy mu.

    "paper"   : wx = wy = 1 (PAPER Eqs. 4, 9 and the merit function).
    "balanced": n wx = m wy and (n wx + m wy)/(n + m) = 1.  With a single mu
    and n != m the perturbed KKT system has no solution (summing
    x_ip graX_ip - y_pj graY_pj over one component vanishes for every (X, Y)
    by the scale invariance of XY, which forces mu (n - m) = 0), so the
    paper's inner loop can only drift along the scaling orbit; the balanced
    weights restore a central path.  Opt-in extension, see DESIGN.md.
    """
    if barrier == "paper":
        return 1.0, 1.0
    if barrier == "balanced":
        return (n + m) / (2.0 * n), (n + m) / (2.0 * m)
    raise ValueError(f"unknown barrier {barrier!r}")


class Problem:
    """M resident on one GPU plus every scratch buffer the solver needs."""

    def __init__(self, M, k, device=None, comm: Comm | None = None, m_capacity: int = 0):
        """M: this rank's row block when ``comm`` spans several GPUs (dist.py).

        m_capacity > m: room for appended columns (streaming, ``append_columns``): M lives
        in one of two pre-allocated n x m_capacity buffers and every scratch buffer is sized
        for m_capacity, so an append allocates nothing."""
        if not torch.cuda.is_available():
            raise NativeLibraryError("no CUDA device: the B200 solver has no CPU fallback")
        self.lib = _lib.load()
        self.launches = 0
        self.instrument = set()
        self.event_log = []  # (start, end) events of instrumented launches
        self.captured_events = []  # pairs recorded inside a graph being captured
        self.event_times = []  # resolved durations (ms) of instrumented launches in graphs
        self.graph_timing_failed = False
        self.graph_kernel_launches = 0  # library kernels executed inside replayed graphs
        self.persist_iters = 0  # IPM iterations run inside persistent launches
        self.persist_seconds = 0.0
        self.persist_prof = None  # optional int64 (4096, 16) phase clocks (scripts/)
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        if isinstance(M, np.ndarray):
            if M.dtype not in (np.float64, np.float32):
                M = M.astype(np.float64)
            M = torch.from_numpy(np.ascontiguousarray(M))
        self.M = M.to(self.dev).contiguous()
        if self.M.dtype not in (torch.float64, torch.float32):
            self.M = self.M.double()
        self.f32 = int(self.M.dtype == torch.float32)
        self.n, self.m = self.M.shape
        self.m_cap = max(int(m_capacity), self.m)
        self._mbuf = None
        if self.m_cap > self.m:
            self._mbuf = [torch.empty(self.n * self.m_cap, dtype=self.M.dtype, device=self.dev)
                          for _ in range(2)]
            self._mcur = 0
            view = self._mbuf[0][: self.n * self.m].view(self.n, self.m)
            view.copy_(self.M)
            self.M = view
        self.comm = comm or Comm.single()
        self.n_global = int(self.comm.sum_float(self.n, self.dev)) if self.comm.active else self.n
        self.k = int(k)
        if not 1 <= self.k <= 16:
            raise ValueError("k must be in [1, 16]")
        n, m, k = self.n, self.m_cap, self.k
        f64 = dict(dtype=torch.float64, device=self.dev)
        L = self.lib
        cw = max(L.nmfb_colprod_work_len(n, m, k), L.nmfb_colprod_work_len(n, k, k),
                 L.nmfb_colprod_work_len(m, k, k), L.nmfb_colprod_work_len(n, m, 1),
                 L.nmfb_rowprod_work_len(n, m, k, self.f32), L.nmfb_rowprod_work_len(n, m, k, 0),
                 4096)
        self.cwork = torch.empty(cw, **f64)
        self.gwork = torch.empty(max(self.lib.nmfb_grams_work_len(max(n, m), k, 4), 1),
                                 **f64)
        nb = L.nmfb_ipm_reduce_blocks()
        self.rwork = torch.empty(max(148 * 2 * NTRIALS, 12 * nb, 3 * ((n + 127) // 128 + nb), 4096),
                                 **f64)
        self.swork1 = torch.empty(max(4096, 3 * ((max(n, m) * k + 255) // 256 + 64)), **f64)
        self.row_n2 = torch.empty(n, **f64)
        self._col_n2 = torch.empty(m, **f64)
        self.col_n2 = self._col_n2[: self.m]
        self._call("nmfb_sqnorms", _p(self.M), self.f32, n, self.m, _p(self.row_n2),
                   _p(self.col_n2), _p(self.cwork), self.cwork.numel(), self.stream)
        self.comm.sum_(self.col_n2)
        self.mnorm2_local = float(self.row_n2.sum().item())  # ||M_rank||^2 (F-free objective)
        self._call("nmfb_blas_init", self.stream)  # cuBLAS handle, outside any graph capture
        # factor table of every passive subset for the NNLS batches: always for k <= 12
        # (<= 4.8 MB); above that (135 MB, ~0.19 ms to build at k = 16) only when a
        # half-sweep's batch is large enough to repay the build (c5: 200000 rows, 40000
        # columns: sweep 22.5 -> 18.2 ms)
        use_tab = os.environ.get("NMFB_NNLS_TABLE", "1") != "0" and (
            k <= 12 or max(n, self.m) >= (2 << k))
        self.ftab_len = int(L.nmfb_nnls_ftab_len(k)) if use_tab else 0
        self.ftab = torch.empty(max(self.ftab_len, 1), **f64) if self.ftab_len else None
        self.dscal = torch.zeros(256, **f64)
        self.iscal = torch.zeros(16, dtype=torch.int32, device=self.dev)
        self.hscal = torch.zeros(256, dtype=torch.float64).pin_memory()
        self.hint = torch.zeros(16, dtype=torch.int32).pin_memory()

    def load(self, Mnew):
        """Replace the data of M in place (same shape): one host-to-device copy into the
        resident buffer (non-blocking from pinned memory), the squared row / column norms
        recomputed on the device.  Buffers, tensor maps' targets and cached IPM engines (with
        their CUDA graphs) stay valid -- the serving pattern for repeated solves."""
        if isinstance(Mnew, np.ndarray):
            Mnew = torch.from_numpy(np.ascontiguousarray(Mnew))
        if tuple(Mnew.shape) != (self.n, self.m):
            raise ValueError(f"load: shape {tuple(Mnew.shape)} != {(self.n, self.m)}")
        self.M.copy_(Mnew.to(dtype=self.M.dtype), non_blocking=True)
        return self.refresh_norms()

    def refresh_norms(self):
        """After the data of M changed in place (``load``, or a copy issued by the caller on
        another stream and already awaited on this one: pipeline.SolvePipeline): squared row /
        column norms, ||M||^2, and the cached engines' incremental products invalidated."""
        self._call("nmfb_sqnorms", _p(self.M), self.f32, self.n, self.m, _p(self.row_n2),
                   _p(self.col_n2), _p(self.cwork), self.cwork.numel(), self.stream)
        self.comm.sum_(self.col_n2)
        self.mnorm2_local = float(self.row_n2.sum().item())
        for eng in self.__dict__.get("_engines", {}).values():
            eng.mvalid = False  # incremental residual-free refresh restarts from M
        return self

    def append_columns(self, Mnew):
        """Append columns (n, c) -- host or device, fp32 or fp64 -- in place: the active
        M moves once into the other pre-allocated buffer with the new columns behind it
        (one device copy, no allocation), the squared row norms advance by the new block's
        and its column norms are appended (csrc nmfb_sqnorms on the block only)."""
        if isinstance(Mnew, np.ndarray):
            Mnew = torch.from_numpy(np.ascontiguousarray(Mnew))
        Mn = Mnew.to(self.dev, dtype=self.M.dtype).contiguous()
        n, c = Mn.shape
        if n != self.n:
            raise ValueError("appended block must have the same rows")
        m0, m1 = self.m, self.m + c
        if self._mbuf is None or m1 > self.m_cap:
            raise ValueError(f"column capacity {self.m_cap} exceeded ({m1})")
        dst = self._mbuf[1 - self._mcur][: n * m1].view(n, m1)
        dst[:, :m0].copy_(self.M)
        dst[:, m0:].copy_(Mn)
        self._mcur = 1 - self._mcur
        self.M, self.m = dst, m1
        rn = self.buf(n)
        self.col_n2 = self._col_n2[:m1]
        self._call("nmfb_sqnorms", _p(Mn), self.f32, n, c, _p(rn), _p(self.col_n2[m0:]),
                   _p(self.cwork), self.cwork.numel(), self.stream)
        self.comm.sum_(self.col_n2[m0:])
        self.row_n2.add_(rn)
        self.mnorm2_local = float(self.row_n2.sum().item())
        return Mn

    # -- plumbing -----------------------------------------------------------
    @property
    def stream(self):
        return torch.cuda.current_stream(self.dev).cuda_stream

    def _call(self, name, *args, tag=None):
        if name in self.instrument or (tag is not None and tag in self.instrument):
            # CUDA events on the launching stream (bench roofline)
            st = torch.cuda.current_stream(self.dev)
            cap = torch.cuda.is_current_stream_capturing()
            ext = dict(external=True) if cap else {}
            e0 = torch.cuda.Event(enable_timing=True, **ext)
            e1 = torch.cuda.Event(enable_timing=True, **ext)
            e0.record(st)
            rc = getattr(self.lib, name)(*args)
            e1.record(st)
            if cap:
                self.captured_events.append((e0, e1))  # re-recorded by every graph replay
            else:
                self.event_log.append((e0, e1))
        else:
            rc = getattr(self.lib, name)(*args)
        self.launches += 1
        if rc != 0:
            why = ""
            if rc == -2:  # NMFB_ELAUNCH: name the CUDA error behind it
                why = " (" + self.lib.nmfb_last_cuda_error().decode() + ")"
            raise NativeLibraryError(f"{name} returned {rc}{why}")

    def readback(self, nd, ni=0):
        """Copy dscal[:nd] / iscal[:ni] to pinned host memory and wait."""
        if nd:
            self.hscal[:nd].copy_(self.dscal[:nd], non_blocking=True)
        if ni:
            self.hint[:ni].copy_(self.iscal[:ni], non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        return self.hscal[:nd].numpy().copy(), self.hint[:ni].numpy().copy()

    def buf(self, *shape, dtype=torch.float64):
        return torch.empty(shape, dtype=dtype, device=self.dev)

    def rowprod(self, A, rows, cols, B, k, out, tol=None, f32=0):
        self._call("nmfb_rowprod", _p(A), f32, rows, cols, _p(B), k, _p(out), _p(tol), 1.0,
                   _p(self.cwork), self.cwork.numel(), self.stream)

    def colprod(self, A, rows, cols, B, k, out, tol=None, f32=0, reduce=False, tag=None):
        """out = A^T B.  reduce=True: A, B are row-sharded -> all-reduce (then tol)."""
        if reduce and self.comm.active:
            self._call("nmfb_colprod", _p(A), f32, rows, cols, _p(B), k, _p(out), None, 1.0,
                       _p(self.cwork), self.cwork.numel(), self.stream, tag=tag)
            self.comm.sum_(out)
            if tol is not None:
                self._call("nmfb_row_tol", _p(out), cols, k, _p(tol), self.stream)
            return
        self._call("nmfb_colprod", _p(A), f32, rows, cols, _p(B), k, _p(out), _p(tol), 1.0,
                   _p(self.cwork), self.cwork.numel(), self.stream, tag=tag)

    def grams(self, triples, rows, k, reduce=False):
        """out_q = A_q^T B_q (k x k) for up to four (A, B, out) over the same rows, one pass.
        reduce=True: rows are sharded -> all-reduce every out."""
        args = []
        for q in range(4):
            if q < len(triples):
                a, b, o = triples[q]
                args += [_p(a), _p(b), _p(o)]
            else:
                args += [None, None, None]
        self._call("nmfb_grams", len(triples), *args, rows, k, _p(self.gwork), self.gwork.numel(),
                   self.stream)
        if reduce and self.comm.active:
            for _, _, o in triples:
                self.comm.sum_(o)

    @property
    def ny_local(self):
        """Replicated (Y-side) terms of mixed reductions are counted on rank 0 only."""
        return 1 if self.comm.root else 0

    def reduce_kkt(self, at=16):
        if self.comm.active:
            self.comm.sum_(self.dscal[at:at + 8])
            self.comm.max_(self.dscal[at + 8:at + 12])

    def to_dev(self, a):
        if isinstance(a, torch.Tensor):
            return a.to(device=self.dev, dtype=torch.float64).contiguous().clone()
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.dev)

    # -- gradients / KKT -----------------------------------------------------
    def gradients(self, X, Yt, F, gX, gY, out_index=0):
        """F = XY - M, graX, graY; dscal[out_index] = ||F||^2."""
        n, m, k = self.n, self.m, self.k
        self._call("nmfb_residual", _p(self.M), self.f32, n, m, k, _p(X), _p(Yt), _p(F), _p(gX),
                   _p(self.dscal[out_index:]), _p(self.rwork), self.stream)
        self.comm.sum_(self.dscal[out_index:out_index + 1])
        self.colprod(F, n, m, X, k, gY, reduce=True, tag="graY")

    @property
    def free_residual_default(self):
        """Use the residual-free formulation when an n x m fp64 residual is large."""
        return self.n * self.m >= (1 << 25)

    def gradients_free(self, X, Yt, gX, gY, ws, out_index=0, passes=True):
        """graX, graY and ||F||^2 without forming F (csrc/ipm.cu "F-free"):
        three small Grams plus M Y^T and X^T M (two streaming passes over M;
        passes=False: ws["MY"], ws["MX"] already hold them at (X, Yt))."""
        n, m, k, s = self.n, self.m, self.k, self.stream
        self.colprod(Yt, m, k, Yt, k, ws["GY"])
        self.colprod(X, n, k, X, k, ws["XX"], reduce=True)
        if passes:
            self.rowprod(self.M, n, m, Yt, k, ws["MY"], None, self.f32)
            self.colprod(self.M, n, m, X, k, ws["MX"], None, self.f32, reduce=True)
        self._call("nmfb_ffree_grad_rows", _p(X), _p(ws["GY"]), _p(ws["MY"]), n, k, _p(gX),
                   _p(ws["part"]), s)
        self._call("nmfb_ffree_fsq", _p(ws["part"]), self.mnorm2_local,
                   _p(ws["XX"]) if self.comm.root else None, _p(ws["GY"]), k,
                   _p(self.dscal[out_index:]), None, s)
        self.comm.sum_(self.dscal[out_index:out_index + 1])
        self._call("nmfb_ffree_grad_rows", _p(Yt), _p(ws["XX"]), _p(ws["MX"]), m, k, _p(gY),
                   _p(ws["part2"]), s)

    def dualprod(self, B1, B2, outR, outC, work, reduce=True):
        """outR = M B1 (rows), outC = M^T B2 (all-reduced over row shards): one pass."""
        self._call("nmfb_dualprod", _p(self.M), self.f32, self.n, self.m, _p(B1), _p(B2), self.k,
                   _p(outR), _p(outC), _p(work), work.numel(), self.stream)
        if reduce:
            self.comm.sum_(outC)

    def free_workspace(self):
        n, m, k = self.n, self.m, self.k
        nb = self.lib.nmfb_ipm_reduce_blocks()
        ws = {"GY": self.buf(k, k), "XX": self.buf(k, k), "MY": self.buf(n, k),
              "MX": self.buf(m, k), "part": self.buf(nb), "part2": self.buf(nb)}
        return ws

    def kkt_sums(self, X, R, gX, Yt, S, gY, mux, muy, at=16):
        self._call("nmfb_kkt_sums", _p(X), _p(R), _p(gX), X.numel(), _p(Yt), _p(S), _p(gY),
                   Yt.numel() * self.ny_local, float(mux), float(muy), _p(self.dscal[at:]),
                   _p(self.rwork), self.stream)
        self.reduce_kkt(at)


def kkt_from_sums(v):
    """(E(.;mu), E(.;0)) from the 12 sums of nmfb_kkt_sums (PAPER Eq. 9)."""
    st = math.sqrt(max(v[0] + v[4], 0.0))
    return max(st, math.sqrt(max(v[1] + v[5], 0.0))), max(st, math.sqrt(max(v[2] + v[6], 0.0)))


# ============================================================================
# stage 1 (Algorithm 1)
# ============================================================================
@_nvtx("nmfb.stage1")
def run_stage1(P: Problem, X, Yt, cfg: Stage1Config | None = None, pX=None, pY=None):
    """SPEC.md:209 run_stage1 on the device.  X (n,k), Yt (m,k) device fp64.

    Returns (X, Yt, pX, pY, Stage1Result-without-host-copies).
    """
    cfg = cfg or Stage1Config()
    t0 = time.perf_counter()
    n, m, k = P.n, P.m, P.k
    X = X.clone()
    Yt = Yt.clone()
    have_carry = pX is not None
    pX = torch.zeros((n, k), dtype=torch.uint8, device=P.dev) if pX is None else pX.to(torch.uint8).clone()
    pY = torch.zeros((m, k), dtype=torch.uint8, device=P.dev) if pY is None else pY.to(torch.uint8).clone()
    Xn, Yn = P.buf(n, k), P.buf(m, k)
    pXn = torch.empty_like(pX)
    pYn = torch.empty_like(pY)
    ctbX, tolX, r2X = P.buf(n, k), P.buf(n), P.buf(n)
    ctbY, tolY, r2Y = P.buf(m, k), P.buf(m), P.buf(m)
    chX = P.buf(n, dtype=torch.int64)
    chY = P.buf(m, dtype=torch.int64)
    stX = P.buf(n, dtype=torch.int8)
    stY = P.buf(m, dtype=torch.int8)
    GY, GX = P.buf(k, k), P.buf(k, k)
    tol_fixed = cfg.tol_kkt
    res = Stage1Result(None, None, None, None, 0, False)
    nsweeps = cfg.fixed_sweeps if cfg.fixed_sweeps > 0 else cfg.max_sweeps
    s = P.stream
    if (cfg.persistent and not P.comm.active and nsweeps > 0
            and P.lib.nmfb_stage1_persist_supported(n, m, k, int(P.f32))):
        return _stage1_persistent(P, X, Yt, pX, pY, Yn, stX, stY, have_carry, cfg, nsweeps, res, t0)
    # fixed sweep count: no per-sweep host synchronisation -- the sweep statistics go to a
    # device log and failures to one first-failure word, both read once at the end (the
    # per-sweep readback cost ~5 % of a c4 sweep on one rank, more on a shard).  Row-sharded:
    # the log holds this rank's partial sums and is all-reduced once, the failure word is
    # the minimum over the ranks (any rank's failure is reported on every rank)
    nosync = cfg.fixed_sweeps > 0
    if nosync:
        slog = P.buf(nsweeps, 3)
        fword = torch.full((1,), -1, dtype=torch.int64, device=P.dev)  # all ones
    # single rank: the subset factor tables (they depend only on the Gram) are built on a
    # side stream while the streaming product computes ctb, and the fixed-sweep statistics
    # run there behind the sweep (the kernels fit beside the persistent product kernels)
    side = None
    if nosync and not P.comm.active and P.ftab_len and os.environ.get("NMFB_S1_FORK", "1") != "0":
        side = P.__dict__.get("_s1_side")
        if side is None:
            side = P._s1_side = torch.cuda.Stream(P.dev)
            P._ftabY = torch.empty_like(P.ftab)
        ftX, ftY = P.ftab, P._ftabY
    ev_stats = None

    def fork(C, rows_c, G, table):
        """side stream: Gram G = C^T C, then its subset factor table (both only needed by
        the NNLS batch, not by the streaming product running meanwhile)."""
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(P.dev))
        side.wait_event(ev)
        with torch.cuda.stream(side):
            # the multi-Gram kernel with its own workspace (P.gwork): the product running on
            # the main stream meanwhile owns P.cwork
            P.grams([(C, C, G)], rows_c, k)
            P._call("nmfb_nnls_ftab_build", _p(G), k, _p(table), P.ftab_len, P.stream)
        ev_t = torch.cuda.Event()
        ev_t.record(side)
        return ev_t

    for sweep in range(nsweeps):
        mode = 2 if (sweep > 0 or have_carry) else 0
        cur = torch.cuda.current_stream(P.dev)
        # X-update: C = Y^T, d = rows of M
        if side is not None:
            ev_t = fork(Yt, m, GY, ftX)
        else:
            ev_t = None
            P.colprod(Yt, m, k, Yt, k, GY)
        P.rowprod(P.M, n, m, Yt, k, ctbX, tolX, P.f32)
        if tol_fixed is not None:
            tolX.fill_(float(tol_fixed))
        if ev_t is not None:
            cur.wait_event(ev_t)
            if ev_stats is not None:  # the previous sweep's statistics read X / stX
                cur.wait_event(ev_stats)
            P._call("nmfb_nnls_batch_ws", _p(GY), _p(ctbX), _p(P.row_n2), _p(pX), mode,
                    _p(tolX), 3 * k, n, k, _p(Xn), _p(pXn), _p(chX), _p(r2X), _p(stX), None,
                    None, _p(ftX), -P.ftab_len, s)
        else:
            P._call("nmfb_nnls_batch_ws", _p(GY), _p(ctbX), _p(P.row_n2), _p(pX), mode,
                    _p(tolX), 3 * k, n, k, _p(Xn), _p(pXn), _p(chX), _p(r2X), _p(stX), None,
                    None, _p(P.ftab), P.ftab_len, s)
        # Y-update: C = X, d = columns of M; row contractions all-reduced
        if side is not None:
            ev_t = fork(Xn, n, GX, ftY)
        else:
            ev_t = None
            P.colprod(Xn, n, k, Xn, k, GX, reduce=True)
        P.colprod(P.M, n, m, Xn, k, ctbY, tolY, P.f32, reduce=True)
        if tol_fixed is not None:
            tolY.fill_(float(tol_fixed))
        if ev_t is not None:
            cur.wait_event(ev_t)
            P._call("nmfb_nnls_batch_ws", _p(GX), _p(ctbY), _p(P.col_n2), _p(pY), mode,
                    _p(tolY), 3 * k, m, k, _p(Yn), _p(pYn), _p(chY), _p(r2Y), _p(stY), None,
                    None, _p(ftY), -P.ftab_len, s)
        elif P.comm.active:
            # columns split over the ranks, then all-gathered (dist.py)
            c0, c1 = row_range(m, P.comm.world, P.comm.rank)
            if c1 > c0:
                P._call("nmfb_nnls_batch_ws", _p(GX), _p(ctbY[c0:]), _p(P.col_n2[c0:]),
                        _p(pY[c0:]), mode, _p(tolY[c0:]), 3 * k, c1 - c0, k, _p(Yn[c0:]),
                        _p(pYn[c0:]), _p(chY[c0:]), _p(r2Y[c0:]), _p(stY[c0:]), None, None,
                        _p(P.ftab), P.ftab_len, s)
            for t_ in (Yn, pYn, r2Y, stY):
                P.comm.allgather_rows(t_)
        else:
            P._call("nmfb_nnls_batch_ws", _p(GX), _p(ctbY), _p(P.col_n2), _p(pY), mode,
                    _p(tolY), 3 * k, m, k, _p(Yn), _p(pYn), _p(chY), _p(r2Y), _p(stY), None, None,
                    _p(P.ftab), P.ftab_len, s)
        ny = P.ny_local
        if nosync:
            if side is not None:  # behind the sweep, on the side stream
                ev = torch.cuda.Event()
                ev.record(cur)
                side.wait_event(ev)
            with torch.cuda.stream(side if side is not None else cur):
                ss = P.stream
                P._call("nmfb_stage1_stats", _p(X), _p(Xn), n * k, _p(Yt), _p(Yn), m * k * ny,
                        _p(r2Y), m * ny, _p(slog[sweep]), _p(P.swork1), P.swork1.numel(), ss)
                P._call("nmfb_first_failure_i8", _p(stX), n, 2 * sweep, _p(fword), ss)
                P._call("nmfb_first_failure_i8", _p(stY), m, 2 * sweep + 1, _p(fword), ss)
            if side is not None:
                ev_stats = torch.cuda.Event()
                ev_stats.record(side)
            X, Xn = Xn, X
            Yt, Yn = Yn, Yt
            pX, pXn = pXn, pX
            pY, pYn = pYn, pY
            res.sweeps = sweep + 1
            continue
        P._call("nmfb_stage1_stats", _p(X), _p(Xn), n * k, _p(Yt), _p(Yn), m * k * ny, _p(r2Y),
                m * ny, _p(P.dscal), _p(P.rwork), P.rwork.numel(), s)
        P._call("nmfb_first_nonzero_i8", _p(stX), n, _p(P.iscal[0:]), s)
        P._call("nmfb_first_nonzero_i8", _p(stY), m, _p(P.iscal[1:]), s)
        P.comm.sum_(P.dscal[0:3])
        if P.comm.active:  # any rank's failing row stops every rank
            flag = (P.iscal[0:1] != _NONE).to(torch.int32)
            P.comm.max_(flag)
            P.iscal[0:1].masked_fill_(flag.bool() & (P.iscal[0:1] == _NONE), -1)
        v, iv = P.readback(3, 2)
        for which, idx, st in (("update_X", int(iv[0]), stX), ("update_Y", int(iv[1]), stY)):
            if idx == -1:
                raise status_error(-1, -1, which + " (another rank)")
            if idx != _NONE:
                raise status_error(int(st[idx].item()), idx, which)
        X, Xn = Xn, X
        Yt, Yn = Yn, Yt
        pX, pXn = pXn, pX
        pY, pYn = pYn, pY
        step, nrm = math.sqrt(v[0]), math.sqrt(v[1])
        res.sweeps = sweep + 1
        res.trace.append((time.perf_counter() - t0, 0.5 * v[2], step))
        if cfg.fixed_sweeps <= 0 and step <= cfg.eps_stol * (1.0 + nrm):
            res.converged = True
            break
    if ev_stats is not None:
        torch.cuda.current_stream(P.dev).wait_event(ev_stats)
    if nosync and nsweeps > 0:
        if P.comm.active:
            P.comm.sum_(slog)
            fword.masked_fill_(fword < 0, (1 << 63) - 1)  # "none" sorts last
            P.comm.min_(fword)
            fword.masked_fill_(fword == (1 << 63) - 1, -1)
        fw = int(fword.item()) & ((1 << 64) - 1)
        if fw != (1 << 64) - 1:
            tag, idx, code = fw >> 40, (fw >> 8) & 0xFFFFFFFF, fw & 0xFF
            code = code - 256 if code >= 128 else code
            raise status_error(code, idx, "update_Y" if tag & 1 else "update_X")
        lg = slog.cpu().numpy()
        t1 = time.perf_counter()
        for i in range(nsweeps):
            res.trace.append(((t1 - t0) * (i + 1) / nsweeps, 0.5 * float(lg[i, 2]),
                              math.sqrt(float(lg[i, 0]))))
    res.seconds = time.perf_counter() - t0
    return X, Yt, pX, pY, res


def _stage1_persistent(P, X, Yt, pX, pY, Yn, stX, stY, have_carry, cfg, nsweeps, res, t0):
    """All sweeps of run_stage1 in one cooperative launch (csrc/stage1_persist.cu)."""
    n, m, k = P.n, P.m, P.k
    log = P.buf(nsweeps, 4)
    stat = torch.zeros(3, dtype=torch.int32, device=P.dev)
    work = P.buf(max(P.lib.nmfb_stage1_persist_work_len(n, m, k), 1))
    tol = -1.0 if cfg.tol_kkt is None else float(cfg.tol_kkt)
    P._call("nmfb_stage1_persist", _p(P.M), P.f32, n, m, k, _p(X), _p(Yt), None, _p(Yn),
            _p(pX), _p(pY), _p(P.row_n2), _p(P.col_n2), _p(stX), _p(stY), tol,
            2 if have_carry else 0, nsweeps, 1 if cfg.fixed_sweeps > 0 else 0, cfg.eps_stol,
            _p(log), _p(stat), _p(work), P.stream, tag="stage1_persist")
    st = stat.cpu().numpy()
    sweeps, conv, failed = int(st[0]), bool(st[1]), bool(st[2])
    if failed:
        for which, arr in (("update_X", stX), ("update_Y", stY)):
            bad = torch.nonzero(arr).flatten()
            if bad.numel():
                i = int(bad[0])
                raise status_error(int(arr[i].item()), i, which)
    lg = log[:sweeps].cpu().numpy()
    t1 = time.perf_counter()
    for i in range(sweeps):
        res.trace.append((t0 + (t1 - t0) * (i + 1) / sweeps - t0, float(lg[i, 0]), float(lg[i, 1])))
    res.sweeps = sweeps
    res.converged = conv
    res.seconds = time.perf_counter() - t0
    P.stage1_persist_sweeps = getattr(P, "stage1_persist_sweeps", 0) + sweeps
    return X, Yt, pX, pY, res


# ============================================================================
# stage 2 (Algorithm 2 + the Hessian switch of Algorithm 3)
# ============================================================================
_GRAPH_DEBUG = bool(os.environ.get("NMFB_GRAPH_DEBUG"))


class IpmEngine:
    """Device state and kernels of one interior-point solve."""

    def __init__(self, P: Problem, X, Yt, R, S, mu, rho, p: IpmParams):
        self.P, self.p = P, p
        n, m, k = P.n, P.m, P.k
        self.n, self.m, self.k = n, m, k
        self.kk = k * (k + 1) // 2
        self.X, self.Yt, self.R, self.S = X, Yt, R, S
        self.mu, self.rho, self.flag = float(mu), float(rho), False
        self.wx, self.wy = barrier_weights(P.n_global, m, p.barrier)
        self.comm = P.comm
        b = P.buf
        self.ffree = (p.residual == "free") or (p.residual == "auto" and P.free_residual_default)
        self.F = [None, None] if self.ffree else [b(n, m), b(n, m)]
        if self.ffree:
            self.fws = P.free_workspace()
            self.MdY = b(n, k)
            # one-pass Armijo products (M dY^T, M^T dX) and the incremental refresh of
            # M Y^T / M^T X (csrc/anls.cu k_dualprod_mma, csrc/ipm.cu k_ffree_advance)
            self.dual = (m % 2 == 0) and os.environ.get("NMFB_DUALPROD", "1") != "0"
            if self.dual:
                self.MtdX = b(m, k)
                self.dwork = b(max(P.lib.nmfb_dualprod_work_len(n, m, k), 1))
            self.mvalid = False  # fws["MY"], fws["MX"] hold M Y^T, M^T X at the current point
            self.A1, self.A2, self.B1, self.B2 = b(k, k), b(k, k), b(k, k), b(k, k)
            self.Dgx, self.Dgy, self.Dmd = b(k, k), b(k, k), b(k, k)
        self.fi = 0  # index of F at the current point
        self.gX, self.gY = b(n, k), b(m, k)
        self.L, self.h, self.g = b(n, k, k), b(n, k), b(n, k)
        self.Apk, self.XXpk = b(n, self.kk), b(n, self.kk)
        self.Z = b(self.kk, self.kk)
        self.GY, self.XtX, self.H, self.Gdy = b(k, k), b(k, k), b(k, k), b(k, k)
        if self.ffree:  # the refresh's Grams at the current point (same buffers)
            self.GY, self.XtX = self.fws["GY"], self.fws["XX"]
        N = m * k
        self.N = N
        self.dense_gn = p.schur_solver == "dense"
        self.A = None  # dense mk x mk reduced matrix: allocated on first full-C / dense use
        self.t4work = None
        self.rhs = b(N)
        self.dYbuf = b(m, k)
        Q = k * k
        self.LD, self.Dinvpk, self.YYpk = b(m, k, k), b(m, self.kk), b(m, self.kk)
        self.Gpk = b(self.kk, self.kk)
        self.LG, self.LH, self.lrwork = b(Q, Q), b(Q, Q), b(2 * Q * Q)
        self.uvec, self.wvec = b(Q), b(Q)
        self.fact_dense = False
        self.dX, self.dR, self.dS = b(n, k), b(n, k), b(m, k)
        self.FtG, self.FdY = b(m, k), b(n, k)
        self.Xf, self.Ytf = b(n, k), b(m, k)
        self.have_fact = False
        self.fact_full = False
        self.fact_F = 0
        self.graphs = {}
        self.mu_dev = None  # [mu, wx mu, wy mu] read by the captured general-path kernels
        self.graph_pool = None
        self.capture_stream = None
        self.use_graphs = p.use_graphs and P.comm.graph_ok and not self.dense_gn
        # fused small-problem iteration (csrc/small.cu) for c1-c3-sized problems
        self.small = bool(P.lib.nmfb_small_supported(n, m, k)) and not P.comm.active \
            and not self.dense_gn and p.fused_small and not self.ffree
        if self.small:
            self.swork = b(max(P.lib.nmfb_small_work_len(n, m, k), 1))
            self.tickets = torch.zeros(8, dtype=torch.int32, device=P.dev)
        # persistent inner loop (csrc/persist.cu): one cooperative launch per inner loop
        self.persist = self.small and p.persistent and \
            bool(P.lib.nmfb_persist_supported(n, m, k, p.persist_grid, int(P.f32)))
        if self.persist:
            self.pwork = b(P.lib.nmfb_persist_work_len(n, m, k, p.persist_grid))
            self.pbar = torch.zeros(160, dtype=torch.int32, device=P.dev)  # barrier flags
            self.pstat = torch.zeros(2, dtype=torch.int32, device=P.dev)
            self.pfc0 = torch.tensor([_NONE, -1, _NONE], dtype=torch.int32, device=P.dev)
            self.plog = None
        self.Pbuf = None
        self.W = None
        aw = max(P.lib.nmfb_atb_work_len(n, self.kk, self.kk),
                 P.lib.nmfb_atb_work_len(m, self.kk, self.kk),
                 0 if self.ffree else P.lib.nmfb_atb_work_len(n, m, k ** 3), 1)
        self.awork = b(aw)
        # the Y-side factor (D_j, the G capacitance Gram) runs on a second stream, concurrent
        # with the X-side row factors / Z Gram (independent until the low-rank factorization);
        # both branches are latency-bound kernels on a few SMs each
        self.fork = (not self.comm.active) and os.environ.get("NMFB_IPM_FORK", "1") != "0"
        self.awork2 = b(aw) if self.fork else None
        self.side = torch.cuda.Stream(P.dev) if self.fork else None
        if self.use_graphs:
            # the capacitance Grams' first cuBLAS calls (library init, kernel load) run
            # eagerly here, not inside the first graph capture (~0.4 s there at c4);
            # the outputs are recomputed by every direction
            self.Apk.zero_()
            self.YYpk.zero_()
            for A_, rows_, B_, O_ in ((self.Apk, n, self.XXpk, self.Z),
                                      (self.YYpk, m, self.Dinvpk, self.Gpk)):
                P._call("nmfb_atb", _p(A_), rows_, self.kk, _p(A_), self.kk, _p(O_),
                        _p(self.awork), self.awork.numel(), P.stream)

    def reset(self, X, Yt, R, S, mu, p: IpmParams):
        """Re-arm a cached engine at a new starting point (same problem, structure and rho):
        buffers, factorizations and captured graphs are reused."""
        self.X.copy_(X)
        self.Yt.copy_(Yt)
        self.R.copy_(R)
        self.S.copy_(S)
        self.mu, self.flag, self.p = float(mu), False, p
        self.fi, self.fact_F, self.have_fact, self.fact_full = 0, 0, False, False
        self.fact_dense = self.last_dense = False
        if self.ffree:
            self.mvalid = False

    # -- helpers -------------------------------------------------------------
    @property
    def Fcur(self):
        return self.F[self.fi]

    def refresh_launch(self):
        """Launch gradients + KKT sums at the current point (no host sync)."""
        P = self.P
        if self.ffree:
            passes = not (self.dual and self.mvalid)
            P.gradients_free(self.X, self.Yt, self.gX, self.gY, self.fws, out_index=0,
                             passes=passes)
            self.mvalid = self.dual
            P.kkt_sums(self.X, self.R, self.gX, self.Yt, self.S, self.gY, self.wx * self.mu,
                       self.wy * self.mu, at=16)
            return
        if self.have_fact and self.fact_F == self.fi:
            self.fi ^= 1  # keep the factorization's residual for the predictor
        P.gradients(self.X, self.Yt, self.Fcur, self.gX, self.gY, out_index=0)
        P.kkt_sums(self.X, self.R, self.gX, self.Yt, self.S, self.gY, self.wx * self.mu,
                   self.wy * self.mu, at=16)

    def refresh(self):
        """Gradients + KKT sums at the current point -> (E_mu, E_0, fsq, sums)."""
        self.refresh_launch()
        v, _ = self.P.readback(28)
        e_mu, e_0 = kkt_from_sums(v[16:28])
        return e_mu, e_0, v[0], v[16:28]

    # -- one Gauss-Newton inner iteration entirely on the device ---------------
    def gn_iteration_launch(self):
        """direction (GN) -> Armijo sums -> device Armijo selection -> update ->
        gradients/KKT at the new point.  No host synchronisation, so the whole
        sequence is captured once per (mu, F buffer) as a CUDA graph and replayed."""
        P, p = self.P, self.p
        n, m, k = self.n, self.m, self.k
        if self.small:
            s = P.stream
            P._call("nmfb_small_direction", _p(self.X), _p(self.R), _p(self.gX), _p(self.Yt),
                    _p(self.S), _p(self.gY), n, m, k, self.wx * self.mu, self.wy * self.mu,
                    self.rho, p.tau, _p(self.L), _p(self.h), _p(self.LD), _p(self.LG),
                    _p(self.LH), _p(self.lrwork), _p(self.Z), _p(self.H), _p(self.XtX),
                    _p(self.dX), _p(self.dR), _p(self.dYbuf), _p(self.dS), _p(self.Gdy),
                    _p(P.dscal), _p(P.iscal[2:]), _p(self.swork), _p(self.tickets), s)
            self.last_dense = False
            self.remember_factorization_host(False)
            fold, fnew = self.F[self.fi], self.F[self.fi ^ 1]
            P._call("nmfb_small_step_refresh", _p(P.M), P.f32, n, m, k, _p(self.X), _p(self.R),
                    _p(self.Yt), _p(self.S), _p(self.dX), _p(self.dR), _p(self.dYbuf),
                    _p(self.dS), _p(self.Xf), _p(self.Ytf), _p(fold), _p(fnew), _p(self.gX),
                    _p(self.gY), self.mu, self.wx, self.wy, p.eta, p.max_backtracks, p.tau,
                    NTRIALS, _p(P.dscal), _p(P.iscal[2:]), _p(self.swork), _p(self.tickets), s)
            self.fi ^= 1
            return
        dY = self.direction(False)
        s = P.stream
        if self.comm.active:
            self.armijo_launch(dY)
            P._call("nmfb_armijo_select", _p(P.dscal), self.mu, self.wx, self.wy, p.eta,
                    p.max_backtracks, _p(P.iscal[2:]), s)
        else:  # quartic, then barrier trials in lazy batches + the device selection
            self.armijo_launch(dY, trials=False)
            P._call("nmfb_armijo_lazy", _p(self.X), _p(self.dX), n * k, _p(self.Yt), _p(dY), m * k,
                    _p(P.dscal), NTRIALS, self.mu, self.wx, self.wy, p.eta, p.max_backtracks,
                    _p(P.iscal[2:]), _p(P.rwork), P.rwork.numel(), s)
        self.remember_factorization(False)  # the factorization's X, Y (before the step)
        self.take_step(dY, P.dscal[1:2], 0.0, P.dscal[3:4], 0.0)
        self.refresh_launch()

    def take_step(self, dY, a1_dev, a1, a2_dev, a2):
        """x, y += a1 (dx, dy); r, s += a2 (dr, ds) with the nudge rule;
        step lengths from device memory (graph path) or host scalars.  Residual-free dual
        mode: M Y^T / M^T X advance with the step unless an entry was nudged (iscal[5]
        then reports it and the host recomputes them, see run_ipm)."""
        P, p = self.P, self.p
        n, m, k, s = self.n, self.m, self.k, P.stream
        fl = my = mdy = mx = mtdx = None
        if self.ffree and self.dual:
            P.iscal[5:6].zero_()
            fl = P.iscal[5:]
            my, mdy, mx, mtdx = self.fws["MY"], self.MdY, self.fws["MX"], self.MtdX
        # one launch: x, y (nudge flag), r, s and the incremental M Y^T / M^T X advance (a
        # nudged step recomputes them: check_advance)
        P._call("nmfb_step_all", _p(self.X), _p(self.dX), n * k, _p(self.Yt), _p(dY), m * k,
                _p(self.R), _p(self.dR), _p(self.S), _p(self.dS), _p(my), _p(mdy), _p(mx),
                _p(mtdx), _p(a1_dev), float(a1 or 0.0), _p(a2_dev), float(a2 or 0.0), p.tau,
                _p(fl), s)
        if fl is not None and self.comm.active:  # a nudge on any rank invalidates M^T X
            self.comm.max_(P.iscal[5:6])

    def check_advance(self, flag=None):
        """After a residual-free dual-mode step: if an entry was nudged (iscal[5], or the
        value ``flag`` already read back), recompute M Y^T and M^T X (two passes) and the
        KKT sums -> new (e_mu, e_0, fsq, sums); None when the incremental refresh held."""
        if not (self.ffree and self.dual):
            return None
        if flag is None:
            flag = int(self.P.readback(0, 6)[1][5])
        if int(flag) == 0:
            return None
        self.mvalid = False
        return self.refresh()

    def gn_iteration_graph(self):
        """Replay (capturing on first use) the GN iteration graph for the current state.

        General path: the barrier value is read from device memory by the captured
        kernels (nmfb_set_mu_source during capture), so one graph per F buffer serves
        every mu; the fused small path bakes mu and is keyed by it."""
        if not self.small:
            if self.mu_dev is None:
                self.mu_dev = self.P.buf(3)
                self.mu_host = torch.zeros(3, dtype=torch.float64).pin_memory()
            self.mu_host[0] = self.mu
            self.mu_host[1] = self.wx * self.mu
            self.mu_host[2] = self.wy * self.mu
            self.mu_dev.copy_(self.mu_host, non_blocking=True)
        key = (self.fi,) if not self.small else (self.fi, self.mu)
        g = self.graphs.get(key)
        state = (self.fi, self.fact_F, self.have_fact, self.fact_full, self.fact_dense)
        if g is None:
            if len(self.graphs) > 8:
                self.graphs.clear()
            g = torch.cuda.CUDAGraph()
            self.P.captured_events = []
            c0 = self.P.lib.nmfb_launch_count()
            # Capture on a side stream directly: torch.cuda.graph() would also
            # synchronize and empty the caching allocator on every capture, which
            # forces the next allocations back through cudaMalloc (tens of ms at
            # c4/c5 sizes, more than the graph saves over a short run).
            if _GRAPH_DEBUG:
                torch.cuda.synchronize(self.P.dev)
                tg = time.perf_counter()
            if self.capture_stream is None:
                self.capture_stream = torch.cuda.Stream(self.P.dev)
            cur = torch.cuda.current_stream(self.P.dev)
            self.capture_stream.wait_stream(cur)
            # no cyclic garbage collection while the stream captures: collecting an old
            # engine there destroys its CUDA graphs (cudaGraphExecDestroy is not permitted
            # during a global-mode capture and invalidates this one)
            gc_on = gc.isenabled()
            gc.disable()
            try:
                with torch.cuda.stream(self.capture_stream):
                    if self.graph_pool is None:
                        g.capture_begin()
                    else:
                        g.capture_begin(pool=self.graph_pool)
                    try:
                        if not self.small:
                            self.P.lib.nmfb_set_mu_source(self.mu_dev.data_ptr())
                        self.gn_iteration_launch()
                    finally:
                        self.P.lib.nmfb_set_mu_source(None)
                        g.capture_end()
            finally:
                if gc_on:
                    gc.enable()
            cur.wait_stream(self.capture_stream)
            if _GRAPH_DEBUG:
                torch.cuda.synchronize(self.P.dev)
                tc = time.perf_counter()
                g.replay()
                torch.cuda.synchronize(self.P.dev)
                print(f"[nmfb graph] capture {1e3 * (tc - tg):.2f} ms, first replay "
                      f"{1e3 * (time.perf_counter() - tc):.2f} ms, pool "
                      f"{torch.cuda.memory_reserved(self.P.dev) / 2**20:.0f} MiB", flush=True)
            nk = self.P.lib.nmfb_launch_count() - c0
            self.graph_pool = g.pool()
            self.graphs[key] = (g, self.P.captured_events, nk)
            self.P.captured_events = []
            self.fi, self.fact_F, self.have_fact, self.fact_full, self.fact_dense = state
        g, _, nk = self.graphs[key]
        g.replay()
        self.P.graph_kernel_launches += nk  # kernels executed by this replay
        self.last_graph = key
        # mirror the host-side bookkeeping the captured sequence performs
        self.fact_F, self.have_fact, self.fact_full, self.fact_dense = state[0], True, False, False
        self.last_dense = False
        self.fi = state[0] ^ 1

    def persist_run(self, eps_mu, tol, budget, res, t0):
        """Run the Gauss-Newton inner loop in one cooperative launch (csrc/persist.cu).

        Appends the iterations to ``res`` and returns (exit code, E_mu, E_0, fsq, sums):
        code 0 = inner loop finished (E(.;mu) <= eps_mu or the budget), 1 = a
        factorization failed at the current point (no step taken), 2 = Armijo stall."""
        P, p = self.P, self.p
        n, m, k = self.n, self.m, self.k
        if self.plog is None or self.plog.shape[0] < budget:
            self.plog = P.buf(budget, 8)
        P.iscal[2:5].copy_(self.pfc0)
        fout = self.F[self.fi ^ 1]
        h0 = time.perf_counter()
        P._call("nmfb_ipm_persist", _p(P.M), P.f32, n, m, k, _p(self.X), _p(self.R),
                _p(self.gX), _p(self.Yt), _p(self.S), _p(self.gY), _p(fout), _p(self.L),
                _p(self.Xf), _p(self.Ytf), _p(self.LD), _p(self.LG), _p(self.LH),
                _p(self.lrwork), self.mu, self.wx, self.wy, self.rho, p.tau, p.eta, eps_mu, tol,
                p.max_backtracks, NTRIALS, budget, _p(P.dscal), _p(P.iscal[2:]), _p(self.plog),
                _p(self.pstat), _p(self.pwork), _p(self.pbar), p.persist_grid,
                _p(P.persist_prof) if P.persist_prof is not None else None, P.stream,
                tag="persist")
        st = self.pstat.cpu().numpy()
        iters, code = int(st[0]), int(st[1])
        nrec = iters + (1 if code == 2 else 0)
        log = self.plog[:nrec].cpu().numpy() if nrec else np.zeros((0, 8))
        v, iv = P.readback(28, 5)
        h1 = time.perf_counter()
        P.persist_iters += iters
        if iters:
            ns_last = log[iters - 1, 6]
            for i in range(iters):
                ti = (h1 - t0) - (ns_last - log[i, 6]) * 1e-9
                res.trace.append((ti, 0.5 * log[i, 3], log[i, 5], self.mu, log[i, 1], log[i, 2],
                                  int(log[i, 0])))
                res.armijo_t.append(int(log[i, 0]))
                res.flags.append(False)
            res.iters += iters
            # the kernel left F at the current point in F[fi ^ 1] and the last
            # Gauss-Newton factorization (L, Xf, Ytf, LD, LG, LH, Zb) for the predictor
            self.fact_F = self.fi
            self.fi ^= 1
            self.have_fact, self.fact_full, self.fact_dense = True, False, False
            self.last_dense = False
        if code == 2:
            res.armijo_t.append(int(log[nrec - 1, 0]))
        e_mu, e_zero = kkt_from_sums(v[16:28])
        P.persist_seconds += h1 - h0
        return code, iters, (e_mu, e_zero, v[0], v[16:28])

    def _ensure_full_buffers(self):
        if self.Pbuf is None:
            self.Pbuf = self.P.buf(self.n, self.k ** 3)
            self.W = self.P.buf(self.m, self.k ** 3)

    def _ensure_dense(self):
        if self.A is None:
            self.A = self.P.buf(self.N, self.N)

    def lowrank_solve(self, rhs, dY, Yt):
        P = self.P
        P._call("nmfb_lowrank_solve", _p(self.LD), _p(Yt), _p(self.LG), _p(self.LH),
                _p(self.lrwork), self.m, self.k, _p(rhs), _p(dY), _p(self.uvec), _p(self.wvec),
                _p(P.cwork), P.cwork.numel(), P.stream)

    def direction(self, full, force_dense=False, rho=None, early=False):
        """Newton direction; scalars land in dscal[4:7], codes in iscal[2:4].

        Gauss-Newton coupling: exact low-rank solve of the reduced system
        (csrc/lowrank.cu); full coupling (or schur_solver="dense"): dense
        mk x mk assembly + blocked Cholesky (csrc/ipm.cu, csrc/dense.cu).
        """
        P = self.P
        n, m, k, N, s = self.n, self.m, self.k, self.N, P.stream
        mux, muy = self.wx * self.mu, self.wy * self.mu
        X, Yt, F = self.X, self.Yt, self.Fcur
        rho = self.rho if rho is None else rho  # rho + inertia shift (frozen semantics 10)
        if not self.ffree:  # residual-free: YY^T and X^T X come from the refresh at this point
            P.colprod(Yt, m, k, Yt, k, self.GY)
            P.colprod(X, n, k, X, k, self.XtX, reduce=True)
        dense = full or self.dense_gn or force_dense
        fork = self.fork and not dense
        if fork:  # Y-side factor on the side stream (joined before nmfb_lowrank_factor)
            cur = torch.cuda.current_stream(P.dev)
            ev = torch.cuda.Event()
            ev.record(cur)
            self.side.wait_event(ev)
            with torch.cuda.stream(self.side):
                ss = P.stream
                P._call("nmfb_d_factor", _p(self.XtX), _p(Yt), _p(self.S), rho, m, k,
                        _p(self.LD), _p(self.Dinvpk), _p(self.YYpk), _p(P.iscal[4:]), ss)
                P._call("nmfb_atb", _p(self.YYpk), m, self.kk, _p(self.Dinvpk), self.kk,
                        _p(self.Gpk), _p(self.awork2), self.awork2.numel(), ss)
            ev_y = torch.cuda.Event()
            ev_y.record(self.side)
        P._call("nmfb_r1_factor", _p(self.GY), _p(X), _p(self.R), _p(self.gX), mux, rho, n,
                k, _p(self.L), _p(self.h), _p(self.g), _p(self.Apk), _p(self.XXpk),
                _p(P.iscal[2:]), s)
        self.comm.min_(P.iscal[2:3])
        ev_rhs = None
        if fork:  # H = X^T g and the Schur right-hand side on the side stream as well
            ev_r1 = torch.cuda.Event()
            ev_r1.record(cur)
            self.side.wait_event(ev_r1)
            with torch.cuda.stream(self.side):
                P.grams([(X, self.g, self.H)], n, k)
                P._call("nmfb_schur_rhs", _p(Yt), _p(self.gY), _p(self.H), None, muy, m, k,
                        _p(self.rhs), P.stream)
            ev_rhs = torch.cuda.Event()
            ev_rhs.record(self.side)
        P._call("nmfb_atb", _p(self.Apk), n, self.kk, _p(self.XXpk), self.kk, _p(self.Z),
                _p(self.awork), self.awork.numel(), s)
        self.comm.sum_(self.Z)
        if not fork:
            P.colprod(X, n, k, self.g, k, self.H, reduce=True)
        W = FtG = None
        if full:
            self._ensure_full_buffers()
            P._call("nmfb_make_p", _p(X), _p(self.Apk), n, k, _p(self.Pbuf), s)
            P._call("nmfb_atb", _p(F), n, m, _p(self.Pbuf), k ** 3, _p(self.W), _p(self.awork),
                    self.awork.numel(), s)
            self.comm.sum_(self.W)
            P.colprod(F, n, m, self.g, k, self.FtG, reduce=True)
            W, FtG = self.W, self.FtG
        if not fork:
            P._call("nmfb_schur_rhs", _p(Yt), _p(self.gY), _p(self.H), _p(FtG), muy, m, k,
                    _p(self.rhs), s)
        dY = self.dYbuf
        if dense:
            self._ensure_dense()
            P._call("nmfb_schur_assemble", _p(Yt), _p(self.S), m, k, _p(self.Z), _p(self.XtX),
                    rho, _p(W), _p(self.A), s)
            if full:
                if self.comm.active and not self.comm.root:
                    self.A.zero_()  # rank 0 carries the replicated part, others only term 4
                if self.t4work is None:
                    self.t4work = P.buf(max(P.lib.nmfb_term4_work_len(n, m, k), 1))
                P._call("nmfb_schur_term4", _p(F), n, m, k, _p(self.Apk), _p(self.A),
                        _p(self.t4work), self.t4work.numel(), s)
                self.comm.sum_(self.A)
            # the right-hand side rides along the factorization (b <- L^{-1} b as one more
            # tile row, csrc/dense_flow.cuh), then the backward half
            dY.copy_(self.rhs.view(m, k))
            P._call("nmfb_dense_cholesky_rhs", _p(self.A), N, _p(dY), _p(P.iscal[3:]), s)
            if early:
                # inertia tries (frozen semantics 10): two of three fail in the factorization;
                # read its code now and skip the back substitution and the direction kernels
                _, iv = P.readback(0, 4)
                if int(iv[2]) != _NONE:
                    raise NotPositiveDefinite("R1 block not positive definite", int(iv[2]))
                if int(iv[3]) >= 0:
                    self.last_dense = dense
                    return None
            P._call("nmfb_dense_solve_back", _p(self.A), N, _p(dY), s)
        else:
            if fork:
                cur.wait_event(ev_y)
            else:
                P._call("nmfb_d_factor", _p(self.XtX), _p(Yt), _p(self.S), rho, m, k,
                        _p(self.LD), _p(self.Dinvpk), _p(self.YYpk), _p(P.iscal[4:]), s)
                P._call("nmfb_atb", _p(self.YYpk), m, self.kk, _p(self.Dinvpk), self.kk,
                        _p(self.Gpk), _p(self.awork), self.awork.numel(), s)
            P._call("nmfb_lowrank_factor", _p(self.Z), _p(self.Gpk), k, _p(self.LG), _p(self.LH),
                    _p(self.lrwork), _p(P.iscal[3:]), s)
            if ev_rhs is not None:
                cur.wait_event(ev_rhs)
            self.lowrank_solve(self.rhs, dY, Yt)
        self.last_dense = dense
        P.colprod(Yt, m, k, dY, k, self.Gdy)
        FdY = None
        if full:
            P.rowprod(F, n, m, dY, k, self.FdY)
            FdY = self.FdY
        P._call("nmfb_direction", _p(self.L), _p(X), _p(self.h), _p(self.Gdy), _p(FdY), _p(X),
                _p(self.R), _p(self.gX), mux, _p(Yt), _p(self.S), _p(self.gY), _p(dY), muy,
                self.p.tau, n, m, k, _p(self.dX), _p(self.dR), _p(self.dS), _p(P.dscal[4:]),
                _p(P.rwork), P.rwork.numel(), s)
        self.reduce_direction()
        return dY

    def reduce_direction(self):
        """[gtp, a1, a2, gtp_rows, gtp_cols] at dscal[4:9]: rows summed, minima min-reduced."""
        if not self.comm.active:
            return
        d = self.P.dscal
        self.comm.sum_(d[7:8])
        self.comm.min_(d[5:7])
        d[4:5].copy_(d[7:8] + d[8:9])

    def armijo_launch(self, dY, trials=True):
        """Quartic coefficients + all backtracking barrier sums in two launches
        (trials=False: quartic only; the caller runs nmfb_armijo_lazy)."""
        P, s = self.P, self.P.stream
        n, m, k = self.n, self.m, self.k
        if self.ffree:
            self._armijo_free(dY, trials)
            return
        P._call("nmfb_quartic", _p(self.Fcur), n, m, k, _p(self.X), _p(self.dX), _p(self.Yt),
                _p(dY), _p(P.dscal[10:]), _p(P.rwork), s)
        if not trials:
            return
        P._call("nmfb_barrier_trials", _p(self.X), _p(self.dX), n * k, _p(self.Yt), _p(dY), m * k,
                _p(P.dscal[5:]), NTRIALS, _p(P.dscal[32:]), _p(P.rwork), P.rwork.numel(), s)
        if self.comm.active:
            self.comm.sum_(P.dscal[10:16])
            bx = P.dscal[32:32 + 2 * NTRIALS].view(NTRIALS, 2)[:, 0].contiguous()
            self.comm.sum_(bx)
            P.dscal[32:32 + 2 * NTRIALS].view(NTRIALS, 2)[:, 0].copy_(bx)

    def _armijo_free(self, dY, trials=True):
        """Quartic coefficients from k x k Grams + one streaming pass over M (M dY^T, and
        with the dual product also M^T dX for the next incremental refresh)."""
        P, s = self.P, self.P.stream
        n, m, k = self.n, self.m, self.k
        X, Yt, dX = self.X, self.Yt, self.dX
        if self.dual:
            P.dualprod(dY, dX, self.MdY, self.MtdX, self.dwork)
        else:
            P.rowprod(P.M, n, m, dY, k, self.MdY, None, P.f32)
        P.grams([(dX, dX, self.A1), (dX, X, self.A2), (dX, self.gX, self.Dgx),
                 (dX, self.MdY, self.Dmd)], n, k, reduce=True)
        P.grams([(dY, dY, self.B1), (Yt, dY, self.B2), (dY, self.gY, self.Dgy)], m, k)
        P._call("nmfb_ffree_quartic", _p(self.A1), _p(self.A2), _p(self.XtX), _p(self.B1),
                _p(self.B2), _p(self.GY), _p(self.Dgx), _p(self.Dgy), _p(self.Dmd), k,
                _p(P.dscal), s)
        if not trials:
            return
        P._call("nmfb_barrier_trials", _p(X), _p(dX), n * k, _p(Yt), _p(dY), m * k,
                _p(P.dscal[5:]), NTRIALS, _p(P.dscal[32:]), _p(P.rwork), P.rwork.numel(), s)
        if self.comm.active:
            bx = P.dscal[32:32 + 2 * NTRIALS].view(NTRIALS, 2)[:, 0].contiguous()
            self.comm.sum_(bx)
            P.dscal[32:32 + 2 * NTRIALS].view(NTRIALS, 2)[:, 0].copy_(bx)

    def remember_factorization_host(self, full):
        """Bookkeeping only (the fused step kernel copies X, Y itself)."""
        self.have_fact = True
        self.fact_full = full
        self.fact_dense = self.last_dense
        self.fact_F = self.fi

    def remember_factorization(self, full):
        self.Xf.copy_(self.X)
        self.Ytf.copy_(self.Yt)
        self.have_fact = True
        self.fact_full = full
        self.fact_dense = self.last_dense
        self.fact_F = self.fi

    def predictor_sigma(self, sums):
        """PAPER Eqs. 7-8 with the last Newton factorization."""
        P, p = self.P, self.p
        n, m, k, N, s = self.n, self.m, self.k, self.N, P.stream
        full = self.fact_full
        Ff = self.F[self.fact_F]
        P._call("nmfb_hg", _p(self.L), _p(self.gX), -1.0, n, k, _p(self.h), _p(self.g), s)
        P.colprod(self.Xf, n, k, self.g, k, self.H, reduce=True)
        FtG = None
        if full:
            P.colprod(Ff, n, m, self.g, k, self.FtG, reduce=True)
            FtG = self.FtG
        P._call("nmfb_schur_rhs", _p(self.Ytf), _p(self.gY), _p(self.H), _p(FtG), 0.0, m, k,
                _p(self.rhs), s)
        dY = self.dYbuf
        if self.fact_dense:
            dY.copy_(self.rhs.view(m, k))
            P._call("nmfb_dense_solve", _p(self.A), N, _p(dY), s)
        else:
            self.lowrank_solve(self.rhs, dY, self.Ytf)
        P.colprod(self.Ytf, m, k, dY, k, self.Gdy)
        FdY = None
        if full:
            P.rowprod(Ff, n, m, dY, k, self.FdY)
            FdY = self.FdY
        P._call("nmfb_direction", _p(self.L), _p(self.Xf), _p(self.h), _p(self.Gdy), _p(FdY),
                _p(self.X), _p(self.R), _p(self.gX), 0.0, _p(self.Yt), _p(self.S), _p(self.gY),
                _p(dY), 0.0, 1.0, n, m, k, _p(self.dX), _p(self.dR), _p(self.dS),
                _p(P.dscal[4:]), _p(P.rwork), P.rwork.numel(), s)
        self.reduce_direction()
        v, _ = P.readback(9)
        a1, a2 = v[5], v[6]
        P._call("nmfb_affine_mu", _p(self.X), _p(self.dX), _p(self.R), _p(self.dR), n * k,
                _p(self.Yt), _p(dY), _p(self.S), _p(self.dS), m * k * P.ny_local, a1, a2,
                _p(P.dscal[0:]), _p(P.rwork), s)
        self.comm.sum_(P.dscal[0:1])
        v, _ = P.readback(1)
        nk = P.n_global * k + m * k
        mu_aff = v[0] / nk
        mu_bar = (sums[3] + sums[7]) / nk
        return min((mu_aff / mu_bar) ** 3, p.sigma_cap)


@_nvtx("nmfb.ipm")
def run_ipm(P: Problem, X, Yt, R, S, mu, rho, p: IpmParams | None = None):
    """SPEC.md:337 run_ipm on the device (Algorithm 2 + Algorithm 3 switch).

    X, Yt, R, S are device tensors updated in place.  Returns (engine, IpmResult).
    """
    p = p or IpmParams()
    t0 = time.perf_counter()
    eng = _engine(P, X, Yt, R, S, mu, rho, p)
    try:
        return eng, _run_ipm(P, eng, p, t0)
    finally:  # the caller's tensors hold the final point (in-place contract)
        for dst, src in ((X, eng.X), (Yt, eng.Yt), (R, eng.R), (S, eng.S)):
            if dst is not src:
                dst.copy_(src)


def _engine(P: Problem, X, Yt, R, S, mu, rho, p: IpmParams):
    """The IpmEngine for this problem and parameter structure, cached on the Problem: a
    repeated solve (bench steps, streaming chunks of the same width, restarts) reuses
    its buffers and captured CUDA graphs instead of re-allocating and re-capturing."""
    key = (P.m, P.M.data_ptr(), float(rho), p.barrier, p.schur_solver, p.residual,
           p.use_graphs, p.fused_small, p.persistent, p.persist_grid, p.tau, p.eta,
           p.max_backtracks)
    cache = P.__dict__.setdefault("_engines", {})
    eng = cache.get(key)
    if eng is None:
        if len(cache) >= 4:
            cache.clear()
        eng = IpmEngine(P, X.clone(), Yt.clone(), R.clone(), S.clone(), mu, rho, p)
        cache[key] = eng
    else:
        eng.reset(X, Yt, R, S, mu, p)
    return eng


def _run_ipm(P: Problem, eng, p: IpmParams, t0):
    cap = p.fixed_iters if p.fixed_iters > 0 else p.max_iter
    tol = 0.0 if p.fixed_iters > 0 else p.eps_tol
    e_mu, e_zero, fsq, sums = eng.refresh()
    res = IpmResult(0, 0, False, e_zero, eng.mu, False)
    delta_last = 0.0
    n, m, k = P.n, P.m, P.k
    while e_zero > tol and res.iters < cap:
        eps_mu = eng.mu
        while e_mu > eps_mu and e_zero > tol and res.iters < cap:  # frozen semantics 8
            used_full = False
            ok = False
            if eng.flag:
                # full coupling C; frozen semantics 10: "paper" clears the
                # flag on the first non-PD / non-descent direction, "inertia" shifts rho
                delta = 0.0
                for _ in range(1 if p.hessian == "paper" else INERTIA_MAX_TRIES):
                    dY = eng.direction(True, rho=eng.rho + delta, early=True)
                    if dY is not None:  # None: the shifted Schur matrix did not factor
                        v, iv = P.readback(9, 4)
                        if int(iv[2]) != _NONE:
                            raise NotPositiveDefinite("R1 block not positive definite", int(iv[2]))
                        if int(iv[3]) < 0 and v[4] < 0.0:
                            ok, used_full = True, True
                            break
                    delta = (delta * INERTIA_GROW if delta > 0.0 else
                             (delta_last / INERTIA_SHRINK if delta_last > 0.0 else eng.rho))
                if ok:
                    delta_last = delta
                    res.deltas.append(delta)
                    eng.armijo_launch(dY)
                    v, iv = P.readback(32 + 2 * NTRIALS, 4)
                    eng.remember_factorization(True)
                else:
                    eng.flag = False
            force_dense = False
            if not ok and eng.persist:
                code, done, kkt = eng.persist_run(eps_mu, tol, cap - res.iters, res, t0)
                if done:
                    e_mu, e_zero, fsq, sums = kkt
                if code == 2:
                    raise LineSearchStall(f"Armijo backtracking exceeded {p.max_backtracks}")
                if code == 0:
                    continue
                # a factorization failed at the current point (no step was taken):
                # redo this iteration eagerly with the dense Schur solve
                force_dense = True
                res.dense_fallbacks += 1
            if force_dense:
                pass
            elif not ok and eng.use_graphs:
                eng.gn_iteration_graph()
                v, iv = P.readback(28, 6)
                for e0, e1 in eng.graphs[eng.last_graph][1]:
                    try:
                        P.event_times.append(e0.elapsed_time(e1))
                    except Exception:  # event nodes not timeable on this stack
                        P.graph_timing_failed = True
                if int(v[2]) == -2 and not eng.ffree:
                    # the rank-k^2 factorization lost positive definiteness by rounding:
                    # no step was taken; redo this iteration with the dense Schur solve
                    force_dense = True
                    res.dense_fallbacks += 1
            if force_dense:
                pass
            elif not ok and eng.use_graphs:
                if int(iv[2]) != _NONE:
                    raise NotPositiveDefinite("R1 block not positive definite", int(iv[2]))
                if int(iv[4]) != _NONE:
                    raise NotPositiveDefinite("R2 block not positive definite", int(iv[4]))
                if int(iv[3]) >= 0:
                    raise NotPositiveDefinite("Gauss-Newton Schur matrix not positive definite",
                                              int(iv[3]))
                t = int(v[2])
                if t > p.max_backtracks:
                    raise LineSearchStall(f"Armijo backtracking exceeded {p.max_backtracks}")
                a1, a2max = v[1], v[3]
                res.iters += 1
                res.armijo_t.append(t)
                res.flags.append(False)
                e_mu, e_zero = kkt_from_sums(v[16:28])
                fsq, sums = v[0], v[16:28]
                redo = eng.check_advance(iv[5])
                if redo is not None:
                    e_mu, e_zero, fsq, sums = redo
                res.trace.append((time.perf_counter() - t0, 0.5 * fsq, e_zero, eng.mu, a1, a2max, t))
                continue
            if not ok:
                dY = eng.direction(False, force_dense=force_dense)
                eng.armijo_launch(dY)
                v, iv = P.readback(32 + 2 * NTRIALS, 5)
                if int(iv[2]) != _NONE:
                    raise NotPositiveDefinite("R1 block not positive definite", int(iv[2]))
                if not eng.last_dense and int(iv[4]) != _NONE:
                    raise NotPositiveDefinite("R2 block not positive definite", int(iv[4]))
                if int(iv[3]) >= 0 and not eng.last_dense and not eng.ffree:
                    # low-rank capacitance lost PD-ness by rounding: dense Schur solve
                    res.dense_fallbacks += 1
                    dY = eng.direction(False, force_dense=True)
                    eng.armijo_launch(dY)
                    v, iv = P.readback(32 + 2 * NTRIALS, 5)
                if int(iv[3]) >= 0:
                    raise NotPositiveDefinite("Gauss-Newton Schur matrix not positive definite",
                                              int(iv[3]))
                eng.remember_factorization(False)
            gtp, a1max, a2max = v[4], v[5], v[6]
            aa, ab, bb, ac, bc, cc = v[10:16]
            bars = v[32:32 + 2 * NTRIALS]
            t = 0
            while True:
                a1 = a1max / (2.0 ** t)
                a2_, a3_ = a1 * a1, a1 * a1 * a1
                quad = a1 * ab + a2_ * (0.5 * bb + ac) + a3_ * bc + 0.5 * (a3_ * a1) * cc
                dphi = quad - eng.mu * (eng.wx * bars[2 * t] + eng.wy * bars[2 * t + 1])
                if dphi <= p.eta * a1 * gtp:
                    break
                t += 1
                if t > p.max_backtracks:
                    raise LineSearchStall(f"Armijo backtracking exceeded {p.max_backtracks}")
            eng.take_step(dY, None, a1, None, a2max)
            res.iters += 1
            res.armijo_t.append(t)
            res.flags.append(used_full)
            e_mu, e_zero, fsq, sums = eng.refresh()
            redo = eng.check_advance()
            if redo is not None:
                e_mu, e_zero, fsq, sums = redo
            res.trace.append((time.perf_counter() - t0, 0.5 * fsq, e_zero, eng.mu, a1, a2max, t))
        res.outer += 1
        if e_zero <= tol or res.iters >= cap:
            break
        if not eng.have_fact:
            eng.direction(False)
            v, iv = P.readback(8, 4)
            eng.remember_factorization(False)
        sigma = eng.predictor_sigma(sums)
        eng.mu = sigma * eng.mu
        # the full-Hessian coupling needs the dense mk x mk system and the residual F;
        # in residual-free mode (very large M) the Gauss-Newton coupling is kept
        eng.flag = sigma <= p.sigma_c and not eng.ffree
        e_mu, e_zero, fsq, sums = eng.refresh()
    res.converged = e_zero <= tol
    res.mu, res.flag = eng.mu, eng.flag
    res.seconds = time.perf_counter() - t0
    return res


@_nvtx("nmfb.transition")
def transition(P: Problem, X, Yt, eps_tol, tp: TransitionParams | None = None):
    """SPEC.md:393 / PAPER Eqs. 14-18 on the device -> (X, Yt, R, S, mu, rho)."""
    tp = tp or TransitionParams()
    n, m, k, s = P.n, P.m, P.k, P.stream
    X, Yt = X.clone(), Yt.clone()
    gX, gY = P.buf(n, k), P.buf(m, k)
    if P.free_residual_default:
        ws = P.free_workspace()
        grad = lambda: P.gradients_free(X, Yt, gX, gY, ws)  # noqa: E731
    else:
        F = P.buf(n, m)
        grad = lambda: P.gradients(X, Yt, F, gX, gY)  # noqa: E731
    # max over the concatenated (x, y)
    grad()
    P.kkt_sums(X, None, gX, Yt, None, gY, 0.0, 0.0, at=16)
    v, _ = P.readback(28)
    big = max(v[26], v[27])
    if not big > 0.0:
        raise DegenerateFactor("X and Y are identically zero: transition undefined")
    rho0 = tp.rho0_scale * big
    P._call("nmfb_clamp_min", _p(X), n * k, rho0, s)
    P._call("nmfb_clamp_min", _p(Yt), m * k, rho0, s)
    grad()
    P.kkt_sums(X, None, gX, Yt, None, gY, 0.0, 0.0, at=16)
    v, _ = P.readback(28)
    R, S = P.buf(n, k), P.buf(m, k)
    P._call("nmfb_fill", _p(R), n * k, float(v[24]), s)
    P._call("nmfb_fill", _p(S), m * k, float(v[25]), s)
    P.kkt_sums(X, R, gX, Yt, S, gY, 0.0, 0.0, at=16)
    v, _ = P.readback(28)
    mu = (v[19] + v[23]) / (P.n_global * k + m * k)
    return X, Yt, R, S, mu, float(eps_tol)


def kkt_error_primal_only_dev(P: Problem, X, Yt):
    """SPEC.md:420 on the device."""
    n, m, k = P.n, P.m, P.k
    gX, gY = P.buf(n, k), P.buf(m, k)
    if P.free_residual_default:
        P.gradients_free(X, Yt, gX, gY, P.free_workspace())
    else:
        P.gradients(X, Yt, P.buf(n, m), gX, gY)
    P.kkt_sums(X, None, gX, Yt, None, gY, 0.0, 0.0, at=16)
    v, _ = P.readback(28)
    return kkt_from_sums(v[16:28])[1], 0.5 * v[0]


@_nvtx("nmfb.two_stage")
def run_two_stage(M, X0, Y0, tol_rel=1e-10, s1: Stage1Config | None = None,
                  ipm: IpmParams | None = None, tp: TransitionParams | None = None,
                  stage="two_stage", pX=None, pY=None, e_scale=None, problem: Problem | None = None,
                  comm: Comm | None = None):
    """SPEC.md:411 run_two_stage (Algorithm 3) on the B200.

    M (n,m) host or device array (fp64, or fp32 storage); X0 (n,k); Y0 (k,m).
    Relative KKT tolerance: eps_abs = tol_rel * max(1, E_primal(X0, Y0)) unless
    ``e_scale`` is given (frozen semantics 5).  With ``comm`` spanning
    several GPUs, M / X0 / pX are this rank's row block (dist.row_range) and the
    returned X / R are the local rows.
    """
    X0n = X0 if isinstance(X0, torch.Tensor) else np.asarray(X0, dtype=np.float64)
    k = X0n.shape[1]
    if problem is not None and M is not None and M is not problem.M:
        problem.load(M)  # new data into the resident problem (no allocation)
    P = problem or Problem(M, k, comm=comm)

    def carry(c):
        if c is None:
            return None
        if isinstance(c, torch.Tensor):
            return c.to(P.dev, dtype=torch.uint8)
        return torch.as_tensor(np.asarray(c, np.uint8)).to(P.dev)

    X = P.to_dev(X0)
    Yt = P.to_dev(Y0.T if not isinstance(Y0, torch.Tensor) else Y0.t())
    if e_scale is None:
        e_scale = max(1.0, kkt_error_primal_only_dev(P, X, Yt)[0])
    eps_abs = tol_rel * e_scale
    p = ipm or IpmParams()
    p.eps_tol = eps_abs
    s1 = s1 or Stage1Config()
    if stage == "ipm_only":
        r1 = Stage1Result(None, None, None, None, 0, False)
        pXd = pYd = None
    else:
        pXd, pYd = carry(pX), carry(pY)
        X, Yt, pXd, pYd, r1 = run_stage1(P, X, Yt, s1, pXd, pYd)
    r1.X, r1.Yt = X.cpu().numpy(), Yt.cpu().numpy()
    r1.pX = None if pXd is None else pXd.bool().cpu().numpy()
    r1.pY = None if pYd is None else pYd.bool().cpu().numpy()
    if stage == "anls_only":
        e0, f = kkt_error_primal_only_dev(P, X, Yt)
        return SolveReport("Converged" if e0 <= eps_abs else "IterationCap", r1.X, r1.Yt, None,
                           None, f, e0, eps_abs, r1, None, r1.seconds, 0.0)
    X, Yt, R, S, mu, rho = transition(P, X, Yt, eps_abs, tp)
    eng, r2 = run_ipm(P, X, Yt, R, S, mu, rho, p)
    e_mu, e_zero, fsq, _ = eng.refresh()
    status = "Converged" if r2.converged else "IterationCap"
    rep = SolveReport(status, eng.X.cpu().numpy(), eng.Yt.cpu().numpy(), eng.R.cpu().numpy(),
                      eng.S.cpu().numpy(), 0.5 * fsq, e_zero, eps_abs, r1, r2, r1.seconds,
                      r2.seconds)
    # device-resident final factors and stage-1 carries (streaming sessions continue from them)
    rep.dev_state = {"X": eng.X, "Yt": eng.Yt, "pX": pXd, "pY": pYd}
    return rep
