"""Solver configuration and report types.

Option names and defaults follow the reference specification so a caller of
the reference's stage drivers can pass the same settings.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Stage1Config:
    """Stage-1 ANLS options (defaults :226-230)."""

    eps_stol: float = 1e-3  # relative step tolerance
    max_sweeps: int = 200
    tol_kkt: float | None = None  # None: 1e-12 * max(1, ||C^T d||_inf) per rhs
    fixed_sweeps: int = 0  # > 0: exactly this many sweeps, no step test (configs c4/c5)
    persistent: bool = True  # small problems: all sweeps in one launch (csrc/stage1_persist.cu)


@dataclass
class IpmParams:
    """Stage-2 interior-point options."""

    tau: float = 0.9
    eta: float = 0.5
    sigma_cap: float = 0.99
    sigma_c: float = 0.01
    eps_tol: float = 1e-6
    max_iter: int = 500
    max_backtracks: int = 60
    fixed_iters: int = 0  # > 0: exactly this many inner iterations (configs c4/c5)
    barrier: str = "balanced"  # "balanced" (default, meets SPEC acceptance 5-7) | "paper" (literal single mu)
    # full-coupling directions while the Algorithm-3 flag is set: "inertia" (default) shifts
    # rho until the Schur matrix factors and the direction is descent; "paper" clears the
    # flag on the first failure (DESIGN.md frozen semantics 10)
    hessian: str = "inertia"
    schur_solver: str = "lowrank"  # Gauss-Newton reduced system: "lowrank" (exact, rank k^2) | "dense"
    use_graphs: bool = True  # replay each Gauss-Newton iteration as a captured CUDA graph
    fused_small: bool = True  # fused 6-kernel iteration when k <= 4 and m k <= 2048 (csrc/small.cu)
    persistent: bool = True  # whole inner loop in one cooperative launch (csrc/persist.cu)
    persist_grid: int = 0  # CTAs of the persistent launch (0: automatic)
    residual: str = "auto"  # "dense" (materialise F) | "free" (Grams + M passes) | "auto" (free if n m >= 2^25)


@dataclass
class TransitionParams:
    """Transition options, Eqs. 14-15."""

    rho0_scale: float = 1e-6


@dataclass
class Stage1Result:
    X: np.ndarray
    Yt: np.ndarray
    pX: np.ndarray
    pY: np.ndarray
    sweeps: int
    converged: bool
    trace: list = field(default_factory=list)  # (seconds, objective, step)
    seconds: float = 0.0


@dataclass
class IpmResult:
    iters: int
    outer: int
    converged: bool
    E0: float
    mu: float
    flag: bool
    trace: list = field(default_factory=list)  # (seconds, objective, E0, mu, a1, a2, t)
    armijo_t: list = field(default_factory=list)
    flags: list = field(default_factory=list)
    deltas: list = field(default_factory=list)  # inertia shift of each full-coupling iteration
    seconds: float = 0.0
    dense_fallbacks: int = 0  # GN iterations re-solved densely after a low-rank PD failure


@dataclass
class SolveReport:
    """SPEC.md:381-386 SolveReport (plus the final factors and duals)."""

    status: str  # "Converged" | "IterationCap" | "Error"
    X: np.ndarray
    Yt: np.ndarray
    R: np.ndarray | None
    S: np.ndarray | None
    final_objective: float
    final_kkt_error: float
    eps_abs: float
    stage1: Stage1Result
    ipm: IpmResult | None
    stage1_time: float
    stage2_time: float
    error: str = ""

    @property
    def Y(self):
        return self.Yt.T

    @property
    def converged(self):
        return self.status == "Converged"
