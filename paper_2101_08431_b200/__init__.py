"""B200-native two-stage NMF (arXiv 2101.08431): warm-started active-set ANLS + primal-dual IPM.

Public entry points keep the reference specification's names and options
(SPEC.md:411 run_two_stage, :209 run_stage1, :337 run_ipm, :393 transition);
the seven reference kernels are available as a drop-in module
(``paper_2101_08431_b200.kernels``).  All numerics run in libnmfb200.so
(sm_100a); there is no CPU fallback.
"""
from .config import IpmParams, SolveReport, Stage1Config, TransitionParams  # noqa: F401
from .errors import *  # noqa: F401,F403


def run_two_stage(M, X0, Y0, tol_rel=1e-10, cfg=None, ipm=None, tp=None, stage="two_stage",
                  s1=None, **kw):
    """SPEC.md:411 run_two_stage on the B200 (see solver.run_two_stage).  ``cfg`` (or its
    alias ``s1``) is the Stage1Config, ``ipm`` the IpmParams, ``tp`` the TransitionParams."""
    from . import solver

    return solver.run_two_stage(M, X0, Y0, tol_rel=tol_rel, s1=s1 or cfg, ipm=ipm, tp=tp,
                                stage=stage, **kw)


def SolvePipeline(*a, **kw):
    """Two resident problem slots; the next instance's host-to-device copy overlaps the
    current solve (see pipeline.SolvePipeline)."""
    from .pipeline import SolvePipeline as _SP

    return _SP(*a, **kw)


__all__ = ["run_two_stage", "SolvePipeline", "Stage1Config", "IpmParams", "TransitionParams", "SolveReport"]
