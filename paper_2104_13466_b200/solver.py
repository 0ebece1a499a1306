"""Jacobi-PCG on the GPU: drop-in for ``sdmefem.solver.pcg`` / ``LinearSolver``.

The reference's ``pcg(a, b, precond, tol, maxit)`` (``solver.py:129-170``)
needs an assembled matrix (``a @ p`` and ``a.diagonal()``), so the drop-in
replaces the *solver*, not just the operator.  The operator is
A = c_k K_T(u_lin) + c_m M, applied matrix-free on the device; the iteration,
its order of checks (pAp <= 0 -> PCGError; recursive-residual stop; maxit ->
PCGError with the true residual) and :class:`SolveStats` are the reference's.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import native
from .errors import PCGError
from .problem import DeviceVector, GpuFemProblem

__all__ = ["SolveStats", "StatsLog", "PCGError", "SolverConfig", "pcg_gpu", "GpuLinearSolver",
           "AssembledLinearSolver", "DriverSolver", "make_solver"]

_PRECOND = {"diagonal": 1, "none": 0, None: 0}
_ASSEMBLED = ("sgs", "gauss-seidel")  # need the assembled CSR (csrc/schur.cu)


@dataclass
class SolveStats:
    """``solver.py:41-47``."""

    iterations: int
    residual: float
    seconds: float
    preconditioner: str
    converged: bool = True


@dataclass
class StatsLog:
    """``solver.py:50-75``: per-linear-solve records of the drivers."""

    rows: list = field(default_factory=list)

    def add(self, step: int, newton_iter: int, solver: str, stats: SolveStats):
        self.rows.append({"step": step, "newton_iter": newton_iter, "solver": solver,
                          "preconditioner": stats.preconditioner, "iterations": stats.iterations,
                          "residual": stats.residual, "seconds": stats.seconds})

    def mean_iterations(self) -> float:
        return float(np.mean([r["iterations"] for r in self.rows])) if self.rows else 0.0

    def total_seconds(self) -> float:
        return float(sum(r["seconds"] for r in self.rows))


@dataclass
class SolverConfig:
    """``dynamics.py:38-43``.  ``precond`` "diagonal" / "none" with
    ``condense=False`` is the matrix-free Jacobi-PCG path (any mesh size, SURVEY
    D3); ``precond="sgs"`` and / or ``condense=True`` select the assembled
    path, the reference's default solver (:class:`~.schur.SchurSolver`: dense
    element matrices, Schur condensation, level-scheduled SGS on the device),
    sized like the reference.  The defaults are the reference's (SGS with
    Schur condensation, tol 1e-12), so ``SolverConfig()`` and drivers called
    without ``cfg`` behave as the reference does; pass ``precond="diagonal",
    condense=False`` for the matrix-free path on large meshes."""

    precond: str = "sgs"
    tol: float = 1e-12
    maxit: int = 200000
    condense: bool = True

    @classmethod
    def coerce(cls, cfg) -> "SolverConfig | None":
        """This class, or any object with the reference ``SolverConfig``'s
        fields (``dynamics.py:38-43``: precond, tol, maxit, condense) --
        e.g. ``sdmefem.dynamics.SolverConfig`` itself -- as a GPU-path config."""
        if cfg is None or isinstance(cfg, cls):
            return cfg
        try:
            return cls(precond=cfg.precond, tol=float(cfg.tol), maxit=int(cfg.maxit), condense=bool(cfg.condense))
        except AttributeError as exc:
            raise TypeError(f"not a solver configuration: {cfg!r}") from exc

    @classmethod
    def reference_default(cls) -> "SolverConfig":
        """``sdmefem.dynamics.SolverConfig()``: SGS, Schur condensation, tol 1e-12."""
        return cls(precond="sgs", tol=1e-12, maxit=200000, condense=True)

    @classmethod
    def matrix_free(cls, tol: float = 1e-10, maxit: int = 200000) -> "SolverConfig":
        """Jacobi-PCG on the matrix-free operator: any mesh size."""
        return cls(precond="diagonal", tol=tol, maxit=maxit, condense=False)

    @property
    def assembled(self) -> bool:
        """True when the solve needs the assembled operator (SGS or condensation)."""
        return bool(self.condense) or self.precond in _ASSEMBLED

    def validate(self):
        if self.precond not in _PRECOND and self.precond not in _ASSEMBLED:
            raise ValueError(f"unknown preconditioner {self.precond!r}")


def pcg_gpu(problem: GpuFemProblem, u_lin, b, c_m: float = 0.0, precond: str = "diagonal",
            tol: float = 1e-8, maxit: int = 10000, c_k: float = 1.0, x: DeviceVector | None = None):
    """Solve (c_k K_T(u_lin) + c_m M) x = b on the device.

    ``u_lin`` / ``b``: free-order ndarrays or :class:`DeviceVector`.  Returns
    (x, SolveStats) with x of the same kind as ``b``.  Raises ``ValueError``
    for a bad tol or non-positive diagonal and :class:`PCGError` exactly where
    the reference does.
    """
    if not 0.0 < tol < 1.0:
        raise ValueError(f"tolerance must lie in (0, 1), got {tol}")
    if precond not in _PRECOND:
        raise ValueError(f"unknown preconditioner {precond!r}")
    tag = "diagonal" if _PRECOND[precond] == 1 else "none"
    t0 = time.perf_counter()
    host = not isinstance(b, DeviceVector)
    bv = problem._scratch("pcg_b").set_free(b) if host else b
    if u_lin is None or c_k == 0.0:
        uv = None
    elif isinstance(u_lin, DeviceVector):
        uv = u_lin
    else:
        uv = problem._scratch("pcg_u").set_free(u_lin)
    xv = x if x is not None else (problem._scratch("pcg_x") if host else DeviceVector(problem))
    its = C.c_int(0)
    rel = C.c_double(0.0)
    rc = native.lib().sdme_pcg(problem._ctx, uv.vid if uv is not None else -1, c_k, c_m, bv.vid, xv.vid,
                               tol, maxit, _PRECOND[precond], C.byref(its), C.byref(rel))
    secs = time.perf_counter() - t0
    if rc in (native.INDEFINITE, native.MAXIT):
        _, _, _, msg = native.last_error(problem._ctx)
        raise PCGError(msg, SolveStats(its.value, rel.value, secs, tag, False))
    native.check(problem._ctx, rc, "pcg")
    stats = SolveStats(its.value, rel.value, secs, tag)
    return (xv.free() if host else xv), stats


@dataclass
class GpuLinearSolver:
    """``LinearSolver`` (solver.py:302-322) for A = c_k K_T(u_lin) + c_m M."""

    problem: GpuFemProblem
    u_lin: DeviceVector | None
    c_m: float = 0.0
    precond: str = "diagonal"
    tol: float = 1e-8
    maxit: int = 50000
    c_k: float = 1.0

    @property
    def condensed(self) -> bool:
        return False

    def solve(self, rhs, x: DeviceVector | None = None):
        return pcg_gpu(self.problem, self.u_lin, rhs, self.c_m, self.precond, self.tol, self.maxit,
                       self.c_k, x=x)


class AssembledLinearSolver:
    """``LinearSolver`` (solver.py:302-322) on the assembled / condensed operator
    c_k K_T(u_lin) + c_m M (:class:`~.schur.SchurSolver`)."""

    def __init__(self, schur, u_lin, c_m: float, c_k: float = 1.0):
        self.schur = schur
        self.schur.factor(u_lin, c_k, c_m)

    @property
    def condensed(self) -> bool:
        return self.schur.condensed

    def solve(self, rhs, x: DeviceVector | None = None):
        return self.schur.solve(rhs, x=x)


def make_solver(problem: GpuFemProblem, u_lin, c_m: float, cfg: SolverConfig,
                c_k: float = 1.0):
    """``make_solver`` (dynamics.py:111-127) without element matrices: the
    operator is defined by its linearisation point and mass coefficient.
    ``cfg`` may be this package's or the reference's ``SolverConfig``; with
    ``condense=True`` or ``precond="sgs"`` the result is the assembled solver
    (the reference's default path), else matrix-free Jacobi-PCG."""
    cfg = SolverConfig.coerce(cfg)
    cfg.validate()
    if cfg.assembled:
        from .schur import SchurSolver

        sch = SchurSolver(problem, cfg.condense, cfg.precond, cfg.tol, cfg.maxit)
        return AssembledLinearSolver(sch, u_lin, c_m, c_k)
    if u_lin is not None and not isinstance(u_lin, DeviceVector):
        u_lin = problem.vector(np.asarray(u_lin, dtype=float))
    return GpuLinearSolver(problem, u_lin, c_m, cfg.precond, cfg.tol, cfg.maxit, c_k)


class DriverSolver:
    """The linear solves of one time-integration run (dynamics.py:186-241):
    matrix-free Jacobi-PCG, or the assembled / condensed solver whose
    structure (CSR pattern, SGS levels, element tables) is built once per run
    and refactored per operator."""

    def __init__(self, problem: GpuFemProblem, cfg: SolverConfig):
        self.pb, self.cfg = problem, cfg
        self._schur = {}

    def solve(self, u_lin, c_k: float, c_m: float, rhs: DeviceVector, x: DeviceVector, slot: str = "k"):
        """x = (c_k K_T(u_lin) + c_m M)^-1 rhs; ``slot`` names a cached factorisation
        reused while (c_k, c_m, u_lin) stay the same object/values."""
        cfg = self.cfg
        if not cfg.assembled:
            return pcg_gpu(self.pb, u_lin, rhs, c_m=c_m, precond=cfg.precond, tol=cfg.tol, maxit=cfg.maxit,
                           c_k=c_k, x=x)
        from .schur import SchurSolver

        ent = self._schur.get(slot)
        key = (c_k, c_m)
        if ent is None:
            ent = self._schur[slot] = [SchurSolver(self.pb, cfg.condense, cfg.precond, cfg.tol, cfg.maxit), None]
        if c_k != 0.0 or ent[1] != key:  # K_T(u) changes every call; mass-only operators factor once
            ent[0].factor(u_lin, c_k, c_m)
            ent[1] = key
        return ent[0].solve(rhs, x=x)
