"""Time integration drivers on device-resident vectors.

``newmark_run`` follows ``sdmefem.dynamics.newmark_run`` (``dynamics.py:173-257``)
step for step -- trial acceleration, residual psi = P - R(u) - M a, Newton
stop relative to the first ||psi|| of the step, effective operator
K_T + b1 M, Newmark v/a update -- with every vector operation on the GPU and
the linear solves done by matrix-free Jacobi-PCG.  With
``contact=`` the residual carries the penalty force, Newton also waits for the
contact pressures to settle, the operator adds the contact stiffness of the
current active set (matrix-free, sdme_pcg_contact) and every accepted step
runs ``accept_step`` -- ``dynamics.py:196-255`` / ``contact.py:103-176``.

``explicit_run`` is the central-difference scheme of ``dynamics.py:130-170``
with the row-sum lumped mass and penalty contact against a rigid plane
(SURVEY D6): m_L = M 1, w = dt^2 psi / m_L, u+ = 2u - u_prev + w,
v = (u+ - u_prev) / (2 dt).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import native
from .errors import NewtonDivergenceError
from .problem import DeviceVector, GpuFemProblem
from .solver import DriverSolver, SolverConfig, StatsLog, pcg_gpu

__all__ = ["NewmarkCoeffs", "TimeState", "Trajectory", "ScaledLoad", "cfl_dt", "newmark_run",
           "explicit_run", "estimate_lambda_max"]


@dataclass
class NewmarkCoeffs:
    """``dynamics.py:46-59``."""

    dt: float
    gamma: float = 0.5
    beta: float = 0.25

    def __post_init__(self):
        if self.dt <= 0.0:
            raise ValueError("time step must be positive")
        self.b1 = 1.0 / (self.beta * self.dt ** 2)
        self.b2 = 1.0 / (self.beta * self.dt)
        self.b3 = (1.0 - 2.0 * self.beta) / (2.0 * self.beta)


@dataclass
class TimeState:
    t: float
    u: np.ndarray
    v: np.ndarray
    a: np.ndarray
    u_prev: np.ndarray | None = None


@dataclass
class Trajectory:
    times: list = field(default_factory=list)
    snapshots: list = field(default_factory=list)
    energy: list = field(default_factory=list)
    state: TimeState | None = None
    stats: StatsLog = field(default_factory=StatsLog)
    newton_iters: list = field(default_factory=list)
    contact_history: list = field(default_factory=list)


class ScaledLoad:
    """external_load(t) = scale(t) * base, kept on the device (one upload).

    Any plain callable returning a free vector is accepted by the drivers too
    (uploaded every evaluation); this form avoids the per-step transfer.
    """

    def __init__(self, base_free: np.ndarray, scale=lambda t: 1.0):
        self.base = np.asarray(base_free, dtype=float)
        self.scale = scale

    def __call__(self, t):
        return self.scale(t) * self.base


_CFL_MODES = ("AsPrinted", "PhysicalSqrt")


def cfl_dt(mesh, mat, delta: float, mode: str = "AsPrinted") -> float:
    """Time-step estimate delta * h_min / c (``dynamics.py:81-101``, host only).

    With E = mu (3 lam + 2 mu)/(lam + mu), nu = lam / (2 (lam + mu)) and
    K = E / (3 (1 - 2 nu)), the wave-speed expression is
    c2 = 3 K (1 - nu) / (rho (1 + nu)) = (lam + 2 mu) / rho, i.e. the squared
    dilatational wave speed.  "PhysicalSqrt" uses c = sqrt(c2); "AsPrinted"
    uses c2 itself (no square root), as the reference's scenario step counts do.
    """
    if not (0.2 < delta < 0.9):
        raise ValueError(f"delta should lie in (0.2, 0.9), got {delta}")
    if mode not in _CFL_MODES:
        raise ValueError(f"unknown CFL mode {mode!r}")
    mu, lam = float(mat.mu), float(mat.lambda_lame)
    young = mu * (3.0 * lam + 2.0 * mu) / (lam + mu)
    poisson = 0.5 * lam / (lam + mu)
    bulk = young / (3.0 - 6.0 * poisson)
    c2 = 3.0 * bulk * (1.0 - poisson) / ((1.0 + poisson) * mat.rho0)
    speed = float(np.sqrt(c2)) if mode == "PhysicalSqrt" else c2
    return delta * mesh.min_edge_length() / speed


class _Load:
    """Evaluates external_load(t) into a device vector."""

    def __init__(self, problem: GpuFemProblem, external_load):
        self.pb = problem
        self.fn = external_load
        self.vec = DeviceVector(problem)
        self.scaled = isinstance(external_load, ScaledLoad)
        if self.scaled:
            self.base = DeviceVector(problem).set_free(external_load.base)
        self._last = None

    def at(self, t: float) -> DeviceVector:
        if self.scaled:
            s = float(self.fn.scale(t))
            if self._last != s:
                self.vec.assign(s, self.base)
                self._last = s
        else:
            self.vec.set_free(np.asarray(self.fn(t), dtype=float))
        return self.vec


def _fused_residual(pb, lib, uk, du, u, v, a, load, t_next, nm, atr, tmp, psi) -> float:
    """``residual`` + ``psi.norm()`` of one Newton iterate without contact, as
    one native call (``sdme_newmark_residual``; bit-identical to the separate calls)."""
    import ctypes as C

    if load.scaled:
        lid, s = load.base.vid, float(load.fn.scale(t_next))
    else:
        lid, s = load.at(t_next).vid, 1.0
    out = C.c_double(0.0)
    native.check(pb._ctx, lib.sdme_newmark_residual(pb._ctx, uk.vid, du.vid if du is not None else -1, u.vid, v.vid,
                                                    a.vid, lid, s, nm.b1, nm.b2, nm.b3, atr.vid, tmp.vid, psi.vid,
                                                    C.byref(out)), "newmark residual")
    return out.value


def _dev(problem, x) -> DeviceVector:
    v = DeviceVector(problem)
    if x is not None:
        v.set_free(np.asarray(x, dtype=float))
    return v


def newmark_run(problem: GpuFemProblem, external_load, dt: float, n_steps: int,
                newton_tol: float = 1e-8, newton_maxit: int = 25, u0=None, v0=None,
                cfg: SolverConfig | None = None, gamma: float = 0.5, beta: float = 0.25,
                contact=None, snapshot_stride: int = 0, track_energy: bool = False) -> Trajectory:
    """Implicit Newmark with Newton-Raphson (``dynamics.py:173-257``)."""
    cfg = SolverConfig.coerce(cfg) or SolverConfig()  # the reference's default: SGS + Schur
    cfg.validate()
    nm = NewmarkCoeffs(dt, gamma, beta)
    pb = problem
    u = _dev(pb, u0)
    v = _dev(pb, v0)
    load = _Load(pb, external_load)
    traj = Trajectory()
    uk, atr, psi, tmp, du, a = (DeviceVector(pb) for _ in range(6))
    fcv = DeviceVector(pb) if contact is not None else None
    lib = native.lib()

    def residual(uk_, atr_, t_next):
        """psi = P(t) - R(uk) - M a_trial (+ f_c(uk))  (dynamics.py:197-203);
        returns (contact settled, any contact point active)."""
        pb.fint_(uk_, tmp)
        pb.mass_(atr_, psi)
        if contact is None:
            psi.assign(1.0, load.at(t_next), -1.0, tmp, -1.0, psi)
            return True, False
        settled, active = contact.evaluate_(uk_, fcv)
        psi.assign(1.0, load.at(t_next), -1.0, tmp, -1.0, psi, 1.0, fcv)
        return settled, active

    # a0 = M^-1 psi0 (mass-only PCG, short-circuits for psi0 = 0)
    solver = DriverSolver(pb, cfg)
    atr.fill(0.0)
    residual(u, atr, 0.0)
    _, st = solver.solve(None, 0.0, 1.0, psi, a, slot="mass")
    traj.stats.add(-1, 0, "newmark-init", st)

    t = 0.0

    def energy_row(tt):
        # (t, kinetic 1/2 v.Mv, strain, penalty) -- dynamics.py:260-265
        kin = 0.5 * v.dot(pb.mass_(v, tmp))
        pen = contact.penalty_energy_(u, fcv) if contact is not None else 0.0
        traj.energy.append((tt, kin, pb.strain_energy_(u), pen))

    if track_energy:
        energy_row(t)
    for step in range(n_steps):
        t_next = t + dt
        uk.copy_from(u)
        psi_ref = None
        n_newton = 0
        pending = False  # uk += du folded into the next fused residual
        for k in range(newton_maxit):
            if contact is None:
                # one enqueued sequence + one host sync (sdme_newmark_residual):
                # [uk += du]; a_trial = b1 (uk - u) - b2 v - b3 a; psi = P - f_int - M a_trial
                rnorm = _fused_residual(pb, lib, uk, du if pending else None, u, v, a, load, t_next, nm,
                                        atr, tmp, psi)
                pending = False
                contact_ok, active = True, False
            else:
                # a_trial = b1 (uk - u) - b2 v - b3 a  (difference first, as dynamics.py:219)
                tmp.assign(1.0, uk, -1.0, u)
                atr.assign(nm.b1, tmp, -nm.b2, v, -nm.b3, a)
                contact_ok, active = residual(uk, atr, t_next)
                rnorm = psi.norm()
            if psi_ref is None:
                psi_ref = rnorm
            if psi_ref == 0.0:
                break
            if rnorm <= newton_tol * psi_ref and contact_ok:
                break
            if k == newton_maxit - 1:
                raise NewtonDivergenceError(
                    f"Newton did not converge in {newton_maxit} iterations at t={t_next:.6g} "
                    f"(residual {rnorm / psi_ref:.3e} relative)", rnorm)
            # effective operator K_T + b1 M (+ K_c on the active set of this
            # residual, dynamics.py:235-241)
            if active and cfg.assembled:
                raise NotImplementedError("implicit contact with the assembled (SGS / Schur) solver; "
                                          "use precond=\"diagonal\", condense=False")
            if active:
                lib.sdme_pcg_contact(pb._ctx, 1)
            try:
                _, st = solver.solve(uk, 1.0, nm.b1, psi, du)
            finally:
                if active:
                    lib.sdme_pcg_contact(pb._ctx, 0)
            traj.stats.add(step, k, "newmark", st)
            if contact is None:
                pending = True
            else:
                uk.assign(1.0, uk, 1.0, du)
            n_newton += 1
        if pending:  # Newton stopped by the iteration cap right after a solve
            uk.assign(1.0, uk, 1.0, du)
        traj.newton_iters.append(n_newton)
        # a_next = b1(uk-u) - b2 v - b3 a ; v += dt((1-g) a + g a_next) ; u = uk
        tmp.assign(1.0, uk, -1.0, u)
        atr.assign(nm.b1, tmp, -nm.b2, v, -nm.b3, a)
        v.assign(1.0, v, dt * (1.0 - gamma), a, dt * gamma, atr)
        a.copy_from(atr)
        u.copy_from(uk)
        t = t_next
        if contact is not None:
            contact.accept_step_(u, fcv)
        if track_energy:
            energy_row(t)
        if snapshot_stride and (step + 1) % snapshot_stride == 0:
            traj.times.append(t)
            traj.snapshots.append(u.free())
    traj.state = TimeState(t, u.free(), v.free(), a.free())
    return traj


def lumped_mass(problem: GpuFemProblem) -> tuple[DeviceVector, DeviceVector]:
    """(m_L, 1/m_L): row sums of the consistent mass over free columns,
    ``mass().sum(axis=1)``, computed as M 1 on the device."""
    ones = DeviceVector(problem).fill(1.0)
    ml = problem.mass_(ones, DeviceVector(problem))
    inv = DeviceVector(problem)
    native.check(problem._ctx, native.lib().sdme_vec_reciprocal(problem._ctx, inv.vid, ml.vid),
                 "lumped mass")
    return ml, inv


def estimate_lambda_max(problem: GpuFemProblem, inv_ml: DeviceVector, contact=None,
                        iters: int = 400, seed: int = 0, rtol: float = 1e-12) -> float:
    """lambda_max(M_L^-1 K_0) at u = 0 by Lanczos on the symmetric form
    S = M_L^-1/2 K_0 M_L^-1/2 (same spectrum), every operator application on
    the device (it sets the explicit time step 2/sqrt(lambda_max)
    of BASELINE config 4, the reference's ``cfl_dt`` role, dynamics.py:81-101).

    The largest Ritz value of the Lanczos tridiagonal converges from below,
    monotonically and much faster than power iteration; iteration stops once
    it changes by less than ``rtol`` (relative) over 10 steps, or after
    ``iters`` steps.  With ``contact`` the penalty stiffness enters as its
    diagonal upper bound eps * sum_q warea N_f^2 on the contact plane.
    """
    from scipy.linalg import eigvalsh_tridiagonal

    pb = problem
    wl = np.sqrt(np.maximum(inv_ml.lattice(), 0.0))
    w = DeviceVector(pb).set_lattice(wl)
    del wl
    rng = np.random.default_rng(seed)
    q = DeviceVector(pb).set_free(rng.standard_normal(pb.n_free))
    q.assign(1.0 / q.norm(), q)
    q_prev = DeviceVector(pb).fill(0.0)
    t1, t2 = DeviceVector(pb), DeviceVector(pb)
    u0 = DeviceVector(pb).fill(0.0)
    alphas, betas = [], []
    beta = 0.0
    lam, history = 0.0, []
    for j in range(max(2, iters)):
        _mul(pb, t1, w, q)
        pb.apply_(u0, t1, t2, 1.0, 0.0)
        _mul(pb, t1, w, t2)                      # t1 = S q
        alpha = t1.dot(q)
        t1.assign(1.0, t1, -alpha, q, -beta, q_prev)
        alphas.append(alpha)
        beta = t1.norm()
        if j >= 1:
            lam = float(eigvalsh_tridiagonal(np.array(alphas), np.array(betas), select="i",
                                             select_range=(j, j))[0])
            history.append(lam)
            if len(history) > 10 and abs(history[-1] - history[-11]) <= rtol * abs(history[-1]):
                break
        if beta <= 1e-300:
            lam = float(eigvalsh_tridiagonal(np.array(alphas), np.array(betas), select="i",
                                             select_range=(j, j))[0]) if j else alpha
            break
        betas.append(beta)
        q_prev.copy_from(q)
        q.assign(1.0 / beta, t1)
    if contact is not None:
        lam += contact.stiffness_bound() * max(inv_ml.lattice().max(), 0.0)
    return float(lam)


def _mul(pb, out, a, b):
    from . import native

    native.check(pb._ctx, native.lib().sdme_vec_mul(pb._ctx, out.vid, a.vid, b.vid), "vec_mul")
    return out


def explicit_run(problem: GpuFemProblem, external_load, dt: float, n_steps: int, u0=None, v0=None,
                 cfg: SolverConfig | None = None, snapshot_stride: int = 0, contact=None,
                 record_every: int = 0, mass: str = "consistent") -> Trajectory:
    """Central difference on the GPU.

    ``mass="consistent"`` (default, as the reference): the
    reference's own scheme (``dynamics.py:130-170``) -- each step solves
    (M/dt^2) w = psi with matrix-free Jacobi-PCG (``cfg``, full system) and
    records SolveStats.  ``mass="lumped"`` (BASELINE config 4):
    row-sum lumped mass with optional penalty contact, no linear solve.
    ``external_load`` may be None (no load), a :class:`ScaledLoad`, or any
    callable of t returning a free vector.  Startup a0 = M^-1 psi0,
    u_-1 = u0 - dt v0 + dt^2/2 a0 (``dynamics.py:152-155``).
    """
    if mass == "consistent":
        if contact is not None:
            raise NotImplementedError("contact with the consistent-mass explicit scheme; "
                                      "pass mass=\"lumped\" (SURVEY D6)")
        return _explicit_consistent(problem, external_load, dt, n_steps, u0, v0, cfg, snapshot_stride)
    if mass != "lumped":
        raise ValueError(f"unknown mass treatment {mass!r}")
    pb = problem
    u = _dev(pb, u0)
    v = _dev(pb, v0)
    traj = Trajectory()
    _, inv_ml = lumped_mass(pb)
    load = _Load(pb, external_load) if external_load is not None else None
    fint = DeviceVector(pb)
    fc = DeviceVector(pb) if contact is not None else None
    u_prev = DeviceVector(pb)
    a0 = DeviceVector(pb)
    # psi0 = P(0) - f_int(u0) + f_c(u0)
    pb.fint_(u, fint)
    terms = [-1.0, fint]
    if load is not None:
        terms += [1.0, load.at(0.0)]
    if contact is not None:
        contact.forces_(u, fc)
        terms += [1.0, fc]
    psi = DeviceVector(pb).assign(*terms)
    _mul(pb, a0, inv_ml, psi)
    u_prev.assign(1.0, u, -dt, v, 0.5 * dt * dt, a0)
    del psi
    t = 0.0
    from . import native

    lib = native.lib()

    def one_step(step, t):
        lid = -1
        if load is not None:
            lid = load.at(t).vid
        fid = -1
        if contact is not None:
            contact.forces_(u, fc, record=(record_every and step % record_every == 0))
            fid = fc.vid
        native.check(pb._ctx, lib.sdme_explicit_step(pb._ctx, u.vid, u_prev.vid, v.vid, lid, 1.0, fid,
                                                     inv_ml.vid, dt, fint.vid), "explicit_step")

    # Steps run in chunks on the device (sdme_explicit_steps: no host round trip
    # per step) between the steps that need the host (contact records,
    # snapshots); a general load callable runs step by step.  An inversion in a
    # chunk is replayed step by step from the chunk's start, so the error names
    # the first inverted step's element as the reference does.
    chunked = load is None or load.scaled
    saved = [DeviceVector(pb) for _ in range(3)] if chunked else None
    step = 0
    while step < n_steps:
        if not chunked:
            one_step(step, t)
            step += 1
            t += dt
        else:
            # the first step of a chunk goes through forces_ (records, contact parameters)
            one_step(step, t)
            step += 1
            t += dt
            end = n_steps
            if record_every:
                end = min(end, (step + record_every - 1) // record_every * record_every)
            if snapshot_stride:
                end = min(end, (step + snapshot_stride - 1) // snapshot_stride * snapshot_stride)
            if snapshot_stride and step % snapshot_stride == 0:
                traj.times.append(t)
                traj.snapshots.append(u.free())
            n = end - step
            if n > 0:
                for dst, src in zip(saved, (u, u_prev, v)):
                    dst.copy_from(src)
                scales = np.array([float(external_load.scale(t + k * dt)) if load is not None else 0.0
                                   for k in range(n)])
                rc = lib.sdme_explicit_steps(pb._ctx, n, u.vid, u_prev.vid, v.vid,
                                             load.base.vid if load is not None else -1, native.dptr(scales),
                                             fc.vid if contact is not None else -1, inv_ml.vid, dt, fint.vid)
                if rc == native.INVERSION:
                    for dst, src in zip((u, u_prev, v), saved):
                        dst.copy_from(src)
                    for k in range(n):  # raises at the first inverted step
                        one_step(step + k, t + k * dt)
                native.check(pb._ctx, rc, "explicit_steps")
                if contact is not None:
                    contact._serial += n
                step += n
                t += n * dt
                if snapshot_stride and step % snapshot_stride == 0:
                    traj.times.append(t)
                    traj.snapshots.append(u.free())
            continue
        if snapshot_stride and step % snapshot_stride == 0:
            traj.times.append(t)
            traj.snapshots.append(u.free())
    traj.state = TimeState(t, u.free(), v.free(), a0.free(), u_prev.free())
    if contact is not None:
        traj.contact_history = list(contact.history)
    return traj


def _explicit_consistent(pb: GpuFemProblem, external_load, dt, n_steps, u0, v0, cfg, snapshot_stride):
    """``explicit_run`` of the reference with a full (uncondensed) Jacobi-PCG
    mass solve per step (``dynamics.py:147-170``)."""
    cfg = SolverConfig.coerce(cfg) or SolverConfig()  # the reference's default: SGS + Schur
    cfg.validate()
    u = _dev(pb, u0)
    v = _dev(pb, v0)
    traj = Trajectory()
    load = _Load(pb, external_load) if external_load is not None else None
    fint, psi, a, w, un, up = (DeviceVector(pb) for _ in range(6))

    def residual(t):
        pb.fint_(u, fint)
        if load is not None:
            psi.assign(1.0, load.at(t), -1.0, fint)
        else:
            psi.assign(-1.0, fint)
        return psi

    solver = DriverSolver(pb, cfg)
    _, st = solver.solve(None, 0.0, 1.0, residual(0.0), a, slot="mass")
    traj.stats.add(-1, 0, "explicit-init", st)
    up.assign(1.0, u, -dt, v, 0.5 * dt * dt, a)
    t = 0.0
    inv_dt2 = 1.0 / dt ** 2
    for step in range(n_steps):
        _, st = solver.solve(None, 0.0, inv_dt2, residual(t), w, slot="mhat")
        traj.stats.add(step, 0, "explicit", st)
        un.assign(2.0, u, -1.0, up, 1.0, w)        # (2u - u_prev) + w
        v.assign(1.0, un, -1.0, up)                # (u_next - u_prev) ...
        v.assign(1.0 / (2.0 * dt), v)              # ... / (2 dt)
        up.copy_from(u)
        u.copy_from(un)
        t += dt
        if snapshot_stride and (step + 1) % snapshot_stride == 0:
            traj.times.append(t)
            traj.snapshots.append(u.free())
    traj.state = TimeState(t, u.free(), v.free(), a.free(), up.free())
    return traj
