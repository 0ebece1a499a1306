"""Penalty contact against a rigid plane, GPU force evaluation.

Mirrors ``sdmefem.contact`` (``contact.py:25-204``): :class:`RigidObstacle`,
:class:`ContactParams`, and :class:`GpuPenaltyContact` with
``evaluate_forces`` (force, pressures, gaps, active set, settled flag),
``accept_step`` (penalty stepping + history) and ``penalty_energy``.  The
contact stiffness (implicit contact, ``contact.py:120-140``) is a matrix-free
operator on the device: ``ContactForces.stiffness`` is a :class:`ContactStiffness`
(``@`` and ``diagonal()``) over the active set of that evaluation, and
``newmark_run(..., contact=...)`` adds it to the PCG operator.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import native
from .basis import gauss_rule
from .lattice import FACE_TAGS
from .problem import DeviceVector, GpuFemProblem

__all__ = ["RigidObstacle", "ContactParams", "ContactForces", "ContactStiffness", "GpuPenaltyContact", "gap"]


@dataclass(frozen=True)
class RigidObstacle:
    """Plane through ``point`` with unit ``outward_normal`` (``contact.py:25-39``)."""

    point: np.ndarray
    outward_normal: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "point", np.asarray(self.point, dtype=float))
        n = np.asarray(self.outward_normal, dtype=float)
        nrm = np.linalg.norm(n)
        if abs(nrm - 1.0) > 1e-12:
            n = n / nrm
        object.__setattr__(self, "outward_normal", n)


def gap(obstacle: RigidObstacle, x: np.ndarray) -> np.ndarray:
    """``contact.py:42-45``."""
    return (np.asarray(x, dtype=float) - obstacle.point) @ obstacle.outward_normal


@dataclass
class ContactParams:
    """``contact.py:48-59``."""

    eps_n: float
    deps_n: float = 0.0
    gap_tol: float = 1e-3
    stress_tol: float = 1e-2

    def __post_init__(self):
        if self.eps_n <= 0.0:
            raise ValueError("penalty stiffness must be positive")
        if self.gap_tol <= 0.0 or self.stress_tol <= 0.0:
            raise ValueError("tolerances must be positive")


@dataclass
class ContactForces:
    force: np.ndarray
    stiffness: object
    pressures: np.ndarray
    gaps: np.ndarray
    active: np.ndarray
    settled: bool


class ContactStiffness:
    """K_c = eps sum_{q active} warea N_f N_g (n n^T) of one force evaluation
    (``contact.py:129-140``), applied matrix-free on the device.  Valid until
    the next evaluation of the same contact (the active set lives on the device)."""

    def __init__(self, contact: "GpuPenaltyContact", serial: int):
        self.contact = contact
        self.serial = serial
        self.shape = (contact.problem.n_free, contact.problem.n_free)

    def _check(self):
        if self.serial != self.contact._serial:
            raise RuntimeError("contact stiffness of an older evaluation (the active set has changed)")

    def __matmul__(self, p: np.ndarray) -> np.ndarray:
        self._check()
        pb = self.contact.problem
        pv = pb._scratch("kc_p").set_free(np.asarray(p, dtype=float))
        y = pb._scratch("kc_y").fill(0.0)
        native.check(pb._ctx, native.lib().sdme_contact_apply(pb._ctx, pv.vid, y.vid), "contact_apply")
        return y.free()

    def diagonal(self) -> np.ndarray:
        self._check()
        pb = self.contact.problem
        d = pb._scratch("kc_y").fill(0.0)
        native.check(pb._ctx, native.lib().sdme_contact_diag(pb._ctx, d.vid), "contact_diag")
        return d.free()


class GpuPenaltyContact:
    """Penalty contact of one box side against a rigid plane (``contact.py:72-204``)."""

    def __init__(self, problem: GpuFemProblem, obstacle: RigidObstacle, params: ContactParams,
                 surface_tag: str, quad_order: int | None = None):
        if surface_tag not in FACE_TAGS:
            raise KeyError(f"unknown boundary tag {surface_tag!r}")
        self.problem = problem
        self.obstacle = obstacle
        self.params = params
        self.surface_tag = surface_tag
        self.side = FACE_TAGS.index(surface_tag)
        self.qf = quad_order if quad_order is not None else problem.P + 1  # contact.py:81-83
        rule = gauss_rule(self.qf)
        v, _ = problem.basis.eval(rule.points)
        self.Bf = np.ascontiguousarray(v.T)
        self.xf = np.ascontiguousarray(rule.points)
        self.wf = np.ascontiguousarray(rule.weights)
        n = C.c_int64(0)
        native.lib().sdme_contact_points(problem._ctx, self.side, self.qf, C.byref(n))
        self.n_points = n.value
        self._last_pressures = None
        self.history = []
        self._fc = None
        self._u = None
        self._serial = 0  # bumped by every device evaluation (active set)

    def forces_(self, u: DeviceVector, fc: DeviceVector, record: bool = False):
        """Device path: fc = contact nodal force at u (no host traffic unless
        ``record`` asks for the gap statistics)."""
        pb = self.problem
        self._serial += 1
        gaps = np.empty(self.n_points) if record else None
        stats = np.zeros(3) if record else None
        rc = native.lib().sdme_contact(
            pb._ctx, u.vid, self.side, self.qf, native.dptr(self.Bf), native.dptr(self.xf),
            native.dptr(self.wf), native.dptr(self.obstacle.point), native.dptr(self.obstacle.outward_normal),
            float(self.params.eps_n), fc.vid,
            native.dptr(gaps) if record else None, native.dptr(stats) if record else None)
        native.check(pb._ctx, rc, "contact")
        if record:
            self.history.append((self.params.eps_n, float(stats[0]), float(stats[1]), int(stats[2])))
        return gaps

    def _gaps(self, u: DeviceVector, fc: DeviceVector):
        self._serial += 1
        gaps = np.empty(self.n_points)
        rc = native.lib().sdme_contact(
            self.problem._ctx, u.vid, self.side, self.qf, native.dptr(self.Bf), native.dptr(self.xf),
            native.dptr(self.wf), native.dptr(self.obstacle.point), native.dptr(self.obstacle.outward_normal),
            float(self.params.eps_n), fc.vid, native.dptr(gaps), None)
        native.check(self.problem._ctx, rc, "contact")
        return gaps

    def _scratch(self):
        if self._fc is None:
            self._fc = DeviceVector(self.problem)
            self._u = DeviceVector(self.problem)
        return self._u, self._fc

    def face_points(self) -> np.ndarray:
        """Reference positions of the face quadrature points, (n_points, 3), in
        the order of the gaps: faces of the side with the first in-plane axis
        d1 fastest, points (a along d1, b along d2) with b fastest
        (``build_face_tables``, femcore.py:215-253)."""
        mesh = self.problem.mesh
        ax, side = divmod(self.side, 2)
        d1, d2 = [d for d in range(3) if d != ax]
        n1, n2 = mesh.divisions[d1], mesh.divisions[d2]
        t = 0.5 * (1.0 + self.xf)
        c1 = mesh.origin[d1] + mesh.h[d1] * (np.arange(n1)[:, None] + t[None, :])  # (face i1, a)
        c2 = mesh.origin[d2] + mesh.h[d2] * (np.arange(n2)[:, None] + t[None, :])  # (face i2, b)
        qf = self.qf
        pts = np.empty((n2, n1, qf, qf, 3))
        pts[..., ax] = mesh.origin[ax] + (mesh.lengths[ax] if side else 0.0)
        pts[..., d1] = c1[None, :, :, None]
        pts[..., d2] = c2[:, None, None, :]
        return pts.reshape(-1, 3)

    def update_active_set(self, u_free: np.ndarray):
        """``contact.py:98-101``: (active flags, gaps), one array per face."""
        u, fc = self._scratch()
        u.set_free(u_free)
        g = self._gaps(u, fc).reshape(-1, self.qf * self.qf)
        gaps = [row.copy() for row in g]
        return [row < 0.0 for row in gaps], gaps

    def pressure_profile(self, u_free: np.ndarray) -> np.ndarray:
        """``contact.py:186-204``: (in-plane distance from the surface's
        minimum corner, pressure) rows sorted by the distance."""
        _, gaps = self.update_active_set(u_free)
        g = np.concatenate(gaps) if gaps else np.zeros(0)
        t_n = np.where(g < 0.0, -self.params.eps_n * g, 0.0)
        pts = self.face_points()
        nrm = np.asarray(self.obstacle.outward_normal, dtype=float)
        inplane = pts - np.outer(pts @ nrm, nrm)
        dist = np.linalg.norm(inplane - inplane.min(axis=0), axis=1)
        order = np.argsort(dist, kind="stable")
        return np.column_stack([dist[order], t_n[order]])

    def evaluate_forces(self, u_free: np.ndarray) -> ContactForces:
        """``contact.py:103-151`` (force, pressures per face point, gaps, active, settled)."""
        u, fc = self._scratch()
        u.set_free(u_free)
        g = self._gaps(u, fc)
        act = g < 0.0
        pressures = np.where(act, -self.params.eps_n * g, 0.0)
        settled = self._pressure_settled(pressures)
        self._last_pressures = pressures
        kc = ContactStiffness(self, self._serial) if act.any() else None
        return ContactForces(fc.free(), kc, pressures, g, act, settled)

    def evaluate_(self, u: DeviceVector, fc: DeviceVector):
        """Device form of :meth:`evaluate_forces` for the Newton loop: fc on
        the device, returns (settled, any_active); the gaps (one value per face
        point) are the only host traffic."""
        g = self._gaps(u, fc)
        act = g < 0.0
        pressures = np.where(act, -self.params.eps_n * g, 0.0)
        settled = self._pressure_settled(pressures)
        self._last_pressures = pressures
        return settled, bool(act.any())

    def _pressure_settled(self, pressures):
        """``contact.py:153-160``."""
        prev = self._last_pressures
        if prev is None or prev.shape != pressures.shape:
            return not pressures.any()
        scale = max(np.abs(pressures).max(), np.abs(prev).max())
        if scale == 0.0:
            return True
        return float(np.abs(pressures - prev).max()) / scale <= self.params.stress_tol

    def accept_step(self, u_free: np.ndarray):
        """``contact.py:162-176``: history row and penalty stepping."""
        u, fc = self._scratch()
        u.set_free(u_free)
        self.accept_step_(u, fc)

    def accept_step_(self, u: DeviceVector, fc: DeviceVector):
        """:meth:`accept_step` on a device vector (fc is scratch)."""
        g = self._gaps(u, fc)
        pen = max(float(-g.min()), 0.0) if g.size else 0.0
        act = g < 0.0
        tn = np.where(act, -self.params.eps_n * g, 0.0)
        t_min = float(tn[act].min()) if act.any() else 0.0
        self.history.append((self.params.eps_n, pen, t_min, int(act.sum())))
        if pen > self.params.gap_tol and self.params.deps_n > 0.0:
            self.params.eps_n += self.params.deps_n
        self._last_pressures = None

    def penalty_energy(self, u_free: np.ndarray) -> float:
        """``contact.py:178-184``: sum over points of eps/2 warea min(g,0)^2."""
        u, fc = self._scratch()
        u.set_free(u_free)
        return self.penalty_energy_(u, fc)

    def penalty_energy_(self, u: DeviceVector, fc: DeviceVector) -> float:
        """:meth:`penalty_energy` at a device vector (fc is scratch)."""
        g = self._gaps(u, fc).reshape(-1, self.qf, self.qf)
        ax = self.side // 2
        d1, d2 = [d for d in range(3) if d != ax]
        h = self.problem.mesh.h
        warea = np.outer(self.wf, self.wf) * 0.25 * h[d1] * h[d2]
        pen = np.minimum(g, 0.0)
        return float(0.5 * self.params.eps_n * (warea[None] * pen ** 2).sum())

    def stiffness_bound(self) -> float:
        """Gershgorin bound of the contact stiffness rows, all points active:
        eps * max_f sum_q warea |N_f| sum_g |N_g| (for the CFL estimate, D7)."""
        ax = self.side // 2
        d1, d2 = [d for d in range(3) if d != ax]
        h = self.problem.mesh.h
        a1 = np.abs(self.Bf)  # (qf, n)
        w = self.wf * 0.5
        # 1D factors: s[l] = sum_a w_a |phi_l(a)| sum_k |phi_k(a)|; neighbours double up
        s = (w[:, None] * a1 * a1.sum(axis=1)[:, None]).sum(axis=0)
        return float(self.params.eps_n * 4.0 * s.max() ** 2 * h[d1] * h[d2])
