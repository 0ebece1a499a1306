"""GpuFemProblem: the drop-in for ``sdmefem.femcore.FemProblem`` on the hot path.

Mirrors the problem-level entry points of ``femcore.py:273-431`` that sit on
the Newmark/Newton/PCG path -- ``internal_force`` (:346), the tangent action
that replaces ``tangent_matrices`` + ``a @ p`` (:351, solver.py:149), the
Jacobi diagonal that replaces ``a.diagonal()`` (solver.py:106), the mass
action ``mass() @ a`` (:367, dynamics.py:198) and ``traction_vector`` (:391) --
for axis-aligned ``gen_box_mesh`` meshes.  All compute runs in
``libsdme.so`` (CUDA, sm_100a); host vectors cross the boundary in the
reference's free-DOF order, device-resident :class:`DeviceVector` handles
are available for inner loops.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import native
from .basis import Basis1D, Rule, constant_coeffs, gauss_rule
from .lattice import (FACE_TAGS, BoxMesh, constrained_lattice, dirichlet_face_masks,
                      reference_free_index)

__all__ = ["NeoHookean", "GpuFemProblem", "DeviceVector"]


@dataclass(frozen=True)
class NeoHookean:
    """Lame parameters (Pa) and reference density (``material.py:32-62``)."""

    mu: float
    lambda_lame: float
    rho0: float = 1.0

    def __post_init__(self):
        if self.mu <= 0.0:
            raise ValueError(f"shear modulus must be positive, got {self.mu}")
        if self.rho0 <= 0.0:
            raise ValueError(f"reference density must be positive, got {self.rho0}")
        if self.lambda_lame + 2.0 * self.mu / 3.0 <= 0.0:
            raise ValueError("bulk modulus must be positive")

    @classmethod
    def from_engineering(cls, E: float, nu: float, rho0: float = 1.0) -> "NeoHookean":
        if E <= 0.0:
            raise ValueError(f"Young's modulus must be positive, got {E}")
        if not -1.0 < nu < 0.5:
            raise ValueError(f"Poisson ratio must lie in (-1, 0.5), got {nu}")
        return cls(E / (2.0 * (1.0 + nu)), E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), rho0)


class DeviceVector:
    """A device-resident lattice vector (3 x Lz x Ly x Lx doubles) owned by a
    problem context.  Dirichlet points are held at zero."""

    __slots__ = ("problem", "vid", "__weakref__")

    def __init__(self, problem: "GpuFemProblem"):
        self.problem = problem
        vid = C.c_int(-1)
        native.check(problem._ctx, native.lib().sdme_vec_alloc(problem._ctx, C.byref(vid)), "vec_alloc")
        self.vid = vid.value

    def __del__(self):
        pb = getattr(self, "problem", None)
        if pb is not None and pb._ctx and self.vid >= 0:
            native.lib().sdme_vec_free(pb._ctx, self.vid)
            self.vid = -1

    # host transfers -----------------------------------------------------
    def set_free(self, values: np.ndarray) -> "DeviceVector":
        a = np.ascontiguousarray(values, dtype=np.float64)
        if a.shape != (self.problem.n_free,):
            raise ValueError(f"expected a free vector of length {self.problem.n_free}, got {a.shape}")
        native.check(self.problem._ctx, native.lib().sdme_vec_upload_free(self.problem._ctx, self.vid,
                                                                          native.dptr(a)), "upload")
        return self

    def free(self, out: np.ndarray | None = None) -> np.ndarray:
        """Download in the reference free-DOF order (into ``out`` if given,
        e.g. a page-locked buffer from :func:`native.pinned_empty`)."""
        if out is None:
            out = np.empty(self.problem.n_free)
        elif out.shape != (self.problem.n_free,) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("out must be a contiguous float64 free vector")
        native.check(self.problem._ctx, native.lib().sdme_vec_download_free(self.problem._ctx, self.vid,
                                                                            native.dptr(out)), "download")
        return out

    def set_lattice(self, values: np.ndarray) -> "DeviceVector":
        a = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        if a.size != self.problem.n_lattice:
            raise ValueError("lattice vector has the wrong size")
        a = a * self.problem.free_mask_flat  # Dirichlet points held at zero
        native.check(self.problem._ctx, native.lib().sdme_vec_upload(self.problem._ctx, self.vid,
                                                                     native.dptr(a)), "upload")
        return self

    def lattice(self) -> np.ndarray:
        out = np.empty(self.problem.n_lattice)
        native.check(self.problem._ctx, native.lib().sdme_vec_download(self.problem._ctx, self.vid,
                                                                       native.dptr(out)), "download")
        return out.reshape(self.problem.lattice_shape)

    # device ops ----------------------------------------------------------
    def fill(self, value: float) -> "DeviceVector":
        native.check(self.problem._ctx, native.lib().sdme_vec_fill(self.problem._ctx, self.vid, value), "fill")
        return self

    def copy_from(self, other: "DeviceVector") -> "DeviceVector":
        native.check(self.problem._ctx, native.lib().sdme_vec_copy(self.problem._ctx, self.vid, other.vid),
                     "copy")
        return self

    def assign(self, *terms) -> "DeviceVector":
        """self = sum c_i x_i for terms (c_0, x_0, c_1, x_1, ...)."""
        cs = np.array(terms[0::2], dtype=np.float64)
        ids = (C.c_int * len(cs))(*[t.vid for t in terms[1::2]])
        native.check(self.problem._ctx, native.lib().sdme_vec_lincomb(
            self.problem._ctx, self.vid, len(cs), native.dptr(cs), ids), "lincomb")
        return self

    def dot(self, other: "DeviceVector") -> float:
        out = C.c_double(0.0)
        native.check(self.problem._ctx, native.lib().sdme_vec_dot(self.problem._ctx, self.vid, other.vid,
                                                                  C.byref(out)), "dot")
        return out.value

    def norm(self) -> float:
        return float(np.sqrt(self.dot(self)))


class GpuFemProblem:
    """Box mesh + basis + material bound to one GPU context.

    ``rule`` defaults to P+1 Gauss-Legendre points per direction, as
    ``FemProblem`` does (``femcore.py:283-293``).  ``dirichlet`` is a sequence
    of (face tag, components) pairs (``build_dofmap``'s argument,
    ``meshdof.py:404-409``); every mode on a tagged face is constrained
    (``boundary_modes``, ``meshdof.py:475-503``).
    """

    def __init__(self, mesh: BoxMesh, basis: Basis1D, mat: NeoHookean, rule: Rule | None = None,
                 dirichlet=None, reference_order: bool = True, tables=None, perm=None, n_free=None):
        """``tables`` = (B, D, w) and ``perm`` / ``n_free`` (lattice -> free
        index) override the ones built here; :func:`interop.from_reference`
        passes the reference problem's own."""
        self.mesh = mesh
        self.basis = basis
        self.mat = mat
        self.P = basis.P
        self.rule = rule if rule is not None else gauss_rule(basis.P + 1)
        self.m = self.rule.n
        self.dirichlet = [(t, tuple(c)) for t, c in (dirichlet or [])]
        self.B, self.D, self.w = basis.tables(self.rule) if tables is None else (
            np.asarray(t, dtype=np.float64) for t in tables)
        lx, ly, lz = mesh.lattice_shape(self.P)
        self.lattice_shape = (3, lz, ly, lx)
        self.n_lattice = 3 * lx * ly * lz
        masks = dirichlet_face_masks(self.dirichlet)
        self.constrained = constrained_lattice(mesh, self.P, masks)
        self.free_mask_flat = (~self.constrained).reshape(-1).astype(np.float64)
        if perm is not None:
            perm = np.asarray(perm).reshape(-1)
            if perm.size != self.n_lattice or n_free is None:
                raise ValueError("perm must cover the lattice and come with n_free")
            if not np.array_equal(perm < 0, self.constrained.reshape(-1)):
                raise ValueError("perm's constrained entries differ from the Dirichlet faces")
            self.perm = perm.astype(np.int32)
            n_free = int(n_free)
        elif reference_order:
            perm, n_free = reference_free_index(mesh, self.P, self.dirichlet)
            self.perm = perm.reshape(-1).astype(np.int32)
        else:
            self.perm = None
            n_free = int((~self.constrained).sum())
        self.n_free = n_free
        d = native.Desc()
        d.P, d.m = self.P, self.m
        d.nx, d.ny, d.nz = mesh.divisions
        d.hx, d.hy, d.hz = mesh.h
        d.origin = (C.c_double * 3)(*mesh.origin)
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (self.B, self.D, self.w)]
        d.B, d.D, d.w = (native.dptr(a) for a in self._keep)
        d.mu, d.lambda_lame, d.rho0 = mat.mu, mat.lambda_lame, mat.rho0
        d.dirichlet_mask = (C.c_int * 3)(*[int(v) for v in masks])
        if self.perm is not None:
            d.perm = self.perm.ctypes.data_as(C.POINTER(C.c_int32))
        d.n_free = n_free
        ctx = C.c_void_p()
        rc = native.lib().sdme_create(C.byref(d), C.byref(ctx))
        if rc != native.OK:
            raise ValueError(f"sdme_create failed with status {rc} (P={self.P}, m={self.m}; "
                             "supported m in {P+1, P+2}, P <= 8)")
        self._ctx = ctx
        self._tmp = {}

    def close(self):
        if getattr(self, "_ctx", None):
            self._tmp.clear()
            native.lib().sdme_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        self.close()

    # ----------------------------------------------------------- vectors
    def vector(self, free: np.ndarray | None = None) -> DeviceVector:
        v = DeviceVector(self)
        if free is not None:
            v.set_free(free)
        return v

    def _scratch(self, name: str) -> DeviceVector:
        v = self._tmp.get(name)
        if v is None:
            v = self._tmp[name] = DeviceVector(self)
        return v

    def to_free(self, lattice: np.ndarray) -> np.ndarray:
        """Host-side lattice -> reference free order."""
        if self.perm is None:
            return lattice.reshape(-1)[self.free_mask_flat > 0].copy()
        out = np.zeros(self.n_free)
        sel = self.perm >= 0
        out[self.perm[sel]] = lattice.reshape(-1)[sel]
        return out

    def to_lattice(self, free: np.ndarray) -> np.ndarray:
        out = np.zeros(self.n_lattice)
        if self.perm is None:
            out[self.free_mask_flat > 0] = free
        else:
            sel = self.perm >= 0
            out[sel] = free[self.perm[sel]]
        return out.reshape(self.lattice_shape)

    # ------------------------------------------------- device operators
    def fint_(self, u: DeviceVector, out: DeviceVector) -> DeviceVector:
        native.check(self._ctx, native.lib().sdme_fint(self._ctx, u.vid, out.vid), "fint")
        return out

    def apply_(self, u: DeviceVector | None, p: DeviceVector, out: DeviceVector, c_k: float = 1.0,
               c_m: float = 0.0) -> DeviceVector:
        uid = u.vid if u is not None else -1
        native.check(self._ctx, native.lib().sdme_apply(self._ctx, uid, p.vid, out.vid, c_k, c_m), "apply")
        return out

    def mass_(self, a: DeviceVector, out: DeviceVector) -> DeviceVector:
        native.check(self._ctx, native.lib().sdme_mass(self._ctx, a.vid, out.vid), "mass")
        return out

    def diag_(self, u: DeviceVector | None, out: DeviceVector, c_k: float = 1.0,
              c_m: float = 0.0) -> DeviceVector:
        uid = u.vid if u is not None else -1
        native.check(self._ctx, native.lib().sdme_diag(self._ctx, uid, c_k, c_m, out.vid), "diag")
        return out

    # ------------------------------------- reference-order host entry points
    def internal_force(self, u_free: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """``FemProblem.internal_force`` (femcore.py:346-349)."""
        u = self._scratch("u").set_free(u_free)
        return self.fint_(u, self._scratch("y")).free(out)

    def apply_tangent(self, u_free: np.ndarray, p_free: np.ndarray, c_m: float = 0.0,
                      out: np.ndarray | None = None) -> np.ndarray:
        """(K_T(u) + c_m M) p: ``element_tangent(...)@p_e`` summed (femcore.py:130-146)."""
        u = self._scratch("u").set_free(u_free)
        p = self._scratch("p").set_free(p_free)
        return self.apply_(u, p, self._scratch("y"), 1.0, c_m).free(out)

    def apply_tangent_batch(self, us, ps, c_m: float = 0.0, outs=None) -> list:
        """[(K_T(u_k) + c_m M) p_k for k]: ``apply_tangent`` over a batch of host
        pairs, pipelined over PCIe (the H2D copies of pair k+1 and the D2H copy of
        result k-1 overlap pair k's operator; ``sdme_apply_batch``).  Inputs and
        ``outs`` should be page-locked (:func:`native.pinned_empty`) for full overlap."""
        n = len(ps)
        if len(us) != n:
            raise ValueError("us and ps must have the same length")
        if outs is None:
            outs = [np.empty(self.n_free) for _ in range(n)]
        arrs = []
        for a in list(us) + list(ps) + list(outs):
            if a.shape != (self.n_free,) or a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ValueError(f"batch vectors must be contiguous float64 free vectors of length {self.n_free}")
            arrs.append(a)
        U = (native._dp * n)(*[native.dptr(a) for a in us])
        Pp = (native._dp * n)(*[native.dptr(a) for a in ps])
        Y = (native._dp * n)(*[native.dptr(a) for a in outs])
        native.check(self._ctx, native.lib().sdme_apply_batch(self._ctx, n, U, Pp, Y, 1.0, c_m), "apply_batch")
        return list(outs)

    def tangent_diagonal(self, u_free: np.ndarray, c_m: float = 0.0) -> np.ndarray:
        """diag(K_T(u) + c_m M) over free dofs (solver.py:106 on the assembled operator)."""
        u = self._scratch("u").set_free(u_free)
        return self.diag_(u, self._scratch("y"), 1.0, c_m).free()

    def strain_energy_(self, u: DeviceVector) -> float:
        """Total strain energy at a device vector (femcore.py:374-378)."""
        out = C.c_double(0.0)
        native.check(self._ctx, native.lib().sdme_strain_energy(self._ctx, u.vid, C.byref(out)), "strain energy")
        return out.value

    def total_strain_energy(self, u_free: np.ndarray) -> float:
        """``FemProblem.total_strain_energy`` (femcore.py:374-378)."""
        return self.strain_energy_(self._scratch("u").set_free(u_free))

    def mass_apply(self, a_free: np.ndarray) -> np.ndarray:
        """``mass() @ a`` (femcore.py:367-372, dynamics.py:198)."""
        a = self._scratch("p").set_free(a_free)
        return self.mass_(a, self._scratch("y")).free()

    # ------------------------------------------------------------ loads
    def traction_lattice(self, tag: str, tvec) -> np.ndarray:
        """Constant-traction load (``traction_vector``, femcore.py:391-397) in
        lattice layout: t_c (h1/2)(h2/2) G1 (x) G2 on the face plane, with
        G[l] = sum_a w_a phi_l(xi_a) assembled along each in-plane line."""
        if tag not in FACE_TAGS:
            raise KeyError(f"unknown boundary tag {tag!r}")
        f = FACE_TAGS.index(tag)
        axis, side = divmod(f, 2)
        d1, d2 = [d for d in range(3) if d != axis]
        P = self.P
        g1d = self.w @ self.B  # (n,), reference function order
        gl = np.empty(P + 1)
        gl[0], gl[P] = g1d[0], g1d[1]
        gl[1:P] = g1d[2:]
        lines = []
        for d in (d1, d2):
            ne = self.mesh.divisions[d]
            line = np.zeros(P * ne + 1)
            for e in range(ne):
                line[P * e:P * e + P + 1] += gl
            lines.append(line * 0.5 * self.mesh.h[d])
        plane = np.outer(lines[0], lines[1])  # [d1, d2]
        out = np.zeros(self.lattice_shape)
        tvec = np.asarray(tvec, dtype=float)
        idx = [slice(None)] * 3
        idx[2 - axis] = -1 if side else 0  # lattice array is [z, y, x]
        for c in range(3):
            if tvec[c] == 0.0:
                continue
            # plane is [d1][d2] with d1 < d2; the lattice face view is [d2][d1]
            out[c][tuple(idx)] = tvec[c] * plane.T
        out[self.constrained] = 0.0
        return out

    def traction_vector(self, tag: str, tvec) -> np.ndarray:
        return self.to_free(self.traction_lattice(tag, tvec))

    def constant_field(self, value) -> np.ndarray:
        """Free coefficients of a constant displacement (exact in every basis:
        tensor product of the 1D constant coefficients, SURVEY §8a notes);
        equals ``l2_project`` of a constant to its 1e-14 tolerance."""
        c1 = constant_coeffs(self.basis)
        cl = np.empty(self.P + 1)
        cl[0], cl[self.P] = c1[0], c1[1]
        cl[1:self.P] = c1[2:]
        lines = []
        for d in range(3):
            ne = self.mesh.divisions[d]
            line = np.empty(self.P * ne + 1)
            for e in range(ne):
                line[self.P * e:self.P * e + self.P + 1] = cl
            lines.append(line)
        cube = np.einsum("z,y,x->zyx", lines[2], lines[1], lines[0])
        out = np.stack([value[c] * cube for c in range(3)])
        out[self.constrained] = 0.0
        return self.to_free(out)

    def launch_count(self) -> int:
        n = C.c_int64(0)
        native.lib().sdme_launch_count(self._ctx, C.byref(n))
        return n.value

    def time_op(self, op: str, u: DeviceVector, p: DeviceVector, y: DeviceVector, c_m: float = 0.0,
                reps: int = 10) -> float:
        """Mean ms per call of one operator, CUDA events on the context stream."""
        code = {"apply": 0, "fint": 1, "mass": 2, "diag": 3, "setup": 4, "apply_pa": 5}[op]
        ms = C.c_double(0.0)
        native.check(self._ctx, native.lib().sdme_time_op(self._ctx, code, u.vid, p.vid, y.vid, c_m, reps,
                                                          C.byref(ms)), "time_op")
        return ms.value

    def sync(self):
        native.check(self._ctx, native.lib().sdme_sync(self._ctx), "sync")
