"""``FemProblem`` on a general hexahedral mesh on the GPU.

:class:`GpuMeshProblem` is the general-mesh counterpart of
:class:`~paper_2104_13466_b200.problem.GpuFemProblem`: the same operator,
vector and solver entry points (``internal_force``, ``apply_tangent``,
``tangent_diagonal``, ``mass_apply``, ``pcg_gpu``, ``newmark_run`` ...), on any
conforming hexahedral mesh with trilinear geometry and oriented modes.  The
host builds the reference numbering and the device tables
(:mod:`paper_2104_13466_b200.mesh`); the device gathers element boxes through
the index table, runs the collocated element kernels with per-point J^-1 and
w det J, and assembles in the reference's element order (``element_gen.cuh``).
Vectors are plain free-DOF arrays in the reference order.  Requires the
reference default rule m = P + 1; contact and strain energy stay on the
box-mesh path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import native
from .basis import Basis1D, Rule, gauss_rule
from .mesh import (HexMesh, FACE_TABLE, MeshError, build_mesh_dofmap, element_tables, kernel_tables, _jacobians,
                   locality_order)
from .problem import GpuFemProblem, NeoHookean

__all__ = ["GpuMeshProblem"]


class GpuMeshProblem(GpuFemProblem):
    """General hexahedral mesh + basis + material bound to one GPU context.

    ``dirichlet``: (boundary tag, components) pairs, as ``build_dofmap``
    (``meshdof.py:404-409``)."""

    def __init__(self, mesh: HexMesh, basis: Basis1D, mat: NeoHookean, rule: Rule | None = None, dirichlet=None,
                 tables=None, locality: bool = True):
        self.mesh = mesh
        self.basis = basis
        self.mat = mat
        self.P = basis.P
        self.rule = rule if rule is not None else gauss_rule(basis.P + 1)
        self.m = self.rule.n
        if self.m != self.P + 1:
            raise ValueError(f"general meshes use the reference default rule m = P + 1 (got m = {self.m})")
        self.dirichlet = [(t, tuple(c)) for t, c in (dirichlet or [])]
        self.B, self.D, self.w = basis.tables(self.rule) if tables is None else (
            np.asarray(t, dtype=np.float64) for t in tables)
        self.dofmap = build_mesh_dofmap(mesh, basis, self.dirichlet)
        self.n_free = self.dofmap.n_free
        self.perm = None
        self.n_lattice = self.n_free
        geom = element_tables(mesh, self.rule)
        dof, ptr, slot = kernel_tables(self.dofmap)
        order = rows = None
        if locality:
            # element boxes along a Morton curve, assembly rows in box order
            # (placement only: per-DOF sums keep the reference element order)
            n_box = 3 * (self.P + 1) ** 3
            order, rows, ptr, slot = locality_order(mesh, self.dofmap, ptr, slot, n_box)
            dof, geom = dof[order], geom[order]
        d = native.MeshDesc()
        d.P, d.m, d.n_elems = self.P, self.m, mesh.n_elems
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (self.B, self.D, self.w)]
        d.B, d.D, d.w = (native.dptr(a) for a in self._keep)
        d.mu, d.lambda_lame, d.rho0 = mat.mu, mat.lambda_lame, mat.rho0
        d.n_free = self.n_free
        tabs = [np.ascontiguousarray(dof, dtype=np.int32), np.ascontiguousarray(ptr, dtype=np.int64),
                np.ascontiguousarray(slot, dtype=np.int32), np.ascontiguousarray(geom, dtype=np.float64)]
        if order is not None:
            tabs += [np.ascontiguousarray(order, dtype=np.int32), np.ascontiguousarray(rows, dtype=np.int32)]
            d.elem_id = tabs[4].ctypes.data_as(C.POINTER(C.c_int32))
            d.asm_rows = tabs[5].ctypes.data_as(C.POINTER(C.c_int32))
        d.dof = tabs[0].ctypes.data_as(C.POINTER(C.c_int32))
        d.asm_ptr = tabs[1].ctypes.data_as(C.POINTER(C.c_int64))
        d.asm_slot = tabs[2].ctypes.data_as(C.POINTER(C.c_int32))
        d.geom = native.dptr(tabs[3])
        ctx = C.c_void_p()
        rc = native.lib().sdme_create_mesh(C.byref(d), C.byref(ctx))
        if rc != native.OK:
            raise ValueError(f"sdme_create_mesh failed with status {rc} (P={self.P}, m={self.m}; P in 2..8)")
        self._ctx = ctx
        self._tmp = {}

    # lattice helpers of the box path do not apply
    def to_free(self, lattice):
        raise NotImplementedError("general meshes have no lattice; vectors are free-DOF arrays")

    to_lattice = to_free
    traction_lattice = to_free

    def traction_vector(self, tag: str, tvec, rule: Rule | None = None) -> np.ndarray:
        """Constant-traction load on a boundary tag: ``build_face_tables`` +
        ``surface_traction`` + ``traction_vector`` (femcore.py:215-253, 256-259,
        391-397) with t(x) = tvec; face rule = the problem rule by default."""
        if tag not in self.mesh.boundary_sides:
            raise KeyError(f"unknown boundary tag {tag!r}")
        rule = rule or self.rule
        x1, w1 = rule.points, rule.weights
        n = self.P + 1
        tvec = np.asarray(tvec, dtype=float)
        out = np.zeros(self.n_free)
        dm = self.dofmap
        for e, lf in self.mesh.boundary_sides[tag]:
            axis, side, d1, d2, _ = FACE_TABLE[lf]
            A, Bq = np.meshgrid(x1, x1, indexing="ij")
            xi = np.zeros((A.size, 3))
            xi[:, axis] = 1.0 if side else -1.0
            xi[:, d1], xi[:, d2] = A.reshape(-1), Bq.reshape(-1)
            w2 = np.outer(w1, w1).reshape(-1)
            sub = HexMesh(self.mesh.coords, self.mesh.elems[e:e + 1])
            jac, _ = _jacobians(sub, xi)
            area = np.linalg.norm(np.cross(jac[0, :, :, d1], jac[0, :, :, d2]), axis=1)
            v, _ = self.basis.eval(xi.reshape(-1))
            v = np.asarray(v).reshape(n, -1, 3)  # (function, point, axis)
            vals = np.ones((len(w2), n, n, n))  # [q][p][q'][r] reference tensor order
            vals *= v[:, :, 0].T[:, :, None, None]
            vals *= v[:, :, 1].T[:, None, :, None]
            vals *= v[:, :, 2].T[:, None, None, :]
            r = np.einsum("q,qf,c->fc", w2 * area, vals.reshape(len(w2), -1), tvec)
            dofs = dm.free_map[dm.gdof[e][:, None] * 3 + np.arange(3)[None, :]]
            sg = dm.gsign[e][:, None] * np.ones((1, 3))
            mask = dofs >= 0
            np.add.at(out, dofs[mask], (r * sg)[mask])
        return out

    def constant_field(self, value) -> np.ndarray:
        """Free coefficients of a constant displacement: vertex coefficients
        value, edge / face / interior coefficients of the 1D constant vector
        (exact in every basis, SURVEY §8a notes)."""
        from .basis import constant_coeffs
        c1 = constant_coeffs(self.basis)
        n = self.P + 1
        t = np.array([c1[i] for i in range(n)])
        coef = np.einsum("p,q,r->pqr", t, t, t).reshape(-1)  # reference local order
        dm = self.dofmap
        out = np.zeros(self.n_free)
        for c in range(3):
            f = dm.free_map[dm.gdof * 3 + c]
            vals = value[c] * coef[None, :] * dm.gsign
            mask = f >= 0
            out[f[mask]] = vals[mask]
        return out
