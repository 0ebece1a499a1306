"""The reference's default linear solver on the GPU: Schur condensation + SGS.

``SolverConfig()`` of the reference is ``precond="sgs", condense=True``
(``dynamics.py:38-43``): ``make_solver`` condenses the element-interior modes
out of the dense element matrices (``condense_elements``,
``solver.py:258-293``) and ``LinearSolver.solve`` runs PCG with the symmetric
Gauss-Seidel preconditioner on the boundary Schur complement, then recovers
the interior (``solver.py:302-322``, ``CondensedSystem``, ``solver.py:179-203``).
:class:`SchurSolver` does all of it on the device (``csrc/schur.cu``): element
matrices of c_k K_T(u) + c_m M, batched per-element Cholesky and Schur
products, deterministic CSR assembly in element order (the reference's
summation order), level-scheduled SGS sweeps and the PCG loop with the
reference's order of checks.  ``condense=False`` assembles the full free-DOF
operator instead (``make_solver``'s CSR branch, ``dynamics.py:118-126``), so
``precond="sgs"`` works uncondensed too.

Box meshes only, and sized like the reference: the dense element matrices
take (3 (P+1)^3)^2 doubles per element (1.1 MB at P = 4).  The matrix-free
Jacobi-PCG path (``pcg_gpu``) is the one for large meshes.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import native
from .errors import PCGError
from .problem import DeviceVector, GpuFemProblem

__all__ = ["SchurSolver", "schur_tables"]

_PREC = {"none": 0, None: 0, "diagonal": 1, "sgs": 2, "gauss-seidel": 2}


def _device_memory():
    """(free, total) bytes of the current device (cudaMemGetInfo via the runtime)."""
    try:
        import ctypes.util

        rt = C.CDLL(ctypes.util.find_library("cudart") or "libcudart.so")
    except OSError:
        return float("inf"), float("inf")
    f, t = C.c_size_t(0), C.c_size_t(0)
    if rt.cudaMemGetInfo(C.byref(f), C.byref(t)) != 0:
        return float("inf"), float("inf")
    return float(f.value), float(t.value)


def schur_tables(pb: GpuFemProblem):
    """(G, N, wdet) of the problem's rule in the reference orders: points
    (a, b, c) with c fastest and a along x (tensorelem.py:156-182), local
    functions (p, q, r) with r fastest (tensorelem.py:97-129).  G holds the
    physical gradients (axis-aligned box elements: dxi/dX = 2/h)."""
    B, D, w = pb.B, pb.D, pb.w  # (m, n) in the reference function order
    m, n = B.shape
    hx, hy, hz = pb.mesh.h
    Bx = B[:, None, None, :, None, None]
    By = B[None, :, None, None, :, None]
    Bz = B[None, None, :, None, None, :]
    Dx = D[:, None, None, :, None, None] * (2.0 / hx)
    Dy = D[None, :, None, None, :, None] * (2.0 / hy)
    Dz = D[None, None, :, None, None, :] * (2.0 / hz)
    G = np.stack([Dx * By * Bz, Bx * Dy * Bz, Bx * By * Dz], axis=-1).reshape(m ** 3, n ** 3, 3)
    N = (Bx * By * Bz).reshape(m ** 3, n ** 3)
    wdet = np.einsum("a,b,c->abc", w, w, w).reshape(-1) * (hx * hy * hz / 8.0)
    return np.ascontiguousarray(G), np.ascontiguousarray(N), np.ascontiguousarray(wdet)


class SchurSolver:
    """Device-resident ``make_solver`` + ``LinearSolver`` for one box problem.

    ``factor(u, c_k, c_m)`` builds the operator c_k K_T(u) + c_m M (element
    matrices, condensation, CSR); ``solve(b)`` returns (x, SolveStats) exactly
    as ``LinearSolver.solve`` does (preconditioner tag "+schur" when condensed)
    and raises PCGError / ValueError where the reference does."""

    def __init__(self, problem: GpuFemProblem, condense: bool = True, precond: str = "sgs", tol: float = 1e-12,
                 maxit: int = 200000):
        if not isinstance(problem, GpuFemProblem) or getattr(problem, "dofmap", None) is not None:
            raise NotImplementedError("the assembled / condensed solve is implemented for box-mesh problems")
        if precond not in _PREC:
            raise ValueError(f"unknown preconditioner {precond!r}")
        if not 0.0 < tol < 1.0:
            raise ValueError(f"tolerance must lie in (0, 1), got {tol}")
        self.problem = pb = problem
        self.condensed = bool(condense)
        self.precond, self.tol, self.maxit = precond, tol, maxit
        P, n = pb.P, pb.P + 1
        nx, ny, nz = pb.mesh.divisions
        lx, ly, lz = pb.mesh.lattice_shape(P)
        perm = pb.perm if pb.perm is not None else None
        if perm is None:
            from .lattice import reference_free_index

            perm = reference_free_index(pb.mesh, P, pb.dirichlet)[0].reshape(-1)
        perm = np.asarray(perm, dtype=np.int64).reshape(3, lz, ly, lx)
        # device addresses of the pitched lattice
        a = C.c_int64(0)
        lib = native.lib()

        def address(c, x, y, z):
            native.check(pb._ctx, lib.sdme_lattice_address(pb._ctx, c, x, y, z, C.byref(a)), "lattice_address")
            return a.value

        base = address(0, 0, 0, 0)
        px = address(0, 1, 0, 0) - base if lx > 1 else 1
        pitch_y = address(0, 0, 1, 0) - base if ly > 1 else lx
        pitch_z = address(0, 0, 0, 1) - base if lz > 1 else lx * ly
        ns = address(1, 0, 0, 0) - base
        assert px == 1
        off = np.array([0, P] + list(range(1, P)))
        t = np.arange(n)
        ei, ej, ek = (g.ravel() for g in np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"))
        order = np.lexsort((ei, ej, ek))  # element e = (k ny + j) nx + i
        ei, ej, ek = ei[order], ej[order], ek[order]
        tp, tq, tr = (g.ravel() for g in np.meshgrid(t, t, t, indexing="ij"))  # local (p, q, r), r fastest
        X = P * ei[:, None] + off[tp][None, :]
        Y = P * ej[:, None] + off[tq][None, :]
        Z = P * ek[:, None] + off[tr][None, :]
        interior = ((tp >= 2) & (tq >= 2) & (tr >= 2))[None, :].repeat(len(ei), axis=0)
        ne, nf = len(ei), n ** 3
        addr = np.empty((ne, nf, 3), dtype=np.int64)
        fidx = np.empty((ne, nf, 3), dtype=np.int64)
        for c in range(3):
            addr[:, :, c] = c * ns + Z * pitch_z + Y * pitch_y + X
            fidx[:, :, c] = perm[c, Z, Y, X]
        cons = fidx < 0
        addr[cons] = -1
        inter = np.broadcast_to(interior[:, :, None], fidx.shape)
        n_free = pb.n_free
        if self.condensed:
            nb = int(np.unique(fidx[~cons & ~inter]).size)
            bfree = fidx[~cons & ~inter]
            if bfree.size and (bfree.max() >= nb or np.unique(fidx[inter]).min() < nb):
                raise AssertionError("free boundary dofs are expected to be contiguous")  # dynamics.py:104-108
            role = np.where(cons, -1, np.where(inter, -2, fidx))
        else:
            nb = n_free
            role = np.where(cons, -1, fidx)
        self.nb = nb
        addr_b = np.full(nb, -1, dtype=np.int64)
        sel = role >= 0
        addr_b[role[sel]] = addr[sel]
        if nb and (addr_b < 0).any():
            raise AssertionError("system DOF without a lattice point")
        G, N, wdet = schur_tables(pb)
        need = 8 * ne * ((3 * nf) ** 2 + G.shape[0] * 3 * nf) * 1.5
        free_b, total_b = _device_memory()
        if need > 0.8 * free_b:
            raise MemoryError(f"the assembled solver needs ~{need / 2**30:.1f} GiB of element matrices "
                              f"({ne} elements of {3 * nf} DOFs; {free_b / 2**30:.1f} GiB free): use the "
                              "matrix-free path, SolverConfig(precond=\"diagonal\", condense=False)")
        self._keep = [np.ascontiguousarray(addr.reshape(ne, -1)), np.ascontiguousarray(role.reshape(ne, -1),
                                                                                        dtype=np.int32),
                      np.ascontiguousarray(addr_b), G, N, wdet]
        d = native.SchurDesc()
        d.n_elems, d.nd, d.nq, d.nb = ne, 3 * nf, G.shape[0], nb
        d.addr = self._keep[0].ctypes.data_as(C.POINTER(C.c_int64))
        d.role = self._keep[1].ctypes.data_as(C.POINTER(C.c_int32))
        d.addr_b = self._keep[2].ctypes.data_as(C.POINTER(C.c_int64))
        d.G, d.N, d.wdet = (native.dptr(x) for x in (G, N, wdet))
        d.mu, d.lambda_lame, d.rho0 = pb.mat.mu, pb.mat.lambda_lame, pb.mat.rho0
        h = C.c_void_p()
        native.check(pb._ctx, lib.sdme_schur_create(pb._ctx, C.byref(d), C.byref(h)), "schur_create")
        self._h = h
        self._x = None

    def close(self):
        if getattr(self, "_h", None):
            native.lib().sdme_schur_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def info(self) -> dict:
        nb, nnz = C.c_int64(0), C.c_int64(0)
        fl, bl = C.c_int(0), C.c_int(0)
        native.lib().sdme_schur_info(self._h, C.byref(nb), C.byref(nnz), C.byref(fl), C.byref(bl))
        return {"nb": nb.value, "nnz": nnz.value, "sgs_levels": (fl.value, bl.value)}

    def factor(self, u, c_k: float = 1.0, c_m: float = 0.0) -> "SchurSolver":
        """Operator c_k K_T(u) + c_m M; ``u`` a DeviceVector, a free ndarray
        or None (c_k = 0)."""
        pb = self.problem
        uid = -1
        if c_k != 0.0:
            uv = u if isinstance(u, DeviceVector) else pb._scratch("schur_u").set_free(np.asarray(u, dtype=float))
            uid = uv.vid
        native.check(pb._ctx, native.lib().sdme_schur_factor(self._h, uid, float(c_k), float(c_m)), "schur_factor")
        return self

    def solve(self, rhs, x: DeviceVector | None = None):
        """``LinearSolver.solve`` (solver.py:312-322): x and SolveStats."""
        from .solver import SolveStats

        pb = self.problem
        t0 = time.perf_counter()
        host = not isinstance(rhs, DeviceVector)
        bv = pb._scratch("schur_b").set_free(np.asarray(rhs, dtype=float)) if host else rhs
        xv = x if x is not None else (pb._scratch("schur_x") if host else DeviceVector(pb))
        its, rel = C.c_int(0), C.c_double(0.0)
        rc = native.lib().sdme_schur_solve(self._h, bv.vid, xv.vid, _PREC[self.precond], self.tol, self.maxit,
                                          C.byref(its), C.byref(rel))
        tag = {0: "none", 1: "diagonal", 2: "sgs"}[_PREC[self.precond]] + ("+schur" if self.condensed else "")
        secs = time.perf_counter() - t0
        if rc in (native.INDEFINITE, native.MAXIT):
            _, _, _, msg = native.last_error(pb._ctx)
            raise PCGError(msg, SolveStats(its.value, rel.value, secs, tag, False))
        if rc == native.BAD_DIAGONAL:
            _, _, _, msg = native.last_error(pb._ctx)
            raise ValueError(msg)
        native.check(pb._ctx, rc, "schur_solve")
        stats = SolveStats(its.value, rel.value, secs, tag)
        return (xv.free() if host else xv), stats

    def matrix(self):
        """(scipy CSR of the assembled system, element 0's dense matrix) -- for tests."""
        import scipy.sparse as sp

        info = self.info()
        nb, nnz = info["nb"], info["nnz"]
        rp = np.empty(nb + 1, dtype=np.int64)
        ci = np.empty(max(nnz, 1), dtype=np.int32)
        v = np.empty(max(nnz, 1))
        nd = 3 * (self.problem.P + 1) ** 3
        k0 = np.empty((nd, nd))
        native.check(self.problem._ctx, native.lib().sdme_schur_matrix(
            self._h, rp.ctypes.data_as(C.POINTER(C.c_int64)), ci.ctypes.data_as(C.POINTER(C.c_int32)),
            native.dptr(v), native.dptr(k0)), "schur_matrix")
        return sp.csr_matrix((v[:nnz], ci[:nnz], rp), shape=(nb, nb)), k0
