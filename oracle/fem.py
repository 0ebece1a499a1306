"""Oracle restatement of the reference FEM path (test infrastructure only).

Structured box meshes and the reference DOF numbering
(``sdmefem/meshdof.py:146-193, 404-503``), per-element dense tables
(``femcore.py:73-81``), the neo-Hookean element kernels
(``femcore.py:87-156``, ``material.py:65-105``), gather/scatter assembly
(``femcore.py:302-333``), boundary face quadrature and tractions
(``femcore.py:215-259, 391-397``) and frictionless penalty contact forces
(``contact.py:87-151``).  Element kernels are the dense reference formulation
(B^T D B + geometric), i.e. the algorithm the GPU replaces, not a copy of the
GPU's sum factorisation.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .basis import Basis, gauss, gll

BITS = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))
VTK_EDGES = ((0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4),
             (0, 4), (1, 5), (2, 6), (3, 7))
TAG_FACE = {"xmin": (0, 0), "xmax": (0, 1), "ymin": (1, 0), "ymax": (1, 1),
            "zmin": (2, 0), "zmax": (2, 1)}


class InversionError(RuntimeError):
    """femcore.py:36-42."""

    def __init__(self, elem_id, qp):
        super().__init__(f"element {elem_id} inverted at quadrature point {qp}")
        self.elem_id, self.qp = elem_id, qp


class Mesh:
    """gen_box_mesh (meshdof.py:146-193) + edge/face tables (meshdof.py:76-98)."""

    def __init__(self, div, lengths, origin=(0.0, 0.0, 0.0)):
        nx, ny, nz = div
        self.div = div
        xs = [origin[a] + np.linspace(0.0, lengths[a], div[a] + 1) for a in range(3)]
        vid = lambda i, j, k: (k * (ny + 1) + j) * (nx + 1) + i
        self.coords = np.array([(xs[0][i], xs[1][j], xs[2][k]) for k in range(nz + 1)
                                for j in range(ny + 1) for i in range(nx + 1)])
        self.elems = np.array([[vid(i + b[0], j + b[1], k + b[2]) for b in BITS]
                               for k in range(nz) for j in range(ny) for i in range(nx)])
        self.ijk = [(i, j, k) for k in range(nz) for j in range(ny) for i in range(nx)]
        self.nv = len(self.coords)
        self.ne = len(self.elems)
        # edges by first appearance over (element, local VTK edge)
        edges = {}
        self.elem_edges = np.zeros((self.ne, 12), dtype=int)
        for e, conn in enumerate(self.elems):
            for le, (a, b) in enumerate(VTK_EDGES):
                key = tuple(sorted((conn[a], conn[b])))
                self.elem_edges[e, le] = edges.setdefault(key, len(edges))
        self.n_edges = len(edges)
        # faces by first appearance over (element, local face 2*axis+side)
        faces = {}
        self.elem_faces = np.zeros((self.ne, 6), dtype=int)
        for e, conn in enumerate(self.elems):
            for lf in range(6):
                axis, side = divmod(lf, 2)
                corners = sorted(conn[v] for v, b in enumerate(BITS) if b[axis] == side)
                self.elem_faces[e, lf] = faces.setdefault(tuple(corners), len(faces))
        self.n_faces = len(faces)

    def boundary_sides(self, tag):
        """(element, local face) pairs on a box side, in face_quads order."""
        axis, side = TAG_FACE[tag]
        out = []
        for e, ijk in enumerate(self.ijk):
            if ijk[axis] == (self.div[axis] - 1 if side else 0):
                out.append((e, 2 * axis + side))
        # reference order: loops b (outer) then a (inner) over the in-plane axes
        d1, d2 = [d for d in range(3) if d != axis]
        out.sort(key=lambda t: (self.ijk[t[0]][d2], self.ijk[t[0]][d1]))
        return out

    def geometry(self, e, xi):
        """isoparametric_map (meshdof.py:286-296): X, J = dX/dxi, det J."""
        xc = self.coords[self.elems[e]]
        n = xi.shape[0]
        g = np.ones((n, 8))
        dg = np.ones((n, 8, 3))
        for v, b in enumerate(BITS):
            for d in range(3):
                f = 0.5 * (1 + xi[:, d]) if b[d] else 0.5 * (1 - xi[:, d])
                df = 0.5 if b[d] else -0.5
                g[:, v] *= f
                for gd in range(3):
                    dg[:, v, gd] *= df if gd == d else f
        x = g @ xc
        jac = np.einsum("pvd,vc->pcd", dg, xc)
        return x, jac, np.linalg.det(jac)


class DofMap:
    """build_dofmap (meshdof.py:404-472) restricted to box meshes, where every
    edge/face orientation is canonical (sign +1); boundary_modes
    (meshdof.py:475-503); free numbering (meshdof.py:364-370)."""

    def __init__(self, mesh: Mesh, P: int, dirichlet=None):
        self.P = P
        n = P + 1
        nep = P - 1
        self.index_map = np.array(list(np.ndindex(n, n, n)))  # r fastest (tensorelem.py:103)
        e_off = mesh.nv
        f_off = e_off + mesh.n_edges * nep
        i_off = f_off + mesh.n_faces * nep * nep
        self.n_modes = i_off + mesh.ne * nep ** 3
        edge_of = {}
        for le, (a, b) in enumerate(VTK_EDGES):
            axis = next(d for d in range(3) if BITS[a][d] != BITS[b][d])
            lo = BITS[a] if BITS[a][axis] == 0 else BITS[b]
            edge_of[(axis, tuple(lo[d] for d in range(3) if d != axis))] = le
        self.gdof = np.zeros((mesh.ne, n ** 3), dtype=int)
        for e in range(mesh.ne):
            conn = mesh.elems[e]
            for f, idx in enumerate(self.index_map):
                internal = [d for d in range(3) if idx[d] >= 2]
                if not internal:
                    self.gdof[e, f] = conn[BITS.index(tuple(int(t) for t in idx))]
                elif len(internal) == 1:
                    ax = internal[0]
                    le = edge_of[(ax, tuple(int(idx[d]) for d in range(3) if d != ax))]
                    self.gdof[e, f] = e_off + mesh.elem_edges[e, le] * nep + idx[ax] - 2
                elif len(internal) == 2:
                    ax = next(d for d in range(3) if idx[d] < 2)
                    lf = 2 * ax + int(idx[ax])
                    m1, m2 = (idx[d] for d in internal)
                    self.gdof[e, f] = (f_off + mesh.elem_faces[e, lf] * nep * nep
                                       + (m1 - 2) * nep + (m2 - 2))
                else:
                    lex = ((idx[0] - 2) * nep + idx[1] - 2) * nep + idx[2] - 2
                    self.gdof[e, f] = i_off + e * nep ** 3 + lex
        constrained = np.zeros((self.n_modes, 3), dtype=bool)
        for tag, comps in dirichlet or ():
            axis, side = TAG_FACE[tag]
            for e, _ in mesh.boundary_sides(tag):
                on = self.index_map[:, axis] == (1 if side else 0)
                for c in comps:
                    constrained[self.gdof[e, on], c] = True
        free = ~constrained.reshape(-1)
        self.free_map = np.where(free, np.cumsum(free) - 1, -1)
        self.n_free = int(free.sum())

    def evdofs(self, e):
        """elem_vector_dofs (meshdof.py:345-350): comp fastest."""
        modes = np.repeat(self.gdof[e], 3) * 3 + np.tile(np.arange(3), len(self.gdof[e]))
        return self.free_map[modes]


class Tables:
    """Per-element quadrature tables (femcore.py:62-81, tensorelem.py:156-182)."""

    def __init__(self, mesh: Mesh, basis: Basis, m: int, share_geometry: bool = False):
        xq, wq = gauss(m)
        v, d = basis.eval(xq)  # (n, m)
        n = basis.P + 1
        self.pts_ref = np.array([(a, b, c) for a in xq for b in xq for c in xq])
        self.w = np.einsum("a,b,c->abc", wq, wq, wq).ravel()
        self.vals = np.einsum("pa,qb,rc->abcpqr", v, v, v).reshape(m ** 3, n ** 3)
        g = [np.einsum("pa,qb,rc->abcpqr", *(d if k == ax else v for k in range(3)))
             for ax, _ in enumerate(range(3))]
        self.dref = np.stack([gi.reshape(m ** 3, n ** 3) for gi in g], axis=-1)
        self.per_elem = []
        shared = {}
        for e in range(mesh.ne):
            x, jac, det = mesh.geometry(e, self.pts_ref)
            key = None
            if share_geometry:
                # large uniform box meshes (test-size memory): elements whose
                # Jacobians agree to 1e-13 reuse one (grad, w det J) pair
                key = np.round(jac / np.abs(jac).max(), 13).tobytes() + np.round(det / np.abs(det).max(), 13).tobytes()
            if key is not None and key in shared:
                grad, wdet = shared[key]
            else:
                grad = np.einsum("qfd,qdc->qfc", self.dref, np.linalg.inv(jac))
                wdet = self.w * det
                if key is not None:
                    shared[key] = (grad, wdet)
            self.per_elem.append((x, grad, wdet))


class Material:
    """NeoHookean (material.py:32-62)."""

    def __init__(self, E, nu, rho):
        self.mu = E / (2.0 * (1.0 + nu))
        self.lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
        self.rho = rho


def _state(grad, ue, e):
    """deformation_state (femcore.py:87-96) + pk2 pieces (material.py:65-81)."""
    f = np.einsum("qfd,fc->qcd", grad, ue) + np.eye(3)
    det = np.linalg.det(f)
    if np.any(det <= 0):
        raise InversionError(e, int(np.argmax(det <= 0)))
    c = np.einsum("qkc,qkd->qcd", f, f)
    ci = np.linalg.inv(c)
    lnj = 0.5 * np.log(np.linalg.det(c))
    return f, ci, lnj


def pk2(mat, ci, lnj):
    return mat.mu * (np.eye(3) - ci) + mat.lam * lnj[:, None, None] * ci


def elem_fint(mat, grad, wdet, ue, e=-1):
    """element_internal_force (femcore.py:99-106)."""
    f, ci, lnj = _state(grad, ue, e)
    p1 = f @ pk2(mat, ci, lnj)
    return np.einsum("q,qfd,qcd->fc", wdet, grad, p1).reshape(-1)


def elem_energy(mat, grad, wdet, ue, e=-1):
    """strain_energy (femcore.py:109-113, material.py:80)."""
    f, _, lnj = _state(grad, ue, e)
    trc = np.einsum("qij,qij->q", f, f)
    psi = 0.5 * mat.mu * (trc - 3.0) - mat.mu * lnj + 0.5 * mat.lam * lnj ** 2
    return float(wdet @ psi)


_VOIGT = ((0, 0), (1, 1), (2, 2), (0, 1), (1, 2), (0, 2))


def elem_tangent(mat, grad, wdet, ue, e=-1):
    """element_tangent (femcore.py:116-146, material.py:84-105): dense
    B^T D B material part plus the geometric part grad S grad^T (x) I3."""
    f, ci, lnj = _state(grad, ue, e)
    s = pk2(mat, ci, lnj)
    nq, nf, _ = grad.shape
    dm = np.empty((nq, 6, 6))
    coef = mat.mu - mat.lam * lnj
    for a, (i, j) in enumerate(_VOIGT):
        for b, (k, l) in enumerate(_VOIGT):
            dm[:, a, b] = (mat.lam * ci[:, i, j] * ci[:, k, l]
                           + coef * (ci[:, i, k] * ci[:, j, l] + ci[:, i, l] * ci[:, j, k]))
    bm = np.zeros((nq, 6, nf, 3))
    for a, (i, j) in enumerate(_VOIGT):
        bm[:, a] = grad[:, :, j, None] * f[:, None, :, i]
        if i != j:
            bm[:, a] += grad[:, :, i, None] * f[:, None, :, j]
    bm = bm.reshape(nq, 6, 3 * nf)
    tmp = (dm * wdet[:, None, None]) @ bm
    k = np.tensordot(bm, tmp, axes=([0, 1], [0, 1]))
    kg = np.tensordot(grad, grad @ (s * wdet[:, None, None]), axes=([0, 2], [0, 2]))
    k4 = k.reshape(nf, 3, nf, 3)
    for c in range(3):
        k4[:, c, :, c] += kg
    return k


def elem_mass(mat, vals, wdet):
    """element_mass (femcore.py:149-156)."""
    ms = (vals * (mat.rho * wdet)[:, None]).T @ vals
    nf = vals.shape[1]
    out = np.zeros((nf, 3, nf, 3))
    for c in range(3):
        out[:, c, :, c] = ms
    return out.reshape(3 * nf, 3 * nf)


class Problem:
    """FemProblem (femcore.py:273-431) on a box mesh."""

    def __init__(self, mesh, basis, mat, m=None, dirichlet=None, share_geometry=False):
        self.mesh, self.basis, self.mat = mesh, basis, mat
        self.m = basis.P + 1 if m is None else m  # femcore.py:283-292
        self.dmap = DofMap(mesh, basis.P, dirichlet)
        self.tab = Tables(mesh, basis, self.m, share_geometry)
        self.n_free = self.dmap.n_free
        self._edofs = [self.dmap.evdofs(e) for e in range(mesh.ne)]

    def gather(self, e, u):
        """femcore.py:302-306 (signs are +1 on box meshes)."""
        d = self._edofs[e]
        return np.where(d >= 0, u[np.maximum(d, 0)], 0.0).reshape(-1, 3)

    def scatter(self, out, e, r):
        d = self._edofs[e]
        ok = d >= 0
        np.add.at(out, d[ok], r[ok])

    def total_strain_energy(self, u):
        """femcore.py:374-378."""
        return sum(elem_energy(self.mat, self.tab.per_elem[e][1], self.tab.per_elem[e][2], self.gather(e, u), e)
                   for e in range(self.mesh.ne))

    def internal_force(self, u):
        out = np.zeros(self.n_free)
        for e in range(self.mesh.ne):
            _, grad, wdet = self.tab.per_elem[e]
            self.scatter(out, e, elem_fint(self.mat, grad, wdet, self.gather(e, u), e))
        return out

    def element_tangents(self, u):
        for e in range(self.mesh.ne):
            _, grad, wdet = self.tab.per_elem[e]
            yield e, elem_tangent(self.mat, grad, wdet, self.gather(e, u), e)

    def apply_tangent(self, u, p, c_m=0.0):
        """sum_e (K_e + c_m M_e) p_e -- the EBE K.p the GPU replaces."""
        out = np.zeros(self.n_free)
        for e, ke in self.element_tangents(u):
            if c_m:
                ke = ke + c_m * elem_mass(self.mat, self.tab.vals, self.tab.per_elem[e][2])
            self.scatter(out, e, ke @ self.gather(e, p).reshape(-1))
        return out

    def assemble(self, u=None, c_k=1.0, c_m=0.0):
        """CSR of c_k K_T(u) + c_m M over free dofs (femcore.py:319-333)."""
        rows, cols, vals = [], [], []
        for e in range(self.mesh.ne):
            _, grad, wdet = self.tab.per_elem[e]
            ke = np.zeros((3 * len(self.dmap.gdof[e]),) * 2)
            if c_k:
                ke = c_k * elem_tangent(self.mat, grad, wdet, self.gather(e, u), e)
            if c_m:
                ke = ke + c_m * elem_mass(self.mat, self.tab.vals, wdet)
            d = self._edofs[e]
            ok = d >= 0
            kd = ke[np.ix_(ok, ok)]
            fr = d[ok]
            rows.append(np.repeat(fr, fr.size))
            cols.append(np.tile(fr, fr.size))
            vals.append(kd.ravel())
        a = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.n_free, self.n_free))
        a.sum_duplicates()
        return a

    def mass(self):
        return self.assemble(None, c_k=0.0, c_m=1.0)

    def lumped_mass(self):
        """Row sums of the assembled mass over free columns,
        ``mass().sum(axis=1)``, accumulated element by element
        (M_e applied to the element's free-DOF mask) without forming the CSR."""
        out = np.zeros(self.n_free)
        for e in range(self.mesh.ne):
            me = elem_mass(self.mat, self.tab.vals, self.tab.per_elem[e][2])
            self.scatter(out, e, me @ (self._edofs[e] >= 0).astype(float))
        return out

    # ---------------------------------------------------------- faces (femcore.py:215-259)
    def face_tables(self, tag, q):
        xq, wq = gauss(q)
        axis, side = TAG_FACE[tag]
        d1, d2 = [d for d in range(3) if d != axis]
        grid = np.array([(a, b) for a in xq for b in xq])
        w2 = np.einsum("a,b->ab", wq, wq).ravel()
        out = []
        for e, _ in self.mesh.boundary_sides(tag):
            xi = np.zeros((len(grid), 3))
            xi[:, axis] = 1.0 if side else -1.0
            xi[:, d1], xi[:, d2] = grid[:, 0], grid[:, 1]
            x, jac, _ = self.mesh.geometry(e, xi)
            nvec = np.cross(jac[:, :, d1], jac[:, :, d2])
            area = np.linalg.norm(nvec, axis=1)
            nvec /= area[:, None]
            outward = (1.0 if side else -1.0) * jac[:, :, axis]
            nvec *= np.sign(np.einsum("qc,qc->q", nvec, outward))[:, None]
            v = [self.basis.eval(xi[:, k])[0] for k in range(3)]
            im = self.dmap.index_map
            vals = v[0][im[:, 0]].T * v[1][im[:, 1]].T * v[2][im[:, 2]].T
            out.append((e, x, vals, w2 * area, nvec))
        return out

    def traction_vector(self, tag, tvec):
        """traction_vector (femcore.py:391-397) with a constant traction."""
        out = np.zeros(self.n_free)
        for e, x, vals, warea, _ in self.face_tables(tag, self.m):
            r = np.einsum("q,qf,c->fc", warea, vals, np.asarray(tvec, dtype=float))
            self.scatter(out, e, r.reshape(-1))
        return out


class Contact:
    """PenaltyContact (contact.py:72-176): forces, assembled stiffness, the
    pressure-settled test and the per-step penalty update."""

    def __init__(self, problem: Problem, point, normal, eps, tag, quad_order=None, deps=0.0, gap_tol=1e-3,
                 stress_tol=1e-2):
        self.pb = problem
        self.point = np.asarray(point, dtype=float)
        n = np.asarray(normal, dtype=float)
        self.normal = n / np.linalg.norm(n)
        self.eps = eps
        self.deps, self.gap_tol, self.stress_tol = deps, gap_tol, stress_tol
        q = quad_order if quad_order is not None else problem.basis.P + 1
        self.faces = problem.face_tables(tag, q)
        self.last_pressures = None
        self.history = []

    def stiffness(self, u):
        """contact.py:129-140: eps sum_{q active} warea N_f N_g (n n^T), CSR."""
        rows, cols, vals = [], [], []
        nn = np.outer(self.normal, self.normal)
        for (e, x, fv, warea, _), g in zip(self.faces, self.gaps(u)):
            act = g < 0.0
            if not act.any():
                continue
            fv = np.where(np.abs(fv).max(axis=0) > 1e-13, fv, 0.0)  # face support (contact.py:121-123)
            kf = np.einsum("q,qf,qg->fg", self.eps * warea * act, fv, fv)
            kc = np.einsum("fg,ce->fcge", kf, nn).reshape(kf.shape[0] * 3, kf.shape[0] * 3)
            d = self.pb._edofs[e]
            ok = d >= 0
            rows.append(np.repeat(d[ok], ok.sum()))
            cols.append(np.tile(d[ok], ok.sum()))
            vals.append(kc[np.ix_(ok, ok)].ravel())
        n = self.pb.n_free
        if not rows:
            return None
        return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))

    def pressures(self, u):
        return np.concatenate([np.where(g < 0.0, -self.eps * g, 0.0) for g in self.gaps(u)])

    def settled(self, p):
        """contact.py:153-160 (and records p as the iteration's pressures)."""
        prev = self.last_pressures
        self.last_pressures = p
        if prev is None or prev.shape != p.shape:
            return not p.any()
        scale = max(np.abs(p).max(), np.abs(prev).max())
        if scale == 0.0:
            return True
        return float(np.abs(p - prev).max()) / scale <= self.stress_tol

    def accept_step(self, u):
        """contact.py:162-176."""
        gs = np.concatenate(self.gaps(u))
        pen = max(float(-gs.min()), 0.0)
        act = gs < 0.0
        tn = np.where(act, -self.eps * gs, 0.0)
        self.history.append((self.eps, pen, float(tn[act].min()) if act.any() else 0.0, int(act.sum())))
        if pen > self.gap_tol and self.deps > 0.0:
            self.eps += self.deps
        self.last_pressures = None

    def gaps(self, u):
        return [(x + vals @ self.pb.gather(e, u) - self.point) @ self.normal
                for e, x, vals, _, _ in self.faces]

    def force(self, u):
        out = np.zeros(self.pb.n_free)
        gs = self.gaps(u)
        for (e, x, vals, warea, _), g in zip(self.faces, gs):
            tn = np.where(g < 0.0, -self.eps * g, 0.0)
            if not np.any(g < 0.0):
                continue
            vals = np.where(np.abs(vals).max(axis=0) > 1e-13, vals, 0.0)  # face support (contact.py:121-123)
            r = np.einsum("q,qf,c->fc", warea * tn, vals, self.normal)
            self.pb.scatter(out, e, r.reshape(-1))
        return out, gs

    def penalty_energy(self, u):
        """contact.py:178-184."""
        return sum(0.5 * self.eps * float(warea @ np.minimum(g, 0.0) ** 2)
                   for (_, _, _, warea, _), g in zip(self.faces, self.gaps(u)))

    def penetration(self, u):
        return max(0.0, max(float(-g.min()) for g in self.gaps(u)))
