"""Oracle restatement of general hexahedral meshes (test infrastructure only).

``Mesh`` with edge / face tables by first appearance (``meshdof.py:41-136``),
``build_dofmap`` with orientation (``meshdof.py:373-472``: ``_oriented_1d``,
``_face_frame``), ``boundary_modes`` (``meshdof.py:475-503``) and the signed
gather / scatter of ``FemProblem`` (``femcore.py:302-321``), written as the
reference's plain loops.  Element kernels, tables and assembly are the box
oracle's (``oracle/fem.py``), which are geometry-general already.
"""

from __future__ import annotations

import numpy as np

from .fem import BITS, VTK_EDGES, Problem, Tables

# local faces 2*axis + side: (axis, side, d1, d2, corners[(ba, bb)]) (tensorelem.py:53-70)
FACES = []
for _axis in range(3):
    _d1, _d2 = [d for d in range(3) if d != _axis]
    for _side in (0, 1):
        _c = {}
        for _ba in (0, 1):
            for _bb in (0, 1):
                _w = [0, 0, 0]
                _w[_axis], _w[_d1], _w[_d2] = _side, _ba, _bb
                _c[(_ba, _bb)] = BITS.index(tuple(_w))
        FACES.append((_axis, _side, _d1, _d2, _c))
QUAD = ((0, 0), (1, 0), (1, 1), (0, 1))


def _edge_table():
    out = []
    for a, b in VTK_EDGES:
        axis = next(d for d in range(3) if BITS[a][d] != BITS[b][d])
        lo, hi = (a, b) if BITS[a][axis] == 0 else (b, a)
        out.append((axis, tuple(BITS[lo][d] for d in range(3) if d != axis), lo, hi))
    return out


EDGES = _edge_table()


class GeneralMesh:
    """meshdof.py:41-136 for 3D hexahedra."""

    def __init__(self, coords, elems, boundary=None):
        self.coords = np.asarray(coords, dtype=float)
        self.elems = np.asarray(elems, dtype=int)
        self.boundary = dict(boundary or {})
        self.nv, self.ne = len(self.coords), len(self.elems)
        lookup = {}
        self.elem_edges = np.zeros((self.ne, 12), dtype=int)
        for e, conn in enumerate(self.elems):
            for le, (_, _, lo, hi) in enumerate(EDGES):
                key = tuple(sorted((conn[lo], conn[hi])))
                self.elem_edges[e, le] = lookup.setdefault(key, len(lookup))
        self.edge_verts = np.array(sorted(lookup, key=lookup.get), dtype=int).reshape(-1, 2)
        self.n_edges = len(lookup)
        flook = {}
        self.elem_faces = np.zeros((self.ne, 6), dtype=int)
        for e, conn in enumerate(self.elems):
            for lf, (_, _, _, _, corners) in enumerate(FACES):
                key = tuple(sorted(conn[corners[bb]] for bb in QUAD))
                self.elem_faces[e, lf] = flook.setdefault(key, len(flook))
        self.n_faces = len(flook)
        owner = {}
        for e in range(self.ne):
            for lf in range(6):
                owner.setdefault(self.elem_faces[e, lf], []).append((e, lf))
        self.sides = {tag: [owner[flook[tuple(sorted(v))]][0] for v in faces] for tag, faces in self.boundary.items()}

    def boundary_sides(self, tag):
        return self.sides[tag]

    def geometry(self, e, xi):
        """isoparametric_map (meshdof.py:286-296)."""
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
        jac = np.einsum("pvd,vc->pcd", dg, xc)
        return g @ xc, jac, np.linalg.det(jac)


def _oriented(m, flipped, basis):
    """_oriented_1d (meshdof.py:373-384)."""
    if not flipped:
        return m, 1.0
    if basis.tag == "LagrangeGLL":
        return basis.P + 2 - m, 1.0
    if basis.internal_parity is None:
        raise ValueError("edge/face reversal needs definite-parity internal modes")
    return m, float(basis.internal_parity[m - 2])


def _face_frame(gvids):
    """_face_frame (meshdof.py:387-401)."""
    a0, b0 = min(gvids, key=gvids.get)
    ga, gb = gvids[(1 - a0, b0)], gvids[(a0, 1 - b0)]
    return (ga > gb), a0 == 1, b0 == 1


class GeneralDofMap:
    """build_dofmap (meshdof.py:404-472) + apply_dirichlet (meshdof.py:364-370)."""

    def __init__(self, mesh: GeneralMesh, basis, dirichlet=None):
        P = basis.P
        n, nep = P + 1, P - 1
        self.P = P
        self.index_map = np.array(list(np.ndindex(n, n, n)))
        e_off = mesh.nv
        f_off = e_off + mesh.n_edges * nep
        i_off = f_off + mesh.n_faces * nep * nep
        self.n_modes = i_off + mesh.ne * nep ** 3
        edge_of = {(ax, fixed): le for le, (ax, fixed, _, _) in enumerate(EDGES)}
        self.gdof = np.zeros((mesh.ne, n ** 3), dtype=int)
        self.gsign = np.ones((mesh.ne, n ** 3))
        for e in range(mesh.ne):
            conn = mesh.elems[e]
            for f, idx in enumerate(self.index_map):
                internal = [d for d in range(3) if idx[d] >= 2]
                if not internal:
                    self.gdof[e, f] = conn[BITS.index(tuple(int(t) for t in idx))]
                elif len(internal) == 1:
                    ax = internal[0]
                    le = edge_of[(ax, tuple(int(idx[d]) for d in range(3) if d != ax))]
                    ge = mesh.elem_edges[e, le]
                    flipped = conn[EDGES[le][2]] != mesh.edge_verts[ge, 0]
                    mc, s = _oriented(int(idx[ax]), flipped, basis)
                    self.gdof[e, f] = e_off + ge * nep + mc - 2
                    self.gsign[e, f] = s
                elif len(internal) == 2:
                    ax = next(d for d in range(3) if idx[d] < 2)
                    lf = 2 * ax + int(idx[ax])
                    m1, m2 = (int(idx[d]) for d in internal)
                    corners = FACES[lf][4]
                    swap, fa, fb = _face_frame({bb: conn[corners[bb]] for bb in corners})
                    ma, sa = _oriented(m1, fa, basis)
                    mb, sb = _oriented(m2, fb, basis)
                    ms, mt = (mb, ma) if swap else (ma, mb)
                    self.gdof[e, f] = f_off + mesh.elem_faces[e, lf] * nep * nep + (ms - 2) * nep + (mt - 2)
                    self.gsign[e, f] = sa * sb
                else:
                    lex = ((idx[0] - 2) * nep + idx[1] - 2) * nep + idx[2] - 2
                    self.gdof[e, f] = i_off + e * nep ** 3 + lex
        constrained = np.zeros((self.n_modes, 3), dtype=bool)
        for tag, comps in dirichlet or ():
            modes = set()
            for e, lf in mesh.boundary_sides(tag):
                conn = mesh.elems[e]
                vids = [FACES[lf][4][bb] for bb in QUAD]
                modes.update(int(conn[v]) for v in vids)
                for le, (_, _, lo, hi) in enumerate(EDGES):
                    if {lo, hi} <= set(vids):
                        modes.update(e_off + mesh.elem_edges[e, le] * nep + j for j in range(nep))
                modes.update(f_off + mesh.elem_faces[e, lf] * nep * nep + j for j in range(nep * nep))
            for c in comps:
                constrained[sorted(modes), c] = True
        free = ~constrained.reshape(-1)
        self.free_map = np.where(free, np.cumsum(free) - 1, -1)
        self.n_free = int(free.sum())

    def evdofs(self, e):
        """elem_vector_dofs (meshdof.py:345-350): free ids and signs, comp fastest."""
        modes = np.repeat(self.gdof[e], 3) * 3 + np.tile(np.arange(3), len(self.gdof[e]))
        return self.free_map[modes], np.repeat(self.gsign[e], 3)


class GeneralProblem(Problem):
    """FemProblem (femcore.py:273-431) on a general hexahedral mesh: the box
    oracle's element kernels with the signed gather / scatter of
    femcore.py:302-321 (and an assembled matrix with sign(i) sign(j))."""

    def __init__(self, mesh: GeneralMesh, basis, mat, m=None, dirichlet=None):
        self.mesh, self.basis, self.mat = mesh, basis, mat
        self.m = basis.P + 1 if m is None else m
        self.dmap = GeneralDofMap(mesh, basis, dirichlet)
        self.tab = Tables(mesh, basis, self.m)
        self.n_free = self.dmap.n_free
        self._sedofs = [self.dmap.evdofs(e) for e in range(mesh.ne)]
        self._edofs = [d for d, _ in self._sedofs]

    def gather(self, e, u):
        d, s = self._sedofs[e]
        return (np.where(d >= 0, u[np.maximum(d, 0)], 0.0) * s).reshape(-1, 3)

    def scatter(self, out, e, r):
        d, s = self._sedofs[e]
        ok = d >= 0
        np.add.at(out, d[ok], (r * s)[ok])

    def assemble(self, u=None, c_k=1.0, c_m=0.0):
        """CSR with the element matrices signed by sign(i) sign(j) (femcore.py:323-333)."""
        import scipy.sparse as sp
        from .fem import elem_mass, elem_tangent
        rows, cols, vals = [], [], []
        for e in range(self.mesh.ne):
            _, grad, wdet = self.tab.per_elem[e]
            d, s = self._sedofs[e]
            ke = np.zeros((len(d), len(d)))
            if c_k:
                ke = c_k * elem_tangent(self.mat, grad, wdet, self.gather(e, u), e)
            if c_m:
                ke = ke + c_m * elem_mass(self.mat, self.tab.vals, wdet)
            ke = ke * np.outer(s, s)
            ok = d >= 0
            fr = d[ok]
            rows.append(np.repeat(fr, fr.size))
            cols.append(np.tile(fr, fr.size))
            vals.append(ke[np.ix_(ok, ok)].ravel())
        a = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.n_free, self.n_free))
        a.sum_duplicates()
        return a
