"""General conforming hexahedral meshes: geometry, entity tables,
the reference's global mode numbering with orientation signs, and the index /
geometry tables the device operators of :class:`GpuMeshProblem` consume.

Restates, vectorised over elements:

* ``Mesh`` and its edge / face tables (``meshdof.py:41-136``): edges and faces
  numbered by first appearance in the (element, local entity) loop;
* ``gen_box_mesh`` / ``read_mesh`` / ``write_mesh`` (``meshdof.py:146-266``);
* the trilinear isoparametric map (``meshdof.py:269-296``): ``J = dX/dxi`` at the
  quadrature points, ``det J > 0`` enforced (``MeshError``);
* ``build_dofmap`` (``meshdof.py:404-472``): vertex modes by vertex id, edge modes
  ``edge_off + ge*(P-1) + m`` with the reversal rule of ``_oriented_1d``
  (``meshdof.py:373-384``: nodal bases reverse the index, modal / SDME bases take
  the reflection parity of the internal function as a sign), face modes with the
  canonical frame of ``_face_frame`` (``meshdof.py:387-401``), element interiors
  last; ``boundary_modes`` (``meshdof.py:475-503``) and the free-DOF compaction of
  ``DofMap.apply_dirichlet`` (``meshdof.py:364-370``).

The device works element by element (no lattice): each element's (P+1)^3
coefficients per component are gathered through an index table in the
kernel's lattice-local order (1D offset 0 = left vertex, P = right vertex,
1..P-1 = internal functions 2..P), and the element results are summed into the
free-DOF vector through a CSR table whose per-DOF order is the element order of
the reference's ``np.add.at`` assembly (``femcore.py:318-321``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .basis import Basis1D, Rule
from .lattice import VERTEX_BITS

__all__ = ["MeshError", "HexMesh", "read_mesh", "write_mesh", "MeshDofMap", "build_mesh_dofmap",
           "element_tables"]

_VTK_EDGE_PAIRS = ((0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4),
                   (0, 4), (1, 5), (2, 6), (3, 7))


class MeshError(ValueError):
    """``meshdof.py:36-37``."""


def _edge_table():
    """Per local edge (axis, lo vertex, hi vertex): lo at bit 0 of the running
    axis (``tensorelem.py:36-50``)."""
    out = []
    for va, vb in _VTK_EDGE_PAIRS:
        axis = next(d for d in range(3) if VERTEX_BITS[va][d] != VERTEX_BITS[vb][d])
        lo, hi = (va, vb) if VERTEX_BITS[va][axis] == 0 else (vb, va)
        out.append((axis, lo, hi))
    return tuple(out)


def _face_table():
    """Face id 2*axis + side: (axis, side, d1, d2, corners[(ba, bb)] -> local
    vertex) with in-plane axes d1 < d2 (``tensorelem.py:53-70``)."""
    out = []
    for axis in range(3):
        d1, d2 = [d for d in range(3) if d != axis]
        for side in (0, 1):
            corners = {}
            for ba in (0, 1):
                for bb in (0, 1):
                    want = [0, 0, 0]
                    want[axis], want[d1], want[d2] = side, ba, bb
                    corners[(ba, bb)] = VERTEX_BITS.index(tuple(want))
            out.append((axis, side, d1, d2, corners))
    return tuple(out)


EDGE_TABLE = _edge_table()
FACE_TABLE = _face_table()
_QUAD = ((0, 0), (1, 0), (1, 1), (0, 1))


def _first_appearance(keys):
    """Ids of ``keys`` (rows) numbered by first appearance; returns (ids, first rows)."""
    uniq, first, inv = np.unique(keys, axis=0, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty(len(order), dtype=np.int64)
    rank[order] = np.arange(len(order))
    return rank[inv.reshape(-1)], first[order]


@dataclass
class HexMesh:
    """Conforming hexahedral mesh: vertex coordinates, VTK-ordered element
    connectivity and boundary tags (tag -> list of vertex quads)."""

    coords: np.ndarray
    elems: np.ndarray
    boundary: dict = field(default_factory=dict)

    def __post_init__(self):
        self.coords = np.asarray(self.coords, dtype=np.float64)
        self.elems = np.asarray(self.elems, dtype=np.int64)
        if self.coords.ndim != 2 or self.coords.shape[1] != 3:
            raise MeshError("coordinates must be (n_vertices, 3)")
        if self.elems.ndim != 2 or self.elems.shape[1] != 8:
            raise MeshError("element connectivity does not match the dimension")
        ne = len(self.elems)
        conn = self.elems
        lo = conn[:, [e[1] for e in EDGE_TABLE]]
        hi = conn[:, [e[2] for e in EDGE_TABLE]]
        keys = np.stack([np.minimum(lo, hi).reshape(-1), np.maximum(lo, hi).reshape(-1)], axis=1)
        ids, first = _first_appearance(keys)
        self.elem_edges = ids.reshape(ne, 12)
        self.edge_verts = keys[first]
        quads = np.stack([conn[:, [f[4][bb] for bb in _QUAD]] for f in FACE_TABLE], axis=1)  # (ne, 6, 4)
        skeys = np.sort(quads.reshape(-1, 4), axis=1)
        fids, ffirst = _first_appearance(skeys)
        self.elem_faces = fids.reshape(ne, 6)
        self.face_verts = quads.reshape(-1, 4)[ffirst]
        self._face_key = {tuple(k): i for i, k in enumerate(skeys[ffirst])}
        owners = np.bincount(self.elem_faces.reshape(-1), minlength=len(ffirst))
        self.boundary_sides = {}
        flat_owner = {}
        for e in range(ne):
            for lf in range(6):
                f = int(self.elem_faces[e, lf])
                if owners[f] == 1:
                    flat_owner[f] = (e, lf)
        for tag, faces in self.boundary.items():
            sides = []
            for verts in faces:
                f = self._face_key.get(tuple(sorted(int(v) for v in verts)))
                if f is None:
                    raise MeshError(f"boundary tag {tag!r} references a missing face {tuple(verts)}")
                if owners[f] != 1:
                    raise MeshError(f"boundary tag {tag!r} face {tuple(verts)} is interior")
                sides.append(flat_owner[f])
            self.boundary_sides[tag] = sides

    @property
    def n_vertices(self) -> int:
        return len(self.coords)

    @property
    def n_elems(self) -> int:
        return len(self.elems)

    @property
    def n_edges(self) -> int:
        return len(self.edge_verts)

    @property
    def n_faces(self) -> int:
        return len(self.face_verts)

    @classmethod
    def box(cls, divisions, lengths, origin=None) -> "HexMesh":
        """``gen_box_mesh`` (``meshdof.py:146-193``): same vertex ids, element
        order and boundary quads."""
        nx, ny, nz = (int(v) for v in divisions)
        if min(nx, ny, nz) < 1:
            raise MeshError("need at least one cell per axis")
        ox, oy, oz = origin if origin is not None else (0.0, 0.0, 0.0)
        xs = ox + np.linspace(0.0, lengths[0], nx + 1)
        ys = oy + np.linspace(0.0, lengths[1], ny + 1)
        zs = oz + np.linspace(0.0, lengths[2], nz + 1)
        Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
        coords = np.stack([X.reshape(-1), Y.reshape(-1), Z.reshape(-1)], axis=1)

        def vid(i, j, k):
            return (k * (ny + 1) + j) * (nx + 1) + i

        k, j, i = (a.reshape(-1) for a in np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij"))
        elems = np.stack([vid(i + bx, j + by, k + bz) for bx, by, bz in VERTEX_BITS], axis=1)

        def face_quads(axis, at_end):
            n = (nx, ny, nz)
            fix = n[axis] if at_end else 0
            r0, r1 = {0: (ny, nz), 1: (nx, nz), 2: (nx, ny)}[axis]
            quads = []
            for b in range(r1):
                for a in range(r0):
                    pts = [(a, b), (a + 1, b), (a + 1, b + 1), (a, b + 1)]
                    if axis == 0:
                        quads.append(tuple(vid(fix, s, t) for s, t in pts))
                    elif axis == 1:
                        quads.append(tuple(vid(s, fix, t) for s, t in pts))
                    else:
                        quads.append(tuple(vid(s, t, fix) for s, t in pts))
            return quads

        boundary = {"xmin": face_quads(0, False), "xmax": face_quads(0, True),
                    "ymin": face_quads(1, False), "ymax": face_quads(1, True),
                    "zmin": face_quads(2, False), "zmax": face_quads(2, True)}
        return cls(coords, elems, boundary)


_SECTIONS = ("VERTICES", "ELEMENTS", "BOUNDARY")


def _numbered_rows(rows, fmt) -> list[str]:
    return [f"{i} {' '.join(fmt(v) for v in row)}" for i, row in enumerate(rows)]


def write_mesh(mesh: HexMesh, path) -> None:
    """Write the reference's plain-text mesh format (``meshdof.py:223-234``):
    a VERTICES block of ``id x y z`` rows (round-trip ``repr`` floats), an
    ELEMENTS block of ``id v0..v7`` rows and a BOUNDARY block of
    ``tag v0..v3`` rows."""
    blocks = {
        "VERTICES": _numbered_rows(np.asarray(mesh.coords, dtype=float).tolist(), lambda c: repr(float(c))),
        "ELEMENTS": _numbered_rows(np.asarray(mesh.elems).tolist(), lambda v: str(int(v))),
        "BOUNDARY": [tag + " " + " ".join(str(int(v)) for v in quad)
                     for tag, quads in mesh.boundary.items() for quad in quads],
    }
    text = "".join(name + "\n" + "".join(row + "\n" for row in blocks[name]) for name in _SECTIONS)
    with open(path, "w") as fh:
        fh.write(text)


def _mesh_tokens(path):
    """(line number, section, fields) of every non-empty, comment-stripped
    data line; ``#`` starts a comment, a bare section name switches section."""
    section = None
    with open(path) as fh:
        for ln, raw in enumerate(fh, 1):
            fields = raw.partition("#")[0].split()
            if not fields:
                continue
            if len(fields) == 1 and fields[0] in _SECTIONS:
                section = fields[0]
                continue
            if section is None:
                raise MeshError(f"{path}:{ln}: content before any section header")
            yield ln, section, fields


def read_mesh(path) -> HexMesh:
    """Read the format of :func:`write_mesh` (the reference's ``read_mesh``,
    ``meshdof.py:237-266``): rows are placed by their id, so ids may appear
    in any order."""
    table = {"VERTICES": {}, "ELEMENTS": {}}
    boundary: dict[str, list] = {}
    for _, section, fields in _mesh_tokens(path):
        if section == "BOUNDARY":
            boundary.setdefault(fields[0], []).append(tuple(map(int, fields[1:])))
        else:
            conv = float if section == "VERTICES" else int
            table[section][int(fields[0])] = list(map(conv, fields[1:]))
    verts, elems = table["VERTICES"], table["ELEMENTS"]
    if not (verts and elems):
        raise MeshError(f"{path}: missing VERTICES or ELEMENTS section")
    coords = np.array([row for _, row in sorted(verts.items())], dtype=float)
    conn = np.array([row for _, row in sorted(elems.items())], dtype=np.int64)
    return HexMesh(coords, conn, boundary)


def _internal_parity(basis: Basis1D):
    """Reflection parity (+1 / -1) of each internal function (2..P), or None
    if some internal function has none (the reference's ``internal_parity``;
    None for the nodal basis, whose orientation is an index reversal)."""
    if basis.kind.is_nodal or basis.P < 2:
        return None
    x = np.linspace(0.1, 0.9, 7)
    v, _ = basis.eval(np.concatenate([x, -x]))
    v = np.asarray(v)
    if v.shape[0] != basis.n:
        v = v.T
    par = []
    for t in range(2, basis.P + 1):
        a, b = v[t, :7], v[t, 7:]
        s = np.abs(a).max()
        if np.abs(a - b).max() <= 1e-10 * s:
            par.append(1.0)
        elif np.abs(a + b).max() <= 1e-10 * s:
            par.append(-1.0)
        else:
            return None
    return np.array(par)


@dataclass
class MeshDofMap:
    """``DofMap`` (``meshdof.py:316-370``) for one mesh and order P."""

    P: int
    gdof: np.ndarray       # (ne, n^3) reference local order (p, q, r), r fastest
    gsign: np.ndarray
    n_modes: int
    free_map: np.ndarray   # (n_modes * 3,) -> free index or -1
    n_free: int


def _oriented(m, flipped, P, nodal, parity):
    """``_oriented_1d`` vectorised over elements: (index, sign)."""
    if nodal:
        return np.where(flipped, P + 2 - m, m), np.ones(flipped.shape)
    if parity is None:
        if np.any(flipped):
            raise MeshError("edge/face reversal needs definite-parity internal modes; "
                            "use symmetric Jacobi weights (alpha == beta) on multi-element meshes")
        return np.full(flipped.shape, m), np.ones(flipped.shape)
    return np.full(flipped.shape, m), np.where(flipped, parity[m - 2], 1.0)


def build_mesh_dofmap(mesh: HexMesh, basis: Basis1D, dirichlet=None) -> MeshDofMap:
    """``build_dofmap`` (``meshdof.py:404-472``) plus ``apply_dirichlet``."""
    P, n = basis.P, basis.P + 1
    nep = P - 1
    ne = mesh.n_elems
    edge_off = mesh.n_vertices
    face_off = edge_off + mesh.n_edges * nep
    interior_off = face_off + mesh.n_faces * nep * nep
    n_modes = interior_off + ne * nep ** 3
    nodal = basis.kind.is_nodal
    parity = _internal_parity(basis)
    conn = mesh.elems
    gdof = np.empty((ne, n ** 3), dtype=np.int64)
    gsign = np.ones((ne, n ** 3))
    edge_lookup = {}
    for le, (axis, lo, _) in enumerate(EDGE_TABLE):
        fixed = tuple(VERTEX_BITS[lo][d] for d in range(3) if d != axis)
        edge_lookup[(axis, fixed)] = le
    face_lookup = {(f[0], f[1]): i for i, f in enumerate(FACE_TABLE)}
    eidx = np.arange(ne)
    for i, idx in enumerate(np.ndindex(n, n, n)):
        internal = tuple(d for d in range(3) if idx[d] >= 2)
        if len(internal) == 0:
            gdof[:, i] = conn[:, VERTEX_BITS.index(tuple(idx))]
        elif len(internal) == 1:
            axis = internal[0]
            le = edge_lookup[(axis, tuple(int(idx[d]) for d in range(3) if d != axis))]
            ge = mesh.elem_edges[:, le]
            flipped = conn[:, EDGE_TABLE[le][1]] != mesh.edge_verts[ge, 0]
            mc, s = _oriented(int(idx[axis]), flipped, P, nodal, parity)
            gdof[:, i] = edge_off + ge * nep + (mc - 2)
            gsign[:, i] = s
        elif len(internal) == 2:
            axis = next(d for d in range(3) if idx[d] < 2)
            lf = face_lookup[(axis, int(idx[axis]))]
            m1, m2 = (int(idx[d]) for d in internal)
            gf = mesh.elem_faces[:, lf]
            corners = FACE_TABLE[lf][4]
            cb = list(corners)  # (ba, bb) keys
            gv = np.stack([conn[:, corners[bb]] for bb in cb], axis=1)  # (ne, 4)
            kmin = np.argmin(gv, axis=1)
            a0 = np.array([cb[k][0] for k in range(4)])[kmin]
            b0 = np.array([cb[k][1] for k in range(4)])[kmin]
            pos = {bb: k for k, bb in enumerate(cb)}
            ka = np.array([[pos[(1 - a, b)] for a, b in cb][k] for k in range(4)])[kmin]
            kb = np.array([[pos[(a, 1 - b)] for a, b in cb][k] for k in range(4)])[kmin]
            ga, gb = gv[eidx, ka], gv[eidx, kb]
            swap = ga > gb
            ma, sa = _oriented(m1, a0 == 1, P, nodal, parity)
            mb, sb = _oriented(m2, b0 == 1, P, nodal, parity)
            ms = np.where(swap, mb, ma)
            mt = np.where(swap, ma, mb)
            gdof[:, i] = face_off + gf * nep * nep + (ms - 2) * nep + (mt - 2)
            gsign[:, i] = sa * sb
        else:
            lex = ((idx[0] - 2) * nep + (idx[1] - 2)) * nep + (idx[2] - 2)
            gdof[:, i] = interior_off + eidx * nep ** 3 + lex
    # positive mapping Jacobian at the element centres (meshdof.py:468-469)
    _, det = _jacobians(mesh, np.zeros((1, 3)))
    bad = np.nonzero(det[:, 0] <= 0.0)[0]
    if len(bad):
        raise MeshError(f"element {int(bad[0])}: non-positive mapping Jacobian")
    cons = np.zeros((n_modes, 3), dtype=bool)
    for tag, comps in dirichlet or []:
        modes = boundary_modes(mesh, P, tag)
        for c in comps:
            cons[modes, c] = True
    mask = ~cons.reshape(-1)
    free_map = np.where(mask, np.cumsum(mask) - 1, -1)
    return MeshDofMap(P, gdof, gsign, n_modes, free_map, int(mask.sum()))


def boundary_modes(mesh: HexMesh, P: int, tag: str) -> np.ndarray:
    """``boundary_modes`` (``meshdof.py:475-503``)."""
    if tag not in mesh.boundary_sides:
        raise MeshError(f"unknown boundary tag {tag!r}")
    nep = P - 1
    edge_off = mesh.n_vertices
    face_off = edge_off + mesh.n_edges * nep
    modes = set()
    for e, lf in mesh.boundary_sides[tag]:
        conn = mesh.elems[e]
        corners = FACE_TABLE[lf][4]
        vids = [corners[bb] for bb in _QUAD]
        modes.update(int(conn[v]) for v in vids)
        for le, (_, lo, hi) in enumerate(EDGE_TABLE):
            if {lo, hi} <= set(vids):
                ge = int(mesh.elem_edges[e, le])
                modes.update(edge_off + ge * nep + j for j in range(nep))
        gf = int(mesh.elem_faces[e, lf])
        modes.update(face_off + gf * nep * nep + j for j in range(nep * nep))
    return np.array(sorted(modes), dtype=np.int64)


def _jacobians(mesh: HexMesh, xi: np.ndarray):
    """J[e, q, c, d] = dX_c / dxi_d of the trilinear map and det J (``meshdof.py:269-296``)."""
    xi = np.atleast_2d(xi)
    bits = np.array(VERTEX_BITS, dtype=float)  # (8, 3)
    f = np.where(bits[None, :, :] > 0, 0.5 * (1 + xi[:, None, :]), 0.5 * (1 - xi[:, None, :]))  # (q, 8, 3)
    df = np.where(bits > 0, 0.5, -0.5)  # (8, 3)
    dg = np.empty(f.shape)  # (q, 8, d)
    for d in range(3):
        dg[:, :, d] = df[None, :, d] * np.prod(np.delete(f, d, axis=2), axis=2)
    xc = mesh.coords[mesh.elems]  # (ne, 8, 3)
    jac = np.einsum("qvd,evc->eqcd", dg, xc)
    return jac, np.linalg.det(jac)


def element_tables(mesh: HexMesh, rule: Rule) -> np.ndarray:
    """Per element and kernel point q = (c m + b) m + a (a along xi_x):
    J^-1[d, c] in slots d*3 + c and w_a w_b w_c det J in slot 9 -> (ne, 10, m^3).
    Raises MeshError on a non-positive Jacobian (``build_tables``, femcore.py:73-81)."""
    x, w = rule.points, rule.weights
    m = len(x)
    C, B, A = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    xi = np.stack([x[A.reshape(-1)], x[B.reshape(-1)], x[C.reshape(-1)]], axis=1)
    wq = w[A.reshape(-1)] * w[B.reshape(-1)] * w[C.reshape(-1)]
    jac, det = _jacobians(mesh, xi)
    bad = np.argwhere(det <= 0.0)
    if len(bad):
        raise MeshError(f"element {int(bad[0, 0])}: non-positive mapping Jacobian")
    jinv = np.linalg.inv(jac)  # (ne, q, d, c)
    out = np.empty((mesh.n_elems, 10, m ** 3))
    out[:, :9, :] = jinv.reshape(mesh.n_elems, m ** 3, 9).transpose(0, 2, 1)
    out[:, 9, :] = wq[None, :] * det
    return out


def kernel_tables(dm: MeshDofMap):
    """Device index tables from a dof map.

    * ``dof`` (ne, 3, n, n, n) int32 in kernel order [e][comp][z][y][x] (lattice-local
      1D offsets): 2 * free index + (sign < 0), or -1 on a constrained DOF;
    * the assembly CSR over free DOFs: ``ptr`` (n_free + 1) int64 and ``slot``
      int32 entries 2 * s + (sign < 0), s = flat index into the element-vector
      buffer, in increasing element order (the reference's ``np.add.at`` order).
    """
    P, n = dm.P, dm.P + 1
    ne = dm.gdof.shape[0]
    t = np.array([0] + list(range(2, P + 1)) + [1])  # lattice offset -> reference 1D index
    tz, ty, tx = np.meshgrid(t, t, t, indexing="ij")
    ref = ((tx * n + ty) * n + tz).reshape(-1)  # kernel point (z, y, x) -> reference local index
    g = dm.gdof[:, ref]  # (ne, n^3)
    s = dm.gsign[:, ref]
    free = dm.free_map[g[:, None, :] * 3 + np.arange(3)[None, :, None]]  # (ne, 3, n^3)
    neg = np.broadcast_to((s < 0)[:, None, :], free.shape)
    dof = np.where(free >= 0, 2 * free + neg, -1).astype(np.int32)
    flat = free.reshape(-1)
    sel = np.nonzero(flat >= 0)[0]
    order = np.argsort(flat[sel], kind="stable")
    slots = sel[order]
    ptr = np.zeros(dm.n_free + 1, dtype=np.int64)
    np.cumsum(np.bincount(flat[sel], minlength=dm.n_free), out=ptr[1:])
    slot = (2 * slots + neg.reshape(-1)[slots]).astype(np.int64)
    if slot.size and slot.max() >= 2 ** 31:
        raise MeshError("mesh too large for 32-bit element-vector slots")
    return dof.reshape(ne, 3, n, n, n), ptr, slot.astype(np.int32)


def locality_order(mesh: HexMesh, dm: MeshDofMap, ptr: np.ndarray, slot: np.ndarray, n_box: int):
    """Storage order of the element boxes and of the assembly rows for memory
    locality (pure data placement: the per-DOF summation order, i.e. the
    reference's element order, is unchanged, so results are bit-identical).

    Elements are stored along a Morton (Z-order) curve of their centroids, so
    the boxes a DOF gathers from lie close together; the assembly CSR rows are
    visited in the order of their first stored element.  Returns (perm, rows,
    ptr2, slot2): storage position -> element id, CSR row -> free DOF, and the
    CSR re-laid in that row order with slots pointing into the permuted boxes
    (``n_box`` = doubles per element box)."""
    cent = mesh.coords[mesh.elems].mean(axis=1)
    lo, hi = cent.min(axis=0), cent.max(axis=0)
    q = np.floor((cent - lo) / np.maximum(hi - lo, 1e-300) * 1023.0).astype(np.int64)

    def spread(v):  # 10 bits -> every third bit
        v = (v | (v << 16)) & 0x030000FF
        v = (v | (v << 8)) & 0x0300F00F
        v = (v | (v << 4)) & 0x030C30C3
        return (v | (v << 2)) & 0x09249249

    code = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
    perm = np.argsort(code, kind="stable")
    pos = np.empty_like(perm)
    pos[perm] = np.arange(len(perm))
    s = slot.astype(np.int64)
    flat = s >> 1
    e, j = flat // n_box, flat % n_box
    s2 = ((pos[e] * n_box + j) << 1) | (s & 1)
    n_free = len(ptr) - 1
    counts = np.diff(ptr)
    first = np.full(n_free, np.iinfo(np.int64).max)
    row_of = np.repeat(np.arange(n_free), counts)
    np.minimum.at(first, row_of, pos[e])
    rows = np.argsort(first, kind="stable")
    ptr2 = np.zeros(n_free + 1, dtype=np.int64)
    np.cumsum(counts[rows], out=ptr2[1:])
    lens = counts[rows]
    take = np.repeat(ptr[rows] - ptr2[:-1], lens) + np.arange(ptr2[-1])
    return perm.astype(np.int32), rows.astype(np.int32), ptr2, s2[take].astype(np.int32)
