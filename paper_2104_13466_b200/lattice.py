"""Structured box meshes and the lattice numbering the GPU works in.

On an axis-aligned ``gen_box_mesh`` (``sdmefem/meshdof.py:146-193``) every
orientation sign of the reference DOF map is +1 and its global modes are in
bijection with a lexicographic lattice of (P*nx+1) x (P*ny+1) x (P*nz+1)
points: element (i, j, k), local tensor index t along an axis, sits at lattice
coordinate ``P*i + off(t)`` with off(0)=0, off(1)=P, off(t>=2)=t-1
(SURVEY §0 finding 6).  The device keeps every vector in that lattice, one
plane of ``Lx*Ly*Lz`` doubles per displacement component (component-major SoA),
with Dirichlet points held at zero.

The only place the reference numbering matters is the drop-in boundary, where
vectors arrive in the reference's *free-DOF* order.  :func:`reference_free_index`
reproduces ``build_dofmap`` (``meshdof.py:404-472``) for box meshes in closed,
vectorised form: vertices by vertex id, then edges and faces numbered by first
appearance in the (element, local entity) loop of ``Mesh._build_edges`` /
``_build_faces`` (``meshdof.py:76-98``), then element interiors, and finally the
Dirichlet compaction of ``DofMap.apply_dirichlet`` (``meshdof.py:364-370``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["BoxMesh", "FACE_TAGS", "dirichlet_face_masks", "reference_free_index",
           "VERTEX_BITS", "LOCAL_EDGES", "LOCAL_FACES"]

FACE_TAGS = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")

# VTK hexahedron corner order as per-axis bits (tensorelem.py:19-24).
VERTEX_BITS = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
               (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))
_VTK_EDGE_PAIRS = ((0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4),
                   (0, 4), (1, 5), (2, 6), (3, 7))


def _local_edges():
    """(axis, bits of the low-end corner) per local edge, reference order."""
    out = []
    for va, vb in _VTK_EDGE_PAIRS:
        ba, bb = VERTEX_BITS[va], VERTEX_BITS[vb]
        axis = next(d for d in range(3) if ba[d] != bb[d])
        lo = ba if ba[axis] == 0 else bb
        out.append((axis, lo))
    return tuple(out)


LOCAL_EDGES = _local_edges()
# Local face id = 2*axis + side (tensorelem.py:53-70); low corner bits.
LOCAL_FACES = tuple((axis, side) for axis in range(3) for side in (0, 1))


@dataclass(frozen=True)
class BoxMesh:
    """Axis-aligned structured hexahedral mesh of ``divisions`` cells."""

    divisions: tuple
    lengths: tuple
    origin: tuple = (0.0, 0.0, 0.0)
    h: tuple = field(init=False)

    def __post_init__(self):
        div = tuple(int(v) for v in self.divisions)
        if len(div) != 3 or min(div) < 1:
            raise ValueError("need at least one cell per axis")
        object.__setattr__(self, "divisions", div)
        object.__setattr__(self, "lengths", tuple(float(v) for v in self.lengths))
        object.__setattr__(self, "origin", tuple(float(v) for v in self.origin))
        object.__setattr__(self, "h", tuple(l / n for l, n in zip(self.lengths, div)))

    @property
    def n_elems(self) -> int:
        nx, ny, nz = self.divisions
        return nx * ny * nz

    def lattice_shape(self, P: int) -> tuple[int, int, int]:
        """(Lx, Ly, Lz) lattice points per axis at order P."""
        return tuple(P * n + 1 for n in self.divisions)

    def n_lattice(self, P: int) -> int:
        lx, ly, lz = self.lattice_shape(P)
        return lx * ly * lz

    def min_edge_length(self) -> float:
        return float(min(self.h))

    def lattice_coords(self, P: int, xi_nodes: np.ndarray | None = None) -> list[np.ndarray]:
        """1D physical coordinates of the lattice lines per axis.

        ``xi_nodes`` (length P+1, function order) places internal lattice
        lines at given reference coordinates (GLL nodes for the nodal basis);
        default puts them equally spaced.
        """
        out = []
        for ax in range(3):
            n, h, o = self.divisions[ax], self.h[ax], self.origin[ax]
            if xi_nodes is None:
                loc = np.linspace(-1.0, 1.0, P + 1)
            else:
                xn = np.asarray(xi_nodes, dtype=float)
                loc = np.concatenate(([xn[0]], xn[2:], [xn[1]]))
            pts = [o + i * h + 0.5 * (loc[:-1] + 1.0) * h for i in range(n)]
            out.append(np.concatenate(pts + [np.array([o + n * h])]))
        return out


def dirichlet_face_masks(dirichlet) -> np.ndarray:
    """Per-component 6-bit masks of clamped faces (bit f = FACE_TAGS[f])."""
    masks = np.zeros(3, dtype=np.int32)
    for tag, comps in dirichlet or ():
        if tag not in FACE_TAGS:
            raise ValueError(f"unknown boundary tag {tag!r}")
        for c in comps:
            if c < 3:
                masks[c] |= 1 << FACE_TAGS.index(tag)
    return masks


def constrained_lattice(mesh: BoxMesh, P: int, masks: np.ndarray) -> np.ndarray:
    """Bool (3, Lz, Ly, Lx): lattice points held by a Dirichlet plane."""
    lx, ly, lz = mesh.lattice_shape(P)
    out = np.zeros((3, lz, ly, lx), dtype=bool)
    for c in range(3):
        m = int(masks[c])
        if m & 1:
            out[c, :, :, 0] = True
        if m & 2:
            out[c, :, :, -1] = True
        if m & 4:
            out[c, :, 0, :] = True
        if m & 8:
            out[c, :, -1, :] = True
        if m & 16:
            out[c, 0, :, :] = True
        if m & 32:
            out[c, -1, :, :] = True
    return out


def _first_appearance_ids(keys: np.ndarray, n_keys: int) -> np.ndarray:
    """id[key] = rank of the key's first position in ``keys`` (loop order)."""
    uniq, first = np.unique(keys, return_index=True)
    order = np.argsort(first, kind="stable")
    ids = np.full(n_keys, -1, dtype=np.int64)
    ids[uniq[order]] = np.arange(uniq.size, dtype=np.int64)
    return ids


def reference_mode_ids(mesh: BoxMesh, P: int) -> np.ndarray:
    """Reference global scalar-mode id of every lattice point, (Lz, Ly, Lx).

    Vertices: ``vid = (k(ny+1)+j)(nx+1)+i`` (``meshdof.py:163-164``).
    Edges/faces: first appearance over elements (x fastest) and local
    edges/faces in table order; mode offsets per ``meshdof.py:413-421``.
    Interior: ``interior_off + e*nep^3 + lex(t-2)``.
    """
    nx, ny, nz = mesh.divisions
    nep = P - 1
    vx, vy, vz = nx + 1, ny + 1, nz + 1
    nv = vx * vy * vz

    ei, ej, ek = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    # element loop order: e = (k*ny + j)*nx + i  -> flatten with i fastest
    ei = ei.transpose(2, 1, 0).ravel()
    ej = ej.transpose(2, 1, 0).ravel()
    ek = ek.transpose(2, 1, 0).ravel()

    def vid(i, j, k):
        return (k * vy + j) * vx + i

    edge_keys = np.empty((ei.size, 12), dtype=np.int64)
    for le, (axis, lo) in enumerate(LOCAL_EDGES):
        edge_keys[:, le] = axis * nv + vid(ei + lo[0], ej + lo[1], ek + lo[2])
    edge_id = _first_appearance_ids(edge_keys.ravel(), 3 * nv)
    n_edges = int((edge_id >= 0).sum())

    face_keys = np.empty((ei.size, 6), dtype=np.int64)
    for lf, (axis, side) in enumerate(LOCAL_FACES):
        b = [0, 0, 0]
        b[axis] = side
        face_keys[:, lf] = axis * nv + vid(ei + b[0], ej + b[1], ek + b[2])
    face_id = _first_appearance_ids(face_keys.ravel(), 3 * nv)
    n_faces = int((face_id >= 0).sum())

    edge_off = nv
    face_off = edge_off + n_edges * nep
    int_off = face_off + n_faces * nep * nep

    lx, ly, lz = mesh.lattice_shape(P)
    X, Y, Z = np.meshgrid(np.arange(lx), np.arange(ly), np.arange(lz), indexing="ij")
    X, Y, Z = X.transpose(2, 1, 0), Y.transpose(2, 1, 0), Z.transpose(2, 1, 0)
    coords = (X, Y, Z)
    # per axis: vertex-type (on an element boundary plane) or internal index t
    vert = [c % P == 0 for c in coords]
    cell = [np.where(v, c // P, c // P) for v, c in zip(vert, coords)]
    tloc = [c % P + 1 for c in coords]  # t in 2..P for internal points
    nvert = vert[0].astype(int) + vert[1] + vert[2]
    out = np.full(X.shape, -1, dtype=np.int64)

    # vertices
    sel = nvert == 3
    out[sel] = vid(X[sel] // P, Y[sel] // P, Z[sel] // P)
    # edges: exactly one internal axis
    for axis in range(3):
        sel = (nvert == 2) & ~vert[axis]
        lo = [coords[d][sel] // P for d in range(3)]
        key = axis * nv + vid(lo[0], lo[1], lo[2])
        out[sel] = edge_off + edge_id[key] * nep + (tloc[axis][sel] - 2)
    # faces: exactly one vertex-type axis (the face normal)
    for axis in range(3):
        sel = (nvert == 1) & vert[axis]
        lo = [coords[d][sel] // P for d in range(3)]
        key = axis * nv + vid(lo[0], lo[1], lo[2])
        d1, d2 = [d for d in range(3) if d != axis]
        out[sel] = (face_off + face_id[key] * nep * nep
                    + (tloc[d1][sel] - 2) * nep + (tloc[d2][sel] - 2))
    # element interiors
    sel = nvert == 0
    e = (cell[2][sel] * ny + cell[1][sel]) * nx + cell[0][sel]
    lex = ((tloc[0][sel] - 2) * nep + (tloc[1][sel] - 2)) * nep + (tloc[2][sel] - 2)
    out[sel] = int_off + e * nep ** 3 + lex
    return out


def reference_free_index(mesh: BoxMesh, P: int, dirichlet) -> tuple[np.ndarray, int]:
    """(perm, n_free): perm[c, z, y, x] = index of that lattice DOF in the
    reference free vector, or -1 when Dirichlet-constrained."""
    modes = reference_mode_ids(mesh, P)
    n_modes = mesh.n_lattice(P)
    cons = constrained_lattice(mesh, P, dirichlet_face_masks(dirichlet))
    # reference free numbering: cumsum over vector dofs d = mode*3 + comp
    dir_flags = np.zeros((n_modes, 3), dtype=bool)
    for c in range(3):
        dir_flags[modes.ravel(), c] = cons[c].ravel()
    free = ~dir_flags.reshape(-1)
    fmap = np.where(free, np.cumsum(free) - 1, -1)
    perm = np.empty((3,) + modes.shape, dtype=np.int64)
    for c in range(3):
        perm[c] = fmap[modes * 3 + c]
    return perm, int(free.sum())
