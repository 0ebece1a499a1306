"""Drop-in adapter: GPU problems built from the reference's own objects.

``from_reference(problem)`` takes a reference ``sdmefem.femcore.FemProblem``
(``femcore.py:273-295``: mesh, TensorElement, DofMap, NeoHookean, rule) and
returns the GPU problem that replaces it on the hot path:

* the device's 1D tables B, D and the weights w are the reference basis
  tabulated at the reference rule, ``element.basis.with_rule(problem.rule)``
  (``basis1d.py:123-126``), not rebuilt;
* the vector numbering is the reference's: on a ``gen_box_mesh`` mesh the
  lattice -> free-index permutation is read off ``dmap.gdof`` (element box
  placement) and ``dmap.free_map`` (``meshdof.py:345-370``); on any other
  hexahedral mesh the general-mesh context is used and its oriented DOF map is
  checked entry for entry against ``gdof`` / ``gsign`` / ``free_map``;
* Dirichlet constraints are read from ``dmap.dirichlet`` and must be whole
  boundary faces per component (what ``build_dofmap`` produces,
  ``meshdof.py:404-409, 475-503``).

Nothing here imports the reference: the argument is duck-typed on the
reference's attribute names, so the adapter works wherever the caller's
objects come from.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .basis import BasisKind, Rule, build_basis
from .lattice import FACE_TAGS, BoxMesh, constrained_lattice, dirichlet_face_masks
from .problem import GpuFemProblem, NeoHookean

__all__ = ["from_reference", "reference_descriptor", "reference_tables", "box_layout", "BoxDescriptor"]


def reference_tables(problem):
    """(B, D, w, rule) of a reference FemProblem: B[a, t] = phi_t(x_a),
    D[a, t] = phi_t'(x_a) at the problem's rule (m x n, reference function
    order), w the rule weights."""
    rb = problem.element.basis.with_rule(problem.rule)
    B = np.ascontiguousarray(np.asarray(rb.values, dtype=float).T)
    D = np.ascontiguousarray(np.asarray(rb.derivs, dtype=float).T)
    w = np.ascontiguousarray(np.asarray(problem.rule.weights, dtype=float))
    kind = str(getattr(problem.rule, "kind", "GaussLegendre"))
    return B, D, w, Rule(kind, np.asarray(problem.rule.points, dtype=float), w)


def _kind_of(basis) -> BasisKind:
    k = basis.kind
    return BasisKind(k.tag, float(k.jacobi_alpha), float(k.jacobi_beta), float(k.k), float(k.lam))


def box_layout(mesh, rtol: float = 1e-12):
    """BoxMesh if ``mesh`` is a ``gen_box_mesh`` mesh (``meshdof.py:146-193``:
    uniform axis-aligned grid, vertex id (k(ny+1)+j)(nx+1)+i, elements
    x-fastest in VTK corner order), else None."""
    coords = np.asarray(mesh.coords, dtype=float)
    elems = np.asarray(mesh.elems)
    if coords.ndim != 2 or coords.shape[1] != 3 or elems.shape[1:] != (8,):
        return None
    lines = [np.unique(coords[:, a]) for a in range(3)]
    div = tuple(len(x) - 1 for x in lines)
    if min(div) < 1 or (div[0] + 1) * (div[1] + 1) * (div[2] + 1) != len(coords) or len(elems) != np.prod(div):
        return None
    origin = tuple(float(x[0]) for x in lines)
    lengths = tuple(float(x[-1] - x[0]) for x in lines)
    box = BoxMesh(div, lengths, origin)
    nx, ny, nz = div
    i, j, k = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    vid = ((k * (ny + 1) + j) * (nx + 1) + i)
    expect = np.zeros_like(coords)
    for a, (idx, x) in enumerate(zip((i, j, k), lines)):
        expect[vid.ravel(), a] = box.origin[a] + box.h[a] * idx.ravel()
    scale = max(1.0, float(np.abs(coords).max()))
    if np.abs(expect - coords).max() > rtol * 10 * scale:
        return None
    bits = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))
    ei, ej, ek = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ei, ej, ek = (a.transpose(2, 1, 0).ravel() for a in (ei, ej, ek))  # e = (k ny + j) nx + i
    conn = np.stack([((ek + b[2]) * (ny + 1) + ej + b[1]) * (nx + 1) + ei + b[0] for b in bits], axis=1)
    if not np.array_equal(conn, elems):
        return None
    return box


def _lattice_modes(box: BoxMesh, P: int, gdof: np.ndarray) -> np.ndarray:
    """Global scalar mode of every lattice point, read from the reference
    ``gdof`` (element e = (k ny + j) nx + i, local function (p, q, r) with r
    fastest, ``tensorelem.py:103``; local 1D index t sits at lattice offset
    0 (t = 0), P (t = 1), t - 1 (t >= 2))."""
    nx, ny, nz = box.divisions
    lx, ly, lz = box.lattice_shape(P)
    n = P + 1
    off = np.array([0, P] + list(range(1, P)))
    modes = np.full((lz, ly, lx), -1, dtype=np.int64)
    ei, ej, ek = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ei, ej, ek = (a.transpose(2, 1, 0).ravel() for a in (ei, ej, ek))
    p, q, r = np.meshgrid(off, off, off, indexing="ij")  # local (p, q, r), r fastest
    X = (P * ei)[:, None] + p.ravel()[None, :]
    Y = (P * ej)[:, None] + q.ravel()[None, :]
    Z = (P * ek)[:, None] + r.ravel()[None, :]
    g = np.asarray(gdof).reshape(len(ei), n ** 3)
    modes[Z, Y, X] = g
    if (modes < 0).any():
        raise ValueError("reference DOF map does not cover the lattice")
    # a conforming map gives every lattice point one mode, whichever element wrote it
    check = np.empty_like(g)
    check[:] = modes[Z, Y, X]
    if not np.array_equal(check, g):
        raise ValueError("reference DOF map is not conforming on the box lattice")
    return modes


def _face_dirichlet(modes: np.ndarray, dirichlet: np.ndarray):
    """(tag, comps) pairs equivalent to the reference's per-mode Dirichlet
    flags, or ValueError if they are not whole faces."""
    planes = {"xmin": (slice(None), slice(None), 0), "xmax": (slice(None), slice(None), -1),
              "ymin": (slice(None), 0, slice(None)), "ymax": (slice(None), -1, slice(None)),
              "zmin": (0, slice(None), slice(None)), "zmax": (-1, slice(None), slice(None))}
    flags = np.asarray(dirichlet, dtype=bool)
    out = []
    for tag in FACE_TAGS:
        comps = tuple(c for c in range(3) if flags[modes[planes[tag]].ravel(), c].all())
        if comps:
            out.append((tag, comps))
    return out


@dataclass
class BoxDescriptor:
    """Everything a :class:`GpuFemProblem` needs, read off a reference
    FemProblem on a ``gen_box_mesh`` mesh (no device context created)."""

    mesh: BoxMesh
    basis: object
    mat: NeoHookean
    rule: Rule
    dirichlet: list
    tables: tuple
    perm: np.ndarray  # (3, Lz, Ly, Lx) lattice -> reference free index, -1 constrained
    n_free: int


def reference_descriptor(problem):
    """BoxDescriptor of a reference FemProblem, or None if its mesh is not a
    ``gen_box_mesh`` box with canonical orientation (then the general-mesh
    context applies).  Raises ``ValueError`` for what the GPU path does not
    cover (2D meshes, non-face Dirichlet sets)."""
    mesh, el, dm = problem.mesh, problem.element, problem.dmap
    if getattr(mesh, "dim", 3) != 3:
        raise ValueError("the GPU path covers 3D hexahedral meshes")
    box = box_layout(mesh)
    if box is None or not np.all(np.asarray(dm.gsign) == 1):
        return None
    P = int(el.P)
    B, D, w, rule = reference_tables(problem)
    modes = _lattice_modes(box, P, dm.gdof)
    dirichlet = _face_dirichlet(modes, dm.dirichlet)
    cons = constrained_lattice(box, P, dirichlet_face_masks(dirichlet))
    flags = np.zeros((int(dm.n_modes), 3), dtype=bool)
    for c in range(3):
        flags[modes.ravel(), c] = cons[c].ravel()
    if not np.array_equal(flags, np.asarray(dm.dirichlet, dtype=bool)):
        raise ValueError("Dirichlet set is not a union of whole boundary faces")
    fmap = np.asarray(dm.free_map)
    perm = np.stack([fmap[modes * 3 + c] for c in range(3)])
    mat = NeoHookean(float(problem.mat.mu), float(problem.mat.lambda_lame), float(problem.mat.rho0))
    return BoxDescriptor(box, build_basis(P, _kind_of(el.basis)), mat, rule, dirichlet, (B, D, w), perm,
                         int(dm.n_free))


def from_reference(problem, reference_order: bool = True):
    """GPU problem for a reference ``FemProblem`` (see the module docstring).

    Box meshes give a :class:`GpuFemProblem` (lattice kernels, TMA element
    boxes); other hexahedral meshes a :class:`GpuMeshProblem`.  Raises
    ``ValueError`` for what the GPU path does not cover (2D meshes,
    non-face Dirichlet sets, general meshes with m != P + 1)."""
    d = reference_descriptor(problem)
    if d is not None:
        return GpuFemProblem(d.mesh, d.basis, d.mat, d.rule, d.dirichlet, reference_order=reference_order,
                             tables=d.tables, perm=d.perm if reference_order else None,
                             n_free=d.n_free if reference_order else None)
    from .mesh import HexMesh, boundary_modes
    from .mesh_problem import GpuMeshProblem

    mesh, el, dm = problem.mesh, problem.element, problem.dmap
    P = int(el.P)
    B, D, w, rule = reference_tables(problem)
    mat = NeoHookean(float(problem.mat.mu), float(problem.mat.lambda_lame), float(problem.mat.rho0))
    boundary = {t: [tuple(int(v) for v in q) for q in quads] for t, quads in mesh.boundary.items()}
    hm = HexMesh(np.asarray(mesh.coords, dtype=float), np.asarray(mesh.elems), boundary)
    flags = np.asarray(dm.dirichlet, dtype=bool)
    dirichlet = []
    for tag in sorted(boundary):
        on = boundary_modes(hm, P, tag) if len(boundary[tag]) else np.zeros(0, dtype=np.int64)
        comps = tuple(c for c in range(3) if on.size and flags[on, c].all())
        if comps:
            dirichlet.append((tag, comps))
    gp = GpuMeshProblem(hm, build_basis(P, _kind_of(el.basis)), mat, rule, dirichlet, tables=(B, D, w))
    ours = gp.dofmap
    if not (np.array_equal(ours.gdof, dm.gdof) and np.array_equal(ours.gsign, dm.gsign)
            and np.array_equal(ours.free_map, dm.free_map)):
        raise ValueError("general-mesh DOF map differs from the reference's (gdof / gsign / free_map)")
    return gp
