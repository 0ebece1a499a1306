"""General hexahedral meshes, host side: the product's mesh tables
and DOF numbering (paper_2104_13466_b200/mesh.py) against the reference's
``build_dofmap`` output on twisted, renumbered and perturbed meshes
(tests/golden/meshes.npz, made by the real reference), mesh file round trip,
and error behaviour."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden
from paper_2104_13466_b200 import build_basis
from paper_2104_13466_b200.basis import BasisKind
from paper_2104_13466_b200.lattice import BoxMesh, reference_free_index
from paper_2104_13466_b200.mesh import (HexMesh, MeshError, build_mesh_dofmap, kernel_tables, read_mesh,
                                        write_mesh)

KINDS = ("LagrangeGLL", "ModalJacobi", "SDME_M", "SDME_K", "SDME_H")
TAGS = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")


def golden_mesh_cases():
    g = load_golden("meshes")
    n = len({k.split("_")[0] for k in g.files})
    return [(g, f"m{i}") for i in range(n)]


def mesh_from(g, key):
    boundary = {str(t): [tuple(q) for q in g[f"{key}_b_{t}"]] for t in g[f"{key}_btags"]}
    return HexMesh(g[f"{key}_coords"], g[f"{key}_elems"], boundary)


def case_setup(g, key):
    kind, P = (int(v) for v in g[f"{key}_meta"])
    dr = {}
    for t, c in g[f"{key}_dir"]:
        dr.setdefault(TAGS[int(t)], []).append(int(c))
    return mesh_from(g, key), build_basis(P, BasisKind(KINDS[kind])), [(t, tuple(c)) for t, c in dr.items()]


@pytest.mark.parametrize("case", golden_mesh_cases(), ids=lambda c: c[1])
def test_dofmap_matches_reference(case):
    g, key = case
    mesh, basis, dr = case_setup(g, key)
    dm = build_mesh_dofmap(mesh, basis, dr)
    assert np.array_equal(dm.gdof, g[f"{key}_gdof"])
    assert np.array_equal(dm.gsign, g[f"{key}_gsign"])
    assert np.array_equal(dm.free_map, g[f"{key}_free_map"])
    assert dm.n_free == len(g[f"{key}_u"])


@pytest.mark.parametrize("case", golden_mesh_cases(), ids=lambda c: c[1])
def test_kernel_tables_are_consistent(case):
    """Every free DOF's CSR entries point back at element slots whose gather
    entry names that DOF with the same sign, in increasing element order."""
    g, key = case
    mesh, basis, dr = case_setup(g, key)
    dm = build_mesh_dofmap(mesh, basis, dr)
    dof, ptr, slot = kernel_tables(dm)
    flat = dof.reshape(-1)
    assert ptr[-1] == np.count_nonzero(flat >= 0)
    for f in range(0, dm.n_free, max(1, dm.n_free // 200)):
        ent = slot[ptr[f]:ptr[f + 1]]
        s = ent >> 1
        assert np.all(np.diff(s) > 0)
        assert np.all(flat[s] >> 1 == f)
        assert np.array_equal(flat[s] & 1, ent & 1)


def test_box_mesh_numbering_matches_lattice_permutation():
    """On an axis-aligned box the general numbering agrees with the closed-form
    lattice permutation used by the box path (lattice.py)."""
    for P in (2, 3, 4):
        box = BoxMesh((3, 2, 2), (1.5, 1.0, 1.0))
        dr = [("xmin", (0, 1, 2)), ("zmax", (2,))]
        perm, n_free = reference_free_index(box, P, dr)
        dm = build_mesh_dofmap(HexMesh.box((3, 2, 2), (1.5, 1.0, 1.0)), build_basis(P, BasisKind("SDME_M")), dr)
        assert dm.n_free == n_free
        assert np.all(dm.gsign == 1.0)
        dof, _, _ = kernel_tables(dm)
        # element (i, j, k) box in lattice order -> the same free ids as the lattice permutation
        Lx, Ly, Lz = (P * d + 1 for d in (3, 2, 2))
        pr = perm.reshape(3, Lz, Ly, Lx)
        for e, (i, j, k) in enumerate([(i, j, k) for k in range(2) for j in range(2) for i in range(3)]):
            box_ids = pr[:, P * k:P * k + P + 1, P * j:P * j + P + 1, P * i:P * i + P + 1]
            got = np.where(dof[e] >= 0, dof[e] >> 1, -1)
            assert np.array_equal(got, box_ids)


def test_mesh_file_round_trip(tmp_path):
    g = load_golden("meshes")
    mesh = mesh_from(g, "m3")
    path = tmp_path / "m.mesh"
    write_mesh(mesh, path)
    back = read_mesh(path)
    assert np.array_equal(back.coords, mesh.coords) and np.array_equal(back.elems, mesh.elems)
    assert back.boundary_sides == mesh.boundary_sides


def test_mesh_errors():
    box = HexMesh.box((1, 1, 1), (1.0, 1.0, 1.0))
    with pytest.raises(MeshError):
        HexMesh(box.coords, box.elems, {"bad": [(0, 1, 6, 7)]})  # not a face
    inverted = box.elems.copy()
    inverted[0] = inverted[0][[4, 5, 6, 7, 0, 1, 2, 3]]  # mirrored: det J < 0
    with pytest.raises(MeshError):
        build_mesh_dofmap(HexMesh(box.coords, inverted), build_basis(2, BasisKind("SDME_M")))
    two = HexMesh.box((2, 1, 1), (2.0, 1.0, 1.0))
    with pytest.raises(MeshError):
        HexMesh(two.coords, two.elems, {"mid": [(1, 4, 10, 7)]})  # interior face


# --- the oracle's general-mesh restatement (oracle/mesh.py), pinned to the
# same reference golden vectors

def oracle_case(g, key):
    from oracle import basis as ob
    from oracle import fem as of
    from oracle.mesh import GeneralMesh, GeneralProblem
    kind, P = (int(v) for v in g[f"{key}_meta"])
    dr = {}
    for t, c in g[f"{key}_dir"]:
        dr.setdefault(TAGS[int(t)], []).append(int(c))
    boundary = {str(t): [tuple(q) for q in g[f"{key}_b_{t}"]] for t in g[f"{key}_btags"]}
    mesh = GeneralMesh(g[f"{key}_coords"], g[f"{key}_elems"], boundary)
    return GeneralProblem(mesh, ob.Basis(KINDS[kind], P), of.Material(1.0e7, 0.3, 1.0e3), P + 1,
                          [(t, tuple(c)) for t, c in dr.items()])


@pytest.mark.parametrize("case", [c for c in golden_mesh_cases() if c[1] != "m6"], ids=lambda c: c[1])
def test_oracle_general_mesh_vs_reference(case):
    from conftest import max_rel_err
    g, key = case
    opb = oracle_case(g, key)
    assert np.array_equal(opb.dmap.gdof, g[f"{key}_gdof"])
    assert np.array_equal(opb.dmap.gsign, g[f"{key}_gsign"])
    assert np.array_equal(opb.dmap.free_map, g[f"{key}_free_map"])
    u, p, cm = g[f"{key}_u"], g[f"{key}_p"], float(g[f"{key}_cm"])
    assert max_rel_err(opb.internal_force(u), g[f"{key}_fint"]) <= 1e-12
    assert max_rel_err(opb.apply_tangent(u, p), g[f"{key}_kp"]) <= 1e-12
    assert max_rel_err(opb.assemble(u, 1.0, cm).diagonal(), g[f"{key}_diag"]) <= 1e-12
    assert max_rel_err(opb.mass() @ p, g[f"{key}_mp"]) <= 1e-12


def test_free_dofs_match_reference_table():
    """test_meshdof.py:88-92: the 8-hex cube clamped on xmin has 300 / 1944 /
    6084 / 13872 free DOFs at P = 2 / 4 / 6 / 8 (box path and general path)."""
    for P, expect in ((2, 300), (4, 1944), (6, 6084), (8, 13872)):
        _, n_free = reference_free_index(BoxMesh((2, 2, 2), (1.0, 1.0, 1.0)), P, [("xmin", (0, 1, 2))])
        assert n_free == expect
        dm = build_mesh_dofmap(HexMesh.box((2, 2, 2), (1.0, 1.0, 1.0)), build_basis(P, BasisKind("SDME_M")),
                               [("xmin", (0, 1, 2))])
        assert dm.n_free == expect


def test_all_dirichlet_empty_system():
    """test_femcore.py:248-253: every face of a single P = 1 hexahedron
    clamped leaves no free DOF (box numbering and general numbering)."""
    tags = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")
    dr = [(t, (0, 1, 2)) for t in tags]
    _, n_free = reference_free_index(BoxMesh((1, 1, 1), (1.0, 1.0, 1.0)), 1, dr)
    assert n_free == 0
    dm = build_mesh_dofmap(HexMesh.box((1, 1, 1), (1.0, 1.0, 1.0)), build_basis(1, BasisKind("ModalJacobi")), dr)
    assert dm.n_free == 0
