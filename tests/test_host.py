"""Host-side logic (no GPU): basis tables, lattice numbering, C-ABI symbols."""

from __future__ import annotations

import os
import re

import numpy as np
import pytest

from conftest import KINDS, ROOT, load_golden, max_rel_err
from oracle import fem as of
from paper_2104_13466_b200 import native
from paper_2104_13466_b200.basis import BasisKind, build_basis, constant_coeffs, gauss_rule
from paper_2104_13466_b200.lattice import BoxMesh, reference_free_index


def test_product_basis_matches_reference_golden():
    """Host 1D tables (the only CPU-side compute input) vs build_basis."""
    g = load_golden("basis")
    for key in g.files:
        if not key.endswith("_T"):
            continue
        tag, P = key.split("_P")[0], int(key.split("_P")[1].split("_")[0])
        b = build_basis(P, BasisKind(tag))
        if tag != "LagrangeGLL":
            assert np.abs(b.transform - g[key]).max() <= 1e-13
        for m in (P + 1, P + 2):
            B, D, w = b.tables(gauss_rule(m))
            assert max_rel_err(B, g[f"{tag}_P{P}_m{m}_B"]) <= 1e-13
            assert max_rel_err(D, g[f"{tag}_P{P}_m{m}_D"]) <= 1e-13


@pytest.mark.parametrize("tag", KINDS)
def test_constant_coefficients_reproduce_one(tag):
    b = build_basis(4, BasisKind(tag))
    x = np.linspace(-1, 1, 11)
    v, _ = b.eval(x)
    assert np.abs(constant_coeffs(b) @ v - 1.0).max() <= 1e-13


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("div,dr", [((1, 1, 1), None), ((2, 3, 2), [("xmin", (0, 1, 2))]),
                                    ((3, 2, 2), [("xmin", (0, 1, 2)), ("zmax", (2,))]),
                                    ((2, 2, 3), [("ymin", (1,)), ("xmax", (0,))])])
def test_lattice_permutation_matches_reference_numbering(P, div, dr):
    """Closed-form lattice <-> reference free-DOF map vs the oracle's
    restatement of build_dofmap (meshdof.py:404-472)."""
    perm, n_free = reference_free_index(BoxMesh(div, (1.0, 1.0, 1.0)), P, dr)
    dm = of.DofMap(of.Mesh(div, (1.0, 1.0, 1.0)), P, dr)
    assert n_free == dm.n_free
    nx, ny, nz = div
    off = lambda t: 0 if t == 0 else (P if t == 1 else t - 1)
    for e in range(nx * ny * nz):
        i, j, k = e % nx, (e // nx) % ny, e // (nx * ny)
        d = dm.evdofs(e).reshape(-1, 3)
        for f, (p, q, r) in enumerate(dm.index_map):
            X, Y, Z = P * i + off(p), P * j + off(q), P * k + off(r)
            assert tuple(perm[:, Z, Y, X]) == tuple(d[f])


def test_free_index_is_a_bijection():
    perm, n_free = reference_free_index(BoxMesh((4, 3, 5), (1, 1, 1)), 3, [("xmin", (0, 1, 2))])
    v = perm[perm >= 0]
    assert v.size == n_free and np.array_equal(np.sort(v), np.arange(n_free))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "sdme.h")).read()
    return sorted(set(re.findall(r"^int\s+(sdme_\w+)\s*\(", src, re.M)))


def test_abi_library_exports_every_header_symbol():
    """libsdme.so loads (no GPU needed) and exports every declared entry point."""
    lib = native.lib()
    names = _header_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(native.SIGNATURES), set(names) ^ set(native.SIGNATURES)


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_p3_swizzled_layout_is_conflict_free():
    """ColLay::SW (csrc/element_col.cuh, P = 3 with one element per half-warp):
    address 16 s + ((4 m + f) ^ 5 s) of a 4x4x4 array (s slowest).  It is a
    bijection, and every pencil access -- 16 lanes over a slice with one
    coordinate fixed -- is one wavefront in the half-warp 64-bit bank model
    (tools/bank_model.py); the natural layout 16 s + 4 m + f is not."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from bank_model import wavefronts

    def sw(s, m, f):
        return 16 * s + ((4 * m + f) ^ (5 * s))

    def natural(s, m, f):
        return 16 * s + 4 * m + f

    R = range(4)
    assert sorted(sw(s, m, f) for s in R for m in R for f in R) == list(range(64))
    # the point slots: qi applies q ^ 5 (q >> 4) to q = 16 s + 4 m + f
    assert all(sw(s, m, f) == (lambda q: q ^ (5 * (q >> 4)))(16 * s + 4 * m + f) for s in R for m in R for f in R)

    def worst(lay):
        w = 0
        for fixed in range(3):
            for v in R:
                addrs = []
                for x in R:
                    for y in R:
                        idx = [x, y]
                        idx.insert(fixed, v)
                        addrs.append(lay(*idx))
                w = max(w, wavefronts(addrs))
        return w

    assert worst(sw) == 1
    assert worst(natural) > 1
