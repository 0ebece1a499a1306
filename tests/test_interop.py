"""Drop-in adapter (host side, no GPU): descriptors built from the reference's
own FemProblem objects (``femcore.py:273-295``) agree with the GPU path's own
builders; reference SolverConfig objects are accepted; the solver rejects
what it does not implement; cfl_dt restates the reference's formula."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import KINDS, global_cases, import_reference
from paper_2104_13466_b200 import BoxMesh, SolverConfig, build_basis, cfl_dt, make_solver
from paper_2104_13466_b200.basis import BasisKind, gauss_rule
from paper_2104_13466_b200.interop import box_layout, reference_descriptor
from paper_2104_13466_b200.lattice import reference_free_index
from paper_2104_13466_b200.problem import NeoHookean


def ref_problem(sd, tag, P, m, div, L, dr=None, origin=None):
    from sdmefem.basis1d import BasisKind as RK, build_basis as rbb
    from sdmefem.femcore import FemProblem
    from sdmefem.material import NeoHookean as RN
    from sdmefem.meshdof import build_dofmap, gen_box_mesh
    from sdmefem.quadrature import gauss_rule as rgr
    from sdmefem.tensorelem import TensorElement

    mesh = gen_box_mesh(div, L, origin)
    el = TensorElement.create(3, rbb(P, RK(tag)))
    return FemProblem(mesh, el, build_dofmap(mesh, el, dr), RN.from_engineering(1e7, 0.3, 1e3), rule=rgr(m))


@pytest.mark.parametrize("case", global_cases(), ids=lambda c: f"{c[1]}-P{c[2]}")
def test_descriptor_from_reference_problem(case):
    """B, D, w from element.basis.with_rule(rule), perm from dmap.gdof +
    free_map, Dirichlet faces from dmap.dirichlet: identical to the GPU
    path's own builders (basis.py, lattice.reference_free_index)."""
    sd = import_reference()
    _, tag, P, m, div, L, dr = case
    prob = ref_problem(sd, tag, P, m, div, L, dr)
    d = reference_descriptor(prob)
    assert d is not None and d.mesh == BoxMesh(div, L)
    assert d.n_free == prob.n_free
    perm, n_free = reference_free_index(d.mesh, P, dr)
    assert n_free == d.n_free and np.array_equal(perm, d.perm)
    B, D, w = build_basis(P, BasisKind(tag)).tables(gauss_rule(m))
    for ours, ref in zip((B, D, w), d.tables):
        assert np.abs(ours - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())
    want = sorted((t, tuple(sorted(c))) for t, c in dr)
    assert sorted(d.dirichlet) == want
    assert d.mat == NeoHookean.from_engineering(1e7, 0.3, 1e3)


def test_general_mesh_is_not_a_box():
    sd = import_reference()
    from sdmefem.meshdof import Mesh, gen_box_mesh

    box = gen_box_mesh((2, 1, 1), (2.0, 1.0, 1.0))
    assert box_layout(box) == BoxMesh((2, 1, 1), (2.0, 1.0, 1.0))
    conn = np.array(box.elems)
    conn[1] = conn[1][[1, 2, 3, 0, 5, 6, 7, 4]]  # rotated local axes
    assert box_layout(Mesh(3, box.coords.copy(), conn, {})) is None
    coords = box.coords.copy()
    coords[4] += 0.01  # perturbed vertex
    assert box_layout(Mesh(3, coords, np.array(box.elems), {})) is None


def test_reference_solver_config_is_accepted():
    """The reference's SolverConfig objects are accepted as they are; its
    default (SGS + Schur condensation) selects the assembled solver
    (csrc/schur.cu), diagonal / none without condensation the matrix-free
    one; unknown preconditioners are rejected like solver.py:122."""
    sd = import_reference()
    from sdmefem.dynamics import SolverConfig as RefCfg

    cfg = SolverConfig.coerce(RefCfg(precond="diagonal", tol=1e-10, maxit=500, condense=False))
    assert cfg == SolverConfig(precond="diagonal", tol=1e-10, maxit=500, condense=False) and not cfg.assembled
    ref_default = SolverConfig.coerce(RefCfg())
    assert ref_default == SolverConfig.reference_default() and ref_default.assembled
    assert SolverConfig(precond="sgs", condense=False).assembled
    with pytest.raises(ValueError, match="preconditioner"):
        make_solver(None, None, 0.0, SolverConfig(precond="ilu", condense=False))
    with pytest.raises(TypeError):
        SolverConfig.coerce(object())


def test_cfl_dt_restates_reference_formula():
    """dynamics.py:81-101, both modes, and its delta / mode validation."""
    sd = import_reference()
    from sdmefem.dynamics import cfl_dt as ref_cfl
    from sdmefem.material import NeoHookean as RN
    from sdmefem.meshdof import gen_box_mesh

    for E, nu, rho in ((1e7, 0.3, 1e3), (100.0, 0.3, 1.0), (2.1e11, 0.29, 7850.0)):
        ours_mat = NeoHookean.from_engineering(E, nu, rho)
        ref_mat = RN.from_engineering(E, nu, rho)
        for div, L in (((80, 16, 16), (1.0, 0.2, 0.2)), ((4, 4, 4), (1.0, 1.0, 1.0))):
            for mode in ("AsPrinted", "PhysicalSqrt"):
                for delta in (0.3, 0.5, 0.85):
                    a = cfl_dt(BoxMesh(div, L), ours_mat, delta, mode)
                    b = ref_cfl(gen_box_mesh(div, L), ref_mat, delta, mode)
                    assert abs(a - b) <= 1e-14 * b
    m = NeoHookean.from_engineering(1e7, 0.3, 1e3)
    with pytest.raises(ValueError):
        cfl_dt(BoxMesh((1, 1, 1), (1, 1, 1)), m, 0.95)
    with pytest.raises(ValueError):
        cfl_dt(BoxMesh((1, 1, 1), (1, 1, 1)), m, 0.5, "Exact")


def test_error_types_subclass_the_reference_when_importable():
    """Run in a fresh interpreter with the reference importable: the GPU
    path's exceptions are caught by except clauses naming the reference's
    classes (femcore.py:36-42, solver.py:33-38, dynamics.py:32-35)."""
    import os
    import subprocess
    import sys

    from conftest import ROOT, reference_src

    import_reference()
    code = ("import sdmefem.femcore as f, sdmefem.solver as s, sdmefem.dynamics as d\n"
            "from paper_2104_13466_b200 import errors as e\n"
            "assert e.REFERENCE_TYPES\n"
            "assert issubclass(e.ElementInversionError, f.ElementInversionError)\n"
            "assert issubclass(e.PCGError, s.PCGError)\n"
            "assert issubclass(e.NewtonDivergenceError, d.NewtonDivergenceError)\n"
            "try:\n    raise e.ElementInversionError(3, 7)\n"
            "except f.ElementInversionError as x:\n    assert (x.elem_id, x.qp) == (3, 7)\n"
            "try:\n    raise e.PCGError('m', 'st')\nexcept s.PCGError as x:\n    assert x.stats == 'st'\n"
            "print('ok')\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, reference_src()]),
               NUMBA_CACHE_DIR=os.path.join("/tmp", "sdme_numba_cache"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
