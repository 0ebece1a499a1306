"""Drop-in on the GPU: problems built from the reference's own objects
(``interop.from_reference``) reproduce the reference's operators and its
Newmark driver, run live beside them.  Needs the reference package (the
offline install under baseline/_ref travels to the GPU box); skipped when it
is absent."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import global_cases, import_reference, max_rel_err
from paper_2104_13466_b200 import GpuMeshProblem, ScaledLoad, newmark_run
from paper_2104_13466_b200.interop import from_reference
from paper_2104_13466_b200.problem import GpuFemProblem

pytestmark = pytest.mark.gpu


def _ref(tag, P, m, mesh, dr=None):
    from sdmefem.basis1d import BasisKind, build_basis
    from sdmefem.femcore import FemProblem
    from sdmefem.material import NeoHookean
    from sdmefem.meshdof import build_dofmap
    from sdmefem.quadrature import gauss_rule
    from sdmefem.tensorelem import TensorElement

    el = TensorElement.create(3, build_basis(P, BasisKind(tag)))
    return FemProblem(mesh, el, build_dofmap(mesh, el, dr), NeoHookean.from_engineering(1e7, 0.3, 1e3),
                      rule=gauss_rule(m))


@pytest.mark.parametrize("case", global_cases(), ids=lambda c: f"{c[1]}-P{c[2]}")
def test_from_reference_box_operators(case):
    import_reference()
    from sdmefem.meshdof import gen_box_mesh

    _, tag, P, m, div, L, dr = case
    prob = _ref(tag, P, m, gen_box_mesh(div, L), dr)
    gp = from_reference(prob)
    assert isinstance(gp, GpuFemProblem) and gp.n_free == prob.n_free
    rng = np.random.default_rng(11)
    u = 1e-3 * min(L) / max(div) * rng.uniform(-1, 1, prob.n_free)
    p = rng.standard_normal(prob.n_free)
    assert max_rel_err(gp.internal_force(u), prob.internal_force(u)) <= 1e-12
    assert max_rel_err(gp.apply_tangent(u, p, 3e4), (prob.tangent(u) + 3e4 * prob.mass()) @ p) <= 1e-12


def test_from_reference_general_mesh_operators():
    import_reference()
    from sdmefem.meshdof import Mesh, gen_box_mesh

    base = gen_box_mesh((2, 1, 1), (2.0, 1.0, 1.0))
    conn = np.array(base.elems)
    conn[1] = conn[1][[1, 2, 3, 0, 5, 6, 7, 4]]  # second hex with rotated local axes
    coords = base.coords.copy()
    coords[:, 2] += 0.05 * coords[:, 0] * coords[:, 1]  # non-affine
    prob = _ref("SDME_M", 3, 4, Mesh(3, coords, conn, {}))
    gp = from_reference(prob)
    assert isinstance(gp, GpuMeshProblem)
    rng = np.random.default_rng(5)
    u = 2e-3 * rng.uniform(-1, 1, prob.n_free)
    p = rng.standard_normal(prob.n_free)
    assert max_rel_err(gp.internal_force(u), prob.internal_force(u)) <= 1e-12
    assert max_rel_err(gp.apply_tangent(u, p), prob.tangent(u) @ p) <= 1e-12


def test_newmark_with_reference_objects_matches_reference_run():
    """newmark_run(from_reference(prob), ..., cfg=<reference SolverConfig>)
    vs the reference's own newmark_run on the same objects."""
    sd = import_reference()
    from sdmefem.dynamics import SolverConfig as RefCfg
    from sdmefem.dynamics import newmark_run as ref_newmark
    from sdmefem.femcore import build_face_tables
    from sdmefem.meshdof import gen_box_mesh

    prob = _ref("SDME_H", 3, 5, gen_box_mesh((3, 1, 1), (1.5, 0.5, 0.5)), [("xmin", (0, 1, 2))])
    faces = build_face_tables(prob.mesh, prob.element, "xmax", prob.rule)
    base = prob.traction_vector(faces, lambda f: np.tile([0.0, 1e5, -2e5], (len(f.pts), 1)))
    cfg = RefCfg(precond="diagonal", tol=1e-10, maxit=100000, condense=False)
    ramp = lambda t: min(t / 4e-4, 1.0)
    ref = ref_newmark(prob, lambda t: base * ramp(t), 1e-4, 4, newton_tol=1e-8, cfg=cfg)
    gp = from_reference(prob)
    got = newmark_run(gp, ScaledLoad(base, ramp), 1e-4, 4, newton_tol=1e-8, cfg=cfg)
    assert got.newton_iters == ref.newton_iters
    its = [r["iterations"] for r in got.stats.rows]
    rits = [r["iterations"] for r in ref.stats.rows]
    assert len(its) == len(rits) and max(abs(a - b) for a, b in zip(its, rits)) <= 1
    assert max_rel_err(got.state.u, ref.state.u) <= 1e-9


def test_contact_helpers_vs_reference():
    """GpuPenaltyContact.update_active_set / pressure_profile / evaluate_forces
    (contact.py:98-151, 186-204) on a problem built by from_reference, against
    the reference's PenaltyContact on the same FemProblem (tilted plane:
    partially active surface)."""
    import_reference()
    from sdmefem.contact import ContactParams as RP
    from sdmefem.contact import PenaltyContact, RigidObstacle as RO
    from sdmefem.meshdof import gen_box_mesh

    from paper_2104_13466_b200 import ContactParams, GpuPenaltyContact, RigidObstacle

    prob = _ref("SDME_M", 3, 4, gen_box_mesh((2, 3, 2), (0.3, 0.45, 0.2)))
    n = np.array([1.0, 0.15, -0.05])
    n /= np.linalg.norm(n)
    point = np.array([1e-4, 0.2, 0.1])
    ref = PenaltyContact(prob, RO(point, n), RP(1e9), "xmin")
    gp = from_reference(prob)
    ours = GpuPenaltyContact(gp, RigidObstacle(point, n), ContactParams(1e9), "xmin")
    u = 1e-4 * np.random.default_rng(3).uniform(-1, 1, prob.n_free)
    ra, rg = ref.update_active_set(u)
    oa, og = ours.update_active_set(u)
    assert len(rg) == len(og)
    for a, b, fa, fb in zip(rg, og, ra, oa):
        assert np.abs(a - b).max() <= 1e-15 + 1e-12 * np.abs(a).max()
        assert np.array_equal(fa, fb)
    assert 0 < sum(int(a.sum()) for a in ra) < sum(a.size for a in ra)  # partially active
    rp, op = ref.pressure_profile(u), ours.pressure_profile(u)
    ko, kr = np.lexsort((op[:, 1], op[:, 0])), np.lexsort((rp[:, 1], rp[:, 0]))
    assert np.abs(op[ko] - rp[kr]).max() <= 1e-12 * np.abs(rp).max()
    fr, fo = ref.evaluate_forces(u), ours.evaluate_forces(u)
    assert max_rel_err(fo.force, fr.force) <= 1e-12
    p = np.random.default_rng(4).standard_normal(prob.n_free)
    assert max_rel_err(fo.stiffness @ p, fr.stiffness @ p) <= 1e-12
