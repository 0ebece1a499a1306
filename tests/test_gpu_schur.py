"""the reference's default solver -- symmetric Gauss-Seidel PCG on
the Schur complement of the element-interior modes (SolverConfig(),
dynamics.py:38-43; make_solver / condense_elements / LinearSolver,
dynamics.py:111-127, solver.py:78-126, 258-322) -- on the GPU
(csrc/schur.cu), against golden vectors of the reference itself
(tests/golden/make_golden.py gen_sgs, gen_config1_default)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN, global_cases, load_golden, max_rel_err
from paper_2104_13466_b200 import (BoxMesh, GpuFemProblem, NeoHookean, ScaledLoad, SolverConfig, build_basis,
                                   explicit_run, gauss_rule, make_solver, newmark_run)
from paper_2104_13466_b200.basis import BasisKind
from paper_2104_13466_b200.schur import SchurSolver

pytestmark = pytest.mark.gpu

MAT = NeoHookean.from_engineering(1.0e7, 0.3, 1.0e3)
CFGS = (("sgs", True), ("sgs", False), ("diagonal", True), ("none", True))


def gpu_problem(tag, P, m, div, L, dr=None):
    return GpuFemProblem(BoxMesh(div, L), build_basis(P, BasisKind(tag)), MAT, gauss_rule(m), dr)


@pytest.mark.parametrize("case", global_cases(), ids=lambda c: f"{c[1]}-P{c[2]}")
@pytest.mark.parametrize("k", range(len(CFGS)), ids=lambda k: f"{CFGS[k][0]}-{'schur' if CFGS[k][1] else 'full'}")
def test_assembled_solver_vs_reference(case, k):
    """make_solver(problem, K_T(u) + c_m M, cfg).solve(b): iterations +-1,
    x within 1e-9, the reference's preconditioner tag ("sgs+schur" ...)."""
    g, s = load_golden("global"), load_golden("sgs")
    i, tag, P, m, div, L, dr = case
    pc, cond = CFGS[k]
    pb = gpu_problem(tag, P, m, div, L, dr)
    cfg = SolverConfig(precond=pc, tol=1e-10, maxit=100000, condense=cond)
    solver = make_solver(pb, g[f"g{i}_u"], float(g[f"g{i}_cm"]), cfg)
    assert solver.condensed == cond
    x, st = solver.solve(g[f"g{i}_pcg_b"])
    ref_its = int(s[f"g{i}_c{k}_iters"])
    assert abs(st.iterations - ref_its) <= max(1, ref_its // 100 if pc == "none" else 1), (st.iterations, ref_its)
    assert st.preconditioner == str(s[f"g{i}_c{k}_tag"])
    assert max_rel_err(x, s[f"g{i}_c{k}_x"]) <= 1e-9


def test_condensed_schur_matrix_vs_reference():
    """The assembled boundary Schur complement (CSR pattern and values) equals
    the reference's CondensedSystem.schur (solver.py:286-293)."""
    g, s = load_golden("global"), load_golden("sgs")
    i, tag, P, m, div, L, dr = global_cases()[2]
    pb = gpu_problem(tag, P, m, div, L, dr)
    sch = SchurSolver(pb, True, "sgs", 1e-10, 1000)
    sch.factor(g[f"g{i}_u"], 1.0, float(g[f"g{i}_cm"]))
    a, _ = sch.matrix()
    a.sort_indices()
    assert np.array_equal(a.indptr, s[f"g{i}_c0_schur_indptr"])
    assert np.array_equal(a.indices, s[f"g{i}_c0_schur_indices"])
    assert max_rel_err(a.data, s[f"g{i}_c0_schur_data"]) <= 1e-12
    info = sch.info()
    assert info["nb"] == a.shape[0] and min(info["sgs_levels"]) >= 1


def test_explicit_run_reference_default_solver():
    """explicit_run with the reference's SolverConfig() (consistent mass,
    SGS + Schur, tol 1e-12): per-step PCG counts +-1, u / v within 1e-9."""
    s = load_golden("sgs")
    pb = gpu_problem("SDME_M", 3, 4, (3, 2, 2), (1.0, 0.5, 0.5), [("xmin", (0, 1, 2))])
    base = pb.traction_vector("xmax", [0.0, 0.0, 2.0e4])
    traj = explicit_run(pb, ScaledLoad(base, lambda t: min(t / 5e-5, 1.0)), 1e-5, 20,
                        cfg=SolverConfig.reference_default())
    ref = s["explicit_rows"]
    got = np.array([(r["step"], r["iterations"]) for r in traj.stats.rows])
    assert got.shape == ref.shape and int(np.abs(got - ref).max()) <= 1
    assert [r["preconditioner"] for r in traj.stats.rows] == [str(t) for t in s["explicit_tags"]]
    assert max_rel_err(traj.state.u, s["explicit_u"]) <= 1e-9
    assert max_rel_err(traj.state.v, s["explicit_v"]) <= 1e-9


def test_newmark_run_reference_default_solver():
    s = load_golden("sgs")
    pb = gpu_problem("SDME_H", 3, 4, (2, 2, 2), (1.0, 1.0, 1.0), [("xmin", (0, 1, 2))])
    base = pb.traction_vector("xmax", [0.0, 1.0e5, -2.0e5])
    assert max_rel_err(base, s["newmark_load"]) <= 1e-12
    traj = newmark_run(pb, ScaledLoad(base, lambda t: min(t / 4e-4, 1.0)), 1e-4, 4, newton_tol=1e-8,
                       cfg=SolverConfig.reference_default())
    assert traj.newton_iters == [int(v) for v in s["newmark_newton"]]
    got = np.array([r["iterations"] for r in traj.stats.rows])
    assert int(np.abs(got - s["newmark_rows"][:, 2]).max()) <= 1
    assert max_rel_err(traj.state.u, s["newmark_u"]) <= 1e-9


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "config1_default.npz")), reason="fixture not generated")
def test_config1_with_reference_default_solver():
    """BASELINE config 1 with the reference's default solver (SGS + Schur,
    tol 1e-12): Newton counts equal, PCG +-1, u within 1e-9."""
    g = load_golden("config1_default")
    pb = gpu_problem("SDME_M", 4, 6, (4, 4, 4), (1.0, 1.0, 1.0), [("xmin", (0, 1, 2))])
    base = pb.traction_vector("xmax", [0.0, 0.0, 1.0e5])
    traj = newmark_run(pb, ScaledLoad(base, lambda t: min(t / 1e-3, 1.0)), 1e-4, 10, newton_tol=1e-8,
                       cfg=SolverConfig.reference_default())
    assert traj.newton_iters == [int(v) for v in g["newton_iters"]]
    got = np.array([r["iterations"] for r in traj.stats.rows])
    assert got.shape[0] == g["pcg_rows"].shape[0]
    assert int(np.abs(got - g["pcg_rows"][:, 2]).max()) <= 1
    assert [r["preconditioner"] for r in traj.stats.rows] == [str(t) for t in g["tags"]]
    assert max_rel_err(traj.state.u, g["u"]) <= 1e-9


def test_condensation_errors_match_reference():
    """A non-SPD interior block raises ValueError (solver.py:284-285); an
    unpreconditioned solve on a negative definite operator raises ValueError
    from the condensation first, like the reference's cho_factor."""
    pb = gpu_problem("SDME_M", 3, 4, (2, 2, 2), (1.0, 1.0, 1.0), [("xmin", (0, 1, 2))])
    with pytest.raises(ValueError, match="not SPD"):
        make_solver(pb, np.zeros(pb.n_free), 0.0, SolverConfig("none", 1e-10, 100, True), c_k=-1.0)
    with pytest.raises(ValueError, match="positive diagonal"):
        make_solver(pb, np.zeros(pb.n_free), 0.0, SolverConfig("sgs", 1e-10, 100, False), c_k=-1.0).solve(
            np.ones(pb.n_free))
