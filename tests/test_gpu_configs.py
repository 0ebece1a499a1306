"""BASELINE configs 4 and 5 at their own parameters, the CFL eigenvalue and
the solver objects -- GPU path (through the C ABI) vs the reference's golden
vectors and the CPU oracle.

* config 5 (implicit large deformation, P = 6, three bases) reduced to 8x1x1
  elements of the same size and aspect ratio: Newton counts equal, PCG counts
  within the reference's own run-to-run spread (+-1 at least), u within 1e-9
  relative (``dynamics.py:173-257``);
* config 4 (explicit impact, 80x16x16 P = 3 SDME, lumped mass, penalty
  contact eps = 1e10) at FULL size: the first steps against the oracle's
  restatement loop, with and without initial penetration;
* ``estimate_lambda_max`` (the dt of config 4) against scipy ``eigsh`` on the
  oracle's assembled M_L^-1 K_0;
* ``make_solver`` / ``GpuLinearSolver`` (``dynamics.py:111-127``,
  ``solver.py:302-322``).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden, max_rel_err
from oracle import basis as ob
from oracle import fem as of
from oracle import solve as osv
from paper_2104_13466_b200 import (BoxMesh, ContactParams, GpuFemProblem, GpuLinearSolver, GpuPenaltyContact,
                                   NeoHookean, RigidObstacle, ScaledLoad, SolverConfig, build_basis,
                                   explicit_run, gauss_rule, make_solver, newmark_run, pcg_gpu)
from paper_2104_13466_b200.basis import BasisKind
from paper_2104_13466_b200.dynamics import estimate_lambda_max, lumped_mass

pytestmark = pytest.mark.gpu

MAT = NeoHookean.from_engineering(1.0e7, 0.3, 1.0e3)
OMAT = of.Material(1.0e7, 0.3, 1.0e3)
TOL = 1e-12
C5_TAGS = ("LagrangeGLL", "ModalJacobi", "SDME_H")


def gpu_problem(tag, P, m, div, L, dr=None, origin=(0.0, 0.0, 0.0)):
    return GpuFemProblem(BoxMesh(div, L, origin), build_basis(P, BasisKind(tag)), MAT, gauss_rule(m), dr)


def c5_reference_runs(g, tag):
    """The reference's PCG counts per solve from its three runs (default
    threads, OPENBLAS_NUM_THREADS = 1 and 4; make_golden.py gen_config5):
    rows = runs, columns = solves."""
    runs = [np.array([int(r[2]) for r in g[f"{tag}_pcg_rows"]])]
    runs += [np.asarray(g[f"{tag}_pcg_iters_t{t}"]) for t in (1, 4)]
    return np.stack(runs)


@pytest.mark.parametrize("tag", C5_TAGS)
def test_config5_large_deformation_newmark_vs_reference(tag):
    """Config 5 regime (P = 6, m = 7, cantilever of aspect 8, x = 0 clamped, tip
    traction -8e5 ramped over 3 steps: ~24% tip deflection, 4-6 Newton
    iterations per step, 200-1800 PCG iterations per solve) for each basis."""
    g = load_golden("config5")
    traction, steps, dt = (float(v) for v in g["meta"])
    steps = int(steps)
    pb = gpu_problem(tag, 6, 7, (8, 1, 1), (0.5, 0.0625, 0.0625), [("xmin", (0, 1, 2))])
    base = pb.traction_vector("xmax", [0.0, 0.0, traction])
    assert max_rel_err(base, g[f"{tag}_load"]) <= TOL
    T = steps * dt
    cfg = SolverConfig(precond="diagonal", tol=1e-10, maxit=200000, condense=False)
    traj = newmark_run(pb, ScaledLoad(base, lambda t: min(t / T, 1.0)), dt, steps, newton_tol=1e-8, cfg=cfg)
    assert traj.newton_iters == [int(v) for v in g[f"{tag}_newton_iters"]]
    assert min(traj.newton_iters) >= 4  # the nonlinear regime the config asks for
    # PCG counts vs the committed reference run: +-1 (the north_star bar), or
    # the reference's own run-to-run spread when that is larger -- the largest
    # per-solve (max - min) over its three runs.  It is 1 for GLL and SDME_H
    # and ~17 for ModalJacobi (~1,500 iterations per solve, where CG's count
    # depends on last-bit rounding of the operator and the dots).
    runs = c5_reference_runs(g, tag)
    slack = max(1, int((runs.max(axis=0) - runs.min(axis=0)).max()))
    got = np.array([r["iterations"] for r in traj.stats.rows])
    assert got.shape == runs[0].shape
    assert int(np.abs(got - runs[0]).max()) <= slack, (got.tolist(), runs.tolist(), slack)
    assert max_rel_err(traj.state.u, g[f"{tag}_u"]) <= 1e-9
    assert max_rel_err(traj.state.v, g[f"{tag}_v"]) <= 1e-8
    # tip deflection (vertex coefficients are point values in every basis)
    tip = pb.to_lattice(traj.state.u)[2, ::6, ::6, -1].mean()
    assert -tip / 0.5 > 0.15


def _c4_problems(share=True):
    P, div, L = 3, (80, 16, 16), (1.0, 0.2, 0.2)
    pb = gpu_problem("SDME_M", P, P + 1, div, L)
    opb = of.Problem(of.Mesh(div, L), ob.Basis("SDME_M", P), OMAT, P + 1, share_geometry=share)
    return pb, opb


@pytest.mark.slow
def test_config4_full_size_first_steps_vs_oracle():
    """Config 4 at its own size (80x16x16 P = 3 SDME, 1,735,923 DOFs): lumped
    mass, v0 = -10 m/s, eps = 1e10, dt = 0.5 * 2 / sqrt(lambda_max); the first
    3 steps against the oracle's restatement loop (oracle/solve.py
    explicit_lumped) -- once with the wall at x = -1e-3 (free flight) and once
    at x = +2e-6 (the xmin face starts in contact: 4,096 active points)."""
    pb, opb = _c4_problems()
    _, inv_ml = lumped_mass(pb)
    ml = opb.lumped_mass()
    assert max_rel_err(1.0 / inv_ml.free(), ml) <= TOL
    v0 = pb.constant_field([-10.0, 0.0, 0.0])
    zero = np.zeros(opb.n_free)
    for wall in (-1e-3, 2e-6):
        c = GpuPenaltyContact(pb, RigidObstacle([wall, 0.0, 0.0], [1.0, 0.0, 0.0]), ContactParams(1e10), "xmin")
        lam = estimate_lambda_max(pb, inv_ml, contact=c)
        dt = 0.5 * 2.0 / np.sqrt(lam)
        traj = explicit_run(pb, None, dt, 3, v0=v0, contact=c, record_every=1, mass="lumped")
        oc = of.Contact(opb, [wall, 0.0, 0.0], [1.0, 0.0, 0.0], 1e10, "xmin")
        ref = osv.explicit_lumped(opb, lambda t: zero, dt, 3, v0=v0, contact=oc)
        if wall > 0:
            assert traj.contact_history[-1][3] == 4096  # every face point active
        assert max_rel_err(traj.state.u, ref["u"]) <= 1e-10
        assert max_rel_err(traj.state.v, ref["v"]) <= 1e-9


def test_lambda_max_vs_eigsh():
    """estimate_lambda_max (device Lanczos) vs scipy eigsh on the oracle's
    assembled M_L^-1/2 K_0 M_L^-1/2, config-4 element size (h = 1/80, P = 3
    SDME) on a 4x2x2 block: within 1e-6 relative."""
    from scipy.sparse import diags
    from scipy.sparse.linalg import eigsh

    div, L = (4, 2, 2), (0.05, 0.025, 0.025)
    pb = gpu_problem("SDME_M", 3, 4, div, L)
    opb = of.Problem(of.Mesh(div, L), ob.Basis("SDME_M", 3), OMAT, 4)
    _, inv_ml = lumped_mass(pb)
    lam = estimate_lambda_max(pb, inv_ml)
    w = diags(1.0 / np.sqrt(opb.lumped_mass()))
    s = (w @ opb.assemble(np.zeros(opb.n_free)) @ w).tocsr()
    ref = float(eigsh(s, k=1, which="LA", tol=1e-14, return_eigenvectors=False)[0])
    assert abs(lam - ref) <= 1e-6 * ref, (lam, ref)


def test_make_solver_and_linear_solver_vs_reference_pcg():
    """make_solver(problem, u_lin, c_m, cfg).solve(rhs) == pcg on the
    reference-assembled K_T(u) + c_m M (golden case g0: iteration count +-1,
    x within 1e-9); GpuLinearSolver reports condensed = False and accepts a
    reference-style SolverConfig."""
    from conftest import global_cases

    g = load_golden("global")
    i, tag, P, m, div, L, dr = global_cases()[0]
    pb = gpu_problem(tag, P, m, div, L, dr)
    cm = float(g[f"g{i}_cm"])
    cfg = SolverConfig(precond="diagonal", tol=1e-10, maxit=100000, condense=False)
    solver = make_solver(pb, g[f"g{i}_u"], cm, cfg)
    assert isinstance(solver, GpuLinearSolver) and not solver.condensed
    x, st = solver.solve(g[f"g{i}_pcg_b"])
    assert abs(st.iterations - int(g[f"g{i}_pcg_iters"])) <= 1
    assert st.preconditioner == "diagonal" and st.converged
    assert max_rel_err(x, g[f"g{i}_pcg_x"]) <= 1e-9
    x2, st2 = pcg_gpu(pb, g[f"g{i}_u"], g[f"g{i}_pcg_b"], c_m=cm, tol=1e-10, maxit=100000)
    assert st2.iterations == st.iterations and np.array_equal(x, x2)
