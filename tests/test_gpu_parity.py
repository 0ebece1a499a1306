"""GPU parity: the CUDA path (through the C ABI) vs the reference's golden
vectors and the CPU oracle.

Bars (north_star): 1e-12 relative on element/global vectors, PCG iteration
counts +-1, displacements within 1e-9 relative, bit-identical reruns.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import element_cases, global_cases, load_golden, max_rel_err, rel_err
from oracle import basis as ob
from oracle import fem as of
from oracle import solve as osv
from paper_2104_13466_b200 import (BoxMesh, ContactParams, ElementInversionError, GpuFemProblem,
                                   GpuPenaltyContact, NeoHookean, PCGError, RigidObstacle, ScaledLoad,
                                   SolverConfig, build_basis, explicit_run, gauss_rule, newmark_run,
                                   pcg_gpu)
from paper_2104_13466_b200.basis import BasisKind

pytestmark = pytest.mark.gpu

MAT = NeoHookean.from_engineering(1.0e7, 0.3, 1.0e3)
OMAT = of.Material(1.0e7, 0.3, 1.0e3)
TOL = 1e-12


def gpu_problem(tag, P, m, div, L, dr=None, origin=(0.0, 0.0, 0.0), mat=None):
    return GpuFemProblem(BoxMesh(div, L, origin), build_basis(P, BasisKind(tag)), mat or MAT, gauss_rule(m), dr)


@pytest.mark.parametrize("case", element_cases(), ids=lambda c: f"{c[1]}-P{c[2]}-m{c[3]}-{c[0]}")
def test_element_vectors_vs_reference(case):
    """Single-element meshes: f_int, K.p, M.p, diag(K + c_m M) vs the
    reference's element_internal_force / element_tangent / element_mass."""
    i, tag, P, m, h = case
    g = load_golden("elements")
    pb = gpu_problem(tag, P, m, (1, 1, 1), h)
    loc = of.DofMap(of.Mesh((1, 1, 1), h), P).evdofs(0)  # local order -> free index
    u, p, cm = g[f"c{i}_u"], g[f"c{i}_p"], float(g[f"c{i}_cm"])
    assert max_rel_err(pb.internal_force(u)[loc], g[f"c{i}_fint"]) <= TOL
    assert max_rel_err(pb.apply_tangent(u, p)[loc], g[f"c{i}_kp"]) <= TOL
    assert max_rel_err(pb.mass_apply(p)[loc], g[f"c{i}_mp"]) <= TOL
    assert max_rel_err(pb.tangent_diagonal(u, cm)[loc], g[f"c{i}_diag"]) <= TOL


@pytest.mark.parametrize("case", global_cases(), ids=lambda c: f"{c[1]}-P{c[2]}")
def test_global_vectors_and_pcg_vs_reference(case):
    i, tag, P, m, div, L, dr = case
    g = load_golden("global")
    pb = gpu_problem(tag, P, m, div, L, dr)
    assert pb.n_free == g[f"g{i}_u"].size
    u, p, cm = g[f"g{i}_u"], g[f"g{i}_p"], float(g[f"g{i}_cm"])
    assert max_rel_err(pb.internal_force(u), g[f"g{i}_fint"]) <= TOL
    assert max_rel_err(pb.apply_tangent(u, p), g[f"g{i}_kp"]) <= TOL
    assert max_rel_err(pb.apply_tangent(u, p, cm), g[f"g{i}_kp"] + cm * g[f"g{i}_mp"]) <= TOL
    assert max_rel_err(pb.mass_apply(p), g[f"g{i}_mp"]) <= TOL
    assert max_rel_err(pb.tangent_diagonal(u, cm), g[f"g{i}_diag"]) <= TOL
    x, st = pcg_gpu(pb, u, g[f"g{i}_pcg_b"], c_m=cm, precond="diagonal", tol=1e-10, maxit=100000)
    assert abs(st.iterations - int(g[f"g{i}_pcg_iters"])) <= 1
    assert max_rel_err(x, g[f"g{i}_pcg_x"]) <= 1e-9


def test_config1_newmark_vs_reference():
    """BASELINE config 1 (4^3, P=4 SDME, (P+2)^3 Gauss, 10 Newmark steps,
    Jacobi-PCG 1e-10): Newton counts equal, PCG iterations +-1, u within 1e-9."""
    g = load_golden("config1")
    pb = gpu_problem("SDME_M", 4, 6, (4, 4, 4), (1.0, 1.0, 1.0), [("xmin", (0, 1, 2))])
    base = pb.traction_vector("xmax", [0.0, 0.0, 1.0e5])
    assert max_rel_err(base, g["load"]) <= TOL
    load = ScaledLoad(base, lambda t: min(t / 1e-3, 1.0))
    cfg = SolverConfig(precond="diagonal", tol=1e-10, maxit=200000, condense=False)
    traj = newmark_run(pb, load, 1e-4, 10, newton_tol=1e-8, cfg=cfg)
    assert traj.newton_iters == [int(v) for v in g["newton_iters"]]
    ref_its = [int(r[2]) for r in g["pcg_rows"] if r[0] >= 0]
    its = [r["iterations"] for r in traj.stats.rows if r["step"] >= 0]
    assert len(its) == len(ref_its)
    assert max(abs(a - b) for a, b in zip(its, ref_its)) <= 1
    assert max_rel_err(traj.state.u, g["u"]) <= 1e-9
    assert max_rel_err(traj.state.v, g["v"]) <= 1e-8


def test_contact_force_vs_reference():
    g = load_golden("contact")
    pb = gpu_problem("SDME_M", 3, 4, (3, 2, 2), (0.3, 0.2, 0.2))
    c = GpuPenaltyContact(pb, RigidObstacle([-1e-3, 0, 0], [1, 0, 0]), ContactParams(1e10), "xmin")
    fc = c.evaluate_forces(g["u"])
    assert fc.stiffness is not None  # active points -> contact stiffness operator
    assert max_rel_err(fc.force, g["force"]) <= TOL
    assert max_rel_err(fc.gaps, g["gaps"]) <= TOL
    assert fc.active.any()


def test_explicit_lumped_contact_vs_reference_pieces():
    """D6 loop: lumped mass + penalty contact, 40 steps, vs the loop built
    from the reference's own internal_force / evaluate_forces / mass."""
    g = load_golden("contact")
    pb = gpu_problem("SDME_M", 3, 4, (3, 2, 2), (0.3, 0.2, 0.2))
    c = GpuPenaltyContact(pb, RigidObstacle([-2e-5, 0, 0], [1, 0, 0]), ContactParams(1e10), "xmin")
    traj = explicit_run(pb, None, float(g["explicit_dt"]), int(g["explicit_steps"]), v0=g["v0"],
                        contact=c, record_every=1, mass="lumped")
    assert max(h[1] for h in traj.contact_history) > 0.0  # contact engaged
    assert max_rel_err(traj.state.u, g["explicit_u"]) <= 1e-10
    assert max_rel_err(traj.state.v, g["explicit_v"]) <= 1e-9


def test_reruns_are_bit_identical():
    pb = gpu_problem("SDME_M", 4, 5, (6, 5, 4), (1.0, 1.0, 1.0), [("xmin", (0, 1, 2))])
    rng = np.random.default_rng(0)
    u = 1e-4 * rng.uniform(-1, 1, pb.n_free)
    p = rng.standard_normal(pb.n_free)
    a = pb.apply_tangent(u, p, 3e4)
    b = pb.apply_tangent(u, p, 3e4)
    assert np.array_equal(a.view(np.int64), b.view(np.int64))
    f1 = pb.internal_force(u)
    f2 = pb.internal_force(u)
    assert np.array_equal(f1.view(np.int64), f2.view(np.int64))
    x1, s1 = pcg_gpu(pb, u, f1, c_m=3e4, tol=1e-10)
    x2, s2 = pcg_gpu(pb, u, f1, c_m=3e4, tol=1e-10)
    assert s1.iterations == s2.iterations and np.array_equal(x1.view(np.int64), x2.view(np.int64))


@pytest.mark.parametrize("tag,P,m", [("SDME_M", 4, 5), ("LagrangeGLL", 3, 4), ("ModalJacobi", 2, 4),
                                     ("SDME_H", 6, 7), ("SDME_K", 8, 9)])
def test_multi_element_vs_oracle_h64(tag, P, m):
    """h = 1/64 (config 2/3 element size) on a small mesh with Dirichlet:
    GPU vs the dense oracle restatement, f_int / K.p / diag."""
    div = (3, 2, 2) if P <= 4 else (2, 2, 1)
    h = 1.0 / 64
    L = tuple(d * h for d in div)
    dr = [("xmin", (0, 1, 2))]
    pb = gpu_problem(tag, P, m, div, L, dr)
    opb = of.Problem(of.Mesh(div, L), ob.Basis(tag, P), OMAT, m, dr)
    rng = np.random.default_rng(11)
    u = 1e-3 * h * rng.uniform(-1, 1, pb.n_free)
    p = rng.standard_normal(pb.n_free)
    assert max_rel_err(pb.internal_force(u), opb.internal_force(u)) <= TOL
    assert max_rel_err(pb.apply_tangent(u, p), opb.apply_tangent(u, p)) <= TOL
    assert max_rel_err(pb.tangent_diagonal(u, 4e8), opb.assemble(u, 1.0, 4e8).diagonal()) <= TOL


def test_inversion_error_reports_first_element_and_point():
    """ElementInversionError carries the smallest element id and its first
    offending point in reference order (femcore.py:93-94)."""
    tag, P, m = "ModalJacobi", 2, 3
    div = (3, 2, 2)
    pb = gpu_problem(tag, P, m, div, (1.0, 1.0, 1.0))
    opb = of.Problem(of.Mesh(div, (1.0, 1.0, 1.0)), ob.Basis(tag, P), OMAT, m)
    u = np.zeros(pb.n_free)
    # large interior (bubble) coefficients on elements 7 and 4: only they invert
    for e, amp in ((7, -30.0), (4, -25.0)):
        d = opb.dmap.evdofs(e).reshape(-1, 3)
        interior = np.all(opb.dmap.index_map >= 2, axis=1)
        u[d[interior, 0]] = amp
    with pytest.raises(of.InversionError) as ref:
        opb.internal_force(u)
    with pytest.raises(ElementInversionError) as err:
        pb.internal_force(u)
    assert (err.value.elem_id, err.value.qp) == (ref.value.elem_id, ref.value.qp) == (4, ref.value.qp)
    # the same state as a PCG linearisation point (stored-quadrature setup and
    # diagonal both see it) and through the K.p and diagonal entry points
    b = np.ones(pb.n_free)
    for call in (lambda: pcg_gpu(pb, u, b, c_m=1e5), lambda: pb.apply_tangent(u, b),
                 lambda: pb.tangent_diagonal(u, c_m=1e5)):
        with pytest.raises(ElementInversionError) as err2:
            call()
        assert (err2.value.elem_id, err2.value.qp) == (ref.value.elem_id, ref.value.qp)


def test_pcg_error_contract():
    pb = gpu_problem("SDME_M", 2, 3, (2, 2, 2), (1.0, 1.0, 1.0), [("xmin", (0, 1, 2))])
    rng = np.random.default_rng(1)
    b = rng.standard_normal(pb.n_free)
    with pytest.raises(ValueError):
        pcg_gpu(pb, np.zeros(pb.n_free), b, tol=1.5)
    x, st = pcg_gpu(pb, np.zeros(pb.n_free), np.zeros(pb.n_free))
    assert st.iterations == 0 and not x.any()
    with pytest.raises(PCGError) as e:
        pcg_gpu(pb, np.zeros(pb.n_free), b, tol=1e-14, maxit=3)
    assert e.value.stats.iterations == 3 and not e.value.stats.converged
    # indefinite: negative mass coefficient dominates
    with pytest.raises((PCGError, ValueError)):
        pcg_gpu(pb, np.zeros(pb.n_free), b, c_m=-1e12, precond="none")


def test_config2_properties_full_size():
    """Config 2 (64^3, P=4, ~51M DOFs) size-independent properties: symmetry
    q.Kp = p.Kq, linearity, FD consistency of K against f_int, determinism."""
    pb = GpuFemProblem(BoxMesh((64, 64, 64), (1.0, 1.0, 1.0)), build_basis(4, BasisKind("SDME_M")), MAT,
                       reference_order=False)
    from bench import config2_fields

    u_lat, p_lat = config2_fields(pb, seed_u=0, seed_p=1)
    u = pb.vector().set_lattice(u_lat)
    p = pb.vector().set_lattice(p_lat)
    q = pb.vector().set_lattice(np.random.default_rng(5).standard_normal(pb.n_lattice))
    kp, kq, t1, t2 = (pb.vector() for _ in range(4))
    pb.apply_(u, p, kp)
    pb.apply_(u, q, kq)
    s1, s2 = q.dot(kp), p.dot(kq)
    assert abs(s1 - s2) <= 1e-10 * max(abs(s1), abs(s2))
    # linearity
    t1.assign(2.5, p)
    pb.apply_(u, t1, t2)
    t2.assign(1.0, t2, -2.5, kp)
    assert t2.norm() <= 1e-13 * kp.norm()
    # FD: (f(u + e p) - f(u - e p)) / 2e ~ K p
    eps = 1e-9
    t1.assign(1.0, u, eps, p)
    pb.fint_(t1, t2)
    t1.assign(1.0, u, -eps, p)
    fm = pb.vector()
    pb.fint_(t1, fm)
    t2.assign(1.0 / (2 * eps), t2, -1.0 / (2 * eps), fm)
    t2.assign(1.0, t2, -1.0, kp)
    assert t2.norm() <= 1e-5 * kp.norm()
    # determinism
    pb.apply_(u, p, t1)
    t1.assign(1.0, t1, -1.0, kp)
    assert t1.norm() == 0.0


def _grad_peak(u_lat, P):
    """(k, j, i) of the element whose vertex differences of u are largest."""
    v = u_lat[:, ::P, ::P, ::P]
    g = np.zeros(tuple(s - 1 for s in v.shape[1:]))
    for c in range(3):
        for ax in range(3):
            d = np.abs(np.diff(v[c], axis=ax))
            sl = [slice(0, s - 1) for s in v.shape[1:]]
            g = np.maximum(g, d[tuple(sl)])
    return np.unravel_index(int(np.argmax(g)), g.shape)


def test_config2_field_vs_oracle_on_sub_boxes():
    """Config 2 at full size (64^3, P = 4 SDME_M, the bench's own inputs:
    0.02 sin(2 pi (x+y+z)) + 1e-3 h noise, |grad u| up to ~0.13) against the
    oracle: on 3x3x3-element sub-boxes -- including the one around the
    steepest gradient -- every lattice point strictly inside the sub-box
    receives contributions from sub-box elements only, so the full-mesh GPU
    K(u).p and f_int(u) there must equal the oracle's (dense element_tangent,
    femcore.py:130-146) on the sub-box to 1e-12."""
    from bench import config2_fields
    from paper_2104_13466_b200.lattice import reference_free_index

    P, h, nb = 4, 1.0 / 64, 3
    pb = GpuFemProblem(BoxMesh((64, 64, 64), (1.0, 1.0, 1.0)), build_basis(P, BasisKind("SDME_M")), MAT,
                       reference_order=False)
    u_lat, p_lat = config2_fields(pb, seed_u=0, seed_p=1)
    u = pb.vector().set_lattice(u_lat)
    p = pb.vector().set_lattice(p_lat)
    y_kp = pb.apply_(u, p, pb.vector()).lattice()
    y_f = pb.fint_(u, pb.vector()).lattice()
    kk, jj, ii = _grad_peak(u_lat, P)
    starts = [(0, 0, 0), (30, 17, 45), (min(kk, 61), min(jj, 61), min(ii, 61))]
    sub = BoxMesh((nb,) * 3, (nb * h,) * 3)
    perm, n_free = reference_free_index(sub, P, None)
    opb = of.Problem(of.Mesh((nb,) * 3, (nb * h,) * 3), ob.Basis("SDME_M", P), OMAT, P + 1)
    assert opb.n_free == n_free
    for k0, j0, i0 in starts:
        box = (slice(None), slice(P * k0, P * (k0 + nb) + 1), slice(P * j0, P * (j0 + nb) + 1),
               slice(P * i0, P * (i0 + nb) + 1))
        uf = np.zeros(n_free)
        pf = np.zeros(n_free)
        uf[perm] = u_lat[box]
        pf[perm] = p_lat[box]
        inner = (slice(None), slice(1, -1), slice(1, -1), slice(1, -1))
        for got, ref in ((y_kp[box], opb.apply_tangent(uf, pf)), (y_f[box], opb.internal_force(uf))):
            ref_l = ref[perm]
            err = np.abs(got[inner] - ref_l[inner]).max() / np.abs(ref_l[inner]).max()
            assert err <= 1e-12, ((k0, j0, i0), err)


def test_explicit_consistent_mass_vs_reference():
    """the reference's own explicit_run (consistent mass, full
    Jacobi-PCG) -- per-step PCG counts +-1, final u, v within 1e-9."""
    g = load_golden("explicit")
    pb = gpu_problem("SDME_M", 3, 4, (3, 2, 2), (1.0, 0.5, 0.5), [("xmin", (0, 1, 2))])
    base = pb.traction_vector("xmax", [0.0, 0.0, 2.0e4])
    assert max_rel_err(base, g["load"]) <= TOL
    cfg = SolverConfig(precond="diagonal", tol=1e-12, maxit=100000, condense=False)
    traj = explicit_run(pb, ScaledLoad(base, lambda t: min(t / 5e-5, 1.0)), float(g["dt"]), int(g["steps"]),
                        cfg=cfg, mass="consistent")
    ref = [int(r[1]) for r in g["pcg_rows"]]
    got = [r["iterations"] for r in traj.stats.rows]
    assert len(ref) == len(got) and max(abs(a - b) for a, b in zip(ref, got)) <= 1
    assert max_rel_err(traj.state.u, g["u"]) <= 1e-9
    assert max_rel_err(traj.state.v, g["v"]) <= 1e-9


# ------------------------------------------------------------------------------
# Property tests mirroring the reference suite (test_femcore.py, test_acceptance.py
# criterion 7, test_dynamics.py), run on the GPU path.

KINDS5 = ("LagrangeGLL", "ModalJacobi", "SDME_M", "SDME_K", "SDME_H")
RMAT = NeoHookean.from_engineering(1000.0, 0.3, 1.0)  # test_femcore.py:13


@pytest.mark.parametrize("tag", KINDS5)
def test_rigid_translation_zero_force(tag):
    """test_femcore.py:30-34: a rigid translation produces no internal force."""
    pb = gpu_problem(tag, 3, 4, (2, 2, 2), (1.0, 1.0, 1.0), mat=RMAT)
    u = pb.constant_field([0.2, -0.1, 0.3])
    assert np.abs(pb.internal_force(u)).max() <= 1e-9
    assert np.abs(pb.internal_force(np.zeros(pb.n_free))).max() <= 1e-14


@pytest.mark.parametrize("tag", KINDS5)
def test_constant_stress_divergence_theorem(tag):
    """test_femcore.py:37-51: homogeneous stretch F = diag(1.1, 1, 1); the
    internal force equals the surface load of the constant first PK stress."""
    P = 3
    pb = gpu_problem(tag, P, P + 1, (2, 2, 2), (1.0, 1.0, 1.0), mat=RMAT)
    # u = (F - I) X is linear and exact in every basis: X = (X0 + h/2) 1 + (h/2) xi
    from paper_2104_13466_b200.basis import constant_coeffs, gll_rule
    if pb.basis.kind.is_nodal:
        nodes = gll_rule(P + 1).points
        lin = np.concatenate(([nodes[0], nodes[-1]], nodes[1:-1]))
    else:
        lin = np.linalg.solve(pb.basis.transform.T, np.array([-1.0, 1.0] + [0.0] * (P - 1)))
    const = constant_coeffs(pb.basis)
    reorder = lambda c: np.concatenate(([c[0]], c[2:], [c[1]]))  # function -> lattice-local order
    xs = np.empty(P * pb.mesh.divisions[0] + 1)
    h = pb.mesh.h[0]
    for e in range(pb.mesh.divisions[0]):
        xs[P * e:P * e + P + 1] = (e * h + 0.5 * h) * reorder(const) + 0.5 * h * reorder(lin)
    ones = [np.tile(reorder(const)[:P], pb.mesh.divisions[d]).tolist() + [const[1]] for d in (1, 2)]
    lat = np.zeros(pb.lattice_shape)
    lat[0] = 0.1 * np.einsum("z,y,x->zyx", ones[1], ones[0], xs)
    u = pb.to_free(lat)
    r = pb.internal_force(u)
    mu, lam = RMAT.mu, RMAT.lambda_lame
    Fh = np.diag([1.1, 1.0, 1.0])
    C = Fh.T @ Fh
    Ci = np.linalg.inv(C)
    S = mu * (np.eye(3) - Ci) + lam * 0.5 * np.log(np.linalg.det(C)) * Ci
    P1 = Fh @ S
    surf = np.zeros(pb.n_free)
    for tagf, nrm in (("xmin", [-1, 0, 0]), ("xmax", [1, 0, 0]), ("ymin", [0, -1, 0]), ("ymax", [0, 1, 0]),
                      ("zmin", [0, 0, -1]), ("zmax", [0, 0, 1])):
        surf += pb.traction_vector(tagf, P1 @ np.array(nrm, dtype=float))
    assert np.abs(r - surf).max() <= 1e-8 * np.abs(r).max()


@pytest.mark.parametrize("tag", KINDS5)
@pytest.mark.parametrize("P", [2, 4])
def test_global_fd_tangent_consistency(tag, P):
    """test_acceptance.py:196-221 (criterion 7): central FD of f_int along a
    random direction vs the matrix-free K_T, <= 1e-5 relative, Dirichlet."""
    pb = gpu_problem(tag, P, P + 1, (2, 2, 2), (1.0, 1.0, 1.0), [("xmin", (0, 1, 2))], mat=RMAT)
    rng = np.random.default_rng(4)
    u0 = 0.01 * rng.uniform(-1, 1, pb.n_free) / P
    du = rng.standard_normal(pb.n_free)
    du /= np.linalg.norm(du)
    eps = 1e-6
    fd = (pb.internal_force(u0 + eps * du) - pb.internal_force(u0 - eps * du)) / (2 * eps)
    kd = pb.apply_tangent(u0, du)
    assert np.linalg.norm(fd - kd) <= 1e-5 * np.linalg.norm(kd)


@pytest.mark.parametrize("tag", KINDS5)
def test_tangent_symmetry_and_mass_conservation(tag):
    """test_femcore.py:92-108: K_T symmetric (q.Kp = p.Kq); c.M c = rho * volume
    for the constant field c (one component)."""
    pb = gpu_problem(tag, 3, 4, (2, 3, 2), (1.0, 1.5, 1.0), [("xmin", (0, 1, 2))], mat=RMAT)
    rng = np.random.default_rng(9)
    u = 1e-3 * rng.uniform(-1, 1, pb.n_free)
    p, q = rng.standard_normal(pb.n_free), rng.standard_normal(pb.n_free)
    a, b = q @ pb.apply_tangent(u, p), p @ pb.apply_tangent(u, q)
    assert abs(a - b) <= 1e-10 * max(abs(a), abs(b))
    pb2 = gpu_problem(tag, 3, 4, (2, 3, 2), (1.0, 1.5, 1.0), mat=RMAT)
    c = pb2.constant_field([1.0, 0.0, 0.0])
    assert c @ pb2.mass_apply(c) == pytest.approx(RMAT.rho0 * 1.5, rel=1e-12)


def test_newmark_rest_state_stays_at_rest():
    """test_dynamics.py:113-118: zero load, zero state -> zero Newton iterations."""
    pb = gpu_problem("SDME_M", 2, 3, (2, 2, 2), (1.0, 1.0, 1.0), mat=RMAT)
    traj = newmark_run(pb, lambda t: np.zeros(pb.n_free), 1e-3, 5)
    assert np.abs(traj.state.u).max() <= 1e-14 and traj.newton_iters == [0] * 5


def test_explicit_momentum_conservation():
    """test_dynamics.py:62-81: uniform initial velocity, no force, lumped mass:
    momentum conserved to 1e-10 and the motion is exactly u(T) = T v0."""
    from paper_2104_13466_b200.dynamics import ScaledLoad
    pb = gpu_problem("SDME_M", 3, 4, (2, 2, 2), (1.0, 1.0, 1.0), mat=RMAT)
    v0 = pb.constant_field([0.0, 0.3, 0.0])
    ey = pb.constant_field([0.0, 1.0, 0.0])
    traj = explicit_run(pb, ScaledLoad(np.zeros(pb.n_free), lambda t: 0.0), 1e-3, 100, v0=v0, mass="lumped")
    p0, p1 = ey @ pb.mass_apply(v0), ey @ pb.mass_apply(traj.state.v)
    assert abs(p1 - p0) <= 1e-10 * abs(p0)
    ut = traj.state.t * v0
    assert np.abs(traj.state.u - ut).max() <= 1e-8 * np.abs(ut).max()


@pytest.mark.parametrize("tag,P,m", [("SDME_M", 4, 6), ("LagrangeGLL", 3, 4), ("ModalJacobi", 2, 3),
                                     ("SDME_H", 6, 7)])
def test_evector_mode_matches_colour_passes(tag, P, m, monkeypatch):
    """Small meshes use one launch + deterministic gather (E-vector mode);
    large ones 8 colour passes with RED.  Both orders of summation agree to
    rounding, and each is bit-reproducible."""
    out = {}
    rng = np.random.default_rng(3)
    for mode in ("0", "1"):
        monkeypatch.setenv("SDME_EV", mode)
        pb = gpu_problem(tag, P, m, (3, 2, 2), (1.5, 1.0, 1.0), [("xmin", (0, 1, 2))])
        if mode == "0":
            u = 1e-3 * rng.uniform(-1, 1, pb.n_free)
            p = rng.standard_normal(pb.n_free)
        out[mode] = [pb.internal_force(u), pb.apply_tangent(u, p, c_m=3.0e4), pb.mass_apply(p),
                     pb.tangent_diagonal(u, c_m=3.0e4)]
        again = pb.apply_tangent(u, p, c_m=3.0e4)
        assert np.array_equal(again, out[mode][1])
    for a, b in zip(out["0"], out["1"]):
        assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()


@pytest.mark.parametrize("tag,P,m", [("SDME_M", 4, 5), ("LagrangeGLL", 2, 3), ("SDME_H", 6, 7)])
def test_pcg_operator_from_stored_quadrature_data_is_bit_identical(tag, P, m, monkeypatch):
    """sdme_pcg stores K = F^-T and ln J once per solve and iterates with them
    (MODE_PA); the solve is bit-identical to iterating with K(u).p from u."""
    rng = np.random.default_rng(11)
    res = {}
    for pa in ("1", "0"):
        monkeypatch.setenv("SDME_PA", pa)
        pb = gpu_problem(tag, P, m, (3, 2, 2), (1.5, 1.0, 1.0), [("xmin", (0, 1, 2))])
        if pa == "1":
            u = 1e-3 * rng.uniform(-1, 1, pb.n_free)
            b = rng.standard_normal(pb.n_free)
        x, st = pcg_gpu(pb, u, b, c_m=2.0e5, precond="diagonal", tol=1e-10, maxit=500)
        res[pa] = (x, st.iterations)
        uv, pv, yv = pb.vector().set_free(u), pb.vector().set_free(b), pb.vector()
        pb.time_op("setup", uv, pv, yv, 0.0, 1)
        pb.time_op("apply_pa", uv, pv, yv, 2.0e5, 1)
        assert np.array_equal(yv.free(), pb.apply_tangent(u, b, c_m=2.0e5))
    assert res["0"][1] == res["1"][1]
    assert np.array_equal(res["0"][0], res["1"][0])


@pytest.mark.parametrize("tag,P,m,div", [("SDME_M", 4, 5, (7, 6, 5)), ("SDME_H", 6, 7, (4, 3, 3)),
                                         ("LagrangeGLL", 3, 4, (6, 5, 4))])
def test_pcg_iteration_sequences_are_bit_identical(tag, P, m, div, monkeypatch):
    """The default PCG iteration on the TMA colour-pass path -- stored point data
    prefetched (P = 4: on the quintet kernel), colour passes linked by
    programmatic dependent launches inside the captured graph, alpha / beta
    evaluated inside the fused update kernels, A p zeroed by the p update (the
    default below 2^24 vector entries, SDME_PCG_CHAIN=9) or by its own launch
    overlapping the first pass (5), the start of the solve fused into two
    launches (SDME_PCG_START=0: separate ones) -- against the plain sequence
    (SDME_PCG_CHAIN=0, SDME_PDL=0: seven kernels per iteration, no PDL edges)
    on the warp-per-element kernel (SDME_VARIANT=12), and against plain
    launches without a graph (SDME_PCG_DIRECT=1): same iterates, bit for bit."""
    monkeypatch.setenv("SDME_EV", "0")
    rng = np.random.default_rng(5)
    res = []
    for env in ({}, {"SDME_PCG_CHAIN": "0", "SDME_PDL": "0", "SDME_VARIANT": "12", "SDME_PCG_START": "0"},
                {"SDME_PCG_DIRECT": "1"},
                {"SDME_PCG_CHAIN": "7"}, {"SDME_PCG_CHAIN": "5"}, {"SDME_PCG_CHAIN": "9", "SDME_PCG_DIRECT": "1"}, {"SDME_PCG_START": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        pb = gpu_problem(tag, P, m, div, tuple(d / 8 for d in div), [("xmin", (0, 1, 2)), ("ymax", (1,))])
        for k in env:
            monkeypatch.delenv(k)
        if not res:
            u = 1e-3 / 8 * rng.uniform(-1, 1, pb.n_free)
            b = rng.standard_normal(pb.n_free)
        x, st = pcg_gpu(pb, u, b, c_m=4.0e8, precond="diagonal", tol=1e-10, maxit=2000)
        x0, st0 = pcg_gpu(pb, u, b, c_m=0.0, precond="diagonal", tol=1e-6, maxit=20000)
        res.append((x, st.iterations, x0, st0.iterations))
    assert res[0][1] > 5 and res[0][3] > 5
    for r in res[1:]:
        assert r[1] == res[0][1] and r[3] == res[0][3]
        assert np.array_equal(r[0], res[0][0])
        assert np.array_equal(r[2], res[0][2])


# ------------------------------------------------------------------------------
# Implicit penalty contact: contact stiffness operator and
# newmark_run(contact=...) against the reference.

def _block(P, gap0=0.0):
    """test_contact.py:14-20: unit block gap0 above the y = 0 plane."""
    return GpuFemProblem(BoxMesh((1, 1, 1), (1.0, 1.0, 1.0), (0.0, gap0, 0.0)), build_basis(P, BasisKind("SDME_M")),
                         NeoHookean.from_engineering(100.0, 0.3, 1.0), gauss_rule(P + 1))


def test_contact_stiffness_is_force_jacobian_psd_and_matches_oracle():
    """test_contact.py:69-94: K_c is the negative force gradient (FD 1e-5),
    symmetric PSD; its action and diagonal equal the assembled oracle K_c."""
    pb = _block(3)
    plane = RigidObstacle(np.zeros(3), np.array([0.0, 1.0, 0.0]))
    c = GpuPenaltyContact(pb, plane, ContactParams(1e4), "ymin")
    rng = np.random.default_rng(0)
    u0 = pb.constant_field([0.0, -2e-3, 0.0]) + 1e-4 * rng.uniform(-1, 1, pb.n_free)
    du = rng.standard_normal(pb.n_free)
    du /= np.linalg.norm(du)
    fc = c.evaluate_forces(u0)
    kd = fc.stiffness @ du
    dg = fc.stiffness.diagonal()
    q = rng.standard_normal(pb.n_free)
    qk, dk = q @ (fc.stiffness @ du), du @ (fc.stiffness @ q)
    assert abs(qk - dk) <= 1e-12 * max(abs(qk), abs(dk))
    assert du @ kd >= 0.0
    h = 1e-7
    fd = (c.evaluate_forces(u0 + h * du).force - c.evaluate_forces(u0 - h * du).force) / (2 * h)
    assert np.abs(fd + kd).max() <= 1e-5 * np.abs(fd).max()
    opb = of.Problem(of.Mesh((1, 1, 1), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)), ob.Basis("SDME_M", 3),
                     of.Material(100.0, 0.3, 1.0), 4)
    oc = of.Contact(opb, [0.0, 0.0, 0.0], [0.0, 1.0, 0.0], 1e4, "ymin")
    ks = oc.stiffness(u0)
    assert max_rel_err(kd, ks @ du) <= TOL
    assert max_rel_err(dg, ks.diagonal()) <= TOL


def test_contact_stiffness_absent_without_penetration():
    """test_contact.py:45-51."""
    pb = _block(2, gap0=0.1)
    c = GpuPenaltyContact(pb, RigidObstacle(np.zeros(3), np.array([0.0, 1.0, 0.0])), ContactParams(1e4), "ymin")
    fc = c.evaluate_forces(np.zeros(pb.n_free))
    assert fc.stiffness is None and not fc.active.any() and fc.settled
    assert np.abs(fc.force).max() == 0.0


def test_implicit_contact_newmark_vs_reference():
    """Reference newmark_run with penalty contact (bar impact, shortened):
    Newton counts equal, PCG counts +-1, penalty stepping history equal,
    final u, v, a within 1e-9."""
    from paper_2104_13466_b200.dynamics import ScaledLoad

    g = load_golden("impact")
    pb = GpuFemProblem(BoxMesh((1, 2, 1), (0.05, 0.1, 0.05), (-0.025, 0.0005, -0.025)),
                       build_basis(3, BasisKind("SDME_H")), NeoHookean.from_engineering(100.0, 0.3, 1.0),
                       gauss_rule(4))
    c = GpuPenaltyContact(pb, RigidObstacle(np.zeros(3), np.array([0.0, 1.0, 0.0])),
                          ContactParams(1e4, deps_n=1e3, gap_tol=3e-5, stress_tol=1e-2), "ymin")
    cfg = SolverConfig(precond="diagonal", tol=1e-12, maxit=100000, condense=False)
    traj = newmark_run(pb, ScaledLoad(np.zeros(pb.n_free), lambda t: 0.0), float(g["dt"]), int(g["steps"]),
                       newton_tol=1e-10, v0=g["v0"], cfg=cfg, contact=c)
    assert traj.newton_iters == list(g["newton_iters"])
    its = np.array([r["iterations"] for r in traj.stats.rows if r["step"] >= 0])
    assert np.all(np.abs(its - g["pcg_rows"][1:, 2]) <= 1)
    hist = np.array(c.history)
    assert np.array_equal(hist[:, 0], g["history"][:, 0])
    assert np.array_equal(hist[:, 3], g["history"][:, 3])
    assert max_rel_err(hist[:, 1], g["history"][:, 1]) <= 1e-8
    assert max_rel_err(traj.state.u, g["u"]) <= 1e-9
    assert max_rel_err(traj.state.v, g["v"]) <= 1e-9
    assert max_rel_err(traj.state.a, g["a"]) <= 1e-9


def test_bar_impact_energy_criterion9_vs_reference():
    """Full bar-impact scenario (scenarios.py:92-113) on the GPU with energy
    tracking: energy rows, penalty history and final state vs the reference
    run; acceptance criterion 9 (test_acceptance.py:249-264) holds."""
    g = load_golden("impact_energy")
    pb = GpuFemProblem(BoxMesh((1, 2, 1), (0.05, 0.1, 0.05), (-0.025, 0.005, -0.025)),
                       build_basis(3, BasisKind("SDME_H")), NeoHookean.from_engineering(100.0, 0.3, 1.0),
                       gauss_rule(4))
    c = GpuPenaltyContact(pb, RigidObstacle(np.zeros(3), np.array([0.0, 1.0, 0.0])),
                          ContactParams(1e4, deps_n=1e3, gap_tol=1e-3, stress_tol=1e-2), "ymin")
    cfg = SolverConfig(precond="diagonal", tol=1e-12, maxit=100000, condense=False)
    traj = newmark_run(pb, ScaledLoad(np.zeros(pb.n_free), lambda t: 0.0), 1e-3, 200, newton_tol=1e-10,
                       v0=g["v0"], cfg=cfg, contact=c, track_energy=True)
    assert traj.newton_iters == list(g["newton_iters"])
    en = np.array(traj.energy)
    assert max_rel_err(en, g["energy"]) <= 1e-8
    assert np.array_equal(np.array(c.history)[:, 0], g["history"][:, 0])
    assert max_rel_err(traj.state.u, g["u"]) <= 1e-9
    total = en[:, 1] + en[:, 2] + en[:, 3]
    drift = float(np.abs(total - total[0]).max() / total[0])
    ey = pb.constant_field([0.0, 1.0, 0.0])
    vy = float(ey @ pb.mass_apply(traj.state.v)) / (0.05 * 0.1 * 0.05)
    pen = max(h[1] for h in c.history)
    assert pen <= 1e-3 and min(h[2] for h in c.history) >= 0.0 and drift <= 0.02 and vy > 0.0
    assert vy == pytest.approx(float(g["vy"]), rel=1e-8)


def test_strain_energy_vs_oracle():
    """total_strain_energy (femcore.py:374-378) at a seeded admissible state."""
    pb = gpu_problem("SDME_K", 3, 4, (3, 2, 2), (1.5, 1.0, 1.0), [("xmin", (0, 1, 2))])
    rng = np.random.default_rng(21)
    u = 1e-3 * rng.uniform(-1, 1, pb.n_free)
    opb = of.Problem(of.Mesh((3, 2, 2), (1.5, 1.0, 1.0)), ob.Basis("SDME_K", 3), OMAT, 4, [("xmin", (0, 1, 2))])
    assert pb.total_strain_energy(u) == pytest.approx(opb.total_strain_energy(u), rel=1e-12)


@pytest.mark.parametrize("tag", KINDS5)
def test_collocated_path_vs_oracle(tag, monkeypatch):
    """P = 4, m = 5 on colour passes runs the collocated kernels
    (element_col.cuh) for f_int, K.p (+ c_m M p) and the PCG operator; all
    agree with the oracle to 1e-12, and with the v3 kernels (SDME_VARIANT=10)."""
    monkeypatch.setenv("SDME_EV", "0")
    div, L = (3, 2, 2), (1.5, 1.0, 1.0)
    opb = of.Problem(of.Mesh(div, L), ob.Basis(tag, 4), OMAT, 5, [("xmin", (0, 1, 2))])
    rng = np.random.default_rng(17)
    u = 1e-3 * rng.uniform(-1, 1, opb.n_free)
    p = rng.standard_normal(opb.n_free)
    ref_f = opb.internal_force(u)
    ref_kp = opb.assemble(u, 1.0, 2.0e5) @ p
    out = {}
    for variant in ("0", "10"):
        monkeypatch.setenv("SDME_VARIANT", variant)
        pb = gpu_problem(tag, 4, 5, div, L, [("xmin", (0, 1, 2))])
        f, kp = pb.internal_force(u), pb.apply_tangent(u, p, c_m=2.0e5)
        assert max_rel_err(f, ref_f) <= TOL
        assert max_rel_err(kp, ref_kp) <= TOL
        uv, pv, yv = pb.vector().set_free(u), pb.vector().set_free(p), pb.vector()
        pb.time_op("setup", uv, pv, yv, 0.0, 1)
        pb.time_op("apply_pa", uv, pv, yv, 2.0e5, 1)
        assert np.array_equal(yv.free(), kp)
        out[variant] = kp
    assert max_rel_err(out["0"], out["10"]) <= 1e-13


@pytest.mark.parametrize("tag,P,div", [("LagrangeGLL", 1, (3, 2, 2)), ("ModalJacobi", 2, (3, 2, 2)),
                                       ("SDME_H", 3, (3, 2, 1)), ("SDME_K", 3, (2, 3, 2)),
                                       ("SDME_M", 4, (3, 2, 2)), ("LagrangeGLL", 4, (2, 3, 1)),
                                       ("ModalJacobi", 5, (3, 1, 2)), ("SDME_H", 6, (2, 2, 1)),
                                       ("SDME_M", 7, (1, 2, 1)), ("SDME_K", 8, (2, 1, 1))])
def test_tma_box_path_vs_oracle(tag, P, div, monkeypatch):
    """Colour passes load each element box with a TMA tensor copy and add the
    result back with a bulk tensor reduce-add (tma.cuh; pitched lattice rows):
    the collocated kernels at even P >= 4, the all-component kernel at P <= 3
    (boxes from the even x at or below the element start, so odd P shifts the
    rows by one); odd P >= 5 keeps the cp.async / RED kernel.  Dirichlet planes on three faces (the
    output box zeroes them), odd and even element counts (the pitch slot of
    the last element is dropped at the lattice edge): f_int and K.p + c_m M p
    agree with the oracle to 1e-12, with the per-lane cp.async / RED kernel
    (SDME_VARIANT=11) to 1e-13, and reruns are bit-identical."""
    monkeypatch.setenv("SDME_EV", "0")
    L = tuple(0.5 * d for d in div)
    dr = [("xmin", (0, 1, 2)), ("xmax", (0,)), ("ymax", (1, 2))]
    opb = of.Problem(of.Mesh(div, L), ob.Basis(tag, P), OMAT, P + 1, dr)
    rng = np.random.default_rng(29)
    u = 1e-3 * rng.uniform(-1, 1, opb.n_free)
    p = rng.standard_normal(opb.n_free)
    ref_f = opb.internal_force(u)
    ref_kp = opb.assemble(u, 1.0, 2.0e5) @ p
    out = {}
    for variant in ("0", "11"):
        monkeypatch.setenv("SDME_VARIANT", variant)
        pb = gpu_problem(tag, P, P + 1, div, L, dr)
        f, kp = pb.internal_force(u), pb.apply_tangent(u, p, c_m=2.0e5)
        assert max_rel_err(f, ref_f) <= TOL
        assert max_rel_err(kp, ref_kp) <= TOL
        assert np.array_equal(pb.apply_tangent(u, p, c_m=2.0e5).view(np.int64), kp.view(np.int64))
        x, st = pcg_gpu(pb, u, f, c_m=2.0e5, tol=1e-10)
        out[variant] = (f, kp, x, st.iterations)
    for a, b in zip(out["0"][:2], out["11"][:2]):
        assert max_rel_err(a, b) <= 1e-13
    assert abs(out["0"][3] - out["11"][3]) <= 1
    assert max_rel_err(out["0"][2], out["11"][2]) <= 1e-9


@pytest.mark.parametrize("tag,div,L", [("SDME_M", (3, 2, 2), (1.5, 1.0, 1.0)), ("LagrangeGLL", (2, 3, 1), (1.0, 1.5, 0.5)),
                                       ("ModalJacobi", (4, 1, 3), (1.0, 0.5, 2.25)), ("SDME_K", (1, 1, 1), (0.5, 0.5, 0.5))])
def test_quintet_diagonal_vs_oracle(tag, div, L, monkeypatch):
    """diag(K_T(u) + c_m M) at P = 4, m = 5 on the colour-pass path runs on the
    quintet kernel (element_q5d.cuh: collocated grad u, point coefficients in
    the rank-one form mu delta + (lam + mu - lam ln J) K K, 6 + 6 + 1 stage
    passes per component, bulk tensor reduce-add).  It agrees with the
    diagonal of the oracle's assembled operator (solver.py:105-110) to 1e-12
    on cubic and non-cubic elements, with Dirichlet planes, ghost elements in
    the last quintet and a finite deformation; with element_diag3
    (SDME_VARIANT=13) to 1e-13; reruns are bit-identical."""
    monkeypatch.setenv("SDME_EV", "0")
    dr = [("xmin", (0, 1, 2)), ("ymax", (1,))]
    opb = of.Problem(of.Mesh(div, L), ob.Basis(tag, 4), OMAT, 5, dr)
    rng = np.random.default_rng(41)
    u = 2e-2 * rng.uniform(-1, 1, opb.n_free)
    out = {}
    for variant in ("0", "13"):
        monkeypatch.setenv("SDME_VARIANT", variant)
        pb = gpu_problem(tag, 4, 5, div, L, dr)
        for cm in (0.0, 2.0e5):
            d = pb.tangent_diagonal(u, cm)
            assert max_rel_err(d, opb.assemble(u, 1.0, cm).diagonal()) <= TOL
            assert np.array_equal(pb.tangent_diagonal(u, cm).view(np.int64), d.view(np.int64))
            out[variant, cm] = d
    for cm in (0.0, 2.0e5):
        assert max_rel_err(out["0", cm], out["13", cm]) <= 1e-13


@pytest.mark.parametrize("ev", ["0", "1"])
def test_apply_batch_matches_single_calls(ev, monkeypatch):
    """apply_tangent_batch (pipelined H2D / operator / D2H, sdme_apply_batch)
    returns exactly the results of one apply_tangent call per pair."""
    monkeypatch.setenv("SDME_EV", ev)
    from paper_2104_13466_b200.native import pinned_empty
    pb = gpu_problem("SDME_M", 4, 5, (3, 2, 2), (1.5, 1.0, 1.0), [("xmin", (0, 1, 2))])
    rng = np.random.default_rng(5)
    us, ps = [], []
    for _ in range(5):
        u, p = pinned_empty(pb.n_free), pinned_empty(pb.n_free)
        u[:] = 1e-3 * rng.uniform(-1, 1, pb.n_free)
        p[:] = rng.standard_normal(pb.n_free)
        us.append(u)
        ps.append(p)
    got = pb.apply_tangent_batch(us, ps, c_m=3.0e4)
    for u, p, y in zip(us, ps, got):
        assert np.array_equal(y.view(np.int64), pb.apply_tangent(u, p, 3.0e4).view(np.int64))


@pytest.mark.parametrize("P,div", [(2, (1, 1, 1)), (3, (1, 3, 1)), (4, (1, 1, 3)), (4, (5, 1, 1)), (3, (4, 2, 1)),
                                   (6, (1, 2, 1)), (8, (1, 1, 1))])
def test_tma_paths_on_thin_meshes(P, div, monkeypatch):
    """Single-element rows / columns / layers on the colour-pass TMA paths:
    boxes at both lattice ends (out-of-tensor slots dropped), every face
    Dirichlet-constrained for one component, the odd-P row shift at odd x."""
    monkeypatch.setenv("SDME_EV", "0")
    L = tuple(0.25 * d for d in div)
    dr = [("xmin", (0,)), ("xmax", (1,)), ("ymin", (2,)), ("zmax", (0, 1))]
    opb = of.Problem(of.Mesh(div, L), ob.Basis("SDME_M", P), OMAT, P + 1, dr)
    pb = gpu_problem("SDME_M", P, P + 1, div, L, dr)
    rng = np.random.default_rng(P * 7 + sum(div))
    u = 1e-3 * rng.uniform(-1, 1, opb.n_free)
    p = rng.standard_normal(opb.n_free)
    assert max_rel_err(pb.internal_force(u), opb.internal_force(u)) <= TOL
    assert max_rel_err(pb.apply_tangent(u, p, 2.0e5), opb.apply_tangent(u, p, 2.0e5)) <= TOL
    assert max_rel_err(pb.mass_apply(p), opb.mass() @ p) <= TOL


def test_explicit_chunks_match_per_step_and_report_first_inversion():
    """explicit_run runs steps in device chunks (sdme_explicit_steps) between
    host-visible steps; the result equals the step-by-step path bitwise, and an
    inversion inside a chunk is replayed so the error names the same element
    and point as the per-step path (the reference raises at the first
    inverted step, femcore.py:92-93)."""
    pb = gpu_problem("SDME_M", 3, 4, (3, 2, 2), (0.3, 0.2, 0.2), [("xmin", (0, 1, 2))])
    v0 = pb.constant_field([0.0, 0.0, 1.0])
    zero = np.zeros(pb.n_free)
    a = explicit_run(pb, None, 1e-6, 40, v0=v0, mass="lumped")             # chunked
    b = explicit_run(pb, lambda t: zero, 1e-6, 40, v0=v0, mass="lumped")   # callable load: per step
    assert np.array_equal(a.state.u.view(np.int64), b.state.u.view(np.int64))
    assert np.array_equal(a.state.v.view(np.int64), b.state.v.view(np.int64))
    fast = pb.constant_field([0.0, 0.0, 3.0e3])
    rng = np.random.default_rng(2)
    fast = fast * (1.0 + rng.uniform(-1, 1, pb.n_free))  # non-uniform: elements invert after some steps
    errs = []
    for load in (None, lambda t: zero):
        with pytest.raises(ElementInversionError) as ei:
            explicit_run(pb, load, 1e-5, 400, v0=fast, mass="lumped")
        errs.append((ei.value.elem_id, ei.value.qp))
    assert errs[0] == errs[1]


def test_gll_collocation_mass_is_diagonal():
    """test_femcore.py:111-116: the nodal basis with the (P+1)-point GLL rule
    (collocation_mass=True, femcore.py:284-288) has an exactly diagonal mass:
    every probed column of M has one non-zero, on the diagonal, positive; and
    M p agrees with (M 1) * p to rounding."""
    from paper_2104_13466_b200 import gll_rule
    pb = GpuFemProblem(BoxMesh((3, 2, 2), (1.5, 1.0, 1.0)), build_basis(3, BasisKind("LagrangeGLL")), MAT,
                       gll_rule(4), [("xmin", (0, 1, 2))])
    rng = np.random.default_rng(4)
    for j in rng.choice(pb.n_free, 12, replace=False):
        e = np.zeros(pb.n_free)
        e[j] = 1.0
        col = pb.mass_apply(e)
        assert np.count_nonzero(col) == 1 and col[j] > 0.0
    d = pb.mass_apply(np.ones(pb.n_free))
    p = rng.standard_normal(pb.n_free)
    assert np.abs(pb.mass_apply(p) - d * p).max() <= 1e-14 * np.abs(d * p).max()


def test_pcg_diagonal_operator_converges_in_one_iteration():
    """test_solver.py:25-31 on the FE operator: the GLL collocation mass is
    diagonal, so Jacobi-PCG on c_m M converges in one iteration to b / diag."""
    from paper_2104_13466_b200 import gll_rule
    pb = GpuFemProblem(BoxMesh((2, 2, 1), (1.0, 1.0, 0.5)), build_basis(3, BasisKind("LagrangeGLL")), MAT,
                       gll_rule(4), [("xmin", (0, 1, 2))])
    b = np.random.default_rng(6).standard_normal(pb.n_free)
    x, st = pcg_gpu(pb, None, b, c_m=2.0, c_k=0.0, precond="diagonal", tol=1e-12)
    assert st.iterations == 1
    d = 2.0 * pb.mass_apply(np.ones(pb.n_free))
    assert np.abs(x - b / d).max() <= 1e-13 * np.abs(b / d).max()


def test_pcg_error_monotone_in_a_norm():
    """test_solver.py:90-105 on the FE operator A = K_T(u) + c_m M: tighter
    tolerances never need fewer iterations nor give a larger A-norm error."""
    pb = gpu_problem("SDME_M", 3, 4, (2, 2, 2), (1.0, 1.0, 1.0), [("xmin", (0, 1, 2))])
    rng = np.random.default_rng(8)
    u = 1e-3 * rng.uniform(-1, 1, pb.n_free)
    b = rng.standard_normal(pb.n_free)
    cm = 1.0e6
    x_ex, _ = pcg_gpu(pb, u, b, c_m=cm, tol=1e-14, maxit=100000)
    errs, iters = [], []
    for tol in (1e-2, 1e-4, 1e-6, 1e-8, 1e-10):
        x, st = pcg_gpu(pb, u, b, c_m=cm, tol=tol, maxit=100000)
        e = x - x_ex
        errs.append(np.sqrt(e @ pb.apply_tangent(u, e, cm)))
        iters.append(st.iterations)
    assert all(i2 >= i1 for i1, i2 in zip(iters, iters[1:]))
    assert all(e2 <= e1 * (1 + 1e-10) for e1, e2 in zip(errs, errs[1:]))


def test_mass_spd_and_tangent_at_reference_state():
    """test_femcore.py:119-125 (p.Mp > 0) and :81-89 (K_T(0) is the linear
    stiffness: compared with the oracle's dense tangent at u = 0)."""
    pb = gpu_problem("SDME_H", 3, 4, (2, 1, 2), (1.0, 0.5, 1.0), [("zmin", (0, 1, 2))])
    opb = of.Problem(of.Mesh((2, 1, 2), (1.0, 0.5, 1.0)), ob.Basis("SDME_H", 3), OMAT, 4, [("zmin", (0, 1, 2))])
    rng = np.random.default_rng(9)
    for _ in range(5):
        p = rng.standard_normal(pb.n_free)
        assert p @ pb.mass_apply(p) > 0.0
    p = rng.standard_normal(pb.n_free)
    zero = np.zeros(pb.n_free)
    assert max_rel_err(pb.apply_tangent(zero, p), opb.apply_tangent(zero, p)) <= TOL
