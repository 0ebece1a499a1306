"""Generate golden vectors from the REAL reference package (sdmefem).

Run in the build container, where the reference tree exists:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes small compressed .npz fixtures next to this file.  Nothing at test or
bench time reads /root/reference; the fixtures are the pin for both the oracle
(tests/test_oracle_golden.py) and the GPU path (tests/test_gpu_parity.py).
All inputs are seeded (numpy default_rng) and stored alongside the outputs.
"""

from __future__ import annotations

import os
import time

import numpy as np

from sdmefem.basis1d import BasisKind, build_basis
from sdmefem.contact import ContactParams, PenaltyContact, RigidObstacle
from sdmefem.dynamics import SolverConfig, newmark_run
from sdmefem.femcore import (FemProblem, build_face_tables, element_internal_force,
                             element_mass, element_tangent)
from sdmefem.material import NeoHookean
from sdmefem.meshdof import Mesh, build_dofmap, gen_box_mesh
from sdmefem.quadrature import gauss_rule
from sdmefem.solver import pcg
from sdmefem.tensorelem import TensorElement

HERE = os.path.dirname(os.path.abspath(__file__))
KINDS = ("LagrangeGLL", "ModalJacobi", "SDME_M", "SDME_K", "SDME_H")
MAT = NeoHookean.from_engineering(1.0e7, 0.3, 1.0e3)


def problem(tag, P, div, lengths, m, dirichlet=None, origin=None):
    mesh = gen_box_mesh(div, lengths, origin)
    el = TensorElement.create(3, build_basis(P, BasisKind(tag)))
    dm = build_dofmap(mesh, el, dirichlet)
    return FemProblem(mesh, el, dm, MAT, rule=gauss_rule(m))


def smooth_plus_noise(prob, amp, noise, seed):
    """Seeded admissible displacement: L2 projection of a smooth field plus
    small i.i.d. coefficient noise (keeps det F > 0)."""
    rng = np.random.default_rng(seed)
    u = prob.l2_project(lambda x: amp * np.column_stack(
        [np.sin(2 * np.pi * (x[:, 0] + x[:, 1] + x[:, 2])),
         np.cos(2 * np.pi * (x[:, 0] - 0.5 * x[:, 2])),
         x[:, 0] * x[:, 1]]))
    return u + noise * rng.uniform(-1.0, 1.0, prob.n_free)


def gen_basis():
    out = {}
    for tag in KINDS:
        for P in (1, 2, 3, 4, 6, 8):
            if P == 1 and tag.startswith("SDME"):
                continue
            b = build_basis(P, BasisKind(tag))
            out[f"{tag}_P{P}_T"] = b.transform
            for m in (P + 1, P + 2):
                bb = b.with_rule(gauss_rule(m))
                out[f"{tag}_P{P}_m{m}_B"] = bb.values.T
                out[f"{tag}_P{P}_m{m}_D"] = bb.derivs.T
    np.savez_compressed(os.path.join(HERE, "basis.npz"), **out)


def gen_elements():
    """Single-element meshes: the global vector is the element vector in
    reference local order (function-major, component fastest)."""
    out = {}
    cases = []
    for tag in KINDS:
        for P in (2, 3, 4, 6, 8):
            for m in (P + 1, P + 2):
                cases.append((tag, P, m, (1 / 64,) * 3))
    cases += [("SDME_M", 4, 5, (0.5, 0.3, 0.7)), ("LagrangeGLL", 3, 5, (0.2, 1.0, 0.4)),
              ("ModalJacobi", 2, 3, (1.0, 1.0, 1.0))]
    for ci, (tag, P, m, h) in enumerate(cases):
        prob = problem(tag, P, (1, 1, 1), h, m)
        rng = np.random.default_rng(100 + ci)
        nf = prob.n_free
        scale = 0.05 * min(h) / P
        u = scale * rng.uniform(-1, 1, nf)
        p = rng.standard_normal(nf)
        tab = prob.tables[0]
        ue = prob.gather(0, u)
        r = element_internal_force(tab, MAT, ue, 0)
        k = element_tangent(tab, MAT, ue, 0)
        mm = element_mass(tab, MAT, 3)
        c_m = 1.0 / (0.25 * 1e-4 ** 2)
        key = f"c{ci}"
        out[key + "_meta"] = np.array([KINDS.index(tag), P, m, *h])
        out[key + "_u"] = u
        out[key + "_p"] = p
        out[key + "_fint"] = r
        pe = prob.gather(0, p).reshape(-1)
        out[key + "_kp"] = k @ pe
        out[key + "_mp"] = mm @ pe
        out[key + "_diag"] = np.diag(k + c_m * mm)
        out[key + "_cm"] = np.array(c_m)
    np.savez_compressed(os.path.join(HERE, "elements.npz"), **out)


def gen_global():
    """Multi-element meshes with Dirichlet faces, reference free order."""
    out = {}
    cases = [("SDME_M", 4, 5, (2, 3, 2), (1.0, 1.5, 1.0), [("xmin", (0, 1, 2))]),
             ("LagrangeGLL", 3, 5, (3, 2, 2), (1.0, 1.0, 0.5), [("xmin", (0, 1, 2)), ("zmax", (2,))]),
             ("ModalJacobi", 2, 3, (2, 2, 3), (0.5, 0.5, 1.0), None),
             ("SDME_H", 3, 4, (2, 2, 2), (1.0, 1.0, 1.0), [("ymin", (1,))])]
    for ci, (tag, P, m, div, L, dr) in enumerate(cases):
        prob = problem(tag, P, div, L, m, dr)
        u = smooth_plus_noise(prob, 0.01, 1e-4, 7 + ci)
        rng = np.random.default_rng(50 + ci)
        p = rng.standard_normal(prob.n_free)
        c_m = 3.0e4
        kt = prob.tangent(u)
        mass = prob.mass()
        eff = kt + c_m * mass
        key = f"g{ci}"
        out[key + "_meta"] = np.array([KINDS.index(tag), P, m, *div, *L])
        out[key + "_dir"] = np.array([[["xmin", "xmax", "ymin", "ymax", "zmin", "zmax"].index(t), c]
                                      for t, cs in (dr or []) for c in cs]).reshape(-1, 2)
        out[key + "_u"] = u
        out[key + "_p"] = p
        out[key + "_fint"] = prob.internal_force(u)
        out[key + "_kp"] = kt @ p
        out[key + "_mp"] = mass @ p
        out[key + "_diag"] = eff.diagonal()
        out[key + "_cm"] = np.array(c_m)
        b = prob.internal_force(u) + 1e3 * p
        x, st = pcg(eff, b, precond="diagonal", tol=1e-10, maxit=100000)
        out[key + "_pcg_b"] = b
        out[key + "_pcg_x"] = x
        out[key + "_pcg_iters"] = np.array(st.iterations)
    np.savez_compressed(os.path.join(HERE, "global.npz"), **out)


def gen_config1():
    """BASELINE config 1: 4^3 P=4 SDME, (P+2)^3 Gauss, Newmark 10 steps,
    Jacobi-PCG 1e-10 full system."""
    P, m = 4, 6
    prob = problem("SDME_M", P, (4, 4, 4), (1.0, 1.0, 1.0), m, [("xmin", (0, 1, 2))])
    faces = build_face_tables(prob.mesh, prob.element, "xmax", prob.rule)
    base = prob.traction_vector(faces, lambda f: np.tile([0.0, 0.0, 1.0e5], (len(f.pts), 1)))
    dt = 1e-4
    ramp = 10 * dt
    load = lambda t: base * min(t / ramp, 1.0)
    cfg = SolverConfig(precond="diagonal", tol=1e-10, maxit=200000, condense=False)
    t0 = time.perf_counter()
    traj = newmark_run(prob, load, dt, 10, newton_tol=1e-8, cfg=cfg)
    wall = time.perf_counter() - t0
    rows = [(r["step"], r["newton_iter"], r["iterations"]) for r in traj.stats.rows]
    np.savez_compressed(os.path.join(HERE, "config1.npz"), u=traj.state.u, v=traj.state.v,
                        a=traj.state.a, load=base, newton_iters=np.array(traj.newton_iters),
                        pcg_rows=np.array(rows), wall_s=np.array(wall))
    print("config1", wall, "s", traj.newton_iters, [r[2] for r in rows])


def gen_contact():
    """Contact force + D6 explicit restatement loop from reference pieces."""
    out = {}
    P = 3
    prob = problem("SDME_M", P, (3, 2, 2), (0.3, 0.2, 0.2), P + 1, None,
                   origin=(0.0, 0.0, 0.0))
    obst = RigidObstacle(np.array([-1e-3, 0.0, 0.0]), np.array([1.0, 0.0, 0.0]))
    cont = PenaltyContact(prob, obst, ContactParams(1e10), "xmin")
    rng = np.random.default_rng(3)
    u = prob.l2_project(lambda x: MAT.rho0 * np.tile([-2e-3, 0.0, 0.0], (len(x), 1)))
    u = u + 1e-4 * rng.uniform(-1, 1, prob.n_free)
    fc = cont.evaluate_forces(u)
    out["u"] = u
    out["force"] = fc.force
    out["gaps"] = fc.gaps
    # D6 explicit loop: lumped mass, contact, v0 = -10 m/s in x
    ml = np.asarray(prob.mass().sum(axis=1)).ravel()
    v0 = prob.l2_project(lambda x: MAT.rho0 * np.tile([-10.0, 0.0, 0.0], (len(x), 1)))
    dt = 2e-7
    n_steps = 40
    uu = np.zeros(prob.n_free)
    obst2 = RigidObstacle(np.array([-2e-5, 0.0, 0.0]), np.array([1.0, 0.0, 0.0]))
    cont2 = PenaltyContact(prob, obst2, ContactParams(1e10), "xmin")

    def psi(uk):
        return -prob.internal_force(uk) + cont2.evaluate_forces(uk).force

    a0 = psi(uu) / ml
    up = uu - dt * v0 + 0.5 * dt * dt * a0
    for _ in range(n_steps):
        un = 2 * uu - up + dt * dt * psi(uu) / ml
        vv = (un - up) / (2 * dt)
        up, uu = uu, un
    out["v0"] = v0
    out["explicit_u"] = uu
    out["explicit_v"] = vv
    out["explicit_dt"] = np.array(dt)
    out["explicit_steps"] = np.array(n_steps)
    out["m_lumped"] = ml
    np.savez_compressed(os.path.join(HERE, "contact.npz"), **out)


def gen_explicit():
    """Reference explicit_run (consistent mass, Jacobi-PCG, condense=False):
    the SURVEY F2 row, pinned against the reference's own explicit path."""
    from sdmefem.dynamics import explicit_run

    P = 3
    prob = problem("SDME_M", P, (3, 2, 2), (1.0, 0.5, 0.5), P + 1, [("xmin", (0, 1, 2))])
    faces = build_face_tables(prob.mesh, prob.element, "xmax", prob.rule)
    base = prob.traction_vector(faces, lambda f: np.tile([0.0, 0.0, 2.0e4], (len(f.pts), 1)))
    load = lambda t: base * min(t / 5e-5, 1.0)
    cfg = SolverConfig(precond="diagonal", tol=1e-12, maxit=100000, condense=False)
    dt, n_steps = 1e-5, 20
    traj = explicit_run(prob, load, dt, n_steps, cfg=cfg)
    rows = [(r["step"], r["iterations"]) for r in traj.stats.rows]
    np.savez_compressed(os.path.join(HERE, "explicit.npz"), u=traj.state.u, v=traj.state.v,
                        u_prev=traj.state.u_prev, load=base, dt=np.array(dt), steps=np.array(n_steps),
                        pcg_rows=np.array(rows))
    print("explicit", [r[1] for r in rows][:6])


def gen_impact():
    """Implicit Newmark with penalty contact: the reference's
    bar-impact scenario (scenarios.py:92-113) shortened -- the bar starts 0.5 mm
    above the plane so contact engages after ~8 steps -- with Jacobi-PCG and
    tight tolerances for displacement parity."""
    mat = NeoHookean.from_engineering(100.0, 0.3, 1.0)
    mesh = gen_box_mesh((1, 2, 1), (0.05, 0.1, 0.05), (-0.025, 0.0005, -0.025))
    el = TensorElement.create(3, build_basis(3, BasisKind("SDME_H")))
    prob = FemProblem(mesh, el, build_dofmap(mesh, el, None), mat, rule=gauss_rule(4))
    v0 = prob.l2_project(lambda x: np.tile([0.0, -0.06, 0.0], (len(x), 1)))
    cont = PenaltyContact(prob, RigidObstacle(np.zeros(3), np.array([0.0, 1.0, 0.0])),
                          ContactParams(1e4, deps_n=1e3, gap_tol=3e-5, stress_tol=1e-2), "ymin")
    cfg = SolverConfig(precond="diagonal", tol=1e-12, maxit=100000, condense=False)
    dt, n_steps = 1e-3, 25
    zero = np.zeros(prob.n_free)
    traj = newmark_run(prob, lambda t: zero, dt, n_steps, newton_tol=1e-10, v0=v0, cfg=cfg, contact=cont)
    rows = [(r["step"], r["newton_iter"], r["iterations"]) for r in traj.stats.rows]
    np.savez_compressed(os.path.join(HERE, "impact.npz"), u=traj.state.u, v=traj.state.v, a=traj.state.a,
                        v0=v0, dt=np.array(dt), steps=np.array(n_steps),
                        newton_iters=np.array(traj.newton_iters), pcg_rows=np.array(rows),
                        history=np.array(cont.history))
    print("impact", traj.newton_iters, cont.history[-3:])


def gen_impact_energy():
    """The full bar-impact scenario (scenarios.py:92-113: 200 steps, contact at
    ~83 steps, rebound) with energy tracking -- acceptance criterion 9
    (test_acceptance.py:249-264) -- Jacobi-PCG and tight tolerances."""
    mat = NeoHookean.from_engineering(100.0, 0.3, 1.0)
    mesh = gen_box_mesh((1, 2, 1), (0.05, 0.1, 0.05), (-0.025, 0.005, -0.025))
    el = TensorElement.create(3, build_basis(3, BasisKind("SDME_H")))
    prob = FemProblem(mesh, el, build_dofmap(mesh, el, None), mat, rule=gauss_rule(4))
    v0 = prob.l2_project(lambda x: np.tile([0.0, -0.06, 0.0], (len(x), 1)))
    cont = PenaltyContact(prob, RigidObstacle(np.zeros(3), np.array([0.0, 1.0, 0.0])),
                          ContactParams(1e4, deps_n=1e3, gap_tol=1e-3, stress_tol=1e-2), "ymin")
    cfg = SolverConfig(precond="diagonal", tol=1e-12, maxit=100000, condense=False)
    zero = np.zeros(prob.n_free)
    traj = newmark_run(prob, lambda t: zero, 1e-3, 200, newton_tol=1e-10, v0=v0, cfg=cfg, contact=cont,
                       track_energy=True)
    en = np.array(traj.energy)
    total = en[:, 1] + en[:, 2] + en[:, 3]
    ey = prob.l2_project(lambda x: np.tile([0.0, 1.0, 0.0], (len(x), 1)))
    vy = float(ey @ (prob.mass() @ traj.state.v)) / (0.05 * 0.1 * 0.05)
    np.savez_compressed(os.path.join(HERE, "impact_energy.npz"), u=traj.state.u, v=traj.state.v, v0=v0,
                        energy=en, history=np.array(cont.history), newton_iters=np.array(traj.newton_iters),
                        vy=np.array(vy))
    print("impact_energy drift", float(np.abs(total - total[0]).max() / total[0]), "vy", vy,
          "pen", max(h[1] for h in cont.history))


# ---------------------------------------------------------------------------
# general hexahedral meshes: twisted / renumbered / perturbed

_BITS = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))


def _rotations():
    """The 24 orientation-preserving maps of the unit cube's corner bits,
    as (perm, flips): local bit d -> physical axis perm[d], reversed if flips[d]."""
    import itertools
    out = []
    for perm in itertools.permutations(range(3)):
        for flips in itertools.product((0, 1), repeat=3):
            m = np.zeros((3, 3))
            for d in range(3):
                m[perm[d], d] = -1.0 if flips[d] else 1.0
            if np.linalg.det(m) > 0:
                out.append((perm, flips))
    return out


def _relabel(conn, rot):
    """Connectivity of the same hexahedron with its local axes rotated."""
    perm, flips = rot
    phys = {b: conn[i] for i, b in enumerate(_BITS)}
    new = []
    for b in _BITS:
        x = [0, 0, 0]
        for d in range(3):
            x[perm[d]] = 1 - b[d] if flips[d] else b[d]
        new.append(phys[tuple(x)])
    return new


def general_mesh(kind, seed):
    """Seeded general meshes: 'twist' = two unit hexes, the second with rotated
    local axes; 'box' = a 3x2x2 box with shuffled vertex ids, every element's
    local axes rotated at random and interior vertices displaced."""
    rng = np.random.default_rng(seed)
    rots = _rotations()
    if kind == "twist":
        base = gen_box_mesh((2, 1, 1), (2.0, 1.0, 1.0))
        elems = [list(base.elems[0]), _relabel(list(base.elems[1]), rots[seed % len(rots)])]
        return Mesh(3, base.coords.copy(), np.array(elems), {})
    base = gen_box_mesh((3, 2, 2), (1.5, 1.0, 1.0))
    coords = base.coords.copy()
    inner = np.all((coords > 1e-12) & (coords < np.array([1.5, 1.0, 1.0]) - 1e-12), axis=1)
    coords[inner] += 0.08 * rng.uniform(-1, 1, (int(inner.sum()), 3))
    # shift boundary-face vertices within their face so faces stay planar
    for ax, hi in ((0, 1.5), (1, 1.0), (2, 1.0)):
        on = (np.abs(coords[:, ax]) < 1e-12) | (np.abs(coords[:, ax] - hi) < 1e-12)
        for other in range(3):
            if other == ax:
                continue
            top = 1.5 if other == 0 else 1.0
            movable = on & (coords[:, other] > 1e-12) & (coords[:, other] < top - 1e-12)
            coords[movable, other] += 0.05 * rng.uniform(-1, 1, int(movable.sum()))
    newid = rng.permutation(len(coords))
    coords2 = np.empty_like(coords)
    coords2[newid] = coords
    elems = [_relabel([int(newid[v]) for v in conn], rots[int(rng.integers(len(rots)))]) for conn in base.elems]
    order = rng.permutation(len(elems))
    elems = [elems[i] for i in order]
    boundary = {tag: [tuple(int(newid[v]) for v in quad) for quad in quads] for tag, quads in base.boundary.items()}
    return Mesh(3, coords2, np.array(elems), boundary)


GENERAL_CASES = [  # (mesh kind, seed, basis, P, dirichlet)
    ("twist", 5, "ModalJacobi", 3, None),
    ("twist", 17, "LagrangeGLL", 4, None),
    ("twist", 22, "SDME_M", 4, None),
    ("box", 1, "SDME_M", 4, [("xmin", (0, 1, 2)), ("zmax", (2,))]),
    ("box", 2, "LagrangeGLL", 2, [("xmin", (0, 1, 2))]),
    ("box", 3, "SDME_H", 3, [("ymin", (1,)), ("xmax", (0, 1, 2))]),
    ("box", 4, "SDME_K", 6, [("xmin", (0, 1, 2))]),
]


def gen_meshes():
    out = {}
    for ci, (kind, seed, tag, P, dr) in enumerate(GENERAL_CASES):
        mesh = general_mesh(kind, seed)
        el = TensorElement.create(3, build_basis(P, BasisKind(tag)))
        dm = build_dofmap(mesh, el, dr)
        prob = FemProblem(mesh, el, dm, MAT)
        rng = np.random.default_rng(100 + ci)
        u = 2e-3 * rng.uniform(-1, 1, prob.n_free)
        p = rng.standard_normal(prob.n_free)
        c_m = 3.0e4
        kt = prob.tangent(u)
        mass = prob.mass()
        eff = kt + c_m * mass
        key = f"m{ci}"
        out[key + "_coords"] = mesh.coords
        out[key + "_elems"] = mesh.elems
        tags = sorted(mesh.boundary)
        out[key + "_btags"] = np.array(tags)
        for t in tags:
            out[key + "_b_" + t] = np.array(mesh.boundary[t])
        out[key + "_meta"] = np.array([KINDS.index(tag), P])
        out[key + "_dir"] = np.array([[["xmin", "xmax", "ymin", "ymax", "zmin", "zmax"].index(t), c]
                                      for t, cs in (dr or []) for c in cs]).reshape(-1, 2)
        out[key + "_gdof"] = dm.gdof
        out[key + "_gsign"] = dm.gsign
        out[key + "_free_map"] = dm.free_map
        out[key + "_u"] = u
        out[key + "_p"] = p
        out[key + "_cm"] = np.array(c_m)
        out[key + "_fint"] = prob.internal_force(u)
        out[key + "_kp"] = kt @ p
        out[key + "_mp"] = mass @ p
        out[key + "_diag"] = eff.diagonal()
        b = prob.internal_force(u) + 1e3 * p
        x, st = pcg(eff, b, precond="diagonal", tol=1e-10, maxit=100000)
        out[key + "_pcg_b"] = b
        out[key + "_pcg_x"] = x
        out[key + "_pcg_iters"] = np.array(st.iterations)
        print(key, kind, tag, P, prob.n_free, "pcg", st.iterations, "signs", int((dm.gsign < 0).sum()))
    np.savez_compressed(os.path.join(HERE, "meshes.npz"), **out)


def gen_mesh_newmark():
    """Implicit Newmark (dynamics.py:173-257) on a general (renumbered,
    rotated, perturbed) mesh with a traction on xmax."""
    mesh = general_mesh("box", 3)
    el = TensorElement.create(3, build_basis(3, BasisKind("SDME_H")))
    dm = build_dofmap(mesh, el, [("xmin", (0, 1, 2))])
    prob = FemProblem(mesh, el, dm, MAT)
    faces = build_face_tables(prob.mesh, prob.element, "xmax", prob.rule)
    base = prob.traction_vector(faces, lambda f: np.tile([0.0, 2.0e5, 1.0e5], (len(f.pts), 1)))
    dt = 1e-4
    load = lambda t: base * min(t / (5 * dt), 1.0)
    cfg = SolverConfig(precond="diagonal", tol=1e-10, maxit=200000, condense=False)
    traj = newmark_run(prob, load, dt, 5, newton_tol=1e-8, cfg=cfg)
    rows = [(r["step"], r["newton_iter"], r["iterations"]) for r in traj.stats.rows]
    np.savez_compressed(os.path.join(HERE, "mesh_newmark.npz"), u=traj.state.u, v=traj.state.v, a=traj.state.a,
                        load=base, newton_iters=np.array(traj.newton_iters), pcg_rows=np.array(rows))
    print("mesh_newmark", traj.newton_iters, [r[2] for r in rows])


# ---------------------------------------------------------------------------
# BASELINE config 5 (implicit large deformation, P = 6), reduced

C5_TAGS = ("LagrangeGLL", "ModalJacobi", "SDME_H")
C5_TRACTION = -8.0e5   # ~24% tip deflection (GLL vertex values) after 3 steps
C5_STEPS = 3
C5_DT = 2.0833e-3      # the 50 x 1.25e-4 s ramp of the scaled beam in 3 steps


def c5_run(tag):
    """Config 5 geometry reduced to 8x1x1 elements with the same element size
    h = 0.0625 and aspect ratio (cantilever [0,0.5]x[0,0.0625]^2, P = 6,
    m = 7, x = 0 clamped), tip traction ramped over 3 Newmark steps so each
    step needs 4-6 Newton iterations (large deformation)."""
    P = 6
    prob = problem(tag, P, (8, 1, 1), (0.5, 0.0625, 0.0625), P + 1, [("xmin", (0, 1, 2))])
    faces = build_face_tables(prob.mesh, prob.element, "xmax", prob.rule)
    base = prob.traction_vector(faces, lambda f: np.tile([0.0, 0.0, C5_TRACTION], (len(f.pts), 1)))
    T = C5_STEPS * C5_DT
    cfg = SolverConfig(precond="diagonal", tol=1e-10, maxit=200000, condense=False)
    traj = newmark_run(prob, lambda t: base * min(t / T, 1.0), C5_DT, C5_STEPS, newton_tol=1e-8, cfg=cfg)
    rows = [(r["step"], r["newton_iter"], r["iterations"]) for r in traj.stats.rows]
    return traj, base, rows


def _spread(kind, arg, threads):
    """Re-run a case in a fresh process with OPENBLAS_NUM_THREADS=threads and
    return its PCG iteration counts (the reference's own run-to-run spread)."""
    import json
    import subprocess
    import sys

    env = dict(os.environ, OPENBLAS_NUM_THREADS=str(threads))
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "_" + kind, str(arg)], env=env,
                         capture_output=True, text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def gen_config5():
    from concurrent.futures import ThreadPoolExecutor

    out = {}
    jobs = {}
    with ThreadPoolExecutor(max_workers=6) as ex:
        for tag in C5_TAGS:
            for th in (1, 4):
                jobs[(tag, th)] = ex.submit(_spread, "c5rows", tag, th)
        for tag in C5_TAGS:
            traj, base, rows = c5_run(tag)
            out[f"{tag}_u"] = traj.state.u
            out[f"{tag}_v"] = traj.state.v
            out[f"{tag}_a"] = traj.state.a
            out[f"{tag}_load"] = base
            out[f"{tag}_newton_iters"] = np.array(traj.newton_iters)
            out[f"{tag}_pcg_rows"] = np.array(rows)
            print("config5", tag, traj.newton_iters, [r[2] for r in rows], flush=True)
        for (tag, th), fut in jobs.items():
            out[f"{tag}_pcg_iters_t{th}"] = np.array(fut.result())
            print("config5 spread", tag, th, fut.result(), flush=True)
    out["meta"] = np.array([C5_TRACTION, C5_STEPS, C5_DT])
    np.savez_compressed(os.path.join(HERE, "config5.npz"), **out)


def _mesh_case_pcg(ci):
    kind, seed, tag, P, dr = GENERAL_CASES[ci]
    mesh = general_mesh(kind, seed)
    el = TensorElement.create(3, build_basis(P, BasisKind(tag)))
    prob = FemProblem(mesh, el, build_dofmap(mesh, el, dr), MAT)
    rng = np.random.default_rng(100 + ci)
    u = 2e-3 * rng.uniform(-1, 1, prob.n_free)
    p = rng.standard_normal(prob.n_free)
    eff = prob.tangent(u) + 3.0e4 * prob.mass()
    _, st = pcg(eff, prob.internal_force(u) + 1e3 * p, precond="diagonal", tol=1e-10, maxit=100000)
    return st.iterations


def gen_meshes_spread():
    """PCG iteration counts of the general-mesh cases (gen_meshes) under
    OPENBLAS_NUM_THREADS = 1, 2, 4, 8: the reference's own spread, which
    bounds the iteration slack of the ill-conditioned m6 case."""
    out = {}
    for th in (1, 2, 4, 8):
        out[f"t{th}"] = np.array(_spread("meshpcg", -1, th))
        print("meshes spread", th, out[f"t{th}"].tolist(), flush=True)
    np.savez_compressed(os.path.join(HERE, "meshes_spread.npz"), **out)


# ---------------------------------------------------------------------------
# the reference's default solver (SGS, Schur condensation)

SGS_CFGS = (("sgs", True), ("sgs", False), ("diagonal", True), ("none", True))


def gen_sgs():
    """make_solver(problem, element_matrices, cfg).solve(b) (dynamics.py:111-127,
    solver.py:258-322) on the global cases for SGS / diagonal with and without
    condensation (tol 1e-10), the condensed Schur CSR of the smallest case,
    and explicit_run / newmark_run with the reference's default SolverConfig()."""
    from sdmefem.dynamics import explicit_run, make_solver

    out = {}
    cases = [("SDME_M", 4, 5, (2, 3, 2), (1.0, 1.5, 1.0), [("xmin", (0, 1, 2))]),
             ("LagrangeGLL", 3, 5, (3, 2, 2), (1.0, 1.0, 0.5), [("xmin", (0, 1, 2)), ("zmax", (2,))]),
             ("ModalJacobi", 2, 3, (2, 2, 3), (0.5, 0.5, 1.0), None),
             ("SDME_H", 3, 4, (2, 2, 2), (1.0, 1.0, 1.0), [("ymin", (1,))])]
    for ci, (tag, P, m, div, L, dr) in enumerate(cases):
        prob = problem(tag, P, div, L, m, dr)
        u = smooth_plus_noise(prob, 0.01, 1e-4, 7 + ci)
        p = np.random.default_rng(50 + ci).standard_normal(prob.n_free)
        c_m = 3.0e4
        eff = [(kt + c_m * mm, d, sg) for (kt, d, sg), (mm, _, _) in zip(prob.tangent_matrices(u),
                                                                           prob.mass_matrices())]
        b = prob.internal_force(u) + 1e3 * p
        for k, (pc, cond) in enumerate(SGS_CFGS):
            solver = make_solver(prob, eff, SolverConfig(precond=pc, tol=1e-10, maxit=100000, condense=cond))
            x, st = solver.solve(b)
            out[f"g{ci}_c{k}_x"] = x
            out[f"g{ci}_c{k}_iters"] = np.array(st.iterations)
            out[f"g{ci}_c{k}_tag"] = np.array(st.preconditioner)
            if ci == 2 and cond:
                cs = solver.operator.schur.tocsr()
                cs.sort_indices()
                out[f"g{ci}_c{k}_schur_indptr"] = cs.indptr
                out[f"g{ci}_c{k}_schur_indices"] = cs.indices
                out[f"g{ci}_c{k}_schur_data"] = cs.data
            print("sgs", ci, pc, cond, st.iterations, st.preconditioner, flush=True)
    # explicit_run with the reference default SolverConfig() (dynamics.py:130-170)
    P = 3
    prob = problem("SDME_M", P, (3, 2, 2), (1.0, 0.5, 0.5), P + 1, [("xmin", (0, 1, 2))])
    faces = build_face_tables(prob.mesh, prob.element, "xmax", prob.rule)
    base = prob.traction_vector(faces, lambda f: np.tile([0.0, 0.0, 2.0e4], (len(f.pts), 1)))
    traj = explicit_run(prob, lambda t: base * min(t / 5e-5, 1.0), 1e-5, 20)
    out["explicit_u"] = traj.state.u
    out["explicit_v"] = traj.state.v
    out["explicit_rows"] = np.array([(r["step"], r["iterations"]) for r in traj.stats.rows])
    out["explicit_tags"] = np.array([r["preconditioner"] for r in traj.stats.rows])
    # newmark_run with SolverConfig() on a 2x2x2 SDME_H P = 3 block under a ramped traction
    prob = problem("SDME_H", 3, (2, 2, 2), (1.0, 1.0, 1.0), 4, [("xmin", (0, 1, 2))])
    faces = build_face_tables(prob.mesh, prob.element, "xmax", prob.rule)
    base = prob.traction_vector(faces, lambda f: np.tile([0.0, 1.0e5, -2.0e5], (len(f.pts), 1)))
    traj = newmark_run(prob, lambda t: base * min(t / 4e-4, 1.0), 1e-4, 4, newton_tol=1e-8)
    out["newmark_u"] = traj.state.u
    out["newmark_v"] = traj.state.v
    out["newmark_load"] = base
    out["newmark_newton"] = np.array(traj.newton_iters)
    out["newmark_rows"] = np.array([(r["step"], r["newton_iter"], r["iterations"]) for r in traj.stats.rows])
    print("sgs explicit", out["explicit_rows"][:4].tolist(), "newmark", traj.newton_iters,
          out["newmark_rows"][:, 2].tolist(), flush=True)
    np.savez_compressed(os.path.join(HERE, "sgs.npz"), **out)


def gen_config1_default():
    """BASELINE config 1 with the reference's DEFAULT solver (SolverConfig():
    SGS + Schur condensation, tol 1e-12), 10 Newmark steps."""
    P, m = 4, 6
    prob = problem("SDME_M", P, (4, 4, 4), (1.0, 1.0, 1.0), m, [("xmin", (0, 1, 2))])
    faces = build_face_tables(prob.mesh, prob.element, "xmax", prob.rule)
    base = prob.traction_vector(faces, lambda f: np.tile([0.0, 0.0, 1.0e5], (len(f.pts), 1)))
    t0 = time.perf_counter()
    traj = newmark_run(prob, lambda t: base * min(t / 1e-3, 1.0), 1e-4, 10, newton_tol=1e-8)
    wall = time.perf_counter() - t0
    rows = [(r["step"], r["newton_iter"], r["iterations"]) for r in traj.stats.rows]
    np.savez_compressed(os.path.join(HERE, "config1_default.npz"), u=traj.state.u, v=traj.state.v,
                        a=traj.state.a, newton_iters=np.array(traj.newton_iters), pcg_rows=np.array(rows),
                        tags=np.array([r["preconditioner"] for r in traj.stats.rows]), wall_s=np.array(wall))
    print("config1_default", wall, "s", traj.newton_iters, [r[2] for r in rows])


if __name__ == "__main__":
    import json
    import sys

    if len(sys.argv) == 3 and sys.argv[1] == "_c5rows":
        print(json.dumps([r[2] for r in c5_run(sys.argv[2])[2]]))
        sys.exit(0)
    if len(sys.argv) == 3 and sys.argv[1] == "_meshpcg":
        print(json.dumps([_mesh_case_pcg(ci) for ci in range(len(GENERAL_CASES))]))
        sys.exit(0)
    which = sys.argv[1:] or ["basis", "elements", "global", "contact", "explicit", "impact", "impact_energy",
                             "config1"]
    for w in which:
        t = time.perf_counter()
        globals()["gen_" + w]()
        print(w, f"{time.perf_counter() - t:.1f}s")
