"""Small invocations of every kernel family, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py [case ...]
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases (default: all): col4 (P = 4 collocated TMA colour passes: f_int, K.p,
c_m M p, mass, diagonal), col6 (P = 6, 2 warps per element), sub3 (P = 3, one
element per half-warp), tmb2 (P = 2 all-component TMA kernel), ev (E-vector
launch + gather), pcg (whole-solve graph with the 16-CTA cluster tail), pcgd
(PCG as plain launches: the 7-kernel iteration), gen (general mesh: gather,
element kernel, assembly, diagonal), contact (penalty force, K_c p, diag K_c),
explicit (lumped explicit chunks).  Each prints one line; a failure raises.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

MAT = None


def _pb(P, div=(3, 2, 2), tag="SDME_M", m=None, dr=(("xmin", (0, 1, 2)),), ev=None):
    from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis
    from paper_2104_13466_b200.basis import BasisKind, gauss_rule

    if ev is not None:
        os.environ["SDME_EV"] = "1" if ev else "0"
    try:
        return GpuFemProblem(BoxMesh(div, (0.3, 0.2, 0.2)), build_basis(P, BasisKind(tag)),
                             NeoHookean.from_engineering(1e7, 0.3, 1e3), gauss_rule(m or P + 1), list(dr))
    finally:
        os.environ.pop("SDME_EV", None)


def _ops(pb, name):
    rng = np.random.default_rng(0)
    u = 1e-3 * 0.1 * rng.uniform(-1, 1, pb.n_free)
    p = rng.standard_normal(pb.n_free)
    f = pb.internal_force(u)
    y = pb.apply_tangent(u, p, 3e4)
    y0 = pb.apply_tangent(u, p)
    mp = pb.mass_apply(p)
    d = pb.tangent_diagonal(u, 3e4)
    assert all(np.isfinite(a).all() for a in (f, y, y0, mp, d))
    print(name, "ok", pb.n_free, float(np.abs(y).max()))


def case_col4():
    _ops(_pb(4, ev=False), "col4")


def case_col6():
    _ops(_pb(6, ev=False), "col6")


def case_sub3():
    _ops(_pb(3, ev=False), "sub3")


def case_tmb2():
    _ops(_pb(2, ev=False), "tmb2")


def case_ev():
    _ops(_pb(4, ev=True), "ev")


def _pcg(direct):
    from paper_2104_13466_b200 import pcg_gpu

    if direct:
        os.environ["SDME_PCG_DIRECT"] = "1"
    try:
        pb = _pb(4, (2, 2, 2))
    finally:
        os.environ.pop("SDME_PCG_DIRECT", None)
    rng = np.random.default_rng(1)
    u = 1e-4 * rng.uniform(-1, 1, pb.n_free)
    b = rng.standard_normal(pb.n_free)
    x, st = pcg_gpu(pb, u, b, c_m=4e8, tol=1e-10)
    r = pb.apply_tangent(u, x, 4e8) - b
    assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(b)
    print("pcgd" if direct else "pcg", "ok", st.iterations)


def case_pcg():
    _pcg(False)


def case_pcgd():
    _pcg(True)


def case_gen():
    from paper_2104_13466_b200 import GpuMeshProblem, HexMesh, NeoHookean, build_basis
    from paper_2104_13466_b200.basis import BasisKind

    box = HexMesh.box((2, 2, 1), (1.0, 1.0, 0.5))
    coords = box.coords.copy()
    coords[:, 2] += 0.05 * coords[:, 0] * coords[:, 1]
    mesh = HexMesh(coords, box.elems, box.boundary)
    pb = GpuMeshProblem(mesh, build_basis(3, BasisKind("SDME_H")), NeoHookean.from_engineering(1e7, 0.3, 1e3),
                        None, [("xmin", (0, 1, 2))])
    _ops(pb, "gen")


def case_contact():
    from paper_2104_13466_b200 import ContactParams, GpuPenaltyContact, RigidObstacle

    pb = _pb(3, (3, 2, 2), dr=())
    c = GpuPenaltyContact(pb, RigidObstacle([2e-6, 0, 0], [1, 0, 0]), ContactParams(1e10), "xmin")
    u = np.zeros(pb.n_free)
    fc = c.evaluate_forces(u)
    kc = c.stiffness_operator(u) if hasattr(c, "stiffness_operator") else None
    assert np.isfinite(fc.force).all()
    print("contact ok", int((fc.gaps < 0).sum()) if hasattr(fc, "gaps") else -1, kc is not None)


def case_explicit():
    from paper_2104_13466_b200 import ContactParams, GpuPenaltyContact, RigidObstacle, explicit_run

    pb = _pb(3, (3, 2, 2), dr=())
    c = GpuPenaltyContact(pb, RigidObstacle([-1e-6, 0, 0], [1, 0, 0]), ContactParams(1e10), "xmin")
    v0 = pb.constant_field([-10.0, 0.0, 0.0])
    tr = explicit_run(pb, None, 2e-8, 30, v0=v0, contact=c, record_every=10, mass="lumped")
    assert np.isfinite(tr.state.u).all()
    print("explicit ok", tr.contact_history[-1])


CASES = ["col4", "col6", "sub3", "tmb2", "ev", "pcg", "pcgd", "gen", "contact", "explicit"]

if __name__ == "__main__":
    for name in sys.argv[1:] or CASES:
        globals()["case_" + name]()
