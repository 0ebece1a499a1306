"""Pin the CPU oracle (oracle/) against golden vectors of the REAL reference.

The fixtures were produced by tests/golden/make_golden.py importing sdmefem
from /root/reference; these tests need neither the reference nor a GPU.
Tolerance: 1e-12 relative (max-norm) on element and global vectors, the
north_star bar.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import KINDS, element_cases, global_cases, load_golden, max_rel_err
from oracle import basis as ob
from oracle import fem as of
from oracle import solve as osv

MAT = of.Material(1.0e7, 0.3, 1.0e3)
TOL = 1e-12


def test_oracle_basis_tables_match_reference():
    g = load_golden("basis")
    worst = 0.0
    for key in g.files:
        if not key.endswith("_T"):
            continue
        tag, ps = key.split("_P")[0], key.split("_P")[1].split("_")[0]
        P = int(ps)
        b = ob.Basis(tag, P)
        if tag != "LagrangeGLL":
            worst = max(worst, float(np.abs(b.T - g[key]).max()))
        for m in (P + 1, P + 2):
            v, d = b.eval(ob.gauss(m)[0])
            worst = max(worst, max_rel_err(v.T, g[f"{tag}_P{P}_m{m}_B"]),
                        max_rel_err(d.T, g[f"{tag}_P{P}_m{m}_D"]))
    assert worst <= 1e-13, worst


def _elem_problem(tag, P, m, h):
    return of.Problem(of.Mesh((1, 1, 1), h), ob.Basis(tag, P), MAT, m)


@pytest.mark.parametrize("case", [c for c in element_cases() if c[2] <= 4], ids=lambda c: f"{c[1]}-P{c[2]}-m{c[3]}")
def test_oracle_element_vectors(case):
    i, tag, P, m, h = case
    g = load_golden("elements")
    pb = _elem_problem(tag, P, m, h)
    loc = pb.dmap.evdofs(0)  # element-local (function-major, comp fastest) -> free index
    u, p, cm = g[f"c{i}_u"], g[f"c{i}_p"], float(g[f"c{i}_cm"])
    assert max_rel_err(pb.internal_force(u)[loc], g[f"c{i}_fint"]) <= TOL
    assert max_rel_err(pb.apply_tangent(u, p)[loc], g[f"c{i}_kp"]) <= TOL
    assert max_rel_err((pb.mass() @ p)[loc], g[f"c{i}_mp"]) <= TOL
    assert max_rel_err(pb.assemble(u, 1.0, cm).diagonal()[loc], g[f"c{i}_diag"]) <= TOL


@pytest.mark.slow
@pytest.mark.parametrize("case", [c for c in element_cases() if c[2] > 4 and c[3] == c[2] + 1],
                         ids=lambda c: f"{c[1]}-P{c[2]}-m{c[3]}")
def test_oracle_element_vectors_high_order(case):
    i, tag, P, m, h = case
    g = load_golden("elements")
    pb = _elem_problem(tag, P, m, h)
    loc = pb.dmap.evdofs(0)
    u, p = g[f"c{i}_u"], g[f"c{i}_p"]
    assert max_rel_err(pb.internal_force(u)[loc], g[f"c{i}_fint"]) <= TOL
    assert max_rel_err(pb.apply_tangent(u, p)[loc], g[f"c{i}_kp"]) <= TOL


@pytest.mark.parametrize("case", global_cases(), ids=lambda c: f"{c[1]}-P{c[2]}")
def test_oracle_global_vectors_and_pcg(case):
    i, tag, P, m, div, L, dr = case
    g = load_golden("global")
    pb = of.Problem(of.Mesh(div, L), ob.Basis(tag, P), MAT, m, dr)
    assert pb.n_free == g[f"g{i}_u"].size
    u, p, cm = g[f"g{i}_u"], g[f"g{i}_p"], float(g[f"g{i}_cm"])
    assert max_rel_err(pb.internal_force(u), g[f"g{i}_fint"]) <= TOL
    assert max_rel_err(pb.apply_tangent(u, p), g[f"g{i}_kp"]) <= TOL
    assert max_rel_err(pb.mass() @ p, g[f"g{i}_mp"]) <= TOL
    eff = pb.assemble(u, 1.0, cm)
    assert max_rel_err(eff.diagonal(), g[f"g{i}_diag"]) <= TOL
    x, its, _ = osv.pcg(eff, g[f"g{i}_pcg_b"], "diagonal", 1e-10, 100000)
    assert abs(its - int(g[f"g{i}_pcg_iters"])) <= 1
    assert max_rel_err(x, g[f"g{i}_pcg_x"]) <= 1e-9


def _contact_problem():
    return of.Problem(of.Mesh((3, 2, 2), (0.3, 0.2, 0.2)), ob.Basis("SDME_M", 3), MAT, 4)


def test_oracle_contact_force():
    g = load_golden("contact")
    pb = _contact_problem()
    c = of.Contact(pb, [-1e-3, 0, 0], [1, 0, 0], 1e10, "xmin")
    f, gaps = c.force(g["u"])
    assert max_rel_err(f, g["force"]) <= TOL
    assert max_rel_err(np.concatenate(gaps), g["gaps"]) <= TOL


def test_oracle_explicit_lumped_contact_loop():
    g = load_golden("contact")
    pb = _contact_problem()
    c = of.Contact(pb, [-2e-5, 0, 0], [1, 0, 0], 1e10, "xmin")
    assert max_rel_err(np.asarray(pb.mass().sum(axis=1)).ravel(), g["m_lumped"]) <= TOL
    assert max_rel_err(pb.lumped_mass(), g["m_lumped"]) <= TOL
    out = osv.explicit_lumped(pb, lambda t: np.zeros(pb.n_free), float(g["explicit_dt"]),
                              int(g["explicit_steps"]), v0=g["v0"], contact=c)
    assert max(out["penetration"]) > 0.0  # contact engaged
    assert max_rel_err(out["u"], g["explicit_u"]) <= 1e-10
    assert max_rel_err(out["v"], g["explicit_v"]) <= 1e-9


@pytest.mark.slow
def test_oracle_config1_newmark():
    """BASELINE config 1 end to end on the oracle: Newton counts equal, PCG
    iterations +-1, final u within 1e-9 relative."""
    g = load_golden("config1")
    pb = of.Problem(of.Mesh((4, 4, 4), (1.0, 1.0, 1.0)), ob.Basis("SDME_M", 4), MAT, 6,
                    [("xmin", (0, 1, 2))])
    base = pb.traction_vector("xmax", [0.0, 0.0, 1.0e5])
    assert max_rel_err(base, g["load"]) <= TOL
    out = osv.newmark(pb, lambda t: base * min(t / 1e-3, 1.0), 1e-4, 10, 1e-8, 25, 1e-10)
    assert out["newton_iters"] == list(g["newton_iters"])
    ref_its = [r[2] for r in g["pcg_rows"] if r[0] >= 0]
    its = [r[2] for r in out["pcg_iters"]]
    assert len(its) == len(ref_its)
    assert max(abs(a - b) for a, b in zip(its, ref_its)) <= 1
    assert max_rel_err(out["u"], g["u"]) <= 1e-9


def _impact_problem():
    return of.Problem(of.Mesh((1, 2, 1), (0.05, 0.1, 0.05), (-0.025, 0.0005, -0.025)), ob.Basis("SDME_H", 3),
                      of.Material(100.0, 0.3, 1.0), 4)


def test_oracle_implicit_contact_newmark():
    """reference newmark_run with penalty contact (bar impact,
    scenarios.py:92-113, shortened): Newton counts, penalty history, state."""
    g = load_golden("impact")
    pb = _impact_problem()
    c = of.Contact(pb, [0.0, 0.0, 0.0], [0.0, 1.0, 0.0], 1e4, "ymin", deps=1e3, gap_tol=3e-5, stress_tol=1e-2)
    out = osv.newmark(pb, lambda t: np.zeros(pb.n_free), float(g["dt"]), int(g["steps"]), newton_tol=1e-10,
                      pcg_tol=1e-12, v0=g["v0"], contact=c)
    assert out["newton_iters"] == list(g["newton_iters"])
    its = [r[2] for r in out["pcg_iters"]]
    assert np.all(np.abs(np.array(its) - g["pcg_rows"][1:, 2]) <= 1)
    hist = np.array(c.history)
    assert np.array_equal(hist[:, 0], g["history"][:, 0])  # penalty stepping
    assert np.array_equal(hist[:, 3], g["history"][:, 3])  # active counts
    assert max_rel_err(hist[:, 1], g["history"][:, 1]) <= 1e-8
    for k in ("u", "v", "a"):
        assert max_rel_err(out[k], g[k]) <= 1e-9, k


def test_oracle_bar_impact_energy_criterion9():
    """Acceptance criterion 9 (test_acceptance.py:249-264) on the full
    bar-impact scenario: energy rows, penalty history and final state."""
    g = load_golden("impact_energy")
    pb = of.Problem(of.Mesh((1, 2, 1), (0.05, 0.1, 0.05), (-0.025, 0.005, -0.025)), ob.Basis("SDME_H", 3),
                    of.Material(100.0, 0.3, 1.0), 4)
    c = of.Contact(pb, [0.0, 0.0, 0.0], [0.0, 1.0, 0.0], 1e4, "ymin", deps=1e3, gap_tol=1e-3, stress_tol=1e-2)
    out = osv.newmark(pb, lambda t: np.zeros(pb.n_free), 1e-3, 200, newton_tol=1e-10, pcg_tol=1e-12,
                      v0=g["v0"], contact=c, track_energy=True)
    assert out["newton_iters"] == list(g["newton_iters"])
    en = np.array(out["energy"])
    assert max_rel_err(en, g["energy"]) <= 1e-8
    assert np.array_equal(np.array(c.history)[:, 0], g["history"][:, 0])
    assert max_rel_err(out["u"], g["u"]) <= 1e-9
