"""Run the BASELINE.json configs 1, 3, 4, 5 on one GPU and print one JSON line each.

    python tools/run_configs.py c1 c3 c4 c5 [--quick] [--cpu]

``--cpu`` adds, in the same run and on the same host, the reference's own CPU
figure beside each GPU number (tools/refcpu.py: sdmefem from baseline/_ref):
c1 the reference's newmark_run per step; c3 per-element element_tangent @ p_e
on every core, scaled to the mesh (extrapolated); c4 the explicit lumped-mass
+ contact restatement loop built from the reference's internal_force /
PenaltyContact at full size, a few steps scaled to 2,000; c5 the reference's
newmark_run on the 8x1x1 reduction of the cantilever, per step, scaled by the
element count (extrapolated).

c1: 4^3 P=4 SDME_M, (P+2)^3 Gauss, 10 Newmark steps (dt 1e-4), traction 1e5 in +z
    on xmax ramped over 10 dt, Jacobi-PCG 1e-10: s/time-step,
    Newton and PCG iteration counts (parity with the reference is in
    tests/test_gpu_parity.py::test_config1_newmark_vs_reference).
c3: P in {2,3,4,6,8} x {LagrangeGLL, ModalJacobi, SDME_M}, N = round(256/P)
    elements per side (D5): K.p and f_int GDOF/s + FP64 roofline fraction.
c4: explicit impact, bar 80x16x16 P=3 SDME_M, v0 = -10 m/s, rigid wall at
    x = -1e-3, eps = 1e10, lumped mass, dt = 0.5 * 2/sqrt(lambda_max) (D6, D7).
c5: cantilever 64x8x8 P=6, 3 bases, 50 Newmark steps dt=1e-3, tip traction
    -1.3e6 in z ramped over the run (D8; calibrated to ~30% tip deflection of
    the 4 m length): PCG iterations per Newton step, s/step.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2104_13466_b200 import (BoxMesh, ContactParams, GpuFemProblem, GpuPenaltyContact,  # noqa: E402
                                   NeoHookean, RigidObstacle, ScaledLoad, SolverConfig, build_basis,
                                   explicit_run, newmark_run)
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402
from paper_2104_13466_b200.dynamics import estimate_lambda_max, lumped_mass  # noqa: E402

MAT = NeoHookean.from_engineering(1.0e7, 0.3, 1.0e3)


CPU = "--cpu" in sys.argv


def emit(d):
    print(json.dumps(d), flush=True)


def _c4_reference_cpu(div, P, steps, dt, v0_val=-10.0, wall=-1e-3, eps=1e10):
    """Config 4's explicit loop (lumped mass, penalty contact, central
    difference) from the reference's own pieces -- FemProblem.internal_force,
    element_mass row sums, PenaltyContact.evaluate_forces -- at full size,
    ``steps`` steps, in a subprocess with SDMEFEM_THREADS = all cores."""
    import subprocess

    from tools import refcpu

    if not refcpu.reference_dir():
        return None
    code = f"""
import json, sys, time
sys.path.insert(0, {refcpu.REF_DIR!r})
import numpy as np
from sdmefem.basis1d import BasisKind, build_basis
from sdmefem.contact import ContactParams, PenaltyContact, RigidObstacle
from sdmefem.femcore import FemProblem, element_mass
from sdmefem.material import NeoHookean
from sdmefem.meshdof import build_dofmap, gen_box_mesh
from sdmefem.quadrature import gauss_rule
from sdmefem.tensorelem import TensorElement
t0 = time.perf_counter()
mesh = gen_box_mesh({tuple(div)!r}, (1.0, 0.2, 0.2))
el = TensorElement.create(3, build_basis({P}, BasisKind("SDME_M")))
prob = FemProblem(mesh, el, build_dofmap(mesh, el, None), NeoHookean.from_engineering(1e7, 0.3, 1e3),
                  rule=gauss_rule({P + 1}))
ml = np.zeros(prob.n_free)
me = element_mass(prob.tables[0], prob.mat, 3)  # identical geometry on the box
for e in range(prob.mesh.n_elems):
    d, sg = prob.dmap.elem_vector_dofs(e)
    ok = d >= 0
    np.add.at(ml, d[ok], (me @ ok.astype(float))[ok])
cont = PenaltyContact(prob, RigidObstacle(np.array([{wall}, 0.0, 0.0]), np.array([1.0, 0.0, 0.0])),
                      ContactParams({eps}), "xmin")
v = np.zeros(prob.n_free); v[0::3] = {v0_val}  # vertex-coefficient constant field, timing only
u = np.zeros(prob.n_free)
psi = lambda uu: -prob.internal_force(uu) + cont.evaluate_forces(uu).force
dt = {dt!r}
t1 = time.perf_counter()
a = psi(u) / ml
up = u - dt * v + 0.5 * dt * dt * a
ts = []
for _ in range({steps}):
    s0 = time.perf_counter()
    un = 2 * u - up + dt * dt * psi(u) / ml
    v = (un - up) / (2 * dt)
    up, u = u, un
    ts.append(time.perf_counter() - s0)
print(json.dumps({{"setup_s": t1 - t0, "step_s": ts}}))
"""
    env = dict(os.environ, SDMEFEM_THREADS=str(os.cpu_count()), NUMBA_CACHE_DIR="/tmp/sdme_numba_cache")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=3600)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-2000:])
    out = json.loads(r.stdout.strip().splitlines()[-1])
    return out


def c1():
    pb = GpuFemProblem(BoxMesh((4, 4, 4), (1.0, 1.0, 1.0)), build_basis(4, BasisKind("SDME_M")), MAT,
                       gauss_rule(6), [("xmin", (0, 1, 2))])
    base = pb.traction_vector("xmax", [0.0, 0.0, 1.0e5])
    load = ScaledLoad(base, lambda t: min(t / 1e-3, 1.0))
    cfg = SolverConfig(precond="diagonal", tol=1e-10, condense=False)
    newmark_run(pb, load, 1e-4, 1, cfg=cfg)  # warm-up (context, first launches)
    t0 = time.perf_counter()
    traj = newmark_run(pb, load, 1e-4, 10, newton_tol=1e-8, cfg=cfg)
    wall = time.perf_counter() - t0
    its = [r["iterations"] for r in traj.stats.rows if r["step"] >= 0]
    row = {"config": "c1", "s_per_step": wall / 10, "total_s": wall, "newton_iters": traj.newton_iters,
           "pcg_iters": its, "max_u": float(np.abs(traj.state.u).max()), "n_free": pb.n_free}
    if CPU:
        from tools import refcpu

        r = refcpu.newmark_step_s((4, 4, 4), (1.0, 1.0, 1.0), 4, 6, "SDME_M", [0.0, 0.0, 1.0e5], 1e-4, 1e-3, 2)
        if r:
            row["cpu"] = {"s_per_step": r["step_s"][-1], "kind": "reference", "cores": r["cores"],
                          "what": "sdmefem newmark_run, 2nd step wall time (no setup), default BLAS threads",
                          "newton": r["newton"], "pcg": r["pcg"]}
            row["speedup"] = r["step_s"][-1] / row["s_per_step"]
    emit(row)


def c3(quick=False):
    peaks = bench.measured_peaks()
    fp = peaks.get("fp64_tflops")
    orders = [2, 3, 4, 6, 8]
    for P in orders:
        n = round(256 / P)
        if quick:
            n = max(2, n // 4)
        for tag in ("LagrangeGLL", "ModalJacobi", "SDME_M"):
            pb = GpuFemProblem(BoxMesh((n,) * 3, (1.0,) * 3), build_basis(P, BasisKind(tag)), MAT,
                               gauss_rule(P + 1), reference_order=False)
            u_lat, p_lat = bench.config2_fields(pb)
            u = pb.vector().set_lattice(u_lat)
            p = pb.vector().set_lattice(p_lat)
            y = pb.vector()
            del u_lat, p_lat
            pb.fint_(u, y)  # admissibility (raises on det F <= 0)
            for _ in range(2):
                pb.apply_(u, p, y)
            t_kp = pb.time_op("apply", u, p, y, 0.0, 5) / 1e3
            t_f = pb.time_op("fint", u, p, y, 0.0, 5) / 1e3
            flops = bench.kp_flops(n ** 3, P + 1, P + 1)
            row = {"config": "c3", "P": P, "basis": tag, "n_elem_side": n, "n_dofs": pb.n_lattice,
                   "kp_ms": t_kp * 1e3, "kp_gdofs": pb.n_lattice / t_kp / 1e9,
                   "kp_tflops": flops / t_kp / 1e12, "kp_frac_fp64": flops / t_kp / 1e12 / fp if fp else None,
                   "fint_ms": t_f * 1e3, "fint_gdofs": pb.n_lattice / t_f / 1e9}
            if CPU and tag == "SDME_M":  # the basis kind does not change the CPU cost
                from tools import refcpu

                with refcpu.ElementSampler(P, tag, P + 1, 1.0 / n) as smp:
                    probe = smp.sample("kp", 2)
                    k = max(1, int(round(1.5 * 2 / probe["worker_busy_s"])))
                    r = smp.sample("kp", k)
                eps = r["elements_per_s"]
                row["cpu"] = {"kp_gdofs": eps * pb.n_lattice / n ** 3 / 1e9, "kind": r["kind"], "cores": r["cores"],
                              "sample": refcpu.describe(r, P, P + 1, 1.0 / n, "kp"), "extrapolated": True}
                row["speedup_kp"] = row["kp_gdofs"] / row["cpu"]["kp_gdofs"]
            emit(row)
            del pb, u, p, y


def c4(quick=False, steps=2000):
    P = 3
    div = (80, 16, 16) if not quick else (20, 4, 4)
    pb = GpuFemProblem(BoxMesh(div, (1.0, 0.2, 0.2)), build_basis(P, BasisKind("SDME_M")), MAT,
                       gauss_rule(P + 1))
    obst = RigidObstacle([-1e-3, 0.0, 0.0], [1.0, 0.0, 0.0])
    contact = GpuPenaltyContact(pb, obst, ContactParams(1e10), "xmin")
    _, inv_ml = lumped_mass(pb)
    lam = estimate_lambda_max(pb, inv_ml, contact=contact)
    dt = 0.5 * 2.0 / np.sqrt(lam)
    v0 = pb.constant_field([-10.0, 0.0, 0.0])
    n_steps = steps if not quick else 200
    explicit_run(pb, None, dt, 5, v0=v0, contact=contact, mass="lumped")  # warm-up
    contact.history.clear()
    t0 = time.perf_counter()
    traj = explicit_run(pb, None, dt, n_steps, v0=v0, contact=contact, record_every=50, mass="lumped")
    pb.sync()
    wall = time.perf_counter() - t0
    hist = traj.contact_history
    row = {"config": "c4", "elements": int(np.prod(div)), "n_dofs": pb.n_free, "dt": dt, "lambda_max": lam,
           "steps": n_steps, "s_per_step": wall / n_steps, "total_s": wall,
           "max_penetration": max(h[1] for h in hist) if hist else 0.0,
           "contact_active_max": max(h[3] for h in hist) if hist else 0,
           "final_mean_vx": float(traj.state.v[0::3].mean()), "history_every50": hist[:8]}
    if CPU:
        r = _c4_reference_cpu(div, P, 3, dt)
        if r:
            sps = float(np.mean(r["step_s"]))
            row["cpu"] = {"s_per_step": sps, "s_2000_steps_extrapolated": 2000 * sps, "kind": "reference",
                          "cores": os.cpu_count(), "setup_s": r["setup_s"],
                          "what": "restatement loop from sdmefem pieces (internal_force with SDMEFEM_THREADS = "
                                  "all cores, element_mass row sums, PenaltyContact.evaluate_forces), "
                                  f"{len(r['step_s'])} full-size steps, scaled to 2000"}
            row["speedup"] = sps / row["s_per_step"]
    emit(row)


def c5(quick=False, traction=-1.3e6, tags=("LagrangeGLL", "ModalJacobi", "SDME_H")):
    out = []
    for tag in tags:
        div = (64, 8, 8) if not quick else (16, 2, 2)
        kind = BasisKind(tag)
        pb = GpuFemProblem(BoxMesh(div, (4.0, 0.5, 0.5)), build_basis(6, kind), MAT, gauss_rule(7),
                           [("xmin", (0, 1, 2))])
        base = pb.traction_vector("xmax", [0.0, 0.0, traction])
        n_steps = 50 if not quick else 5
        load = ScaledLoad(base, lambda t, T=n_steps * 1e-3: min(t / T, 1.0))
        cfg = SolverConfig(precond="diagonal", tol=1e-10, condense=False, maxit=200000)
        t0 = time.perf_counter()
        traj = newmark_run(pb, load, 1e-3, n_steps, newton_tol=1e-8, cfg=cfg)
        wall = time.perf_counter() - t0
        its = [r["iterations"] for r in traj.stats.rows if r["step"] >= 0]
        lat = pb.to_lattice(traj.state.u)
        # vertex coefficients are point values in every basis (internal modes vanish there)
        tip = float(lat[2, ::6, ::6, -1].mean())
        row = {"config": "c5", "basis": tag, "n_free": pb.n_free, "steps": n_steps, "s_per_step": wall / n_steps,
               "newton_iters_mean": float(np.mean(traj.newton_iters)), "pcg_iters_mean": float(np.mean(its)),
               "pcg_iters_max": int(max(its)), "tip_uz_mean": tip, "tip_deflection_over_length": -tip / 4.0,
               "traction": traction}
        if CPU:
            from tools import refcpu

            # the reference on the 8x1x1 reduction (same h, aspect, P, rule;
            # tests/golden config5), 2 steps, scaled by the element count
            r = refcpu.newmark_step_s((8, 1, 1), (0.5, 0.0625, 0.0625), 6, 7, tag, [0.0, 0.0, -8.0e5],
                                      2.0833e-3, 3 * 2.0833e-3, 2)
            if r:
                sps = r["step_s"][-1]
                row["cpu"] = {"s_per_step_8_elements": sps, "s_per_step_extrapolated": sps * int(np.prod(div)) / 8,
                              "kind": "reference", "cores": r["cores"], "newton": r["newton"], "pcg": r["pcg"],
                              "what": "sdmefem newmark_run on 8x1x1 elements (h = 0.0625, P = 6, m = 7), 2nd step "
                                      "wall time, scaled by 4096 / 8 elements (Newton / PCG counts differ from "
                                      "the full mesh: extrapolated)"}
                row["speedup_extrapolated"] = row["cpu"]["s_per_step_extrapolated"] / row["s_per_step"]
        emit(row)


if __name__ == "__main__":
    quick = "--quick" in sys.argv
    for a in sys.argv[1:]:
        if a.startswith("--"):
            continue
        if a.startswith("c5:"):  # c5:<traction>[:<basis>] calibration runs
            parts = a.split(":")
            c5(quick, float(parts[1]), tuple(parts[2:]) or ("SDME_H",))
            continue
        {"c1": c1, "c3": lambda: c3(quick), "c4": lambda: c4(quick), "c5": lambda: c5(quick)}[a]()
