"""Run the BASELINE.json configs 1, 3, 4, 5 on one GPU and print one JSON line each.

    python tools/run_configs.py c1 c3 c4 c5 [--quick]

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


def emit(d):
    print(json.dumps(d), flush=True)


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
    emit({"config": "c1", "s_per_step": wall / 10, "total_s": wall, "newton_iters": traj.newton_iters,
          "pcg_iters": its, "max_u": float(np.abs(traj.state.u).max()), "n_free": pb.n_free})


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
            emit({"config": "c3", "P": P, "basis": tag, "n_elem_side": n, "n_dofs": pb.n_lattice,
                  "kp_ms": t_kp * 1e3, "kp_gdofs": pb.n_lattice / t_kp / 1e9,
                  "kp_tflops": flops / t_kp / 1e12, "kp_frac_fp64": flops / t_kp / 1e12 / fp if fp else None,
                  "fint_ms": t_f * 1e3, "fint_gdofs": pb.n_lattice / t_f / 1e9})
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
    emit({"config": "c4", "elements": int(np.prod(div)), "n_dofs": pb.n_free, "dt": dt, "lambda_max": lam,
          "steps": n_steps, "s_per_step": wall / n_steps, "total_s": wall,
          "max_penetration": max(h[1] for h in hist) if hist else 0.0,
          "contact_active_max": max(h[3] for h in hist) if hist else 0,
          "final_mean_vx": float(traj.state.v[0::3].mean()), "history_every50": hist[:8]})


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
        emit({"config": "c5", "basis": tag, "n_free": pb.n_free, "steps": n_steps, "s_per_step": wall / n_steps,
              "newton_iters_mean": float(np.mean(traj.newton_iters)), "pcg_iters_mean": float(np.mean(its)),
              "pcg_iters_max": int(max(its)), "tip_uz_mean": tip, "tip_deflection_over_length": -tip / 4.0,
              "traction": traction})


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
