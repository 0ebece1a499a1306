"""A/B of the P = 4 quintet kernel (element_q5.cuh, default) against the
warp-per-element kernel (SDME_VARIANT=12): the results must be bit-identical
(same arithmetic per pencil and point, same colour-pass order), on meshes
whose colour classes are not multiples of five (ghost elements), with
Dirichlet faces, for f_int, K.p (with and without c_m M), mass and the PCG
operator (setup + stored-data apply through one solve)."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis, pcg_gpu  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402


def problem(div, tag, variant, dr, hs=(1.0, 1.0, 1.0)):
    os.environ["SDME_EV"] = "0"
    # one z-slab schedule for both kernels (their defaults differ; the order of
    # the colour passes fixes the summation order at shared points)
    os.environ["SDME_SLABS"] = "4"
    if variant:
        os.environ["SDME_VARIANT"] = str(variant)
    try:
        h = 1.0 / 64
        return GpuFemProblem(BoxMesh(div, tuple(d * h * f for d, f in zip(div, hs))), build_basis(4, BasisKind(tag)),
                             NeoHookean.from_engineering(1e7, 0.3, 1e3), gauss_rule(5), list(dr))
    finally:
        os.environ.pop("SDME_EV", None)
        os.environ.pop("SDME_VARIANT", None)
        os.environ.pop("SDME_SLABS", None)


def run(pb, seed):
    rng = np.random.default_rng(seed)
    u = 1e-3 / 64 * rng.uniform(-1, 1, pb.n_free)
    p = rng.standard_normal(pb.n_free)
    out = {"fint": pb.internal_force(u), "kp": pb.apply_tangent(u, p), "kpm": pb.apply_tangent(u, p, 4e8),
           "mass": pb.mass_apply(p)}
    x, st = pcg_gpu(pb, u, p, c_m=4e8, tol=1e-10)
    out["pcg_x"] = x
    out["pcg_it"] = np.array([st.iterations])
    x0, st0 = pcg_gpu(pb, u, p, c_m=0.0, tol=1e-8, maxit=50000)
    out["pcg0_x"] = x0
    out["pcg0_it"] = np.array([st0.iterations])
    return out


# variants to compare (argv: A B; default the quintet kernel against SDME_VARIANT=12;
# "14 12": the stored-data operator on the quintet kernel against the warp-per-element one)
VA, VB = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (0, 12)


def main():
    bad = 0
    cases = [((3, 2, 2), "SDME_M", (("xmin", (0, 1, 2)),)),
             ((7, 6, 5), "LagrangeGLL", (("xmin", (0, 1, 2)), ("ymax", (1,)))),
             ((1, 1, 1), "SDME_M", (("zmin", (0, 1, 2)),)),
             ((11, 3, 9), "ModalJacobi", (("xmax", (0, 1, 2)), ("zmin", (2,)))),
             ((16, 16, 16), "SDME_M", (("xmin", (0, 1, 2)),))]
    # cubic elements take the one-derivative-table instance (ISO), others the
    # general one (tables re-read per component loop): cover both
    cases = [c + ((1.0, 1.0, 1.0),) for c in cases] + [((7, 6, 5), "SDME_M", cases[1][2], (1.0, 0.75, 1.5)),
                                                        ((3, 2, 2), "LagrangeGLL", cases[0][2], (2.0, 1.0, 1.0))]
    for div, tag, dr, hs in cases:
        a = run(problem(div, tag, VA, dr, hs), 1)
        b = run(problem(div, tag, VB, dr, hs), 1)
        for k in a:
            same = np.array_equal(a[k], b[k])
            rel = float(np.abs(a[k] - b[k]).max() / max(np.abs(b[k]).max(), 1e-300))
            print(div, hs, tag, k, "bit-identical" if same else f"DIFF rel {rel:.3e}", flush=True)
            bad += not same
    print("q5_check", "FAILED" if bad else "ok")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
