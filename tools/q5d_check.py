"""A/B of the P = 4 quintet diagonal kernel (element_q5d.cuh, default) against
element_diag3 (SDME_VARIANT=13): same point coefficients and tables, the x'
stage sums the six chains in a different order, so the two agree to rounding
(<= 1e-13 relative), on meshes with ghost elements, Dirichlet faces, cubic
and non-cubic elements, with and without the mass term."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from q5_check import problem  # noqa: E402


def main():
    bad = 0
    dr1 = (("xmin", (0, 1, 2)),)
    cases = [((3, 2, 2), "SDME_M", dr1, (1.0, 1.0, 1.0)),
             ((7, 6, 5), "LagrangeGLL", (("xmin", (0, 1, 2)), ("ymax", (1,))), (1.0, 1.0, 1.0)),
             ((1, 1, 1), "SDME_M", (("zmin", (0, 1, 2)),), (1.0, 1.0, 1.0)),
             ((11, 3, 9), "ModalJacobi", (("xmax", (0, 1, 2)), ("zmin", (2,))), (1.0, 0.75, 1.5)),
             ((16, 16, 16), "SDME_M", dr1, (1.0, 1.0, 1.0))]
    for div, tag, dr, hs in cases:
        a, b = problem(div, tag, 0, dr, hs), problem(div, tag, 13, dr, hs)
        rng = np.random.default_rng(2)
        u = 2e-2 / 64 * rng.uniform(-1, 1, a.n_free)
        for cm in (0.0, 4e8):
            da, db = a.tangent_diagonal(u, cm), b.tangent_diagonal(u, cm)
            rel = float(np.abs(da - db).max() / np.abs(db).max())
            ok = rel <= 1e-13 and np.array_equal(a.tangent_diagonal(u, cm), da)
            print(div, hs, tag, "c_m", cm, f"rel {rel:.2e}", "ok" if ok else "MISMATCH", flush=True)
            bad += not ok
    print("q5d_check", "FAILED" if bad else "ok")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
