"""E-vector vs colour-pass operator times on a few mesh sizes (sets kEvMaxElements)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.run_configs import MAT  # noqa: E402
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

CASES = [((64, 8, 8), 6, 7, (4.0, 0.5, 0.5)), ((16, 16, 16), 4, 5, (1.0,) * 3), ((24, 24, 24), 4, 5, (1.0,) * 3),
         ((32, 32, 32), 4, 5, (1.0,) * 3), ((32, 16, 16), 3, 4, (1.0,) * 3)]
for div, P, m, L in CASES:
    row = {"div": div, "P": P}
    for ev in ("1", "0"):
        os.environ["SDME_EV"] = ev
        pb = GpuFemProblem(BoxMesh(div, L), build_basis(P, BasisKind("SDME_H")), MAT, gauss_rule(m),
                           [("xmin", (0, 1, 2))])
        rng = np.random.default_rng(0)
        u = pb.vector().set_free(1e-5 * rng.uniform(-1, 1, pb.n_free))
        p = pb.vector().set_free(rng.standard_normal(pb.n_free))
        y = pb.vector()
        pb.time_op("setup", u, p, y, 0.0, 1)
        for op in ("apply", "apply_pa", "diag"):
            pb.time_op(op, u, p, y, 1e5, 2)
            row[f"{op}_ev{ev}_us"] = round(1e3 * pb.time_op(op, u, p, y, 1e5, 10), 1)
        del pb, u, p, y
    print(row, flush=True)
