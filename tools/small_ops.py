"""Operator latencies on small meshes (E-vector mode) vs colour passes."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.run_configs import MAT  # noqa: E402
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

for ev in ("1", "0"):
    os.environ["SDME_EV"] = ev
    for div, m in (((4, 4, 4), 6), ((8, 8, 8), 6), ((16, 16, 16), 5)):
        pb = GpuFemProblem(BoxMesh(div, (1.0, 1.0, 1.0)), build_basis(4, BasisKind("SDME_M")), MAT,
                           gauss_rule(m), [("xmin", (0, 1, 2))])
        rng = np.random.default_rng(0)
        u = pb.vector().set_free(1e-4 * rng.uniform(-1, 1, pb.n_free))
        p = pb.vector().set_free(rng.standard_normal(pb.n_free))
        y = pb.vector()
        row = {"ev": ev, "div": div[0], "m": m}
        for op, cm in (("apply", 0.0), ("apply", 4e8), ("fint", 0.0), ("mass", 0.0), ("diag", 4e8)):
            pb.time_op(op, u, p, y, c_m=cm, reps=3)
            row[f"{op}{'+M' if cm and op == 'apply' else ''}_us"] = round(1e3 * pb.time_op(op, u, p, y, c_m=cm,
                                                                                              reps=50), 2)
        print(row)
