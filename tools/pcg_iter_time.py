"""Per-iteration cost of the device PCG on the config-1 mesh (and others):
time a solve capped at k1 and at k2 iterations (tol too small to converge)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.run_configs import MAT  # noqa: E402
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402
from paper_2104_13466_b200.errors import PCGError  # noqa: E402
from paper_2104_13466_b200.solver import pcg_gpu  # noqa: E402


def run(div, P, m):
    pb = GpuFemProblem(BoxMesh(div, (1.0, 1.0, 1.0)), build_basis(P, BasisKind("SDME_M")), MAT,
                       gauss_rule(m), [("xmin", (0, 1, 2))])
    rng = np.random.default_rng(0)
    u = pb.vector().set_free(1e-4 * rng.uniform(-1, 1, pb.n_free))
    b = pb.vector().set_free(rng.standard_normal(pb.n_free))
    x = pb.vector()
    res = {}
    for k in (5, 5, 105):
        t0 = time.perf_counter()
        for _ in range(5):
            try:
                pcg_gpu(pb, u, b, c_m=4e8, precond="diagonal", tol=1e-300, maxit=k, x=x)
            except PCGError:
                pass
        res[k] = (time.perf_counter() - t0) / 5
    per = (res[105] - res[5]) / 100
    print({"div": div, "P": P, "m": m, "n_dofs": pb.n_free, "solve_overhead_ms": 1e3 * (res[5] - 5 * per),
           "per_iter_us": 1e6 * per})


if __name__ == "__main__":
    if len(sys.argv) > 1:  # e.g. 64 4 5: per-iteration cost at config-2 size
        n, P, m = (int(a) for a in sys.argv[1:4])
        run((n, n, n), P, m)
    else:
        run((4, 4, 4), 4, 6)
        run((8, 8, 8), 4, 6)
    run((16, 16, 16), 4, 5)
    run((32, 32, 32), 4, 5)
