"""ncu driver: a few PCG iterations at config-5 size (64x8x8, P = 6, SDME_H), plain launches
(SDME_PCG_DIRECT=1) so every kernel of an iteration appears in the launch list:
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file x.csv python tools/prof_pcg_c5.py
Without ncu it also prints the per-iteration time of the graph path."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from tools.run_configs import MAT  # noqa: E402
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402
from paper_2104_13466_b200.errors import PCGError  # noqa: E402
from paper_2104_13466_b200.solver import pcg_gpu  # noqa: E402


def run(direct, maxit):
    if direct:
        os.environ["SDME_PCG_DIRECT"] = "1"
    else:
        os.environ.pop("SDME_PCG_DIRECT", None)
    pb = GpuFemProblem(BoxMesh((64, 8, 8), (4.0, 0.5, 0.5)), build_basis(6, BasisKind("SDME_H")), MAT, gauss_rule(7),
                       [("xmin", (0, 1, 2))])
    rng = np.random.default_rng(0)
    u = pb.vector().set_free(1e-6 * rng.uniform(-1, 1, pb.n_free))
    b = pb.vector().set_free(rng.standard_normal(pb.n_free))
    x = pb.vector()
    ts = []
    for mi in maxit:
        t0 = time.perf_counter()
        try:
            pcg_gpu(pb, u, b, c_m=4e6, precond="diagonal", tol=1e-300, maxit=mi, x=x)
        except PCGError:
            pass
        pb.sync()
        ts.append(time.perf_counter() - t0)
    return ts


run(True, [3])
if "--time" in sys.argv:
    ts = run(False, [10, 10, 210])
    print(f"graph path: {(ts[2] - ts[1]) / 200 * 1e6:.1f} us per iteration", flush=True)
print("ok")
