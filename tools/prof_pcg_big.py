"""ncu driver: a few PCG iterations at 64^3 P = 4 (config-2 size)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from tools.run_configs import MAT  # noqa: E402
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402
from paper_2104_13466_b200.errors import PCGError  # noqa: E402
from paper_2104_13466_b200.solver import pcg_gpu  # noqa: E402

os.environ.setdefault("SDME_PCG_DIRECT", "1")
pb = GpuFemProblem(BoxMesh((64,) * 3, (1.0,) * 3), build_basis(4, BasisKind("SDME_M")), MAT, gauss_rule(5),
                   [("xmin", (0, 1, 2))], reference_order=False)
rng = np.random.default_rng(0)
u = pb.vector().set_lattice(1e-6 * rng.uniform(-1, 1, pb.n_lattice))
b = pb.vector().set_lattice(rng.standard_normal(pb.n_lattice))
x = pb.vector()
try:
    pcg_gpu(pb, u, b, c_m=4e8, precond="diagonal", tol=1e-300, maxit=3, x=x)
except PCGError:
    pass
print("ok")
