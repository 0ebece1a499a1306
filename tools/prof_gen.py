"""ncu driver: one general-mesh K.p (gather, element, assembly) at 48^3, P = 4."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import gen_mesh_bench as gb  # noqa: E402
from paper_2104_13466_b200 import BasisKind, GpuMeshProblem, build_basis  # noqa: E402

n = int(os.environ.get("PROF_N", "48"))
pb = GpuMeshProblem(gb.general_box(n), build_basis(4, BasisKind("SDME_M")), gb.MAT, dirichlet=[("xmin", (0, 1, 2))])
rng = np.random.default_rng(0)
u = pb.vector(1e-3 / n * rng.uniform(-1, 1, pb.n_free))
p = pb.vector(rng.standard_normal(pb.n_free))
y = pb.vector()
for _ in range(2):
    pb.apply_(u, p, y)
pb.sync()
print("ok", pb.launch_count())
