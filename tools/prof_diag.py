"""ncu driver: config 2 (64^3, P = 4, m = 5) Jacobi diagonal diag(K_T(u) + c_m M), twice."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

pb = GpuFemProblem(BoxMesh((64,) * 3, (1.0,) * 3), build_basis(4, BasisKind("SDME_M")),
                   NeoHookean.from_engineering(1e7, 0.3, 1e3), gauss_rule(5), reference_order=False)
u_lat, _ = bench.config2_fields(pb)
u = pb.vector().set_lattice(u_lat)
y = pb.vector()
for _ in range(2):
    pb.diag_(u, y, 1.0, 4e8)
pb.sync()
print("ok")
