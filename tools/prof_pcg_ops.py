"""ncu driver: config 2, the PCG-side operators -- quadrature-data setup,
K.p from stored data (+ c_m M p), Jacobi diagonal (launch order: setup 0,
PA 1-8, diag 9-16)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

pb = GpuFemProblem(BoxMesh((64,) * 3, (1.0,) * 3), build_basis(4, BasisKind("SDME_M")),
                   NeoHookean.from_engineering(1e7, 0.3, 1e3), gauss_rule(5), reference_order=False)
u_lat, p_lat = bench.config2_fields(pb)
u = pb.vector().set_lattice(u_lat)
p = pb.vector().set_lattice(p_lat)
y = pb.vector()
pb.time_op("setup", u, p, y, 0.0, 1)
pb.time_op("apply_pa", u, p, y, 4.0e8, 1)
pb.time_op("diag", u, p, y, 4.0e8, 1)
pb.sync()
print("ok")
