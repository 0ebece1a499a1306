"""ncu driver: config 2, K.p + mass + f_int with the schedule variant in SDME_VARIANT."""
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
pb.apply_(u, p, y)   # launches 0-7
pb.mass_(p, y)       # 8-15
pb.fint_(u, y)       # 16-23
pb.sync()
print("ok")
