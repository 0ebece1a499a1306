"""ncu driver: one K(u).p per order of the config-3 sweep (SDME_M, N = round(256/P))."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from tools.run_configs import MAT  # noqa: E402
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

for P in [int(a) for a in sys.argv[1:]] or [2, 3, 6, 8]:
    n = round(256 / P)
    pb = GpuFemProblem(BoxMesh((n,) * 3, (1.0,) * 3), build_basis(P, BasisKind("SDME_M")), MAT, gauss_rule(P + 1),
                       reference_order=False)
    u_lat, p_lat = bench.config2_fields(pb)
    u = pb.vector().set_lattice(u_lat)
    p = pb.vector().set_lattice(p_lat)
    y = pb.vector()
    pb.apply_(u, p, y)
    pb.sync()
    del pb, u, p, y
print("ok")
