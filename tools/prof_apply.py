"""Small driver for ncu: config 2 (64^3, P=4, m=5) -> 2 K.p + 1 f_int."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

P = int(os.environ.get("PROF_P", "4"))
N = int(os.environ.get("PROF_N", str(256 // P)))
pb = GpuFemProblem(BoxMesh((N,) * 3, (1.0,) * 3), build_basis(P, BasisKind("SDME_M")),
                   NeoHookean.from_engineering(1e7, 0.3, 1e3), gauss_rule(P + 1), reference_order=False)
u_lat, p_lat = bench.config2_fields(pb)
u = pb.vector().set_lattice(u_lat)
p = pb.vector().set_lattice(p_lat)
y = pb.vector()
for _ in range(2):
    pb.apply_(u, p, y)
pb.fint_(u, y)
pb.sync()
print("ok", pb.launch_count())
