"""ms per call of each operator at config-2 size (64^3, P = 4, m = 5): K.p, f_int, mass, PCG setup/operator."""
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
out = {}
for op in ("apply", "fint", "mass", "setup", "apply_pa", "diag"):
    pb.time_op(op, u, p, y, 1e3 if op == "mass" else 0.0, 2)
    out[op] = round(pb.time_op(op, u, p, y, 1e3 if op == "mass" else 0.0, 10), 4)
# the Newmark operators: K.p + c_m M p from u and from the stored quadrature data
for op in ("apply", "apply_pa"):
    pb.time_op(op, u, p, y, 4e8, 2)
    out[op + "+m"] = round(pb.time_op(op, u, p, y, 4e8, 10), 4)
print(os.environ.get("SDME_VARIANT", "0"), out)
