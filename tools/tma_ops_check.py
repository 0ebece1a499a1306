"""Debug aid: each operator separately through the colour-pass path for one P."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SDME_EV", "0")
import numpy as np  # noqa: E402

from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

P = int(sys.argv[1])
op = sys.argv[2]
div = tuple(int(x) for x in sys.argv[3].split(",")) if len(sys.argv) > 3 else (3, 2, 2)
pb = GpuFemProblem(BoxMesh(div, (1.0, 1.0, 1.0)), build_basis(P, BasisKind("SDME_M" if P > 1 else "LagrangeGLL")),
                   NeoHookean.from_engineering(1e7, 0.3, 1e3), gauss_rule(P + 1), [("xmin", (0, 1, 2))])
u = 1e-3 * np.random.default_rng(0).uniform(-1, 1, pb.n_free)
try:
    f = {"fint": lambda: pb.internal_force(u), "apply": lambda: pb.apply_tangent(u, u, 0.0),
         "mass": lambda: pb.mass_apply(u), "applym": lambda: pb.apply_tangent(u, u, 1.0)}[op]()
    print("P", P, op, div, os.environ.get("SDME_VARIANT"), "ok", float(np.abs(f).max()))
except Exception as e:  # noqa: BLE001
    print("P", P, op, div, os.environ.get("SDME_VARIANT"), "error", e)
