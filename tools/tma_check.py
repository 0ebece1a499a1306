"""Run f_int / K.p on a small mesh through the colour-pass (TMA) path for one
order P (argv[1]); prints ok or the native error.  Debug aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SDME_EV", "0")
import numpy as np  # noqa: E402

from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

P = int(sys.argv[1])
div = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else (3, 2, 2)
pb = GpuFemProblem(BoxMesh(div, (1.0, 1.0, 1.0)), build_basis(P, BasisKind("SDME_M")),
                   NeoHookean.from_engineering(1e7, 0.3, 1e3), gauss_rule(P + 1), [("xmin", (0, 1, 2))])
u = 1e-3 * np.random.default_rng(0).uniform(-1, 1, pb.n_free)
try:
    f = pb.internal_force(u)
    y = pb.apply_tangent(u, u, 1.0)
    print("P", P, "ok", float(np.abs(f).max()), float(np.abs(y).max()))
except Exception as e:  # noqa: BLE001
    print("P", P, "error", e)
