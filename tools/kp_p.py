"""K.p ms at one order P on an ~50M-DOF box (config-3 sizing), for A/B of variants."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

P = int(sys.argv[1])
n = round(256 / P)
pb = GpuFemProblem(BoxMesh((n,) * 3, (1.0,) * 3), build_basis(P, BasisKind("SDME_M")),
                   NeoHookean.from_engineering(1e7, 0.3, 1e3), gauss_rule(P + 1), reference_order=False)
rng = np.random.default_rng(0)
u = pb.vector().set_lattice(1e-3 / n * rng.uniform(-1, 1, pb.n_lattice))
p = pb.vector().set_lattice(rng.standard_normal(pb.n_lattice))
y = pb.vector()
pb.time_op("apply", u, p, y, 0.0, 3)
ms = pb.time_op("apply", u, p, y, 0.0, 10)
print(f"P {P} variant {os.environ.get('SDME_VARIANT', '0')} K.p {ms:.3f} ms {pb.n_lattice / ms * 1e-6:.2f} GDOF/s")
