"""K.p and f_int ms at one order P over several box sizes (crossover of two kernels;
SDME_VARIANT selects the alternative).  python tools/kp_size.py P n1 n2 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

P = int(sys.argv[1])
for n in map(int, sys.argv[2:]):
    pb = GpuFemProblem(BoxMesh((n,) * 3, (1.0,) * 3), build_basis(P, BasisKind("SDME_M")),
                       NeoHookean.from_engineering(1e7, 0.3, 1e3), gauss_rule(P + 1), reference_order=False)
    rng = np.random.default_rng(0)
    u = pb.vector().set_lattice(1e-3 / n * rng.uniform(-1, 1, pb.n_lattice))
    p = pb.vector().set_lattice(rng.standard_normal(pb.n_lattice))
    y = pb.vector()
    pb.time_op("apply", u, p, y, 0.0, 3)
    kp = pb.time_op("apply", u, p, y, 0.0, 20)
    pb.time_op("fint", u, p, y, 0.0, 3)
    fi = pb.time_op("fint", u, p, y, 0.0, 20)
    print(f"P {P} n {n} elems {n ** 3} variant {os.environ.get('SDME_VARIANT', '0')} "
          f"K.p {kp * 1e3:.1f} us f_int {fi * 1e3:.1f} us", flush=True)
    del pb
