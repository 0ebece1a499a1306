"""P = 2 all-component TMA kernel (element_v3 TMB) at config-3 size: K.p and
f_int from the colour passes, timed, with a checksum of the results so two
builds (e.g. SDME_LIB=<register-cap variant>) can be compared bit for bit.

    python tools/tmb_check.py [n_elem_side=128] [out.npz]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import hashlib  # noqa: E402

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
P = int(os.environ.get("TMB_P", "2"))
pb = GpuFemProblem(BoxMesh((n,) * 3, (1.0,) * 3), build_basis(P, BasisKind("SDME_M")),
                   NeoHookean.from_engineering(1e7, 0.3, 1e3), gauss_rule(P + 1), reference_order=False)
u_lat, p_lat = bench.config2_fields(pb)
u = pb.vector().set_lattice(u_lat)
p = pb.vector().set_lattice(p_lat)
y = pb.vector()
out = {}
for name, fn in (("kp", lambda: pb.apply_(u, p, y)), ("fint", lambda: pb.fint_(u, y)),
                 ("kpm", lambda: pb.apply_(u, p, y, 1.0, 3e4))):
    fn()
    a = y.lattice()
    out[name] = hashlib.sha256(a.tobytes()).hexdigest()[:16]
    out[name + "_max"] = float(np.abs(a).max())
t_kp = pb.time_op("apply", u, p, y, 0.0, 10)
t_f = pb.time_op("fint", u, p, y, 0.0, 10)
print({"n": n, "P": P, "lib": os.environ.get("SDME_LIB", "default"), "kp_ms": t_kp, "fint_ms": t_f, **out})
