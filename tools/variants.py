"""Time the P=4 schedule variants (SDME_VARIANT) on config 2 and check they
agree with variant 0.  Usage: python tools/variants.py 0 8

Current variants: 0 = default (component-serial, staged, even-odd), 8 =
column-fused v5.  The earlier variants in profiles/variants_r01.txt (1-5) were
template arguments of the v3 kernel and the removed column-resident v4; they are
recorded there, not selectable any more."""
import json
import os
import subprocess
import sys

CHILD = r'''
import os, sys, json, numpy as np
sys.path.insert(0, os.getcwd())
import bench
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis
from paper_2104_13466_b200.basis import BasisKind, gauss_rule
pb = GpuFemProblem(BoxMesh((64,)*3, (1.0,)*3), build_basis(4, BasisKind("SDME_M")),
                   NeoHookean.from_engineering(1e7, 0.3, 1e3), gauss_rule(5), reference_order=False)
u_lat, p_lat = bench.config2_fields(pb)
u = pb.vector().set_lattice(u_lat); p = pb.vector().set_lattice(p_lat); y = pb.vector()
for _ in range(3): pb.apply_(u, p, y)
t_kp = pb.time_op("apply", u, p, y, 0.0, 10)
t_kpm = pb.time_op("apply", u, p, y, 4e8, 10)
t_f = pb.time_op("fint", u, p, y, 0.0, 10)
t_m = pb.time_op("mass", u, p, y, 0.0, 10)
pb.apply_(u, p, y); kp = y.lattice().ravel()
np.save("gpurun_out/kp_variant_%s.npy" % os.environ.get("SDME_VARIANT", "0"), kp[::97])
print(json.dumps({"variant": os.environ.get("SDME_VARIANT", "0"), "kp_ms": t_kp, "kp_cm_ms": t_kpm,
                  "fint_ms": t_f, "mass_ms": t_m, "gdofs": pb.n_lattice / t_kp / 1e6}))
'''

if __name__ == "__main__":
    import numpy as np
    os.makedirs("gpurun_out", exist_ok=True)
    for v in sys.argv[1:]:
        env = dict(os.environ, SDME_VARIANT=v)
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-2000:], flush=True)
    base = np.load("gpurun_out/kp_variant_%s.npy" % sys.argv[1])
    for v in sys.argv[2:]:
        try:
            o = np.load("gpurun_out/kp_variant_%s.npy" % v)
            print(v, "max rel diff vs", sys.argv[1], float(np.abs(o - base).max() / np.abs(base).max()))
        except Exception as e:
            print(v, e)
