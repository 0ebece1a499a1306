"""Config 1: host-side time per Newmark step split by call (PCG solves, f_int, mass,
vector updates, norms), by wrapping the driver's calls with perf_counter timers."""
import sys, time, os
sys.path.insert(0, '.')
import numpy as np
from tools.run_configs import MAT
from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, build_basis, ScaledLoad, SolverConfig, newmark_run
from paper_2104_13466_b200.basis import BasisKind, gauss_rule
import paper_2104_13466_b200.dynamics as dyn
import paper_2104_13466_b200.solver as sol
pb = GpuFemProblem(BoxMesh((4, 4, 4), (1.0, 1.0, 1.0)), build_basis(4, BasisKind("SDME_M")), MAT, gauss_rule(6), [("xmin", (0, 1, 2))])
base = pb.traction_vector("xmax", [0.0, 0.0, 1.0e5])
load = ScaledLoad(base, lambda t: min(t / 1e-3, 1.0))
cfg = SolverConfig(precond="diagonal", tol=1e-10, condense=False)
newmark_run(pb, load, 1e-4, 1, cfg=cfg)
acc = {}
orig_pcg = sol.pcg_gpu
def timed(name, fn):
    def w(*a, **k):
        t = time.perf_counter(); r = fn(*a, **k); acc[name] = acc.get(name, 0) + time.perf_counter() - t; return r
    return w
sol.pcg_gpu = timed("pcg", orig_pcg)
from paper_2104_13466_b200 import problem as prb
GpuFemProblem.fint_ = timed("fint", GpuFemProblem.fint_)
GpuFemProblem.mass_ = timed("mass", GpuFemProblem.mass_)
from paper_2104_13466_b200.problem import DeviceVector
DeviceVector.norm = timed("norm", DeviceVector.norm)
DeviceVector.assign = timed("assign", DeviceVector.assign)
t0 = time.perf_counter()
newmark_run(pb, load, 1e-4, 10, newton_tol=1e-8, cfg=cfg)
tot = time.perf_counter() - t0
print({k: round(v / 10 * 1e3, 4) for k, v in acc.items()}, "total ms/step", round(tot / 10 * 1e3, 4))
