"""Config 1, one Newmark step after warm-up (ncu launch-list driver)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.run_configs import MAT  # noqa: E402
from paper_2104_13466_b200 import (BoxMesh, GpuFemProblem, ScaledLoad, SolverConfig, build_basis,  # noqa: E402
                                   newmark_run)
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402

pb = GpuFemProblem(BoxMesh((4, 4, 4), (1.0, 1.0, 1.0)), build_basis(4, BasisKind("SDME_M")), MAT,
                   gauss_rule(6), [("xmin", (0, 1, 2))])
base = pb.traction_vector("xmax", [0.0, 0.0, 1.0e5])
load = ScaledLoad(base, lambda t: min(t / 1e-3, 1.0))
cfg = SolverConfig(precond="diagonal", tol=1e-10, condense=False)
newmark_run(pb, load, 1e-4, int(sys.argv[1]) if len(sys.argv) > 1 else 1, cfg=cfg)
pb.sync()
