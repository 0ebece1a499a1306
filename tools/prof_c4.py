"""Config-4 explicit steps (80x16x16, P = 3, lumped mass, penalty contact) for an ncu launch list:
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/prof_c4.py
profiles 3 steps after a warm-up; without ncu it prints the wall time per step of a 500-step chunk."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tools.run_configs import MAT  # noqa: E402
from paper_2104_13466_b200 import (BoxMesh, ContactParams, GpuFemProblem, GpuPenaltyContact,  # noqa: E402
                                   RigidObstacle, build_basis)
from paper_2104_13466_b200.basis import BasisKind, gauss_rule  # noqa: E402
from paper_2104_13466_b200.dynamics import estimate_lambda_max, explicit_run, lumped_mass  # noqa: E402

P = 3
pb = GpuFemProblem(BoxMesh((80, 16, 16), (1.0, 0.2, 0.2)), build_basis(P, BasisKind("SDME_M")), MAT, gauss_rule(P + 1))
contact = GpuPenaltyContact(pb, RigidObstacle([-1e-3, 0.0, 0.0], [1.0, 0.0, 0.0]), ContactParams(1e10), "xmin")
_, inv_ml = lumped_mass(pb)
dt = 0.5 * 2.0 / np.sqrt(estimate_lambda_max(pb, inv_ml, contact=contact))
v0 = pb.constant_field([-10.0, 0.0, 0.0])
explicit_run(pb, None, dt, 5, v0=v0, contact=contact, mass="lumped")
pb.sync()
torch.cuda.profiler.start()
explicit_run(pb, None, dt, 3, v0=v0, contact=contact, mass="lumped")
pb.sync()
torch.cuda.profiler.stop()
for rec in (500, 50):
    t0 = time.perf_counter()
    explicit_run(pb, None, dt, 500, v0=v0, contact=contact, record_every=rec, mass="lumped")
    pb.sync()
    print(f"record_every {rec}: {(time.perf_counter() - t0) / 500 * 1e6:.1f} us per step", flush=True)
