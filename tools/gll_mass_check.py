"""Debug aid: diagonality of the GLL collocation mass on the GPU."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2104_13466_b200 import BoxMesh, GpuFemProblem, NeoHookean, build_basis, gll_rule  # noqa: E402
from paper_2104_13466_b200.basis import BasisKind  # noqa: E402

pb = GpuFemProblem(BoxMesh((3, 2, 2), (1.5, 1.0, 1.0)), build_basis(3, BasisKind("LagrangeGLL")),
                   NeoHookean.from_engineering(1e7, 0.3, 1e3), gll_rule(4), [("xmin", (0, 1, 2))])
d = pb.mass_apply(np.ones(pb.n_free))
p = np.random.default_rng(4).standard_normal(pb.n_free)
mp = pb.mass_apply(p)
rel = np.abs(mp - d * p) / np.abs(d * p).max()
print("min d", d.min(), "max rel", rel.max(), "argmax", rel.argmax())
e = np.zeros(pb.n_free)
e[int(rel.argmax())] = 1.0
col = pb.mass_apply(e)
nz = np.nonzero(col)[0]
print("column nonzeros", len(nz), col[nz][:10])
