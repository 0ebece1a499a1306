"""Debug aid: GPU PCG iterations / solution error against the reference golden on the general-mesh
cases m5, m6 (tests/golden/meshes.npz).  Run from the repo root on a GPU box."""
import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np
from test_gpu_mesh import gpu_case, golden_mesh_cases
from conftest import max_rel_err
from paper_2104_13466_b200 import pcg_gpu
for i in (5, 6):
    g, key, pb = gpu_case(golden_mesh_cases()[i])
    u, cm = g[f"{key}_u"], float(g[f"{key}_cm"])
    for tol in (1e-10,):
        x, st = pcg_gpu(pb, u, g[f"{key}_pcg_b"], c_m=cm, precond="diagonal", tol=tol, maxit=100000)
        print(key, "gpu its", st.iterations, "ref", int(g[f"{key}_pcg_iters"]), "x err", max_rel_err(x, g[f"{key}_pcg_x"]), "res", st.residual)
