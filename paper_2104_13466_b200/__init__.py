"""B200-native matrix-free neo-Hookean f_int / K.p + Jacobi-PCG for SDME high-order FEM.

Drop-in GPU path for the hot loop of the reference package ``sdmefem``
(arXiv 2104.13466): host code stays Python and keeps the reference entry
points; every operator and vector update runs in ``libsdme.so`` (hand-written
sm_100a FP64 CUDA behind the C ABI of ``include/sdme.h``).
"""

from .basis import Basis1D, BasisKind, build_basis, gauss_rule, gll_rule
from .errors import ElementInversionError, NativeError, NewtonDivergenceError, PCGError
from .lattice import BoxMesh, reference_free_index
from .problem import DeviceVector, GpuFemProblem, NeoHookean
from .solver import GpuLinearSolver, SolverConfig, SolveStats, StatsLog, make_solver, pcg_gpu
from .dynamics import ScaledLoad, cfl_dt, explicit_run, newmark_run
from .contact import ContactParams, GpuPenaltyContact, RigidObstacle
from .mesh import HexMesh, MeshError, read_mesh, write_mesh
from .mesh_problem import GpuMeshProblem

__all__ = [
    "Basis1D", "BasisKind", "build_basis", "gauss_rule", "gll_rule",
    "ElementInversionError", "NativeError", "NewtonDivergenceError", "PCGError",
    "BoxMesh", "reference_free_index",
    "DeviceVector", "GpuFemProblem", "NeoHookean",
    "GpuLinearSolver", "SolverConfig", "SolveStats", "StatsLog", "make_solver", "pcg_gpu",
    "ScaledLoad", "cfl_dt", "explicit_run", "newmark_run",
    "ContactParams", "GpuPenaltyContact", "RigidObstacle",
    "HexMesh", "MeshError", "read_mesh", "write_mesh", "GpuMeshProblem",
]
