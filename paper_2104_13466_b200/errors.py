"""Exception types of the path, mirroring the reference's failure contract
(femcore.py:36-42, solver.py:33-38, dynamics.py:32-35)."""

from __future__ import annotations


class ElementInversionError(RuntimeError):
    """det F <= 0 at a quadrature point (``femcore.py:36-42``).

    ``elem_id`` is the smallest offending element id (reference element loop
    order) and ``qp`` the first offending point in the reference point order
    (a, b, c with c fastest), exactly as the reference reports it.
    """

    def __init__(self, elem_id: int, qp: int):
        super().__init__(f"element {elem_id} inverted at quadrature point {qp}")
        self.elem_id = elem_id
        self.qp = qp


class PCGError(RuntimeError):
    """PCG failure carrying the stats gathered so far (``solver.py:33-38``)."""

    def __init__(self, message, stats=None):
        super().__init__(message)
        self.stats = stats


class NewtonDivergenceError(RuntimeError):
    """``dynamics.py:32-35``."""

    def __init__(self, message, residual):
        super().__init__(message)
        self.residual = residual


class NativeError(RuntimeError):
    """CUDA library missing or a CUDA runtime failure (no CPU fallback)."""
