"""Exception types of the path, mirroring the reference's failure contract
(femcore.py:36-42, solver.py:33-38, dynamics.py:32-35).

When the reference package ``sdmefem`` is importable, each class here
*subclasses* the reference's own type, so ``except sdmefem.solver.PCGError``
clauses written against the reference keep catching the GPU path's errors
after the drop-in swap.  Without the reference they derive from
``RuntimeError`` exactly as the reference's classes do.  Constructor
signatures and attributes are the reference's.
"""

from __future__ import annotations

import importlib.util


def _reference_types():
    """(ElementInversionError, PCGError, NewtonDivergenceError) of the
    reference, or RuntimeError for each when sdmefem is not installed."""
    try:
        if importlib.util.find_spec("sdmefem") is None:
            raise ImportError
        from sdmefem.dynamics import NewtonDivergenceError as _nd
        from sdmefem.femcore import ElementInversionError as _ei
        from sdmefem.solver import PCGError as _pcg
        return _ei, _pcg, _nd, True
    except Exception:  # not installed, or its import fails (e.g. no numba)
        return RuntimeError, RuntimeError, RuntimeError, False


_RefInversion, _RefPCG, _RefNewton, REFERENCE_TYPES = _reference_types()


class ElementInversionError(_RefInversion):
    """det F <= 0 at a quadrature point (``femcore.py:36-42``).

    ``elem_id`` is the smallest offending element id (reference element loop
    order) and ``qp`` the first offending point in the reference point order
    (a, b, c with c fastest), exactly as the reference reports it.
    """

    def __init__(self, elem_id: int, qp: int):
        RuntimeError.__init__(self, f"element {elem_id} inverted at quadrature point {qp}")
        self.elem_id = elem_id
        self.qp = qp


class PCGError(_RefPCG):
    """PCG failure carrying the stats gathered so far (``solver.py:33-38``)."""

    def __init__(self, message, stats=None):
        RuntimeError.__init__(self, message)
        self.stats = stats


class NewtonDivergenceError(_RefNewton):
    """``dynamics.py:32-35``."""

    def __init__(self, message, residual):
        RuntimeError.__init__(self, message)
        self.residual = residual


class NativeError(RuntimeError):
    """CUDA library missing or a CUDA runtime failure (no CPU fallback)."""
