"""Shared fixtures.  ``-m gpu`` tests need a B200 and the in-tree libsdme.so;
``-m "not gpu"`` tests run on any CPU box (oracle vs golden vectors, host
logic, ABI symbol table)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
KINDS = ("LagrangeGLL", "ModalJacobi", "SDME_M", "SDME_K", "SDME_H")
FACES = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")


def reference_src():
    """Directory holding the reference package ``sdmefem`` (the offline
    install under baseline/_ref, which also travels to the GPU box, else the
    read-only tree of the build container), or None.  Only tests import it,
    as the pin of the drop-in adapter; nothing on the product path does."""
    for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "sdmefem")):
            return cand
    return None


def import_reference():
    """Import sdmefem from :func:`reference_src` (numba cache redirected to a
    writable directory), or skip the calling test."""
    src = reference_src()
    if src is None:
        pytest.skip("reference package sdmefem not available")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "sdme_numba_cache"))
    if src not in sys.path:
        sys.path.append(src)
    try:
        import sdmefem  # noqa: F401
    except Exception as exc:  # e.g. numba missing
        pytest.skip(f"reference package not importable: {exc}")
    import sdmefem.dynamics
    import sdmefem.femcore
    return sdmefem


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and libsdme.so")
    config.addinivalue_line("markers", "slow: longer-running oracle checks")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="session")
def golden():
    return load_golden


def element_cases():
    g = load_golden("elements")
    n = len({k.split("_")[0] for k in g.files})
    out = []
    for i in range(n):
        meta = g[f"c{i}_meta"]
        out.append((i, KINDS[int(meta[0])], int(meta[1]), int(meta[2]), tuple(meta[3:6])))
    return out


def global_cases():
    g = load_golden("global")
    n = len({k.split("_")[0] for k in g.files})
    out = []
    for i in range(n):
        meta = g[f"g{i}_meta"]
        dr = {}
        for f, c in g[f"g{i}_dir"].reshape(-1, 2):
            dr.setdefault(FACES[int(f)], []).append(int(c))
        out.append((i, KINDS[int(meta[0])], int(meta[1]), int(meta[2]), tuple(int(v) for v in meta[3:6]),
                    tuple(meta[6:9]), [(t, tuple(c)) for t, c in dr.items()]))
    return out


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def max_rel_err(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))
