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
