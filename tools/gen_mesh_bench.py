"""General-mesh (F4) operator throughput: a perturbed n^3 box (interior
vertices moved by up to 20% of h, every element's local axes rotated at
random, vertex ids shuffled) at P = 4; K.p / f_int / PCG-operator times by
CUDA events (GpuFemProblem.time_op), next to the box-mesh path on the same
element count.  python tools/gen_mesh_bench.py [n ...]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_13466_b200 import (BasisKind, BoxMesh, GpuFemProblem, GpuMeshProblem, HexMesh, NeoHookean,  # noqa: E402
                                   build_basis)
from paper_2104_13466_b200.basis import gauss_rule  # noqa: E402

MAT = NeoHookean.from_engineering(1e7, 0.3, 1e3)
BITS = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))


def rotations():
    import itertools
    out = []
    for perm in itertools.permutations(range(3)):
        for flips in itertools.product((0, 1), repeat=3):
            m = np.zeros((3, 3))
            for d in range(3):
                m[perm[d], d] = -1.0 if flips[d] else 1.0
            if np.linalg.det(m) > 0:
                out.append((perm, flips))
    return out


def general_box(n, seed=0):
    rng = np.random.default_rng(seed)
    box = HexMesh.box((n, n, n), (1.0, 1.0, 1.0))
    coords = box.coords.copy()
    inner = np.all((coords > 1e-12) & (coords < 1 - 1e-12), axis=1)
    coords[inner] += 0.2 / n * rng.uniform(-1, 1, (int(inner.sum()), 3))
    rots = rotations()
    # local-axis rotation per element: new local corner b -> old corner index
    tabs = []
    for perm, flips in rots:
        t = []
        for b in BITS:
            x = [0, 0, 0]
            for d in range(3):
                x[perm[d]] = 1 - b[d] if flips[d] else b[d]
            t.append(BITS.index(tuple(x)))
        tabs.append(t)
    tabs = np.array(tabs)
    choice = rng.integers(len(rots), size=box.n_elems)
    elems = np.take_along_axis(box.elems, tabs[choice], axis=1)
    newid = rng.permutation(len(coords))
    c2 = np.empty_like(coords)
    c2[newid] = coords
    boundary = {t: [tuple(int(newid[v]) for v in q) for q in qs] for t, qs in box.boundary.items()}
    return HexMesh(c2, newid[elems], boundary)


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [32]
    P = 4
    basis = build_basis(P, BasisKind("SDME_M"))
    for n in sizes:
        t0 = time.perf_counter()
        mesh = general_box(n)
        pb = GpuMeshProblem(mesh, basis, MAT, dirichlet=[("xmin", (0, 1, 2))],
                            locality=os.environ.get("GEN_LOCALITY", "1") == "1")
        setup_s = time.perf_counter() - t0
        rng = np.random.default_rng(0)
        u = pb.vector(1e-3 / n * rng.uniform(-1, 1, pb.n_free))
        p = pb.vector(rng.standard_normal(pb.n_free))
        y = pb.vector()
        row = {"mesh": f"general {n}^3 perturbed/rotated", "P": P, "n_free": pb.n_free, "host_setup_s": setup_s}
        pb.time_op("setup", u, p, y, 0.0, 1)
        for op in ("apply", "fint", "apply_pa"):
            pb.time_op(op, u, p, y, 0.0, 2)
            ms = pb.time_op(op, u, p, y, 0.0, 10)
            row[op + "_ms"] = ms
            row[op + "_gdofs"] = pb.n_free / ms * 1e-6
        box = GpuFemProblem(BoxMesh((n, n, n), (1.0,) * 3), basis, MAT, gauss_rule(P + 1), [("xmin", (0, 1, 2))])
        ub = box.vector(1e-3 / n * rng.uniform(-1, 1, box.n_free))
        pbv = box.vector(rng.standard_normal(box.n_free))
        yb = box.vector()
        box.time_op("apply", ub, pbv, yb, 0.0, 2)
        row["box_apply_ms"] = box.time_op("apply", ub, pbv, yb, 0.0, 10)
        print(json.dumps(row), flush=True)
        del pb, u, p, y, box, ub, pbv, yb


if __name__ == "__main__":
    main()
