"""CPU baselines: the reference's OWN code timed on this box's host cores.

The reference package ``sdmefem`` is installed offline under baseline/_ref
(``pip install --no-index --no-deps --target baseline/_ref``; git-ignored,
travels to the GPU box with the snapshot).  Every figure here runs the
reference's functions unmodified; when the install is absent the oracle's
restatement (oracle/) stands in and the result says ``kind: "port"``.

Throughput samples run in worker PROCESSES (spawned, one per core, each with
OPENBLAS_NUM_THREADS = SDMEFEM_THREADS = 1), not GIL-bound threads.  The
parent measures the wall time from dispatch until the last worker returns, so
the throughput is what all cores together sustain.

* ``kp_sample`` / ``fint_sample``: element-by-element K.p
  (``element_tangent(tab, mat, u_e) @ p_e``, femcore.py:130-146) or f_int
  (``element_internal_force``, femcore.py:99-106) on elements of the target
  mesh's size h, order P and rule m -- the per-element cost is independent of
  the values, so GDOF/s = elements/s x DOFs per element of the
  target mesh (labelled extrapolated).
* ``newmark_step_s``: the reference's ``newmark_run`` on a given problem; the
  time of one step is read between the first external_load calls of two
  consecutive steps (no setup in it).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
_ONE_THREAD = {"OPENBLAS_NUM_THREADS": "1", "OMP_NUM_THREADS": "1", "MKL_NUM_THREADS": "1", "SDMEFEM_THREADS": "1"}


def reference_dir():
    return REF_DIR if os.path.isdir(os.path.join(REF_DIR, "sdmefem")) else None


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------ worker side
_W = {}


def _setup_reference(P, tag, m, h, seed):
    sys.path.insert(0, REF_DIR)
    import numpy as np
    from sdmefem.basis1d import BasisKind, build_basis
    from sdmefem.femcore import FemProblem, element_internal_force, element_tangent
    from sdmefem.material import NeoHookean
    from sdmefem.meshdof import build_dofmap, gen_box_mesh
    from sdmefem.quadrature import gauss_rule
    from sdmefem.tensorelem import TensorElement

    mesh = gen_box_mesh((2, 2, 2), (2 * h,) * 3)
    el = TensorElement.create(3, build_basis(P, BasisKind(tag)))
    prob = FemProblem(mesh, el, build_dofmap(mesh, el, None), NeoHookean.from_engineering(1e7, 0.3, 1e3),
                      rule=gauss_rule(m))
    rng = np.random.default_rng(seed)
    u = 1e-3 * h * rng.uniform(-1, 1, prob.n_free)
    p = rng.standard_normal(prob.n_free)
    ue = [prob.gather(e, u) for e in range(prob.mesh.n_elems)]
    pe = [prob.gather(e, p).reshape(-1) for e in range(prob.mesh.n_elems)]
    kp = lambda e: element_tangent(prob.tables[e], prob.mat, ue[e], e) @ pe[e]
    fi = lambda e: element_internal_force(prob.tables[e], prob.mat, ue[e], e)
    return prob.mesh.n_elems, kp, fi


def _setup_port(P, tag, m, h, seed):
    sys.path.insert(0, ROOT)
    import numpy as np
    from oracle import basis as ob
    from oracle import fem as of

    pb = of.Problem(of.Mesh((2, 2, 2), (2 * h,) * 3), ob.Basis(tag, P), of.Material(1e7, 0.3, 1e3), m)
    rng = np.random.default_rng(seed)
    u = 1e-3 * h * rng.uniform(-1, 1, pb.n_free)
    p = rng.standard_normal(pb.n_free)
    ue = [pb.gather(e, u) for e in range(pb.mesh.ne)]
    pe = [pb.gather(e, p).reshape(-1) for e in range(pb.mesh.ne)]

    def kp(e):
        _, grad, wdet = pb.tab.per_elem[e]
        return of.elem_tangent(pb.mat, grad, wdet, ue[e], e) @ pe[e]

    def fi(e):
        _, grad, wdet = pb.tab.per_elem[e]
        return of.elem_fint(pb.mat, grad, wdet, ue[e], e)

    return pb.mesh.ne, kp, fi


def _init(kind, P, tag, m, h, seed):
    n, kp, fi = (_setup_reference if kind == "reference" else _setup_port)(P, tag, m, h, seed)
    _W.update(n=n, kp=kp, fi=fi)
    for e in range(n):  # warm (imports, BLAS / numba first calls)
        kp(e)
        fi(e)


def _run(args):
    op, count = args
    f = _W[op]
    n = _W["n"]
    t0 = time.perf_counter()
    for k in range(count):
        f(k % n)
    return time.perf_counter() - t0


# ------------------------------------------------------------ parent side
class ElementSampler:
    """A pool of spawned single-threaded worker processes, each holding one
    2x2x2-element problem of element size h (reference code, or the port)."""

    def __init__(self, P, tag="SDME_M", m=None, h=1.0 / 64, workers=None, seed=0):
        import multiprocessing as mp

        self.kind = "reference" if reference_dir() else "port"
        self.workers = workers or os.cpu_count() or 1
        self.P, self.tag, self.m, self.h = P, tag, m or P + 1, h
        saved = {k: os.environ.get(k) for k in list(_ONE_THREAD) + ["NUMBA_CACHE_DIR"]}
        os.environ.update(_ONE_THREAD)
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/sdme_numba_cache")
        try:  # children inherit this environment at spawn (before they import numpy)
            ctx = mp.get_context("spawn")
            self.pool = ctx.Pool(self.workers, initializer=_init,
                                 initargs=(self.kind, P, tag, self.m, h, seed))
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        self.pool.map(_run, [("kp", 1)] * self.workers)  # all workers initialised

    def sample(self, op: str, per_worker: int) -> dict:
        """Wall time for every worker to evaluate ``per_worker`` elements
        (op "kp" or "fi"); returns elements, seconds, elements/s."""
        t0 = time.perf_counter()
        busy = self.pool.map(_run, [(op, per_worker)] * self.workers, chunksize=1)
        dt = time.perf_counter() - t0
        n = per_worker * self.workers
        return {"elements": n, "seconds": dt, "elements_per_s": n / dt, "worker_busy_s": max(busy),
                "cores": self.workers, "kind": self.kind}

    def close(self):
        self.pool.terminate()
        self.pool.join()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def describe(s: dict, P: int, m: int, h: float, op: str) -> str:
    what = ("element_tangent(tab, mat, u_e) @ p_e (femcore.py:130-146)" if op == "kp"
            else "element_internal_force (femcore.py:99-106)")
    src = "sdmefem from baseline/_ref" if s["kind"] == "reference" else "oracle restatement (oracle/fem.py)"
    return (f"{s['elements']} elements (P={P}, m={m}, h={h:.5g}) of {what}, {src}, "
            f"{s['cores']} single-threaded worker processes, {s['seconds']:.2f} s; "
            f"per-element cost scaled to the full mesh (extrapolated)")


# ------------------------------------------------------------ whole-run figures (subprocess)
_NEWMARK_SNIPPET = r'''
import json, sys, time
sys.path.insert(0, {ref!r})
import numpy as np
from sdmefem.basis1d import BasisKind, build_basis
from sdmefem.dynamics import SolverConfig, newmark_run
from sdmefem.femcore import FemProblem, build_face_tables
from sdmefem.material import NeoHookean
from sdmefem.meshdof import build_dofmap, gen_box_mesh
from sdmefem.quadrature import gauss_rule
from sdmefem.tensorelem import TensorElement
spec = json.loads({spec!r})
mesh = gen_box_mesh(tuple(spec["div"]), tuple(spec["L"]))
el = TensorElement.create(3, build_basis(spec["P"], BasisKind(spec["tag"])))
prob = FemProblem(mesh, el, build_dofmap(mesh, el, [("xmin", (0, 1, 2))]),
                  NeoHookean.from_engineering(1e7, 0.3, 1e3), rule=gauss_rule(spec["m"]))
faces = build_face_tables(prob.mesh, prob.element, "xmax", prob.rule)
base = prob.traction_vector(faces, lambda f: np.tile(spec["traction"], (len(f.pts), 1)))
T, dt = spec["ramp"], spec["dt"]
stamps = {{}}
def load(t):
    stamps.setdefault(round(t / dt), time.perf_counter())
    return base * min(t / T, 1.0)
cfg = SolverConfig(precond="diagonal", tol=1e-10, maxit=200000, condense=False)
t0 = time.perf_counter()
traj = newmark_run(prob, load, dt, spec["steps"], newton_tol=1e-8, cfg=cfg)
t1 = time.perf_counter()
ks = sorted(k for k in stamps if k >= 1)
steps = [stamps[b] - stamps[a] for a, b in zip(ks, ks[1:])] + [t1 - stamps[ks[-1]]]
print(json.dumps({{"step_s": steps, "total_s": t1 - t0, "newton": traj.newton_iters,
                  "pcg": [r["iterations"] for r in traj.stats.rows]}}))
'''


def newmark_step_s(div, L, P, m, tag, traction, dt, ramp, steps, timeout=1800) -> dict | None:
    """Run the reference's newmark_run (x = 0 clamped, constant traction on
    xmax ramped over ``ramp`` seconds, Jacobi-PCG 1e-10, condense=False) in a
    subprocess with the reference's default BLAS threading; per-step wall
    times exclude the setup.  None when the reference is not installed."""
    if not reference_dir():
        return None
    spec = json.dumps({"div": list(div), "L": list(L), "P": P, "m": m, "tag": tag, "traction": list(traction),
                       "dt": dt, "ramp": ramp, "steps": steps})
    code = _NEWMARK_SNIPPET.format(ref=REF_DIR, spec=spec)
    env = dict(os.environ)
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/sdme_numba_cache")
    for k in _ONE_THREAD:
        env.pop(k, None)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError(f"reference newmark run failed: {r.stderr[-2000:]}")
    out = json.loads(r.stdout.strip().splitlines()[-1])
    out["cores"] = os.cpu_count()
    out["kind"] = "reference"
    return out
