"""Build the sm_100a shared library in-tree (nvcc cross-compiles without a GPU).

    python -m paper_2104_13466_b200.build        # -> paper_2104_13466_b200/libsdme.so

The library is plain CUDA C++ behind the C ABI of include/sdme.h; no torch
types cross the boundary.  The operator kernels are compiled once per
polynomial order (csrc/ops.cu with -DSDME_ORDER=P) in parallel, then linked
with the ABI translation unit.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsdme.so")
OBJDIR = os.path.join(HERE, "build_obj")
# checked build (-DSDME_CHECKED: device bounds / alignment asserts, csrc/check.cuh)
CHECKED_LIB = os.path.join(HERE, "libsdme_checked.so")
CHECKED_OBJDIR = os.path.join(HERE, "build_obj_checked")
ORDERS = range(1, 9)
ABI_UNITS = ["sdme_abi.cu", "schur.cu"]  # host-side ABI translation units (operator units: ops.cu per order)
DEPS = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.cu")) +
              [os.path.join(ROOT, "include", "sdme.h")])

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "128"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in DEPS)


def _compile(args):
    src, obj, defs = args
    cmd = [nvcc(), *NVCC_FLAGS, *defs, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(obj)}:\n{r.stderr[-6000:]}")
    return obj


def build(force: bool = False, verbose: bool = True, jobs: int | None = None, only=None, defs=(),
          checked: bool = False) -> str:
    """Compile every translation unit (or, with ``only``, just those orders'
    operator units -- a development shortcut that relinks the other existing
    objects) and link libsdme.so.  ``defs``: extra -D flags for the operator units.
    ``checked``: the -DSDME_CHECKED variant, libsdme_checked.so (load it with
    SDME_LIB=paper_2104_13466_b200/libsdme_checked.so)."""
    lib, objdir = (CHECKED_LIB, CHECKED_OBJDIR) if checked else (LIB, OBJDIR)
    if checked:
        defs = (*defs, "-DSDME_CHECKED")
    if not force and not checked and up_to_date():
        return LIB
    os.makedirs(objdir, exist_ok=True)
    units = [(os.path.join(CSRC, u), os.path.join(objdir, u.replace(".cu", ".o")), list(defs if checked else []))
             for u in ABI_UNITS]
    units += [(os.path.join(CSRC, "ops.cu"), os.path.join(objdir, f"ops_p{p}.o"), [f"-DSDME_ORDER={p}", *defs])
              for p in ORDERS]
    objs_all = [u[1] for u in units]
    if only is not None:
        units = [u for u in units[len(ABI_UNITS):] if int(u[1].rsplit("_p", 1)[1][:-2]) in only]
    if verbose:
        print(f"nvcc {' '.join(NVCC_FLAGS)} : {len(units)} translation units", flush=True)
    with ThreadPoolExecutor(max_workers=jobs or min(len(units), os.cpu_count() or 4)) as ex:
        list(ex.map(_compile, units))
    cmd = [nvcc(), *ARCH, "-shared", "-o", lib + ".tmp", *objs_all]
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    only = [int(a.split("=", 1)[1]) for a in sys.argv if a.startswith("--only=")]
    defs = [a for a in sys.argv if a.startswith("-D")]
    build(force="--force" in sys.argv or bool(only) or bool(defs), only=only or None, defs=defs,
          checked="--checked" in sys.argv)
