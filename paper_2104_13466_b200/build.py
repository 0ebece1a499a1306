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
ORDERS = range(1, 9)
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


def build(force: bool = False, verbose: bool = True, jobs: int | None = None, only=None, defs=()) -> str:
    """Compile every translation unit (or, with ``only``, just those orders'
    operator units -- a development shortcut that relinks the other existing
    objects) and link libsdme.so.  ``defs``: extra -D flags for the operator units."""
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    units = [(os.path.join(CSRC, "sdme_abi.cu"), os.path.join(OBJDIR, "sdme_abi.o"), [])]
    units += [(os.path.join(CSRC, "ops.cu"), os.path.join(OBJDIR, f"ops_p{p}.o"), [f"-DSDME_ORDER={p}", *defs])
              for p in ORDERS]
    objs_all = [u[1] for u in units]
    if only is not None:
        units = [u for u in units[1:] if int(u[1].rsplit("_p", 1)[1][:-2]) in only]
    if verbose:
        print(f"nvcc {' '.join(NVCC_FLAGS)} : {len(units)} translation units", flush=True)
    with ThreadPoolExecutor(max_workers=jobs or min(len(units), os.cpu_count() or 4)) as ex:
        list(ex.map(_compile, units))
    cmd = [nvcc(), *ARCH, "-shared", "-o", LIB + ".tmp", *objs_all]
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    only = [int(a.split("=", 1)[1]) for a in sys.argv if a.startswith("--only=")]
    defs = [a for a in sys.argv if a.startswith("-D")]
    build(force="--force" in sys.argv or bool(only) or bool(defs), only=only or None, defs=defs)
