"""Build the sm_100a shared library in-tree (nvcc cross-compiles without a GPU).

    python -m paper_2104_13466_b200.build        # -> paper_2104_13466_b200/libsdme.so

The library is plain CUDA C++ behind the C ABI of include/sdme.h; no torch
types cross the boundary.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libsdme.so")
SOURCES = [os.path.join(HERE, "csrc", "sdme_abi.cu")]
HEADERS = [os.path.join(HERE, "csrc", f) for f in
           ("element_kernels.cuh", "element_v3.cuh", "element_v4.cuh", "vector_kernels.cuh", "contact_kernels.cuh")] + \
          [os.path.join(ROOT, "include", "sdme.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "128"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and up_to_date():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp", *SOURCES]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
