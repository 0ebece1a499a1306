"""ctypes binding of the C ABI (include/sdme.h) and the error mapping.

Status codes map 1:1 onto the reference's exception types:
SDME_INVERSION -> ElementInversionError(elem_id, qp) (femcore.py:36-42),
SDME_INDEFINITE / SDME_MAXIT -> PCGError(msg, stats) (solver.py:33-38),
SDME_BAD_DIAGONAL -> ValueError (solver.py:107-108).

There is no CPU fallback: if the shared library is missing or cannot be
loaded, :func:`lib` raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import ElementInversionError, NativeError

HERE = os.path.dirname(os.path.abspath(__file__))
# SDME_LIB: an alternative build of the same library (A/B and sanitizer
# experiments, e.g. a different register cap); default the in-tree build
LIB_PATH = os.environ.get("SDME_LIB") or os.path.join(HERE, "libsdme.so")

OK, INVERSION, INDEFINITE, MAXIT, BAD_DIAGONAL, BAD_ARGUMENT, CUDA_ERROR = range(7)

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)


class Desc(C.Structure):
    _fields_ = [("P", C.c_int), ("m", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("hx", C.c_double), ("hy", C.c_double), ("hz", C.c_double),
                ("origin", C.c_double * 3), ("B", _dp), ("D", _dp), ("w", _dp),
                ("mu", C.c_double), ("lambda_lame", C.c_double), ("rho0", C.c_double),
                ("dirichlet_mask", C.c_int * 3), ("perm", _i32p), ("n_free", C.c_int64)]


_i64p = C.POINTER(C.c_int64)


class MeshDesc(C.Structure):
    """``sdme_mesh_desc`` (include/sdme.h): general hexahedral mesh context."""
    _fields_ = [("P", C.c_int), ("m", C.c_int), ("n_elems", C.c_int64), ("B", _dp), ("D", _dp), ("w", _dp),
                ("mu", C.c_double), ("lambda_lame", C.c_double), ("rho0", C.c_double), ("n_free", C.c_int64),
                ("dof", _i32p), ("asm_ptr", _i64p), ("asm_slot", _i32p), ("geom", _dp),
                ("elem_id", _i32p), ("asm_rows", _i32p)]


class SchurDesc(C.Structure):
    """``sdme_schur_desc`` (include/sdme.h): the assembled / condensed solve."""
    _fields_ = [("n_elems", C.c_int64), ("nd", C.c_int), ("nq", C.c_int), ("nb", C.c_int64),
                ("addr", _i64p), ("role", _i32p), ("addr_b", _i64p), ("G", _dp), ("N", _dp), ("wdet", _dp),
                ("mu", C.c_double), ("lambda_lame", C.c_double), ("rho0", C.c_double)]


# name -> argtypes (restype c_int for all)
SIGNATURES = {
    "sdme_create": [C.POINTER(Desc), C.POINTER(C.c_void_p)],
    "sdme_create_mesh": [C.POINTER(MeshDesc), C.POINTER(C.c_void_p)],
    "sdme_destroy": [C.c_void_p],
    "sdme_lattice_size": [C.c_void_p, C.POINTER(C.c_int64)],
    "sdme_last_error": [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int), C.c_char_p, C.c_size_t],
    "sdme_vec_alloc": [C.c_void_p, C.POINTER(C.c_int)],
    "sdme_vec_free": [C.c_void_p, C.c_int],
    "sdme_vec_upload": [C.c_void_p, C.c_int, _dp],
    "sdme_vec_download": [C.c_void_p, C.c_int, _dp],
    "sdme_vec_upload_free": [C.c_void_p, C.c_int, _dp],
    "sdme_vec_download_free": [C.c_void_p, C.c_int, _dp],
    "sdme_vec_fill": [C.c_void_p, C.c_int, C.c_double],
    "sdme_vec_copy": [C.c_void_p, C.c_int, C.c_int],
    "sdme_vec_lincomb": [C.c_void_p, C.c_int, C.c_int, _dp, C.POINTER(C.c_int)],
    "sdme_vec_mul": [C.c_void_p, C.c_int, C.c_int, C.c_int],
    "sdme_vec_dot": [C.c_void_p, C.c_int, C.c_int, _dp],
    "sdme_vec_reciprocal": [C.c_void_p, C.c_int, C.c_int],
    "sdme_fint": [C.c_void_p, C.c_int, C.c_int],
    "sdme_apply": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double],
    "sdme_apply_batch": [C.c_void_p, C.c_int, C.POINTER(_dp), C.POINTER(_dp), C.POINTER(_dp), C.c_double,
                         C.c_double],
    "sdme_mass": [C.c_void_p, C.c_int, C.c_int],
    "sdme_diag": [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int],
    "sdme_newmark_residual": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                              C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, _dp],
    "sdme_pcg": [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                 C.c_int, C.POINTER(C.c_int), _dp],
    "sdme_explicit_step": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                           C.c_double, C.c_int],
    "sdme_explicit_steps": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.c_int, C.c_int,
                            C.c_double, C.c_int],
    "sdme_contact": [C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_int,
                     _dp, _dp],
    "sdme_contact_points": [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int64)],
    "sdme_contact_apply": [C.c_void_p, C.c_int, C.c_int],
    "sdme_contact_diag": [C.c_void_p, C.c_int],
    "sdme_pcg_contact": [C.c_void_p, C.c_int],
    "sdme_strain_energy": [C.c_void_p, C.c_int, C.POINTER(C.c_double)],
    "sdme_time_op": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _dp],
    "sdme_schur_create": [C.c_void_p, C.POINTER(SchurDesc), C.POINTER(C.c_void_p)],
    "sdme_schur_destroy": [C.c_void_p],
    "sdme_schur_info": [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int),
                        C.POINTER(C.c_int)],
    "sdme_schur_factor": [C.c_void_p, C.c_int, C.c_double, C.c_double],
    "sdme_schur_solve": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.POINTER(C.c_int), _dp],
    "sdme_schur_matrix": [C.c_void_p, _i64p, _i32p, _dp, _dp],
    "sdme_lattice_address": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64)],
    "sdme_host_alloc": [C.c_size_t, C.POINTER(C.c_void_p)],
    "sdme_host_free": [C.c_void_p],
    "sdme_sync": [C.c_void_p],
    "sdme_launch_count": [C.c_void_p, C.POINTER(C.c_int64)],
}

_LIB = None


def lib() -> C.CDLL:
    """Load libsdme.so (fails loudly: there is no fallback path)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"CUDA library missing: {LIB_PATH} (run python -m paper_2104_13466_b200.build)")
        h = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(h, name)
            fn.argtypes = args
            fn.restype = C.c_int
        _LIB = h
    return _LIB


class _Pinned:
    """Owner of a page-locked host buffer (freed with the last numpy view)."""

    def __init__(self, nbytes):
        p = C.c_void_p()
        rc = lib().sdme_host_alloc(nbytes, C.byref(p))
        if rc != OK:
            raise NativeError(f"cudaMallocHost({nbytes}) failed")
        self.ptr = p

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().sdme_host_free(self.ptr)
            self.ptr = None


class PinnedArray(np.ndarray):
    """ndarray view of page-locked memory; holds the allocation alive."""


def pinned_empty(n: int) -> np.ndarray:
    """float64 numpy array of length n in page-locked host memory."""
    owner = _Pinned(max(8, 8 * n))
    buf = (C.c_double * n).from_address(owner.ptr.value)
    arr = np.ctypeslib.as_array(buf).view(PinnedArray)
    arr._owner = owner
    return arr


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def last_error(ctx) -> tuple[int, int, int, str]:
    elem = C.c_int64(-1)
    qp = C.c_int(-1)
    buf = C.create_string_buffer(512)
    code = lib().sdme_last_error(ctx, C.byref(elem), C.byref(qp), buf, 512)
    return code, elem.value, qp.value, buf.value.decode(errors="replace")


def check(ctx, rc: int, what: str = ""):
    """Raise the reference-equivalent exception for a non-zero status."""
    if rc == OK:
        return
    code, elem, qp, msg = last_error(ctx) if ctx else (rc, -1, -1, "")
    if rc == INVERSION:
        raise ElementInversionError(elem, qp)
    if rc == BAD_DIAGONAL:
        raise ValueError("diagonal preconditioner needs positive diagonal entries")
    if rc == BAD_ARGUMENT:
        raise ValueError(f"{what}: {msg or 'bad argument'}")
    raise NativeError(f"{what}: status {rc}: {msg}")
