"""ctypes binding of the sm_100a C ABI (include/paracycle_b200.h).

The product path has no CPU fallback: if the in-tree library is missing this
module raises at import-of-use time with the build command to run.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_size_t, c_void_p

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libparacycle_b200.so")
# experiment switch (same-box A/B of two builds): load another in-tree build
if os.environ.get("PC_LIB_PATH"):
    LIB_PATH = os.path.join(_HERE, "_lib", os.path.basename(os.environ["PC_LIB_PATH"]))

PC_OK = 0
PC_E_INVALID, PC_E_INDEFINITE, PC_E_DIVERGED, PC_E_BLOWUP, PC_E_CAP = 1, 2, 3, 4, 5
PC_E_CUDA, PC_E_NCCL, PC_E_DOMAIN, PC_E_NOTCONV = 6, 7, 8, 9
LAYOUT_AOS, LAYOUT_SOA = 0, 1
PC_JACOBI, PC_LINE_R = 0, 1
TEST_POSITIVE, TEST_NONNEG, TEST_FINITE = 0, 1, 2
RKL2, RKG2, BE, EULER = 0, 1, 2, 3
FLOOR_EULER, FLOOR_FRACTION = 0, 1


class CycleRecord(ctypes.Structure):
    _fields_ = [("cycle", c_int64), ("dt", c_double), ("ptl_raw", c_double), ("relres", c_double),
                ("limited", c_int32), ("iters", c_int32)]


_lib = None
_shutting_down = False


def _mark_shutdown():
    global _shutting_down
    _shutting_down = True


import atexit  # noqa: E402

atexit.register(_mark_shutdown)


def alive() -> bool:
    """False once the interpreter is exiting (destructors must not call CUDA)."""
    return _lib is not None and not _shutting_down

_SIGS = {
    "pc_last_error": (ctypes.c_char_p, []),
    "pc_last_error_info": (c_int64, []),
    "pc_version": (c_int, []),
    "pc_ctx_create": (c_int, [c_int, c_int, c_int, c_void_p, POINTER(c_void_p)]),
    "pc_ctx_create_detached": (c_int, [c_int, c_int, c_int, POINTER(c_void_p)]),
    "pc_op_set_preconditioner": (c_int, [c_void_p, c_int]),
    "pc_op_set_refresh": (c_int, [c_void_p, c_int]),
    "pc_field_set_ghost": (c_int, [c_void_p, c_int, POINTER(c_double)]),
    "pc_field_set_ghost_cols": (c_int, [c_void_p, POINTER(c_double)]),
    "pc_ctx_set_decomposition": (c_int, [c_void_p, c_int]),
    "pc_ctx_destroy": (c_int, [c_void_p]),
    "pc_ctx_sync": (c_int, [c_void_p]),
    "pc_nccl_unique_id": (c_int, [c_void_p]),
    "pc_grid_table_size": (c_int64, [POINTER(c_int64)]),
    "pc_grid_create": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int32), POINTER(c_double), c_int64,
                               POINTER(c_void_p)]),
    "pc_grid_destroy": (c_int, [c_void_p]),
    "pc_field_create": (c_int, [c_void_p, c_int, POINTER(c_void_p)]),
    "pc_field_destroy": (c_int, [c_void_p]),
    "pc_field_upload": (c_int, [c_void_p, POINTER(c_double), c_int]),
    "pc_field_download": (c_int, [c_void_p, POINTER(c_double), c_int]),
    "pc_field_download_planes": (c_int, [c_void_p, c_int64, c_int64, POINTER(c_double)]),
    "pc_field_copy": (c_int, [c_void_p, c_void_p]),
    "pc_field_fill": (c_int, [c_void_p, c_double]),
    "pc_field_exchange_halo": (c_int, [c_void_p]),
    "pc_field_count": (c_int, [c_void_p, c_int, POINTER(c_int64)]),
    "pc_field_upload_async": (c_int, [c_void_p, POINTER(c_double), c_int]),
    "pc_field_download_async": (c_int, [c_void_p, POINTER(c_double), c_int]),
    "pc_field_wait": (c_int, [c_void_p]),
    "pc_host_register": (c_int, [c_void_p, c_size_t]),
    "pc_host_unregister": (c_int, [c_void_p]),
    "pc_host_alloc": (c_int, [c_size_t, POINTER(c_void_p)]),
    "pc_host_free": (c_int, [c_void_p]),
    "pc_op_create_scalar": (c_int, [c_void_p, c_int, c_int, c_double, c_void_p, c_void_p, POINTER(c_void_p)]),
    "pc_op_create_viscous": (c_int, [c_void_p, c_int, c_int, c_double, c_void_p, POINTER(c_void_p)]),
    "pc_op_create_aligned": (c_int, [c_void_p, c_void_p, c_void_p, c_double, c_double, POINTER(c_double),
                                     c_double, POINTER(c_void_p)]),
    "pc_op_freeze": (c_int, [c_void_p, c_void_p]),
    "pc_op_destroy": (c_int, [c_void_p]),
    "pc_op_apply": (c_int, [c_void_p, c_void_p, c_void_p]),
    "pc_op_euler_dt": (c_int, [c_void_p, POINTER(c_double)]),
    "pc_op_diagonal": (c_int, [c_void_p, c_void_p]),
    "pc_ptl": (c_int, [c_void_p, c_void_p, c_void_p, c_double, c_int, POINTER(c_double), POINTER(c_int),
                       POINTER(c_int64)]),
    "pc_sts_count": (c_int, [c_int, c_double, c_double, c_int]),
    "pc_sts_table": (c_int, [c_int, c_int, c_double, POINTER(c_double)]),
    "pc_step_sts": (c_int, [c_void_p, c_void_p, c_double, c_int, c_int, c_void_p]),
    "pc_step_euler": (c_int, [c_void_p, c_void_p, c_double]),
    "pc_step_be": (c_int, [c_void_p, c_void_p, c_double, c_double, c_int, POINTER(c_int), POINTER(c_double),
                           POINTER(c_int)]),
    "pc_pcg_solve": (c_int, [c_void_p, c_double, c_void_p, c_void_p, c_void_p, c_double, c_int, POINTER(c_int),
                             POINTER(c_double), POINTER(c_int)]),
    "pc_cycle": (c_int, [c_void_p, c_void_p, c_double, c_int, c_int, c_double, c_int, c_double, c_int, c_int,
                         c_int, c_double, c_int64, c_double, POINTER(CycleRecord), c_int64, POINTER(c_int64)]),
    "pc_gen_temperature": (c_int, [c_void_p, ctypes.c_uint64, c_int, c_double, POINTER(c_double)]),
    "pc_gen_dipole": (c_int, [c_void_p, ctypes.c_uint64, c_int, c_double, POINTER(c_double), POINTER(c_double),
                              POINTER(c_double)]),
    "pc_gen_harmonic": (c_int, [c_void_p, POINTER(c_double), c_double]),
    "pc_gen_radial": (c_int, [c_void_p, POINTER(c_double)]),
    "pc_ctx_stats": (c_int, [c_void_p, POINTER(c_double), POINTER(c_int64), POINTER(c_int64)]),
    "pc_ctx_reset_stats": (c_int, [c_void_p]),
    "pc_ctx_stats_kind": (c_int, [c_void_p, c_int, POINTER(c_double), POINTER(c_int64), POINTER(c_int64)]),
    "pc_ctx_enable_timing": (c_int, [c_void_p, c_int]),
    "pc_ctx_mark": (c_int, [c_void_p, c_int]),
    "pc_ctx_elapsed": (c_int, [c_void_p, c_int, c_int, POINTER(c_double)]),
}

EXPORTED = tuple(_SIGS)


def lib() -> ctypes.CDLL:
    """Load the in-tree CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise errors.NativeLibraryMissing(
                f"{LIB_PATH} not found: build it with `python -m paper_2403_01004_b200.build` "
                "(the product path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().pc_last_error().decode(errors="replace")


def check(rc: int, what: str = "", **ctx):
    """Map a C status code to the SPEC's Python exceptions."""
    if rc == PC_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    info = lib().pc_last_error_info()
    if rc == PC_E_INVALID:
        raise ValueError(msg)
    if rc == PC_E_INDEFINITE:
        raise errors.IndefiniteOperatorError(msg)
    if rc == PC_E_DIVERGED:
        raise errors.DivergenceError(msg)
    if rc == PC_E_BLOWUP:
        raise errors.BlowUpError(int(info), msg)
    if rc == PC_E_CAP:
        raise errors.CycleCapError(msg, ctx.get("report"))
    if rc == PC_E_DOMAIN:
        raise errors.DomainError(msg)
    if rc == PC_E_NOTCONV:
        raise errors.NotConvergedError(msg, ctx.get("report"))
    if rc == PC_E_NCCL:
        raise errors.CommError(msg)
    raise errors.DeviceError(msg)


def dptr(a):
    return a.ctypes.data_as(POINTER(c_double))
