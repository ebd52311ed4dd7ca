"""ctypes binding of libbloch_b200.so (include/bloch_b200.h).

Loading fails loudly: there is no CPU fallback anywhere in the product path.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_uint8, c_uint32, c_void_p

from .errors import DeviceError, InvalidParameter, WorkerPanic

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbloch_b200.so")

BLOCH_OK = 0
BLOCH_E_INVALID = -1
BLOCH_E_CUDA = -2
BLOCH_E_STATE = -3
BLOCH_E_NOMEM = -4
BLOCH_PREC_F32 = 32
BLOCH_PREC_F64 = 64
BLOCH_IN_DEVICE = 1
BLOCH_OUT_DEVICE = 2
BLOCH_NO_SYNC = 4
BLOCH_HOST_ONLY = -1


class BoxT(ctypes.Structure):
    """bloch_box_t"""
    _fields_ = [("base", c_double * 3), ("step", c_double * 3), ("count", c_int64 * 3), ("m0", c_double),
                ("t1", c_double), ("t2", c_double), ("dw", c_double), ("shape_begin", c_int32),
                ("shape_count", c_int32)]


class ShapeT(ctypes.Structure):
    """bloch_shape_t"""
    _fields_ = [("c", c_double * 3), ("ax", c_double * 3), ("cos_a", c_double), ("sin_a", c_double),
                ("m0", c_double), ("t1", c_double), ("t2", c_double), ("dw", c_double)]


class FieldT(ctypes.Structure):
    """bloch_field_t"""
    _fields_ = [("const_dw", c_double), ("n_poly", c_int32), ("n_bumps", c_int32), ("poly", POINTER(c_double)),
                ("poly_len", c_double), ("poly_scale", c_double), ("poly_peak", c_double),
                ("bumps", POINTER(c_double))]


class CoilT(ctypes.Structure):
    """bloch_coil_t"""
    _fields_ = [("c", c_double * 3), ("sigma", c_double), ("cos_p", c_double), ("sin_p", c_double)]


# every symbol the header declares, with (restype, argtypes)
_PD = POINTER(c_double)
SIGNATURES = {
    "bloch_version": (c_char_p, []),
    "bloch_abi_version": (c_int, []),
    "bloch_last_error": (c_char_p, []),
    "bloch_device_count": (c_int, [POINTER(c_int)]),
    "bloch_create": (c_int, [c_int, c_int, POINTER(c_void_p)]),
    "bloch_destroy": (c_int, [c_void_p]),
    "bloch_create_multi": (c_int, [POINTER(c_int32), c_int32, c_int, POINTER(c_void_p)]),
    "bloch_device_count_of": (c_int, [c_void_p, POINTER(c_int32), POINTER(c_int32)]),
    "bloch_last_device_times": (c_int, [c_void_p, c_int32, POINTER(c_float), POINTER(c_float)]),
    "bloch_set_stream": (c_int, [c_void_p, c_void_p]),
    "bloch_set_tables": (
        c_int,
        [c_void_p, c_int32, POINTER(c_int64), POINTER(c_uint8), _PD, POINTER(c_int32), _PD, _PD,
         POINTER(c_uint8), POINTER(c_int32), c_int32, c_int32, c_int32],
    ),
    "bloch_program_stats": (
        c_int,
        [c_void_p, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64), POINTER(c_int64),
         POINTER(c_int64), POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)],
    ),
    "bloch_program_layout": (
        c_int, [c_void_p, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]),
    "bloch_program_classes": (
        c_int, [c_void_p] + [POINTER(c_int64)] * 5),
    "bloch_compute_block": (
        c_int,
        [c_void_p, c_int64, _PD, _PD, _PD, _PD, _PD, _PD, _PD, _PD, _PD, c_int32, _PD, _PD,
         POINTER(c_uint8), c_uint32],
    ),
    "bloch_last_timing": (c_int, [c_void_p, POINTER(c_float), POINTER(c_float), POINTER(c_int32)]),
    "bloch_last_launch": (c_int, [c_void_p] + [POINTER(c_int32)] * 5),
    "bloch_last_segments": (c_int, [c_void_p, POINTER(c_int32)]),
    "bloch_set_contraction": (c_int, [c_void_p, c_int32]),
    "bloch_set_resident": (c_int, [c_void_p, c_int32]),
    "bloch_last_resident": (c_int, [c_void_p, POINTER(c_int32), POINTER(c_int32)]),
    "bloch_program_groups": (c_int, [c_void_p, POINTER(c_int32), POINTER(c_int64), POINTER(c_int64)]),
    "bloch_program_ops": (c_int, [c_void_p, c_int32, c_int32] + [POINTER(c_int32)] * 7),
    "bloch_last_phases": (c_int, [c_void_p, POINTER(c_float), POINTER(c_float), POINTER(c_int32), POINTER(c_int64)]),
    "bloch_synchronize": (c_int, [c_void_p]),
    "bloch_set_kernel_gate": (c_int, [c_void_p, c_void_p, c_void_p]),
    "bloch_rasterize": (
        c_int,
        [c_void_p, POINTER(BoxT), c_int32, POINTER(ShapeT), c_int32, POINTER(FieldT), POINTER(CoilT), c_int32,
         c_double, c_int64, _PD, _PD, _PD, _PD, _PD, _PD, _PD, _PD, _PD, POINTER(c_int64)],
    ),
}

_lib = None


def load(path: str = None) -> ctypes.CDLL:
    """Load and type the library once; raises ImportError if it is missing.

    ``BLOCH_LIB`` overrides the path (A/B timing of two builds on one box)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("BLOCH_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_1305_6861_b200.build` "
            "(the Bloch engine has no CPU fallback)"
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().bloch_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str, block_index=0) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if status == BLOCH_OK:
        return
    msg = f"{what}: {last_error()}"
    if status == BLOCH_E_INVALID:
        raise InvalidParameter(msg)
    if status == BLOCH_E_CUDA:
        raise WorkerPanic(block_index, msg)
    raise DeviceError(msg)


def device_count() -> int:
    n = c_int(0)
    check(load().bloch_device_count(ctypes.byref(n)), "bloch_device_count")
    return n.value


def dptr(arr):
    """double* of a C-contiguous float64 numpy array (or None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(_PD)
