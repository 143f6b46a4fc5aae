"""ctypes binding of libpt_b200.so (include/pt_b200.h), the C-ABI drop-in boundary.

The product path: every device op of this package goes through these symbols.
There is no fallback — if the shared library is missing or no sm_100 device is
present, calls fail loudly (LibraryMissing / BackendError).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBDIR = os.path.join(_HERE, "lib")
LIBPATH = os.path.join(LIBDIR, "libpt_b200.so")

PT_OK, PT_EVALIDATION, PT_EBACKEND = 0, 2, 3
PT_MATH_TF32, PT_MATH_FP32, PT_MATH_3XTF32 = 0, 1, 2
PT_CONV_FWD, PT_CONV_BWD_DATA, PT_CONV_BWD_FILTER, PT_CONV_BWD = 0, 1, 2, 3
PT_REDUCE_SUM, PT_REDUCE_MAX, PT_REDUCE_MIN = 0, 1, 2


class LibraryMissing(RuntimeError):
    """libpt_b200.so is not built (run __graft_entry__.build() / make)."""


class ValidationError(ValueError):
    """Mirror of portten::ValidationError (proj/include/portten/errors.hpp:29-33)."""


class BackendError(RuntimeError):
    """Mirror of portten::BackendError (proj/include/portten/errors.hpp:35-40)."""


class PtConvGeom(C.Structure):
    # field order == conv::ConvGeometry (proj/include/portten/conv_geometry.hpp:29-39)
    _fields_ = [(n, C.c_int64) for n in
                ("N", "C", "H", "W", "K", "kH", "kW", "padH", "padW", "strideH", "strideW")]


class PtView(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("sizes", C.c_int64 * 8), ("strides", C.c_int64 * 8),
                ("offset", C.c_int64)]


class PtDeviceDesc(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("maxWorkgroupSize", C.c_int32),
                ("localMemBytes", C.c_int64), ("smCount", C.c_int32), ("ccMajor", C.c_int32),
                ("ccMinor", C.c_int32), ("globalMemBytes", C.c_int64)]


_lock = threading.Lock()
_lib = None

_P = C.c_void_p
_F = C.POINTER(C.c_float)
_SIGS = {
    "pt_b200_abi_version": (C.c_int, []),
    "pt_b200_last_error": (C.c_char_p, []),
    "pt_b200_device_count": (C.c_int, []),
    "pt_b200_device_info": (C.c_int, [C.c_int, C.POINTER(PtDeviceDesc)]),
    "pt_b200_set_device": (C.c_int, [C.c_int]),
    "pt_b200_get_device": (C.c_int, [C.POINTER(C.c_int)]),
    "pt_b200_malloc": (C.c_int, [C.POINTER(C.c_void_p), C.c_size_t]),
    "pt_b200_free": (C.c_int, [_P]),
    "pt_b200_memcpy_h2d": (C.c_int, [_P, _P, C.c_size_t, _P]),
    "pt_b200_memcpy_d2h": (C.c_int, [_P, _P, C.c_size_t, _P]),
    "pt_b200_stream_sync": (C.c_int, [_P]),
    "pt_b200_stream_query": (C.c_int, [_P]),
    "pt_b200_fill_uniform": (C.c_int, [_P, C.c_int64, C.c_uint64, C.c_float, C.c_float, _P]),
    "pt_b200_conv_validate": (C.c_int, [C.POINTER(PtConvGeom)]),
    "pt_b200_conv_workspace_bytes": (C.c_size_t, [C.POINTER(PtConvGeom), C.c_int, C.c_int]),
    "pt_b200_conv_fwd": (C.c_int, [C.POINTER(PtConvGeom), _P, _P, _P, _P, C.c_int, _P,
                                   C.c_size_t, _P]),
    "pt_b200_conv_bwd_data": (C.c_int, [C.POINTER(PtConvGeom), _P, _P, _P, C.c_int, _P,
                                        C.c_size_t, _P]),
    "pt_b200_conv_bwd_filter": (C.c_int, [C.POINTER(PtConvGeom), _P, _P, _P, _P, C.c_float,
                                          C.c_int, C.c_int, _P, C.c_size_t, _P]),
    "pt_b200_conv_bwd": (C.c_int, [C.POINTER(PtConvGeom), _P, _P, _P, _P, _P, _P, C.c_float,
                                   C.c_int, C.c_int, _P, C.c_size_t, _P]),
    "pt_b200_conv_finput_bytes": (C.c_size_t, [C.POINTER(PtConvGeom), C.c_int]),
    "pt_b200_conv_fwd_finput": (C.c_int, [C.POINTER(PtConvGeom), _P, _P, _P, _P, C.c_int, _P,
                                          C.c_size_t, _P, _P]),
    "pt_b200_conv_bwd_finput": (C.c_int, [C.POINTER(PtConvGeom), _P, _P, _P, _P, _P, _P,
                                          C.c_float, C.c_int, C.c_int, _P, C.c_size_t, _P, _P]),
    "pt_b200_winograd_workspace_bytes": (C.c_size_t, [C.POINTER(PtConvGeom), C.c_int]),
    "pt_b200_conv_fwd_winograd": (C.c_int, [C.POINTER(PtConvGeom), _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "pt_b200_conv_bwd_data_winograd": (C.c_int, [C.POINTER(PtConvGeom), _P, _P, _P, _P, C.c_size_t, _P]),
    "pt_b200_im2col": (C.c_int, [C.POINTER(PtConvGeom), _P, _P, _P]),
    "pt_b200_im2col_batched": (C.c_int, [C.POINTER(PtConvGeom), _P, C.c_int64, C.c_int64, _P,
                                         _P]),
    "pt_b200_col2im": (C.c_int, [C.POINTER(PtConvGeom), _P, _P, _P]),
    "pt_b200_gemm": (C.c_int, [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_float, _P,
                               C.c_int64, _P, C.c_int64, C.c_float, _P, C.c_int64, C.c_int, _P]),
    "pt_b200_expression_compile": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_int32), C.c_int32,
                                             C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                             C.c_char_p, C.c_size_t]),
    "pt_b200_apply": (C.c_int, [C.POINTER(C.c_int32), C.c_int32, C.c_int, C.POINTER(C.c_void_p),
                                C.POINTER(PtView), C.c_float, _P]),
    "pt_b200_bias_add": (C.c_int, [_P, _P, C.c_int64, C.c_int64, C.c_int64, _P]),
    "pt_b200_reduce_all": (C.c_int, [C.c_int, _P, C.POINTER(PtView), _P, _P]),
    "pt_b200_reduce_dim": (C.c_int, [C.c_int, _P, C.POINTER(PtView), C.c_int, _P, _P]),
    "pt_b200_relu_fwd": (C.c_int, [_P, _P, C.c_int64, _P]),
    "pt_b200_relu_bwd": (C.c_int, [_P, _P, _P, C.c_int64, _P]),
    "pt_b200_maxpool_fwd": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, C.c_int64, C.c_int64] +
                            [C.c_int] * 6 + [_P]),
    "pt_b200_maxpool_bwd": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, C.c_int64, C.c_int64] +
                            [C.c_int] * 6 + [_P]),
    "pt_b200_launch_count": (C.c_int64, []),
    "pt_b200_plan_cache_stats": (None, [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "pt_b200_tf32_mma_peak": (C.c_double, []),
    "pt_b200_profile_enable": (C.c_int, [C.c_int]),
    "pt_b200_set_bwd_streams": (C.c_int, [C.c_int]),
    "pt_b200_profile_reset": (C.c_int, []),
    "pt_b200_profile_tag": (C.c_int, [C.c_char_p]),
    "pt_b200_profile_read": (C.c_int, [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load libpt_b200.so (once). Raises LibraryMissing when it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIBPATH):
                raise LibraryMissing(f"{LIBPATH} not built; run `make` or __graft_entry__.build()")
            h = C.CDLL(LIBPATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def check(status: int) -> None:
    """Map a pt_status to the reference's exception classes."""
    if status == PT_OK:
        return
    msg = lib().pt_b200_last_error().decode(errors="replace")
    if status == PT_EVALIDATION:
        raise ValidationError(msg)
    raise BackendError(msg)


def geom(N, C_, H, W, K, kH, kW, padH=0, padW=0, strideH=1, strideW=1) -> PtConvGeom:
    return PtConvGeom(N, C_, H, W, K, kH, kW, padH, padW, strideH, strideW)


def profile_read(kernel_class: str):
    """(total_ms, launches, flops, bytes) recorded for a kernel class since the last reset."""
    ms, n, fl, by = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
    check(lib().pt_b200_profile_read(kernel_class.encode(), C.byref(ms), C.byref(n), C.byref(fl),
                                     C.byref(by)))
    return ms.value, n.value, fl.value, by.value
