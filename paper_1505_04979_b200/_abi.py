"""ctypes binding of include/pbp.h (libpbp.so). Loads the in-tree library or fails loudly."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PBP_LIB", os.path.join(PKG, "_lib", "libpbp.so"))

PBP_OK, PBP_EINVAL, PBP_ERUNTIME, PBP_ECUDA, PBP_ENODEV, PBP_ENOMEM = range(6)


class PbpCode(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("k", C.c_int32),
                ("frozen", C.POINTER(C.c_uint8))]


class PbpFrameOut(C.Structure):
    _fields_ = [("u_hat_bits", C.POINTER(C.c_uint32)), ("iterations", C.POINTER(C.c_int32)),
                ("pe", C.POINTER(C.c_int64)), ("stop", C.POINTER(C.c_uint8)),
                ("n_events", C.POINTER(C.c_int32))]


class PbpCounters(C.Structure):
    _fields_ = [("frames", C.c_int64), ("bit_errors", C.c_int64), ("frame_errors", C.c_int64),
                ("sum_iters", C.c_int64), ("sum_iters_sq", C.c_int64), ("sum_pe", C.c_int64),
                ("sum_events", C.c_int64), ("stop_hist", C.c_int64 * 3)]


def _ptr(t):
    def f(a):
        if a is None:
            return None
        if isinstance(a, int):  # raw device pointer
            return C.cast(C.c_void_p(a), C.POINTER(t))
        return a.ctypes.data_as(C.POINTER(t))
    return f


u8p, u32p, i32p, i64p, f32p, f64p = (_ptr(C.c_uint8), _ptr(C.c_uint32), _ptr(C.c_int32),
                                     _ptr(C.c_int64), _ptr(C.c_float), _ptr(C.c_double))

_P = C.c_void_p
_CP = C.POINTER(PbpCode)
# name -> (restype, argtypes); every symbol declared in include/pbp.h
SIGNATURES = {
    "pbp_last_error": (C.c_char_p, []),
    "pbp_version": (C.c_int, []),
    "pbp_device_count": (C.c_int, []),
    "pbp_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "pbp_ctx_destroy": (C.c_int, [_P]),
    "pbp_ctx_stream": (C.c_void_p, [_P]),
    "pbp_ctx_synchronize": (C.c_int, [_P]),
    "pbp_construct": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.POINTER(C.c_uint8)]),
    "pbp_polar_transform": (C.c_int, [C.POINTER(C.c_uint8), C.c_int32]),
    "pbp_encode": (C.c_int, [_CP, C.POINTER(C.c_uint8), C.POINTER(C.c_uint8), C.POINTER(C.c_uint8)]),
    "pbp_noise_variance": (C.c_int, [C.c_double, C.c_double, C.POINTER(C.c_double)]),
    "pbp_decode_batch": (C.c_int, [_P, _CP, C.c_int, C.POINTER(C.c_float), C.c_int64, C.c_float,
                                   C.c_int32, C.POINTER(PbpFrameOut)]),
    "pbp_decode_batch_device": (C.c_int, [_P, _CP, C.c_int, C.POINTER(C.c_float), C.c_int64,
                                          C.c_float, C.c_int32, C.POINTER(PbpFrameOut), _P]),
    "pbp_decode_trace": (C.c_int, [_P, _CP, C.c_int, C.POINTER(C.c_float), C.c_float, C.c_int32,
                                   C.POINTER(C.c_uint8), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                   C.c_int32]),
    "pbp_decode_trace_x": (C.c_int, [_P, _CP, C.c_int, C.POINTER(C.c_float), C.c_float, C.c_int32,
                                     C.POINTER(C.c_uint8), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                     C.c_int32, C.POINTER(C.c_uint32)]),
    "pbp_decode_trace_f64_x": (C.c_int, [_P, _CP, C.c_int, C.POINTER(C.c_double), C.c_double, C.c_int32,
                                         C.POINTER(C.c_uint8), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                         C.c_int32, C.POINTER(C.c_uint32)]),
    "pbp_decode_batch_f64": (C.c_int, [_P, _CP, C.c_int, C.POINTER(C.c_double), C.c_int64, C.c_double,
                                       C.c_int32, C.POINTER(PbpFrameOut)]),
    "pbp_decode_batch_f64_device": (C.c_int, [_P, _CP, C.c_int, C.POINTER(C.c_double), C.c_int64,
                                              C.c_double, C.c_int32, C.POINTER(PbpFrameOut), _P]),
    "pbp_decode_trace_f64": (C.c_int, [_P, _CP, C.c_int, C.POINTER(C.c_double), C.c_double, C.c_int32,
                                       C.POINTER(C.c_uint8), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.c_int32]),
    "pbp_simulate_point_f64": (C.c_int, [_P, _CP, C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_double,
                                         C.c_int, C.c_double, C.c_int32, C.POINTER(PbpCounters)]),
    "pbp_generate_device": (C.c_int, [_P, _CP, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_int,
                                      C.POINTER(C.c_float), C.POINTER(C.c_double),
                                      C.POINTER(C.c_uint32), _P]),
    "pbp_generate": (C.c_int, [_P, _CP, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_int,
                               C.POINTER(C.c_float), C.POINTER(C.c_double), C.POINTER(C.c_uint32)]),
    "pbp_simulate_point": (C.c_int, [_P, _CP, C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_double,
                                     C.c_int, C.c_float, C.c_int32, C.POINTER(PbpCounters)]),
    "pbp_simulate_point_device": (C.c_int, [_P, _CP, C.c_int, C.c_uint64, C.c_int64, C.c_int64,
                                            C.c_double, C.c_int, C.c_float, C.c_int32,
                                            C.POINTER(C.c_int64), _P]),
    "pbp_decode_count_device": (C.c_int, [_P, _CP, C.c_int, C.POINTER(C.c_float),
                                          C.POINTER(C.c_uint32), C.c_int64, C.c_float, C.c_int32,
                                          C.POINTER(C.c_int64), _P]),
    "pbp_simulate_batches": (C.c_int, [_P, _CP, C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_int32,
                                       C.c_double, C.c_int, C.c_double, C.c_int32, C.c_int,
                                       C.POINTER(C.c_int64)]),
    "pbp_simulate_sweep_multi": (C.c_int, [C.POINTER(C.c_int), C.c_int, _CP, C.c_int, C.c_uint64, C.c_int64,
                                           C.POINTER(C.c_double), C.c_int, C.c_int, C.c_float, C.c_int32,
                                           C.POINTER(PbpCounters)]),
    "pbp_decode_count_batches_device": (C.c_int, [_P, _CP, C.c_int, C.POINTER(C.c_float),
                                                  C.POINTER(C.c_uint32), C.c_int64, C.c_int64, C.c_float,
                                                  C.c_int32, C.POINTER(C.c_int64), _P]),
    "pbp_kernel_path": (C.c_int, [C.c_int32]),
    "pbp_kernel_cluster": (C.c_int, [C.c_int32, C.c_int]),
    "pbp_ctx_force_generic": (C.c_int, [_P, C.c_int]),
    "pbp_kernel_info": (C.c_int, [C.c_int32, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "pbp_last_launch_info": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
}


def load(path: str = LIB_PATH):
    """Load libpbp.so. Raises (no fallback) when the extension has not been built."""
    if not os.path.exists(path):
        raise ImportError(
            f"libpbp.so not found at {path}: build it with `python paper_1505_04979_b200/build.py` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class PbpError(RuntimeError):
    pass


def check(lib, rc: int):
    if rc == PBP_OK:
        return
    msg = (lib.pbp_last_error() or b"").decode()
    if rc == PBP_EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    if rc == PBP_ERUNTIME:
        raise RuntimeError(msg)
    raise PbpError(f"libpbp status {rc}: {msg}")
