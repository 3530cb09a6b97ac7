"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU oracles.

* ``C`` -- the plain-C restatement (oracle/pbp_oracle.c, built to
  oracle/_build/liboracle.so), functions ``orc_*``.
* ``REF`` -- the reference core compiled in place from /root/reference
  (oracle/ref_wrap.cpp, built to oracle/_ref/libpbp_ref.so), functions
  ``ref64_*`` (shipped fp64) and ``ref32_*`` (same sources in fp32). It is
  built in the dev container and travels to the GPU box as a prebuilt .so;
  ``REF`` is None where it is absent.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this package, and only as the checker / the timed CPU reference.
"""
from __future__ import annotations

import ctypes as C_
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpbp_ref.so")

_u8p = C_.POINTER(C_.c_uint8)
_i32p = C_.POINTER(C_.c_int)
_i64p = C_.POINTER(C_.c_longlong)
_f32p = C_.POINTER(C_.c_float)
_f64p = C_.POINTER(C_.c_double)
_u64p = C_.POINTER(C_.c_uint64)

KIND = {"baseline": 0, "gmatrix": 1, "csfg": 2}
# decode/decode_batch use this library when none is passed (None: the C restatement);
# tests/conftest.py points it at the compiled reference (REF) for the GPU parity tests
DEFAULT_LIB = None
STOP_NAMES = ("max_iter", "gmatrix_converged", "csfg_complete")


def build():
    """Build the oracle libraries (C restatement always, reference when present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _load(path):
    return C_.CDLL(path) if os.path.exists(path) else None


def _setup_decode(fn, real_p, real_t):
    fn.argtypes = [C_.c_int, C_.c_int, _u8p, real_p, real_t, C_.c_int, _u8p, _i32p, _i64p,
                   _i32p, _i32p, _i32p, C_.c_int]
    fn.restype = C_.c_int


def _setup_batch(fn, real_p, real_t):
    fn.argtypes = [C_.c_int, C_.c_int, _u8p, real_p, C_.c_longlong, real_t, C_.c_int, C_.c_int,
                   _u8p, _i32p, _i64p, _i32p, _i32p]
    fn.restype = C_.c_int


C = _load(ORACLE_SO)
if C is not None:
    C.orc_polar_transform.argtypes = [_u8p, C_.c_int]
    C.orc_construct.argtypes = [C_.c_int, C_.c_int, C_.c_double, _u8p]
    C.orc_encode.argtypes = [C_.c_int, _u8p, _u8p, _u8p, _u8p]
    C.orc_trial_frame.argtypes = [C_.c_uint64, C_.c_uint64, C_.c_int, _u8p, C_.c_double,
                                  C_.c_int, _u8p, _f64p]
    C.orc_noise_variance.argtypes = [C_.c_double, C_.c_double]
    C.orc_noise_variance.restype = C_.c_double
    C.orc_pe_update_f32.argtypes = [_f32p, C_.c_float, _f32p]
    C.orc_pe_update_f64.argtypes = [_f64p, C_.c_double, _f64p]
    _setup_decode(C.orc_decode_f32, _f32p, C_.c_float)
    _setup_decode(C.orc_decode_f64, _f64p, C_.c_double)
    _setup_batch(C.orc_decode_batch_f32, _f32p, C_.c_float)
    _setup_batch(C.orc_decode_batch_f64, _f64p, C_.c_double)

REF = _load(REF_SO)
if REF is not None:
    REF.ref64_last_error.restype = C_.c_char_p
    REF.ref32_last_error.restype = C_.c_char_p
    REF.ref64_construct.argtypes = [C_.c_int, C_.c_int, C_.c_double, _u8p]
    REF.ref64_polar_transform.argtypes = [_u8p, C_.c_int]
    REF.ref64_rng_raw.argtypes = [C_.c_uint64, C_.c_uint64, C_.c_int, _u64p]
    REF.ref64_rng_gaussian.argtypes = [C_.c_uint64, C_.c_uint64, C_.c_int, _f64p]
    REF.ref64_noise_variance.argtypes = [C_.c_double, C_.c_double]
    REF.ref64_noise_variance.restype = C_.c_double
    REF.ref64_trials.argtypes = [C_.c_uint64, C_.c_longlong, C_.c_longlong, C_.c_int, _u8p,
                                 C_.c_double, C_.c_int, C_.c_int, _u8p, _f64p]
    REF.ref64_pe_update.argtypes = [_f64p, C_.c_double, _f64p]
    REF.ref32_pe_update.argtypes = [_f32p, C_.c_float, _f32p]
    _setup_decode(REF.ref64_decode, _f64p, C_.c_double)
    _setup_decode(REF.ref32_decode, _f32p, C_.c_float)
    _setup_batch(REF.ref64_decode_batch, _f64p, C_.c_double)
    _setup_batch(REF.ref32_decode_batch, _f32p, C_.c_float)


# --------------------------------------------------------------------------
# numpy-level helpers (lib = C or REF; prec = 32 / 64)

def construct(n, k, z, lib=None):
    lib = lib or C
    out = np.zeros(n, np.uint8)
    fn = lib.orc_construct if lib is C else lib.ref64_construct
    if fn(n, k, z, _p(out, _u8p)) != 0:
        raise ValueError(f"construct({n},{k},{z}) rejected")
    return out


def trials(seed, first, count, frozen, ebn0, noiseless=False, threads=None, lib=None):
    """(info bits [count,k] u8, fp64 LLRs [count,n]) of trials first..first+count-1."""
    n = frozen.size
    k = int(n - frozen.sum())
    info = np.zeros((count, k), np.uint8)
    llr = np.zeros((count, n), np.float64)
    lib = lib or REF or C
    if lib is REF:
        rc = REF.ref64_trials(seed, first, count, n, _p(frozen, _u8p), ebn0, int(noiseless),
                              threads or os.cpu_count() or 1, _p(info, _u8p), _p(llr, _f64p))
        if rc:
            raise RuntimeError(REF.ref64_last_error().decode())
    else:
        fz = np.ascontiguousarray(frozen, np.uint8)
        for i in range(count):
            C.orc_trial_frame(seed, first + i, n, _p(fz, _u8p), ebn0, int(noiseless),
                              _p(info[i], _u8p), _p(llr[i], _f64p))
    return info, llr


def decode(kind, frozen, llr, alpha=0.9375, max_iter=40, prec=32, lib=None, ev_cap=4096):
    """One frame through the oracle. Returns dict(u_hat, iterations, pe, stop, n_events, events)."""
    lib = lib or DEFAULT_LIB or C
    n = frozen.size
    if prec == 32:
        llr = np.ascontiguousarray(llr, np.float32)
        fn = lib.orc_decode_f32 if lib is C else lib.ref32_decode
        lp = _p(llr, _f32p)
    else:
        llr = np.ascontiguousarray(llr, np.float64)
        fn = lib.orc_decode_f64 if lib is C else lib.ref64_decode
        lp = _p(llr, _f64p)
    u = np.zeros(n, np.uint8)
    it, sp, ne = C_.c_int(), C_.c_int(), C_.c_int()
    pe = C_.c_longlong()
    ev = np.zeros(5 * ev_cap, np.int32)
    rc = fn(KIND.get(kind, kind), n, _p(np.ascontiguousarray(frozen, np.uint8), _u8p), lp, alpha,
            max_iter, _p(u, _u8p), C_.byref(it), C_.byref(pe), C_.byref(sp), C_.byref(ne),
            _p(ev, _i32p), ev_cap)
    if rc:
        raise ValueError("oracle decode rejected its arguments")
    nev = ne.value
    return {"u_hat": u, "iterations": it.value, "pe": pe.value, "stop": sp.value,
            "n_events": nev, "events": ev[: 5 * min(nev, ev_cap)].reshape(-1, 5)}


def decode_batch(kind, frozen, llr, alpha=0.9375, max_iter=40, prec=32, lib=None,
                 threads=None, want_u=True, want_events=True):
    """Batched oracle decode (frames x n). Returns dict of per-frame arrays.
    want_events=False passes no event counter, so csfg records no FreezeEvent
    list (the reference's decode_trial does that only with --trace,
    sim_harness.cpp:84-90); "n_events" is then None."""
    lib = lib or DEFAULT_LIB or C
    llr = np.ascontiguousarray(llr, np.float32 if prec == 32 else np.float64)
    frames, n = llr.shape
    if lib is C:
        fn = C.orc_decode_batch_f32 if prec == 32 else C.orc_decode_batch_f64
    else:
        fn = lib.ref32_decode_batch if prec == 32 else lib.ref64_decode_batch
    u = np.zeros((frames, n), np.uint8) if want_u else None
    it = np.zeros(frames, np.int32)
    sp = np.zeros(frames, np.int32)
    ne = np.zeros(frames, np.int32) if want_events else None
    pe = np.zeros(frames, np.int64)
    rc = fn(KIND.get(kind, kind), n, _p(np.ascontiguousarray(frozen, np.uint8), _u8p),
            _p(llr, _f32p if prec == 32 else _f64p), frames, alpha, max_iter,
            threads or os.cpu_count() or 1, _p(u, _u8p), _p(it, _i32p), _p(pe, _i64p),
            _p(sp, _i32p), _p(ne, _i32p))
    if rc:
        raise RuntimeError("oracle batch decode failed")
    return {"u_hat": u, "iterations": it, "pe": pe, "stop": sp, "n_events": ne}
