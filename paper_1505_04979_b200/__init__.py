"""B200-native batched polar-code BP decoder (baseline / G-matrix stop / CSFG freezing).

Python mirror of the reference's public interface (/root/reference/proj/include/polarbp/*.hpp)
on top of the C ABI in include/pbp.h (libpbp.so, built in-tree by
``paper_1505_04979_b200.build``). Names, argument meaning and error behaviour follow
the reference: ``PolarCode.construct``, ``polar_transform``, ``encode``,
``noise_variance``, ``decode_baseline`` / ``decode_gmatrix`` / ``decode_csfg`` returning a
``DecodeOutcome``, ``run_point`` / ``run_sweep`` returning ``PointStats`` rows. Batched entry
points (``decode_batch``, ``generate``, ``simulate_point``) are the B200 additions.

There is no CPU fallback: decoding needs a CUDA device and the extension; without them
every decode call raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi

__all__ = [
    "PolarCode", "Codeword", "DecodeOutcome", "FreezeEvent", "PointStats", "SimConfig",
    "StopReason", "DecoderKind", "polar_transform", "encode", "extract_info_bits",
    "noise_variance", "bhattacharyya_profile", "decode_baseline", "decode_gmatrix",
    "decode_csfg", "decode_batch", "generate", "simulate_point", "simulate_batches", "simulate_sweep_multi",
    "run_point", "run_sweep",
    "Context", "default_context", "LLR_CAP", "lib",
]

LLR_CAP = 1e30
lib = _abi.load()


class StopReason:
    """StopReason (bp_core.hpp:48)."""
    max_iter = 0
    gmatrix_converged = 1
    csfg_complete = 2
    names = ("max_iter", "gmatrix_converged", "csfg_complete")

    @staticmethod
    def to_string(v: int) -> str:
        return StopReason.names[v] if 0 <= v < 3 else "?"


class DecoderKind:
    """DecoderKind (sim_harness.hpp:19)."""
    baseline = 0
    gmatrix = 1
    csfg = 2
    names = ("baseline", "gmatrix", "csfg")

    @staticmethod
    def parse(name: str) -> int:
        # parse_decoder (sim_harness.cpp:43-48)
        if name in DecoderKind.names:
            return DecoderKind.names.index(name)
        raise ValueError(f"unknown decoder '{name}'")

    @staticmethod
    def to_string(v: int) -> str:
        return DecoderKind.names[v] if 0 <= v < 3 else "?"


def _kind(k) -> int:
    return DecoderKind.parse(k) if isinstance(k, str) else int(k)


def _check(rc: int):
    _abi.check(lib, rc)


# ---------------------------------------------------------------- codes

def bhattacharyya_profile(n: int, design_z: float) -> np.ndarray:
    """bhattacharyya_profile (polar_code.cpp:27-43), host-side, fp64."""
    if n <= 0 or n & (n - 1):
        raise ValueError("bhattacharyya_profile: n must be a power of two")
    if not (0.0 < design_z < 1.0):
        raise ValueError("bhattacharyya_profile: design_z must be in (0,1)")
    z = np.full(n, float(design_z))
    half = n // 2
    while half >= 1:
        idx = np.arange(n)
        lo = idx[(idx & half) == 0]
        zi = z[lo].copy()
        z[lo] = 2.0 * zi - zi * zi
        z[lo + half] = zi * zi
        half //= 2
    return z


@dataclass
class PolarCode:
    """PolarCode (polar_code.hpp:27-40): n = 2^m, k info rows, frozen[r] = 1 marks a frozen row."""
    n: int
    m: int
    k: int
    frozen: np.ndarray

    def is_frozen(self, pos: int) -> bool:
        return bool(self.frozen[pos])

    def frozen_positions(self) -> List[int]:
        return [int(i) for i in np.flatnonzero(self.frozen)]

    @staticmethod
    def construct(n: int, k: int, design_z: float = 0.5) -> "PolarCode":
        out = np.zeros(max(int(n), 1), np.uint8)
        _check(lib.pbp_construct(int(n), int(k), float(design_z), _abi.u8p(out)))
        return PolarCode.from_frozen_mask(n, out)

    @staticmethod
    def from_frozen_mask(n: int, mask) -> "PolarCode":
        # from_frozen_mask (polar_code.cpp:68-80)
        if n <= 0 or n & (n - 1):
            raise ValueError("from_frozen_mask: n must be a power of two")
        mask = np.ascontiguousarray(np.asarray(mask, dtype=np.uint8) != 0, dtype=np.uint8)
        if mask.size != n:
            raise ValueError("from_frozen_mask: mask length != n")
        k = int(n - int(mask.sum()))
        if k < 1:
            raise ValueError("from_frozen_mask: no information positions")
        return PolarCode(int(n), int(n).bit_length() - 1, k, mask)

    def c_struct(self) -> _abi.PbpCode:
        return _abi.PbpCode(self.n, self.m, self.k, _abi.u8p(self.frozen))


@dataclass
class Codeword:
    u: np.ndarray
    x: np.ndarray


def polar_transform(v) -> np.ndarray:
    """x = u F^{(x)m}, natural order, self-inverse (polar_code.cpp:13-25)."""
    a = np.ascontiguousarray(np.asarray(v, dtype=np.uint8) & 1, dtype=np.uint8).copy()
    _check(lib.pbp_polar_transform(_abi.u8p(a), int(a.size)))
    return a


def encode(code: PolarCode, info_bits) -> Codeword:
    """encode (polar_code.cpp:82-91)."""
    info = np.ascontiguousarray(np.asarray(info_bits, dtype=np.uint8))
    if info.size != code.k:
        raise ValueError("encode: info length != k")
    u = np.zeros(code.n, np.uint8)
    x = np.zeros(code.n, np.uint8)
    cs = code.c_struct()
    _check(lib.pbp_encode(C.byref(cs), _abi.u8p(info), _abi.u8p(u), _abi.u8p(x)))
    return Codeword(u, x)


def extract_info_bits(code: PolarCode, u) -> np.ndarray:
    """extract_info_bits (polar_code.cpp:93-101)."""
    u = np.asarray(u, dtype=np.uint8)
    if u.size != code.n:
        raise ValueError("extract_info_bits: length != n")
    return u[code.frozen == 0].copy()


def noise_variance(ebn0_db: float, rate: float) -> float:
    """noise_variance (channel.cpp:9-15)."""
    out = C.c_double()
    _check(lib.pbp_noise_variance(float(ebn0_db), float(rate), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- device context

class Context:
    """One CUDA device context (include/pbp.h pbp_ctx): stream + device buffers."""

    def __init__(self, device: int = 0):
        self._p = C.c_void_p()
        _check(lib.pbp_ctx_create(int(device), C.byref(self._p)))
        self.device = device

    @property
    def handle(self):
        return self._p

    def close(self):
        if self._p:
            lib.pbp_ctx_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stream(self) -> int:
        return lib.pbp_ctx_stream(self._p) or 0

    def synchronize(self):
        _check(lib.pbp_ctx_synchronize(self._p))

    def force_generic(self, on: bool = True):
        _check(lib.pbp_ctx_force_generic(self._p, 1 if on else 0))

    def last_launch_info(self):
        n = C.c_int32()
        r = C.c_int64()
        _check(lib.pbp_last_launch_info(self._p, C.byref(n), C.byref(r)))
        return n.value, r.value


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("PBP_DEVICE", "0")))
    return _default_ctx


def device_count() -> int:
    return int(lib.pbp_device_count())


# ---------------------------------------------------------------- decoding

@dataclass
class FreezeEvent:
    """FreezeEvent (csfg_freeze.hpp:28-35): x_hat = the block's hard decisions at freeze time."""
    iteration: int
    stage: int
    block: int
    start: int
    size: int
    x_hat: Optional[np.ndarray] = None


@dataclass
class DecodeOutcome:
    """DecodeOutcome (bp_core.hpp:51-57)."""
    u_hat: np.ndarray
    info_bits: np.ndarray
    iterations_used: int
    pe_activations: int
    stop_reason: int
    n_events: int = 0


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    """(frames, ceil(n/32)) uint32 -> (frames, n) uint8 bits, row r = bit r%32 of word r/32."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    b = np.unpackbits(w.view(np.uint8).reshape(*w.shape[:-1], -1), axis=-1, bitorder="little")
    return b[..., :n]


def pack_bits(bits: np.ndarray) -> np.ndarray:
    bits = np.asarray(bits, dtype=np.uint8)
    n = bits.shape[-1]
    nw = (n + 31) // 32
    pad = np.zeros((*bits.shape[:-1], nw * 32), np.uint8)
    pad[..., :n] = bits
    by = np.packbits(pad, axis=-1, bitorder="little")
    return by.view(np.uint32).reshape(*bits.shape[:-1], nw)


def decode_batch(code: PolarCode, decoder, llrs, alpha: float = 0.9375, max_iter: int = 40,
                 ctx: Optional[Context] = None, precision: str = "f32"):
    """Batched decode of frames x n LLRs (host arrays) through pbp_decode_batch
    (precision "f32": fp32 in the reference's operation order, the fast path) or
    pbp_decode_batch_f64 ("f64": double, the reference as shipped).

    Returns dict: u_hat_bits (frames, ceil(n/32)) uint32, iterations, pe, stop, n_events.
    """
    ctx = ctx or default_context()
    f64 = _precision(precision)
    llr = np.ascontiguousarray(np.asarray(llrs, dtype=np.float64 if f64 else np.float32))
    if llr.ndim == 1:
        llr = llr.reshape(1, -1)
    if llr.shape[1] != code.n:
        raise ValueError("init_state: LLR length != n")
    frames = llr.shape[0]
    nw = (code.n + 31) // 32
    out = {
        "u_hat_bits": np.zeros((frames, nw), np.uint32),
        "iterations": np.zeros(frames, np.int32),
        "pe": np.zeros(frames, np.int64),
        "stop": np.zeros(frames, np.uint8),
        "n_events": np.zeros(frames, np.int32),
    }
    fo = _abi.PbpFrameOut(_abi.u32p(out["u_hat_bits"]), _abi.i32p(out["iterations"]),
                          _abi.i64p(out["pe"]), _abi.u8p(out["stop"]), _abi.i32p(out["n_events"]))
    cs = code.c_struct()
    if f64:
        _check(lib.pbp_decode_batch_f64(ctx.handle, C.byref(cs), _kind(decoder), _abi.f64p(llr), frames,
                                        float(alpha), int(max_iter), C.byref(fo)))
    else:
        _check(lib.pbp_decode_batch(ctx.handle, C.byref(cs), _kind(decoder), _abi.f32p(llr), frames,
                                    float(alpha), int(max_iter), C.byref(fo)))
    return out


def _precision(p: str) -> bool:
    if p not in ("f32", "f64"):
        raise ValueError(f"precision must be 'f32' or 'f64', got {p!r}")
    return p == "f64"


def _decode_one(code: PolarCode, kind: int, llrs, alpha, max_iter, events=None, ctx=None, precision="f32"):
    ctx = ctx or default_context()
    f64 = _precision(precision)
    llr = np.ascontiguousarray(np.asarray(llrs, dtype=np.float64 if f64 else np.float32).reshape(-1))
    if llr.size != code.n:
        raise ValueError("init_state: LLR length != n")
    cap = max(1, int(max_iter) * code.m)  # one commit per stage per iteration at most: never truncated
    u = np.zeros(code.n, np.uint8)
    ev = np.zeros(cap * 5, np.int32)
    it, sp, ne = C.c_int32(), C.c_int32(), C.c_int32()
    pe = C.c_int64()
    cs = code.c_struct()
    nw = (code.n + 31) // 32
    xw = np.zeros(cap * nw if events is not None else 1, np.uint32)  # each event's x_hat
    xp = xw.ctypes.data_as(C.POINTER(C.c_uint32)) if events is not None else None
    fn, lp = (lib.pbp_decode_trace_f64_x, _abi.f64p(llr)) if f64 else (lib.pbp_decode_trace_x, _abi.f32p(llr))
    _check(fn(ctx.handle, C.byref(cs), kind, lp, float(alpha), int(max_iter), _abi.u8p(u), C.byref(it),
              C.byref(pe), C.byref(sp), C.byref(ne), _abi.i32p(ev), cap, xp))
    if events is not None:
        events.clear()
        for i in range(min(ne.value, cap)):
            it_, st_, bl_, sa_, sz_ = (int(x) for x in ev[5 * i: 5 * i + 5])
            bits = unpack_bits(xw[i * nw:(i + 1) * nw], code.n)[sa_:sa_ + sz_].copy()
            events.append(FreezeEvent(it_, st_, bl_, sa_, sz_, bits))
    return DecodeOutcome(u, extract_info_bits(code, u), it.value, pe.value, sp.value, ne.value)


def decode_baseline(code: PolarCode, llrs, alpha: float, max_iter: int, ctx=None,
                    precision: str = "f32") -> DecodeOutcome:
    """decode_baseline (bp_core.hpp:84) on the GPU."""
    return _decode_one(code, 0, llrs, alpha, max_iter, ctx=ctx, precision=precision)


def decode_gmatrix(code: PolarCode, llrs, alpha: float, max_iter: int, ctx=None,
                   precision: str = "f32") -> DecodeOutcome:
    """decode_gmatrix (bp_core.hpp:86) on the GPU."""
    return _decode_one(code, 1, llrs, alpha, max_iter, ctx=ctx, precision=precision)


def decode_csfg(code: PolarCode, llrs, alpha: float, max_iter: int,
                events: Optional[list] = None, ctx=None, precision: str = "f32") -> DecodeOutcome:
    """decode_csfg (csfg_freeze.hpp:109-111) on the GPU; `events` receives FreezeEvents."""
    return _decode_one(code, 2, llrs, alpha, max_iter, events=events, ctx=ctx, precision=precision)


# ---------------------------------------------------------------- channel / Monte Carlo

def generate(code: PolarCode, seed: int, first_trial: int, count: int, ebn0_db: float,
             noiseless: bool = False, want64: bool = False, ctx=None):
    """Frames of decode_trial (sim_harness.cpp:67-73) generated on the GPU.

    Returns (llr fp32 [count, n], u bits [count, ceil(n/32)], llr fp64 or None)."""
    ctx = ctx or default_context()
    nw = (code.n + 31) // 32
    llr = np.zeros((count, code.n), np.float32)
    u = np.zeros((count, nw), np.uint32)
    l64 = np.zeros((count, code.n), np.float64) if want64 else None
    cs = code.c_struct()
    _check(lib.pbp_generate(ctx.handle, C.byref(cs), C.c_uint64(seed), int(first_trial), int(count),
                            float(ebn0_db), int(bool(noiseless)), _abi.f32p(llr),
                            _abi.f64p(l64) if want64 else None, _abi.u32p(u)))
    return llr, u, l64


COUNTER_FIELDS = ("frames", "bit_errors", "frame_errors", "sum_iters", "sum_iters_sq", "sum_pe",
                  "sum_events", "stop_max_iter", "stop_gmatrix", "stop_csfg")


def simulate_point(code: PolarCode, decoder, seed: int, first_trial: int, frames: int,
                   ebn0_db: float, alpha: float = 0.9375, max_iter: int = 40,
                   noiseless: bool = False, ctx=None, precision: str = "f32") -> dict:
    """Counters (Accumulator, sim_harness.cpp:56-63) over trials [first, first+frames);
    precision "f64" decodes the reference's double LLRs in double (as shipped)."""
    ctx = ctx or default_context()
    c = _abi.PbpCounters()
    cs = code.c_struct()
    fn = lib.pbp_simulate_point_f64 if _precision(precision) else lib.pbp_simulate_point
    _check(fn(ctx.handle, C.byref(cs), _kind(decoder), C.c_uint64(seed), int(first_trial), int(frames),
              float(ebn0_db), int(bool(noiseless)), float(alpha), int(max_iter), C.byref(c)))
    vals = [c.frames, c.bit_errors, c.frame_errors, c.sum_iters, c.sum_iters_sq, c.sum_pe,
            c.sum_events, c.stop_hist[0], c.stop_hist[1], c.stop_hist[2]]
    return dict(zip(COUNTER_FIELDS, [int(v) for v in vals]))


def simulate_batches(code: PolarCode, decoder, seed: int, first_trial: int, frames: int, ebn0_db: float,
                     batch: int = 256, alpha: float = 0.9375, max_iter: int = 40, noiseless: bool = False,
                     ctx=None, precision: str = "f32") -> np.ndarray:
    """One counter set per `batch` consecutive trials (ceil(frames/batch) x 10 int64, the
    COUNTER_FIELDS order): run_point's batches (sim_harness.cpp:136-178) on the device."""
    ctx = ctx or default_context()
    nb = (int(frames) + int(batch) - 1) // int(batch)
    out = np.zeros((max(nb, 1), 10), np.int64)
    cs = code.c_struct()
    _check(lib.pbp_simulate_batches(ctx.handle, C.byref(cs), _kind(decoder), C.c_uint64(seed), int(first_trial),
                                    int(frames), int(batch), float(ebn0_db), int(bool(noiseless)), float(alpha),
                                    int(max_iter), int(_precision(precision)), _abi.i64p(out)))
    return out[:nb]


def simulate_sweep_multi(code: PolarCode, decoder, seed: int, frames_per_point: int, snrs: Sequence[float],
                         devices: Optional[Sequence[int]] = None, alpha: float = 0.9375, max_iter: int = 40,
                         noiseless: bool = False) -> List[dict]:
    """run_sweep's counters with fixed frame counts over several GPUs of this process
    (pbp_simulate_sweep_multi: one host thread per device, contiguous trial ranges, one
    NCCL int64 all-reduce). devices: default every visible GPU."""
    devs = list(range(device_count())) if devices is None else [int(d) for d in devices]
    if not devs:
        raise RuntimeError("simulate_sweep_multi: no CUDA device")
    try:  # libpbp.so resolves NCCL at first use: let it bind to torch's copy (a newer
        import torch  # noqa: F401  NCCL than the system one, which torch cannot load over)
    except ImportError:
        pass
    dv = (C.c_int * len(devs))(*devs)
    sv = (C.c_double * len(snrs))(*[float(x) for x in snrs])
    out = (_abi.PbpCounters * len(snrs))()
    cs = code.c_struct()
    _check(lib.pbp_simulate_sweep_multi(dv, len(devs), C.byref(cs), _kind(decoder), C.c_uint64(seed),
                                        int(frames_per_point), sv, len(snrs), int(bool(noiseless)), float(alpha),
                                        int(max_iter), out))
    rows = []
    for c in out:
        vals = [c.frames, c.bit_errors, c.frame_errors, c.sum_iters, c.sum_iters_sq, c.sum_pe,
                c.sum_events, c.stop_hist[0], c.stop_hist[1], c.stop_hist[2]]
        rows.append(dict(zip(COUNTER_FIELDS, [int(v) for v in vals])))
    return rows


@dataclass
class SimConfig:
    """SimConfig (sim_harness.hpp:23-36)."""
    code: PolarCode
    code_source: str = ""
    decoders: Sequence[int] = (0, 1, 2)
    snr_db: Sequence[float] = ()
    alpha: float = 0.9375
    max_iter: int = 40
    min_frame_errors: int = 100
    max_frames: int = 100000
    seed: int = 1
    workers: int = 1
    noiseless: bool = False
    precision: str = "f32"   # B200 addition: "f64" decodes in double, as shipped


@dataclass
class PointStats:
    """PointStats (sim_harness.hpp:38-52)."""
    decoder: int = 0
    snr_db: float = 0.0
    frames: int = 0
    bit_errors: int = 0
    frame_errors: int = 0
    ber: float = 0.0
    fer: float = 0.0
    fer_ci95: float = 0.0
    avg_iters: float = 0.0
    iters_ci95: float = 0.0
    avg_pe_activations: float = 0.0
    norm_computations: float = 0.0
    low_confidence: bool = False


def make_stats(cfg: SimConfig, kind: int, snr: float, acc: dict) -> PointStats:
    """make_stats (sim_harness.cpp:101-125): double arithmetic on the integer sums."""
    row = PointStats(decoder=kind, snr_db=snr, frames=acc["frames"], bit_errors=acc["bit_errors"],
                     frame_errors=acc["frame_errors"])
    frames = float(acc["frames"])
    row.ber = acc["bit_errors"] / (frames * cfg.code.k)
    row.fer = acc["frame_errors"] / frames
    row.fer_ci95 = 1.96 * math.sqrt(row.fer * (1.0 - row.fer) / frames)
    row.avg_iters = acc["sum_iters"] / frames
    if acc["frames"] > 1:
        mean = row.avg_iters
        var = (float(acc["sum_iters_sq"]) - frames * mean * mean) / (frames - 1.0)
        row.iters_ci95 = 1.96 * math.sqrt(max(var, 0.0) / frames)
    row.avg_pe_activations = acc["sum_pe"] / frames
    full = float(cfg.max_iter) * cfg.code.m * (cfg.code.n // 2)
    row.norm_computations = row.avg_pe_activations / full if full > 0.0 else 0.0
    row.low_confidence = acc["frame_errors"] < cfg.min_frame_errors
    return row


K_BATCH = 256  # kBatchSize (sim_harness.cpp:21)


def run_point(cfg: SimConfig, snr_db: float, ctx=None) -> List[PointStats]:
    """run_point (sim_harness.cpp:129-186) on the GPU, 256-frame batch stop rule included.

    Chunks of whole batches are generated and decoded on the device, which returns one
    counter set per 256-trial batch (pbp_simulate_batches); the batches are merged in trial
    order and the stop rule is evaluated on the same boundaries as the reference, so the
    frame counts (and every sum) are identical."""
    if not cfg.decoders:
        raise ValueError("run_point: no decoders")
    if cfg.max_frames < 1:
        raise ValueError("run_point: max_frames < 1")
    accs = [dict.fromkeys(COUNTER_FIELDS, 0) for _ in cfg.decoders]
    frames = 0
    chunk = K_BATCH * 16
    while frames < cfg.max_frames:
        c = min(chunk, cfg.max_frames - frames)
        per = [simulate_batches(cfg.code, kind, cfg.seed, frames, c, snr_db, K_BATCH, cfg.alpha, cfg.max_iter,
                                cfg.noiseless, ctx, precision=cfg.precision) for kind in cfg.decoders]
        for b in range(per[0].shape[0]):
            for d in range(len(cfg.decoders)):
                for i, key in enumerate(COUNTER_FIELDS):
                    accs[d][key] += int(per[d][b, i])
            if all(a["frame_errors"] >= cfg.min_frame_errors for a in accs):
                return [make_stats(cfg, kind, snr_db, a) for kind, a in zip(cfg.decoders, accs)]
        frames += c
        chunk = min(chunk * 2, K_BATCH * 1024)
    return [make_stats(cfg, kind, snr_db, a) for kind, a in zip(cfg.decoders, accs)]


def run_sweep(cfg: SimConfig, ctx=None) -> List[PointStats]:
    """run_sweep (sim_harness.cpp:188-196)."""
    if not cfg.snr_db:
        raise ValueError("run_sweep: no SNR points")
    rows: List[PointStats] = []
    for snr in cfg.snr_db:
        rows.extend(run_point(cfg, snr, ctx))
    return rows
