"""GPU parity at the configs' scale, against the reference compiled in place (ref32 /
ref64 on all host threads): every frame of 10^4 trials per config-2 Eb/N0 point, 2x10^3
frames of config 3 (n = 4096), 200 frames of config 4 at n = 16384 and 2x10^3 at n = 256,
and the bench sweep's per-point aggregates (FER, average iterations, PE activations)
against ref64 (proj/tests/acceptance.cpp:129-171, proj/test_output.txt:10-20)."""
import math
import os

import numpy as np
import pytest

import oracle as O
import paper_1505_04979_b200 as P

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built")]
Z0 = math.exp(-0.5)
THREADS = os.cpu_count() or 1
SNRS = [1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0]


def _same(got, exp, n, tag):
    u = P.unpack_bits(got["u_hat_bits"], n)
    bad = np.flatnonzero((u != exp["u_hat"]).any(1))
    assert bad.size == 0, f"{tag}: u_hat differs on {bad.size} frames, first {bad[:5]}"
    for f in ("iterations", "pe", "stop", "n_events"):
        g, e = got[f].astype(np.int64), exp[f].astype(np.int64)
        bad = np.flatnonzero(g != e)
        assert bad.size == 0, f"{tag}: {f} differs on {bad.size} frames, first {bad[:5]}"


def _gpu_frames(code, seed, first, count, ebn0, ctx):
    llr, _, _ = P.generate(code, seed, first, count, ebn0, ctx=ctx)
    return llr


@pytest.mark.parametrize("snr", SNRS)
def test_config2_every_frame_of_1e4_trials_per_point(ctx, snr):
    code = P.PolarCode.construct(1024, 512, Z0)
    llr = _gpu_frames(code, 2, 0, 10_000, snr, ctx)
    got = P.decode_batch(code, "csfg", llr, 0.9375, 40, ctx=ctx)
    exp = O.decode_batch("csfg", code.frozen, llr, 0.9375, 40, prec=32, lib=O.REF, threads=THREADS)
    _same(got, exp, 1024, f"config2 {snr} dB")


@pytest.mark.parametrize("n,frames,snr,max_iter,seed", [(4096, 2000, 2.5, 60, 4), (16384, 200, 2.5, 40, 5),
                                                        (256, 2000, 2.5, 40, 5)],
                         ids=["config3_n4096", "config4_n16384", "config4_n256"])
def test_large_and_small_codes_every_frame(ctx, n, frames, snr, max_iter, seed):
    code = P.PolarCode.construct(n, n // 2, Z0)
    llr = _gpu_frames(code, seed, 0, frames, snr, ctx)
    got = P.decode_batch(code, "csfg", llr, 0.9375, max_iter, ctx=ctx)
    exp = O.decode_batch("csfg", code.frozen, llr, 0.9375, max_iter, prec=32, lib=O.REF, threads=THREADS)
    _same(got, exp, n, f"n={n}")


def test_bench_sweep_aggregates_against_ref64(ctx):
    """Per point of the bench sweep (config 2, seed 2, trials 0..1999): the fp64 GPU path
    (device generation + double decode) reproduces ref64's frame errors, bit errors,
    iteration and PE sums on the host's glibc frames; the fp32 path (the bench's) equals
    ref32 decoding the same fp32 frames, whose LLRs equal (float) of the host's fp64 LLRs
    (CUDA's double log/cos are within 2 ulp of glibc's, so a mismatch needs a value within
    a few ulp of a float rounding boundary: counted, expected ~1e-8 per LLR)."""
    code = P.PolarCode.construct(1024, 512, Z0)
    n_tr = 2000
    mism = 0
    for snr in SNRS:
        info, llr64 = O.trials(2, 0, n_tr, code.frozen, snr, lib=O.REF, threads=THREADS)
        llr32, _, _ = P.generate(code, 2, 0, n_tr, snr, ctx=ctx)
        mism += int((llr32 != llr64.astype(np.float32)).sum())
        for prec, frames in (("f64", llr64), ("f32", llr32)):
            r = O.decode_batch("csfg", code.frozen, frames, 0.9375, 40, prec=64 if prec == "f64" else 32,
                               lib=O.REF, threads=THREADS)
            be = (r["u_hat"][:, code.frozen == 0] != info).sum(1)
            it = r["iterations"].astype(np.int64)
            exp = {"frames": n_tr, "bit_errors": int(be.sum()), "frame_errors": int((be > 0).sum()),
                   "sum_iters": int(it.sum()), "sum_iters_sq": int((it * it).sum()), "sum_pe": int(r["pe"].sum()),
                   "sum_events": int(r["n_events"].sum())}
            g = P.simulate_point(code, "csfg", 2, 0, n_tr, snr, ctx=ctx, precision=prec)
            for k, v in exp.items():
                assert g[k] == v, (snr, prec, k, g[k], v)
    assert mism <= 2, f"{mism} fp32 LLRs differ from (float) of the glibc fp64 LLRs"
