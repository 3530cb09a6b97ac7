"""fp64 decode (pbp_*_f64): the reference as shipped, frame by frame.

The frames come from the oracle's host channel (glibc log/cos, the reference's
own arithmetic), are decoded on the GPU in double and compared field by field
with the oracle's fp64 decoder, which tests/test_oracle.py pins against the
reference compiled in place (ref64) and its golden outcomes. Non-converged
frames are included: unlike the fp32 path, fp64 must match them too.
"""
import math

import numpy as np
import pytest

import oracle as O
import paper_1505_04979_b200 as P

pytestmark = pytest.mark.gpu
Z0 = math.exp(-0.5)


def _oracle_batch(kind, fz, llr64, max_iter):
    return O.decode_batch(kind, fz, llr64, 0.9375, max_iter, prec=64)


@pytest.mark.parametrize("n,kind,ebn0,frames,max_iter,seed", [
    (1024, "csfg", 2.0, 96, 40, 2),
    (1024, "gmatrix", 1.5, 64, 40, 2),
    (1024, "baseline", 3.0, 16, 40, 1),
    (256, "csfg", 2.5, 128, 40, 5),
    (128, "csfg", 1.0, 64, 25, 7),
    (4096, "csfg", 2.5, 8, 60, 4),
    (16384, "csfg", 2.5, 2, 40, 5),
])
def test_f64_batch_matches_ref64(ctx, n, kind, ebn0, frames, max_iter, seed):
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    _, llr64 = O.trials(seed, 0, frames, fz, ebn0, lib=O.C)
    got = P.decode_batch(code, kind, llr64, 0.9375, max_iter, ctx=ctx, precision="f64")
    exp = _oracle_batch(kind, fz, llr64, max_iter)
    assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"])
    for f in ("iterations", "pe", "stop", "n_events"):
        assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), f


def test_f64_differs_from_f32_where_the_reference_does(ctx):
    """At 1 dB some non-converged frames decode differently in fp32 and fp64; the
    GPU reproduces each precision's own outcome (so the two paths are not aliases)."""
    n = 1024
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    _, llr64 = O.trials(2, 0, 64, fz, 1.0, lib=O.C)
    g64 = P.decode_batch(code, "csfg", llr64, 0.9375, 40, ctx=ctx, precision="f64")
    g32 = P.decode_batch(code, "csfg", llr64.astype(np.float32), 0.9375, 40, ctx=ctx)
    e64 = _oracle_batch("csfg", fz, llr64, 40)
    e32 = O.decode_batch("csfg", fz, llr64.astype(np.float32), 0.9375, 40, prec=32)
    assert (e64["u_hat"] != e32["u_hat"]).any(1).sum() > 0      # the precisions do disagree here
    assert np.array_equal(g64["pe"], e64["pe"]) and np.array_equal(g32["pe"], e32["pe"])
    assert np.array_equal(P.unpack_bits(g64["u_hat_bits"], n), e64["u_hat"])
    assert np.array_equal(P.unpack_bits(g32["u_hat_bits"], n), e32["u_hat"])


def test_f64_event_trace(ctx):
    n = 1024
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    _, llr64 = O.trials(2, 0, 6, fz, 2.5, lib=O.C)
    for i in range(llr64.shape[0]):
        events = []
        out = P.decode_csfg(code, llr64[i], 0.9375, 40, events=events, ctx=ctx, precision="f64")
        exp = O.decode("csfg", fz, llr64[i], 0.9375, 40, prec=64)
        got = np.array([[e.iteration, e.stage, e.block, e.start, e.size] for e in events], np.int64)
        assert np.array_equal(got.reshape(-1, 5), np.asarray(exp["events"], np.int64).reshape(-1, 5)), i
        assert (out.iterations_used, out.pe_activations, out.stop_reason, out.n_events) == \
            (exp["iterations"], exp["pe"], exp["stop"], exp["n_events"]), i
        assert np.array_equal(out.u_hat, exp["u_hat"]), i


def test_f64_simulate_point_counters(ctx):
    """simulate_point(precision='f64') = the oracle's fp64 decode of the same device-generated
    fp64 frames, counted like decode_trial (sim_harness.cpp:65-99)."""
    n, frames, ebn0 = 256, 400, 2.0
    code = P.PolarCode.construct(n, n // 2, Z0)
    got = P.simulate_point(code, "csfg", 11, 0, frames, ebn0, ctx=ctx, precision="f64")
    _, u, llr64 = P.generate(code, 11, 0, frames, ebn0, want64=True, ctx=ctx)
    exp = O.decode_batch("csfg", code.frozen, llr64, 0.9375, 40, prec=64)
    truth = P.unpack_bits(u, n)
    info = code.frozen == 0
    berr = (exp["u_hat"][:, info] != truth[:, info]).sum(1)
    it = exp["iterations"].astype(np.int64)
    assert got["frames"] == frames
    assert got["bit_errors"] == int(berr.sum()) and got["frame_errors"] == int((berr > 0).sum())
    assert got["sum_iters"] == int(it.sum()) and got["sum_iters_sq"] == int((it * it).sum())
    assert got["sum_pe"] == int(exp["pe"].sum()) and got["sum_events"] == int(exp["n_events"].sum())
    for s, key in enumerate(("stop_max_iter", "stop_gmatrix", "stop_csfg")):
        assert got[key] == int((exp["stop"] == s).sum()), key


# proj/test_output.txt:10-20: the reference's acceptance run (tests/acceptance.cpp:129-150:
# (1024,512) construct(.., 0.5), alpha 0.9375, 40 iterations, >= 100 frame errors or 1e5
# frames per point, seed 61803), printed as frames / fer %.4g / avg_iters %.2f / avg_pe %.0f.
REF_ACCEPTANCE = {
    2.0: [(512, "0.3184", "40.00", "204800"), (512, "0.3184", "35.41", "181280"), (512, "0.3184", "35.39", "176176")],
    2.5: [(1280, "0.08203", "40.00", "204800"), (1280, "0.08125", "29.70", "152056"),
          (1280, "0.08125", "29.70", "147734")],
    3.0: [(7168, "0.01465", "40.00", "204800"), (7168, "0.01409", "24.70", "126442"),
          (7168, "0.01423", "24.69", "123124")],
}


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_run_point_reproduces_reference_acceptance_output(ctx, precision):
    """run_point on the GPU prints the reference's own captured rows: exactly in fp64 (the
    shipped arithmetic); the fp32 path gives the same rows here as well."""
    cfg = P.SimConfig(code=P.PolarCode.construct(1024, 512, 0.5), decoders=(0, 1, 2), alpha=0.9375,
                      max_iter=40, min_frame_errors=100, max_frames=100_000, seed=61803, precision=precision)
    for snr, rows in REF_ACCEPTANCE.items():
        got = P.run_point(cfg, snr, ctx=ctx)
        for r, (frames, fer, it, pe) in zip(got, rows):
            assert (r.frames, f"{r.fer:.4g}", f"{r.avg_iters:.2f}", f"{r.avg_pe_activations:.0f}") == \
                (frames, fer, it, pe), (snr, r.decoder, precision)
