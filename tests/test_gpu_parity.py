"""GPU parity: the CUDA decoders through the C ABI against the oracle.

Bar (north star): hard decisions, iteration counts, PE-activation counts, stop
reasons and freeze-event counts bit-exact against the reference's fp32
operation order ("ref32"), on the golden frames and on random inputs; both the
warp-resident kernel and the generic kernel; property checks at full size.
"""
import math

import numpy as np
import pytest

import oracle as O
import paper_1505_04979_b200 as P
from conftest import load_manifest

pytestmark = pytest.mark.gpu
MAN = load_manifest()
Z0 = math.exp(-0.5)


def _cmp(r, golden, name, tag="ref32"):
    n = golden[name + "/frozen"].size
    got_u = P.unpack_bits(r["u_hat_bits"], n)
    exp_u = np.unpackbits(golden[f"{name}/{tag}/u_hat"], axis=1, bitorder="little")[:, :n]
    bad = np.flatnonzero((got_u != exp_u).any(1))
    assert bad.size == 0, f"{name}: u_hat differs on frames {bad[:10]}"
    for f in ("iterations", "pe", "stop", "n_events"):
        g = r[f].astype(np.int64)
        e = golden[f"{name}/{tag}/{f}"].astype(np.int64)
        assert np.array_equal(g, e), f"{name}: {f} differs at {np.flatnonzero(g != e)[:10]}"


@pytest.mark.parametrize("generic", [False, True], ids=["auto", "generic"])
@pytest.mark.parametrize("case", MAN["cases"], ids=lambda c: c["name"])
def test_golden_case(ctx, golden, case, generic):
    name = case["name"]
    code = P.PolarCode.from_frozen_mask(case["n"], golden[name + "/frozen"])
    ctx.force_generic(generic)
    try:
        r = P.decode_batch(code, case["decoder"], golden[name + "/llr32"], 0.9375, case["max_iter"], ctx=ctx)
    finally:
        ctx.force_generic(False)
    _cmp(r, golden, name)


@pytest.mark.timeout(600, method="thread")  # a hung kernel blocks the signal method
def test_golden_cases_back_to_back(ctx, golden):
    """Every golden case twice in a row on one context, fast and generic kernels
    interleaved: each launch starts on the shared and tensor memory the previous
    kernels left behind, so a read of uninitialised per-warp state (it once diverged
    the n = 1024 kernel's collectives and hung it) shows up as a wrong result or a
    timeout here."""
    for _ in range(2):
        for case in MAN["cases"]:
            name = case["name"]
            code = P.PolarCode.from_frozen_mask(case["n"], golden[name + "/frozen"])
            for generic in (False, True):
                ctx.force_generic(generic)
                try:
                    r = P.decode_batch(code, case["decoder"], golden[name + "/llr32"], 0.9375, case["max_iter"],
                                       ctx=ctx)
                finally:
                    ctx.force_generic(False)
                _cmp(r, golden, name)


@pytest.mark.parametrize("generic", [False, True], ids=["auto", "generic"])
def test_event_traces(ctx, golden, generic):
    ctx.force_generic(generic)
    try:
        for ec in MAN["event_cases"]:
            for i in range(ec["frames"]):
                p = f"{ec['name']}/{i}"
                fz = golden[p + "/frozen"]
                code = P.PolarCode.from_frozen_mask(fz.size, fz)
                events = []
                out = P.decode_csfg(code, golden[p + "/llr32"], 0.9375, ec["max_iter"], events=events, ctx=ctx)
                exp = golden[p + "/events"].reshape(-1, 5)
                got = np.array([[e.iteration, e.stage, e.block, e.start, e.size] for e in events],
                               np.int64).reshape(-1, 5)
                assert np.array_equal(got, exp), p
                assert [out.iterations_used, out.pe_activations, out.stop_reason, out.n_events] == \
                    list(golden[p + "/meta"]), p
                assert np.array_equal(out.u_hat, golden[p + "/u_hat"]), p
    finally:
        ctx.force_generic(False)


def test_reference_known_answers(ctx):
    # test_bp_core.cpp:185-204, test_csfg_freeze.cpp:222-246
    code = P.PolarCode.construct(8, 4, 0.5)
    o = P.decode_baseline(code, np.full(8, 2.0), 0.9375, 40, ctx=ctx)
    assert (o.iterations_used, o.pe_activations, o.stop_reason) == (40, 480, 0)
    assert not o.u_hat.any() and not o.info_bits.any()
    o = P.decode_gmatrix(code, np.full(8, 2.0), 0.9375, 40, ctx=ctx)
    assert (o.iterations_used, o.pe_activations, o.stop_reason) == (1, 12, 1)
    ev = []
    o = P.decode_csfg(code, np.full(8, 5.0), 0.9375, 40, events=ev, ctx=ctx)
    assert (o.iterations_used, o.pe_activations, o.stop_reason) == (1, 7, 1)
    assert [(e.stage, e.start, e.size) for e in ev] == [(0, 0, 4), (1, 4, 2), (2, 6, 1)]
    with pytest.raises(ValueError):
        P.decode_csfg(code, np.zeros(7), 0.9375, 40, ctx=ctx)  # init_state: LLR length != n


@pytest.mark.parametrize("n", [2, 8, 32, 64, 128, 256, 512, 1024, 2048])
@pytest.mark.parametrize("kind", ["baseline", "gmatrix", "csfg"])
def test_random_llrs_vs_oracle(ctx, n, kind):
    """Gaussian LLRs at several scales, exact zeros and exact ties, vs the C oracle (fp32)."""
    rng = np.random.default_rng(1000 * n + len(kind))
    fz = O.construct(n, max(1, n // 2), Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    frames = 64 if n <= 1024 else 8
    llr = rng.normal(1.0, 1.5, size=(frames, n)).astype(np.float32)
    llr[: frames // 4] *= 8.0
    llr[frames // 4: frames // 2, ::5] = 0.0
    llr[frames // 2: 3 * frames // 4] = np.round(llr[frames // 2: 3 * frames // 4])  # ties
    exp = O.decode_batch(kind, fz, llr, 0.9375, 25, prec=32)
    got = P.decode_batch(code, kind, llr, 0.9375, 25, ctx=ctx)
    assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"])
    for f in ("iterations", "pe", "stop", "n_events"):
        assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), f


def _random_frozen(rng, n, k):
    """A frozen set with the information rows anywhere (not a polar construction):
    info rows at low indices, unfrozen rows 0..31, odd block patterns."""
    fz = np.ones(n, np.uint8)
    fz[rng.choice(n, size=k, replace=False)] = 0
    return fz


@pytest.mark.parametrize("n", [128, 256, 512, 1024])
@pytest.mark.parametrize("kind", ["gmatrix", "csfg"])
@pytest.mark.parametrize("rate", [0.25, 0.5, 0.875])
def test_random_frozen_sets_vs_oracle(ctx, n, kind, rate):
    """Random frozen sets and channel-like LLRs at several SNRs: the csfg walks (window,
    re-covered rows, G-check filter preconditions) against the oracle, both kernels."""
    rng = np.random.default_rng(int(7000 * rate) + n + len(kind))
    k = max(1, int(n * rate))
    fz = _random_frozen(rng, n, k)
    code = P.PolarCode.from_frozen_mask(n, fz)
    frames = 96
    scale = rng.choice([1.0, 2.0, 4.0, 8.0], size=(frames, 1))
    llr = (scale * (1.0 + rng.normal(0.0, 1.0, size=(frames, n)))).astype(np.float32)
    exp = O.decode_batch(kind, fz, llr, 0.9375, 30, prec=32)
    for generic in (False, True):
        ctx.force_generic(generic)
        try:
            got = P.decode_batch(code, kind, llr, 0.9375, 30, ctx=ctx)
        finally:
            ctx.force_generic(False)
        assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"]), generic
        for f in ("iterations", "pe", "stop", "n_events"):
            assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), (f, generic)


@pytest.mark.parametrize("alpha,max_iter", [(0.5, 12), (1.0, 20), (0.75, 60)])
def test_other_alpha_and_iteration_caps(ctx, alpha, max_iter):
    n = 1024
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    _, llr64 = O.trials(3, 0, 64, fz, 2.0, lib=O.C)
    llr = llr64.astype(np.float32)
    for kind in ("baseline", "gmatrix", "csfg"):
        exp = O.decode_batch(kind, fz, llr, alpha, max_iter, prec=32)
        got = P.decode_batch(code, kind, llr, alpha, max_iter, ctx=ctx)
        assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"]), kind
        for f in ("iterations", "pe", "stop", "n_events"):
            assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), (kind, f)


@pytest.mark.parametrize("n", [256, 1024])
def test_clamp_and_nonfinite_frames_rerouted(ctx, n):
    """Frames the clamp-free fast path cannot take go to the generic kernel (clamps kept)."""
    rng = np.random.default_rng(7)
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    llr = rng.normal(1.0, 1.0, size=(16, n)).astype(np.float32)
    llr[1, 3] = 1e30
    llr[2, :] *= 1e28
    llr[3, 10] = -3e38
    llr[4, 0] = 2e14
    for kind in ("baseline", "gmatrix", "csfg"):
        exp = O.decode_batch(kind, fz, llr, 0.9375, 20, prec=32)
        got = P.decode_batch(code, kind, llr, 0.9375, 20, ctx=ctx)
        launches, rerouted = ctx.last_launch_info()
        assert rerouted == 4
        assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"]), kind
        for f in ("iterations", "pe", "stop", "n_events"):
            assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), (kind, f)


def test_chunked_batch_matches_single_launches(ctx):
    """pbp_decode_batch pipelines large batches over several streams (chunks of
    >= 16384 frames); results and the re-route count equal one launch per part."""
    n, frames = 256, 70_000
    code = P.PolarCode.construct(n, n // 2, Z0)
    llr, _, _ = P.generate(code, 9, 0, frames, 2.0, ctx=ctx)
    big = [5, 16_400, 33_000, 52_001, 69_999]          # re-routed frames in several chunks
    llr[big, 7] = 1e30
    for kind in ("gmatrix", "csfg"):
        whole = P.decode_batch(code, kind, llr, 0.9375, 30, ctx=ctx)
        launches, rerouted = ctx.last_launch_info()
        assert rerouted == len(big) and launches >= 3, (launches, rerouted)
        for a, b in ((0, 16_000), (16_000, 30_000), (30_000, frames)):
            part = P.decode_batch(code, kind, llr[a:b], 0.9375, 30, ctx=ctx)
            for f in whole:
                assert np.array_equal(whole[f][a:b], part[f]), (kind, f, a)
    exp = O.decode_batch("csfg", code.frozen, llr[big], 0.9375, 30, prec=32)
    assert np.array_equal(P.unpack_bits(whole["u_hat_bits"][big], n), exp["u_hat"])


@pytest.mark.parametrize("n,seed,ebn0", [(64, 4242, 2.0), (1024, 2, 3.0), (256, 5, 2.5), (4096, 4, 2.5)])
def test_channel_generation_matches_reference_stream(ctx, n, seed, ebn0):
    fz = O.construct(n, n // 2, Z0 if n != 64 else 0.5)
    code = P.PolarCode.from_frozen_mask(n, fz)
    count = 48 if n <= 1024 else 8
    llr, u, l64 = P.generate(code, seed, 3, count, ebn0, want64=True, ctx=ctx)
    info, ref64 = O.trials(seed, 3, count, fz, ebn0, lib=O.C)
    # transmitted words: bit-exact (integer RNG + GF(2) encode)
    ref_u = np.zeros((count, n), np.uint8)
    ref_u[:, fz == 0] = info
    assert np.array_equal(P.unpack_bits(u, n), ref_u)
    # fp32 LLRs the decoder consumes: exact; fp64 may differ in the last ulp (CUDA vs glibc log/cos)
    assert np.array_equal(llr, ref64.astype(np.float32))
    # y = s + sigma*g cancels near 0, so measure in ulps of the LLR scale 2/sigma^2
    scale = 2.0 / P.noise_variance(ebn0, 0.5)
    err = np.abs(l64 - ref64) / np.spacing(np.maximum(np.abs(ref64), scale))
    assert err.max() <= 8.0


@pytest.mark.parametrize("n,frames", [(1024, 384), (256, 512), (2048, 64), (4096, 48), (16384, 6)])
def test_simulate_point_counters_match_oracle(ctx, n, frames):
    """run_point's counters (device generation, decode, bit errors against the sent
    words) for every kernel against the oracle."""
    seed, ebn0 = 2, 2.5
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    info, llr = O.trials(seed, 0, frames, fz, ebn0, lib=O.C)
    for kind in ("baseline", "gmatrix", "csfg"):
        c = P.simulate_point(code, kind, seed, 0, frames, ebn0, ctx=ctx)
        r = O.decode_batch(kind, fz, llr.astype(np.float32), 0.9375, 40, prec=32)
        be = (r["u_hat"][:, fz == 0] != info).sum(1)
        it = r["iterations"].astype(np.int64)
        assert c["frames"] == frames
        assert c["bit_errors"] == int(be.sum())
        assert c["frame_errors"] == int((be > 0).sum())
        assert c["sum_iters"] == int(it.sum()) and c["sum_iters_sq"] == int((it * it).sum())
        assert c["sum_pe"] == int(r["pe"].sum())
        assert c["sum_events"] == int(r["n_events"].sum())
        assert [c["stop_max_iter"], c["stop_gmatrix"], c["stop_csfg"]] == \
            [int((r["stop"] == s).sum()) for s in range(3)]


def test_sharded_counters_sum_to_whole(ctx):
    """Trial-range sharding (the multi-GPU split) leaves the integer sums unchanged."""
    code = P.PolarCode.construct(1024, 512, Z0)
    whole = P.simulate_point(code, "csfg", 5, 0, 6000, 2.5, ctx=ctx)
    parts = [P.simulate_point(code, "csfg", 5, a, b - a, 2.5, ctx=ctx) for a, b in ((0, 1500), (1500, 4100), (4100, 6000))]
    for k in whole:
        assert whole[k] == sum(p[k] for p in parts), k


def test_full_size_properties(ctx):
    """Config 2 at 3 dB, 1e5 frames: size-independent invariants."""
    n, frames = 1024, 100_000
    code = P.PolarCode.construct(n, 512, Z0)
    llr, u, _ = P.generate(code, 2, 0, frames, 3.0, ctx=ctx)
    r = P.decode_batch(code, "csfg", llr, 0.9375, 40, ctx=ctx)
    bits = P.unpack_bits(r["u_hat_bits"], n)
    assert not bits[:, code.frozen == 1].any()                      # frozen-bit safety
    it, pe, stop = r["iterations"], r["pe"], r["stop"]
    assert ((it >= 1) & (it <= 40)).all()
    assert (pe <= it.astype(np.int64) * 10 * 512).all() and (pe > 0).all()
    assert ((stop != 0) | (it == 40)).all()                            # max_iter stop => 40 iterations
    truth = P.unpack_bits(u, n)
    fer = (bits != truth).any(1).mean()
    assert fer < 0.03                                                 # reference FER ~0.014 at 3 dB
    r2 = P.decode_batch(code, "csfg", llr, 0.9375, 40, ctx=ctx)      # determinism
    for f in r:
        assert np.array_equal(r[f], r2[f]), f
    # sample parity against the oracle on a strided subset of the full batch
    idx = np.arange(0, frames, 997)
    exp = O.decode_batch("csfg", code.frozen, llr[idx], 0.9375, 40, prec=32)
    assert np.array_equal(bits[idx], exp["u_hat"])
    assert np.array_equal(it[idx], exp["iterations"]) and np.array_equal(pe[idx], exp["pe"])


def test_noiseless_all_decoders(ctx):
    code = P.PolarCode.construct(1024, 512, Z0)
    llr, u, _ = P.generate(code, 1, 0, 256, 1.0, noiseless=True, ctx=ctx)
    for kind, it in (("baseline", 40), ("gmatrix", 1), ("csfg", 1)):
        r = P.decode_batch(code, kind, llr, 0.9375, 40, ctx=ctx)
        assert np.array_equal(r["u_hat_bits"], u), kind
        assert (r["iterations"] == it).all(), kind


def test_edge_cases(ctx):
    code = P.PolarCode.construct(1024, 512, Z0)
    llr = np.random.default_rng(3).normal(1, 1, size=(4, 1024)).astype(np.float32)
    for kind in ("baseline", "gmatrix", "csfg"):
        for mi in (0, 1, 2):
            exp = O.decode_batch(kind, code.frozen, llr, 0.9375, mi, prec=32)
            got = P.decode_batch(code, kind, llr, 0.9375, mi, ctx=ctx)
            assert np.array_equal(P.unpack_bits(got["u_hat_bits"], 1024), exp["u_hat"]), (kind, mi)
            for f in ("iterations", "pe", "stop", "n_events"):
                assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), (kind, mi, f)
    empty = P.decode_batch(code, "csfg", np.zeros((0, 1024), np.float32), 0.9375, 40, ctx=ctx)
    assert empty["iterations"].size == 0
    # n = 1 and n = 2 codes
    for n in (1, 2):
        c = P.PolarCode.construct(n, 1, 0.5)
        l = np.array([[-1.0] * n, [1.0] * n], np.float32)
        for kind in ("baseline", "gmatrix", "csfg"):
            exp = O.decode_batch(kind, c.frozen, l, 0.9375, 5, prec=32)
            got = P.decode_batch(c, kind, l, 0.9375, 5, ctx=ctx)
            assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"]), (n, kind)
            assert np.array_equal(got["iterations"], exp["iterations"]), (n, kind)


def test_concurrent_device_calls_on_two_streams(ctx):
    """Device-pointer decodes queued on two streams of one context at once: each call gets
    its own launch resources (rotated slots, ordered by events), results unchanged."""
    import ctypes as C
    import torch
    n, frames = 1024, 20000
    code = P.PolarCode.construct(n, n // 2, Z0)
    cs = code.c_struct()
    llr, _, _ = P.generate(code, 21, 0, 2 * frames, 2.5, ctx=ctx)
    ref = P.decode_batch(code, "csfg", llr, 0.9375, 40, ctx=ctx)
    dev = torch.device("cuda", 0)
    d_llr = torch.from_numpy(llr).to(dev)
    nw = n // 32
    outs, streams = [], [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    torch.cuda.synchronize()
    for i, st in enumerate(streams):
        o = {"u": torch.empty((frames, nw), dtype=torch.int32, device=dev),
             "it": torch.empty(frames, dtype=torch.int32, device=dev),
             "pe": torch.empty(frames, dtype=torch.int64, device=dev),
             "st": torch.empty(frames, dtype=torch.uint8, device=dev),
             "ne": torch.empty(frames, dtype=torch.int32, device=dev)}
        fo = P._abi.PbpFrameOut(P._abi.u32p(o["u"].data_ptr()), P._abi.i32p(o["it"].data_ptr()),
                                P._abi.i64p(o["pe"].data_ptr()), P._abi.u8p(o["st"].data_ptr()),
                                P._abi.i32p(o["ne"].data_ptr()))
        part = d_llr[i * frames:(i + 1) * frames]
        P._check(P.lib.pbp_decode_batch_device(ctx.handle, C.byref(cs), 2, P._abi.f32p(part.data_ptr()),
                                               frames, 0.9375, 40, C.byref(fo), C.c_void_p(st.cuda_stream)))
        outs.append(o)
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        sl = slice(i * frames, (i + 1) * frames)
        assert np.array_equal(o["u"].cpu().numpy().view(np.uint32), ref["u_hat_bits"][sl])
        assert np.array_equal(o["it"].cpu().numpy(), ref["iterations"][sl])
        assert np.array_equal(o["pe"].cpu().numpy(), ref["pe"][sl])
        assert np.array_equal(o["ne"].cpu().numpy(), ref["n_events"][sl])


def test_concurrent_simulate_point_device(ctx):
    """Two asynchronous simulate_point calls on two streams of one context (each generates
    into its own slot's staging) give the counters of the calls run one after another."""
    import ctypes as C
    import torch
    code = P.PolarCode.construct(1024, 512, Z0)
    cs = code.c_struct()
    exp = [P.simulate_point(code, "csfg", 2, a, 30000, e, ctx=ctx) for a, e in ((0, 2.0), (30000, 3.0))]
    dev = torch.device("cuda", 0)
    cnt = torch.zeros((2, 10), dtype=torch.int64, device=dev)
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    torch.cuda.synchronize()
    for i, (st, (a, e)) in enumerate(zip(streams, ((0, 2.0), (30000, 3.0)))):
        P._check(P.lib.pbp_simulate_point_device(ctx.handle, C.byref(cs), 2, C.c_uint64(2), a, 30000, e, 0,
                                                 0.9375, 40, P._abi.i64p(cnt[i].data_ptr()),
                                                 C.c_void_p(st.cuda_stream)))
    torch.cuda.synchronize()
    got = cnt.cpu().numpy()
    for i in range(2):
        assert [int(x) for x in got[i]] == [exp[i][k] for k in P.COUNTER_FIELDS], i


@pytest.mark.parametrize("n", [2048, 4096, 8192])
@pytest.mark.parametrize("kind", ["baseline", "gmatrix", "csfg"])
def test_cta_kernel_vs_oracle(ctx, n, kind):
    """n = 2048..16384 run on the CTA-per-frame register-pass kernel (pbp_kernel_path 2)."""
    assert P.lib.pbp_kernel_path(n) == 2
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    _, llr64 = O.trials(4, 0, 8 if n <= 4096 else 4, fz, 2.5, lib=O.C)
    llr = llr64.astype(np.float32)
    exp = O.decode_batch(kind, fz, llr, 0.9375, 30, prec=32)
    got = P.decode_batch(code, kind, llr, 0.9375, 30, ctx=ctx)
    assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"])
    for f in ("iterations", "pe", "stop", "n_events"):
        assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), f


def test_cta_kernel_reroute_and_events(ctx):
    n = 4096
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    _, llr64 = O.trials(4, 0, 6, fz, 2.5, lib=O.C)
    llr = llr64.astype(np.float32)
    llr[1, 5] = 1e30          # re-routed to the generic kernel (clamps kept)
    llr[4, :] *= 1e25
    exp = O.decode_batch("csfg", fz, llr, 0.9375, 40, prec=32)
    got = P.decode_batch(code, "csfg", llr, 0.9375, 40, ctx=ctx)
    assert ctx.last_launch_info()[1] == 2  # frames 1 and 4 went to the generic kernel
    assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"])
    for f in ("iterations", "pe", "stop", "n_events"):
        assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), f
    for i in (0, 2):
        events = []
        out = P.decode_csfg(code, llr[i], 0.9375, 40, events=events, ctx=ctx)
        e = O.decode("csfg", fz, llr[i], 0.9375, 40, prec=32)
        got_ev = np.array([[x.iteration, x.stage, x.block, x.start, x.size] for x in events], np.int64)
        assert np.array_equal(got_ev.reshape(-1, 5), np.asarray(e["events"], np.int64).reshape(-1, 5)), i
        assert out.pe_activations == e["pe"] and out.iterations_used == e["iterations"], i


@pytest.mark.parametrize("n", [2048, 4096, 8192, 16384])
@pytest.mark.parametrize("kind", ["gmatrix", "csfg"])
@pytest.mark.parametrize("rate", [0.25, 0.875])
def test_cta_kernel_random_frozen_sets(ctx, n, kind, rate):
    """The CTA-per-frame kernel on random frozen sets and channel-like LLRs at several
    SNRs (commit patterns of every stage of a pass, re-covered rows, early G-stops)."""
    rng = np.random.default_rng(int(9000 * rate) + n + len(kind))
    k = max(1, int(n * rate))
    fz = _random_frozen(rng, n, k)
    code = P.PolarCode.from_frozen_mask(n, fz)
    frames = 12 if n <= 4096 else 6
    scale = rng.choice([2.0, 4.0, 8.0, 16.0], size=(frames, 1))
    llr = (scale * (1.0 + rng.normal(0.0, 1.0, size=(frames, n)))).astype(np.float32)
    exp = O.decode_batch(kind, fz, llr, 0.9375, 30, prec=32)
    assert P.lib.pbp_kernel_path(n) == 2
    got = P.decode_batch(code, kind, llr, 0.9375, 30, ctx=ctx)
    assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"])
    for f in ("iterations", "pe", "stop", "n_events"):
        assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), f


@pytest.mark.parametrize("n", [64, 256, 1024, 4096])
def test_event_xhat_consistent(ctx, n):
    """FreezeEvent.x_hat from every kernel (generic, warp-resident, CTA) and both
    precisions: the fast and the generic kernel report the same blocks and bits, each
    block's polar_transform(x_hat) is 0 at its frozen rows, and replaying the events'
    decisions in order gives u_hat's decided prefix (acceptance.cpp:209-245)."""
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    _, llr64 = O.trials(11, 0, 6, fz, 3.0 if n >= 1024 else 2.5, lib=O.C)
    seen = 0
    for i in range(llr64.shape[0]):
        for prec in ("f32", "f64"):
            runs = []
            for generic in ((False, True) if prec == "f32" else (False,)):
                ctx.force_generic(generic)
                try:
                    ev = []
                    out = P.decode_csfg(code, llr64[i], 0.9375, 40, events=ev, ctx=ctx, precision=prec)
                finally:
                    ctx.force_generic(False)
                runs.append((out, ev))
            out, ev = runs[0]
            if len(runs) == 2:
                assert [(e.iteration, e.stage, e.start, e.size) for e in ev] == \
                       [(e.iteration, e.stage, e.start, e.size) for e in runs[1][1]]
                assert all(np.array_equal(a.x_hat, b.x_hat) for a, b in zip(ev, runs[1][1]))
            decided = np.zeros(n, np.uint8)
            f = 0
            for e in ev:
                assert e.x_hat is not None and len(e.x_hat) == e.size
                ub = P.polar_transform(e.x_hat)
                assert not np.any(ub & fz[e.start:e.start + e.size])
                decided[e.start:e.start + e.size] = ub
                f = e.start + e.size
            assert np.array_equal(out.u_hat[:f], decided[:f])
            seen += len(ev)
    assert seen > 0


@pytest.mark.parametrize("n", [32768, 65536])
def test_generic_kernel_beyond_cta_sizes(ctx, n):
    """n > 16384 decodes on the generic kernel (global-memory messages): parity with the
    oracle for all three decoders."""
    assert P.lib.pbp_kernel_path(n) == 0
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    _, llr64 = O.trials(13, 0, 2, fz, 3.0, lib=O.C)
    llr = llr64.astype(np.float32)
    for kind in ("baseline", "gmatrix", "csfg"):
        exp = O.decode_batch(kind, fz, llr, 0.9375, 12, prec=32)
        got = P.decode_batch(code, kind, llr, 0.9375, 12, ctx=ctx)
        assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"]), kind
        for f in ("iterations", "pe", "stop", "n_events"):
            assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), (kind, f)


def test_code_length_limit(ctx):
    """n above 131072 is refused with a message (the generic kernel's bit state lives in
    shared memory), not a failed launch."""
    n = 1 << 18
    code = P.PolarCode.from_frozen_mask(n, np.r_[np.ones(n // 2, np.uint8), np.zeros(n // 2, np.uint8)])
    with pytest.raises((ValueError, P._abi.PbpError), match="131072"):
        P.decode_batch(code, "csfg", np.zeros((1, n), np.float32), 0.9375, 2, ctx=ctx)


@pytest.mark.parametrize("n", [2048, 4096, 8192, 16384])
def test_cta_kernel_iteration_caps_and_alpha(ctx, n):
    """The CTA-per-frame kernel at max_iter 0/1/2/7 and other alphas."""
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    llr = np.random.default_rng(n).normal(2.0, 1.5, size=(3, n)).astype(np.float32)
    for kind in ("baseline", "gmatrix", "csfg"):
        for alpha, mi in ((0.9375, 0), (0.9375, 1), (0.9375, 2), (0.5, 7), (1.0, 7)):
            exp = O.decode_batch(kind, fz, llr, alpha, mi, prec=32)
            got = P.decode_batch(code, kind, llr, alpha, mi, ctx=ctx)
            assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"]), (kind, alpha, mi)
            for f in ("iterations", "pe", "stop", "n_events"):
                assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), (kind, alpha, mi, f)


def test_chunked_batch_cta_kernel(ctx):
    """The host pipeline at n = 4096 (CTA-per-frame kernel): several chunks, re-routed
    frames in later chunks (frame_base of the batch-wide list), results equal to
    one launch per part."""
    n, frames = 4096, 9000
    code = P.PolarCode.construct(n, n // 2, Z0)
    llr, _, _ = P.generate(code, 4, 0, frames, 2.5, ctx=ctx)
    big = [3, 4_500, 8_999]
    llr[big, 11] = -1e30
    whole = P.decode_batch(code, "csfg", llr, 0.9375, 20, ctx=ctx)
    launches, rerouted = ctx.last_launch_info()
    assert rerouted == len(big) and launches >= 2, (launches, rerouted)
    for a, b in ((0, 4_000), (4_000, frames)):
        part = P.decode_batch(code, "csfg", llr[a:b], 0.9375, 20, ctx=ctx)
        for f in whole:
            assert np.array_equal(whole[f][a:b], part[f]), (f, a)
    exp = O.decode_batch("csfg", code.frozen, llr[big], 0.9375, 20, prec=32)
    assert np.array_equal(P.unpack_bits(whole["u_hat_bits"][big], n), exp["u_hat"])
    for f in ("iterations", "pe", "stop", "n_events"):
        assert np.array_equal(whole[f][big].astype(np.int64), exp[f].astype(np.int64)), f


@pytest.mark.parametrize("n", [64, 1024, 4096])
@pytest.mark.parametrize("k_of", ["all", "one", "last"])
def test_degenerate_frozen_sets(ctx, n, k_of):
    """k = n (every candidate check accepts), k = 1 with the free row first or last:
    every decoder against the oracle."""
    fz = np.ones(n, np.uint8)
    if k_of == "all":
        fz[:] = 0
    elif k_of == "one":
        fz[0] = 0
    else:
        fz[n - 1] = 0
    code = P.PolarCode.from_frozen_mask(n, fz)
    llr = np.random.default_rng(n + len(k_of)).normal(1.5, 2.0, size=(5, n)).astype(np.float32)
    for kind in ("baseline", "gmatrix", "csfg"):
        exp = O.decode_batch(kind, fz, llr, 0.9375, 15, prec=32)
        got = P.decode_batch(code, kind, llr, 0.9375, 15, ctx=ctx)
        assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"]), kind
        for f in ("iterations", "pe", "stop", "n_events"):
            assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), (kind, f)


@pytest.mark.parametrize("n", [2048, 4096, 16384])
def test_cta_kernel_special_llr_values(ctx, n):
    """Exact zeros, -0, denormals, values at the clamp-free bound (kept on the fast path)
    and just above it (re-routed): the CTA-per-frame kernel against the oracle."""
    fz = O.construct(n, n // 2, Z0)
    code = P.PolarCode.from_frozen_mask(n, fz)
    rng = np.random.default_rng(n)
    llr = rng.normal(1.0, 2.0, size=(4, n)).astype(np.float32)
    llr[0, ::7] = 0.0
    llr[0, 3::7] = -0.0
    llr[1, ::5] = np.float32(1e-42)
    llr[1, 2::5] = -np.float32(1e-42)
    llr[2, ::97] = np.float32(1e14)
    llr[2, 1::97] = -np.float32(1e14)
    llr[3, 17] = np.nextafter(np.float32(1e14), np.float32(np.inf))
    for kind in ("gmatrix", "csfg"):
        exp = O.decode_batch(kind, fz, llr, 0.9375, 25, prec=32)
        got = P.decode_batch(code, kind, llr, 0.9375, 25, ctx=ctx)
        assert ctx.last_launch_info()[1] == 1  # frame 3 only
        assert np.array_equal(P.unpack_bits(got["u_hat_bits"], n), exp["u_hat"]), kind
        for f in ("iterations", "pe", "stop", "n_events"):
            assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), (kind, f)


@pytest.mark.parametrize("n,frames", [(4096, 9000), (16384, 2600)])
def test_chunked_batch_large_codes(ctx, n, frames):
    """At n >= 2048 the host pipeline's chunks are sized in bytes (16 MB of LLRs
    first, growing 1.3x): a multi-chunk call on the CTA kernel (n = 4096) and on the
    2-CTA cluster kernel (n = 16384), with re-routed frames in several chunks, equals
    one launch per part."""
    code = P.PolarCode.construct(n, n // 2, Z0)
    llr, _, _ = P.generate(code, 5, 0, frames, 4.0, ctx=ctx)
    big = [3, frames // 3, frames - 2]
    llr[big, 11] = 1e30
    whole = P.decode_batch(code, "csfg", llr, 0.9375, 40, ctx=ctx)
    launches, rerouted = ctx.last_launch_info()
    assert rerouted == len(big) and launches >= 4, (launches, rerouted)
    step = frames // 4
    for a in range(0, frames, step):
        b = min(frames, a + step)
        part = P.decode_batch(code, "csfg", llr[a:b], 0.9375, 40, ctx=ctx)
        for f in whole:
            assert np.array_equal(whole[f][a:b], part[f]), (f, a)
