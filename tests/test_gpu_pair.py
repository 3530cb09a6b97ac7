"""GPU parity of the 2-CTA cluster ("pair") layout of n = 16384 csfg decodes: each CTA
holds half of the frame on its SM; the frame's stage 0 crosses the pair through
distributed shared memory; the half holding the frontier runs the candidate checks
(csfg_freeze.cpp:99-152), the other half takes over when the frontier crosses n/2.

The paths that only this layout has are forced with constructed inputs and checked
against the oracle (ref32 when oracle/_ref is built): the first half frozen whole at
the frame's stage 0 (the frontier crosses in the cross phase), the frontier crossing
inside a pass, the second half completing the frame mid-sweep (the first half's later
stages are then not counted), and frames that stop on the pinned G-check. The same
frames through one CTA per frame (PBP_PAIR=0) must give identical results."""
import math

import numpy as np
import pytest

import oracle as O
import paper_1505_04979_b200 as P

pytestmark = pytest.mark.gpu
Z0 = math.exp(-0.5)
N = 16384


def _same(got, exp, tag):
    u = P.unpack_bits(got["u_hat_bits"], N)
    bad = np.flatnonzero((u != exp["u_hat"]).any(1))
    assert bad.size == 0, f"{tag}: u_hat differs on frames {bad[:10]}"
    for f in ("iterations", "pe", "stop", "n_events"):
        g, e = got[f].astype(np.int64), exp[f].astype(np.int64)
        bad = np.flatnonzero(g != e)
        assert bad.size == 0, f"{tag}: {f} differs on frames {bad[:10]} ({g[bad[:3]]} vs {e[bad[:3]]})"


def _same_gpu(a, b, tag):
    assert np.array_equal(a["u_hat_bits"], b["u_hat_bits"]), tag
    for f in ("iterations", "pe", "stop", "n_events"):
        assert np.array_equal(a[f], b[f]), (tag, f)


@pytest.fixture
def pair(monkeypatch):
    monkeypatch.setenv("PBP_PAIR", "1")
    assert P.lib.pbp_kernel_cluster(N, 2) == 2 and P.lib.pbp_kernel_cluster(N, 1) == 2
    assert P.lib.pbp_kernel_cluster(N, 0) == 2 and P.lib.pbp_kernel_cluster(8192, 2) == 1


def _oracle(fz, llr, max_iter):
    return O.decode_batch("csfg", fz, llr, 0.9375, max_iter, prec=32)


def _code(fz):
    return P.PolarCode.from_frozen_mask(N, fz)


@pytest.mark.parametrize("snr", [2.5, 3.5, 5.0, 7.0])
def test_pair_channel_frames(ctx, pair, snr):
    """config-4 style frames: at 2.5 dB the frontier stays in the first half; at 5-7 dB
    it crosses into the second half and frames complete."""
    fz = O.construct(N, N // 2, Z0)
    _, llr64 = O.trials(5, 0, 6, fz, snr, lib=O.C)
    llr = llr64.astype(np.float32)
    exp = _oracle(fz, llr, 40)
    got = P.decode_batch(_code(fz), "csfg", llr, 0.9375, 40, ctx=ctx)
    _same(got, exp, f"{snr} dB")


def test_pair_constructed_crossings(ctx, pair):
    """All-zero codeword with the halves at different reliabilities: strong everywhere
    (the first half freezes whole at stage 0 in iteration 1, then the second), strong
    first half + noisy second half, noisy first half + strong second half, a few weak
    rows placed so that the frontier crosses at several stages of a pass."""
    fz = O.construct(N, N // 2, Z0)
    rng = np.random.default_rng(16384)
    frames = []
    frames.append(np.full(N, 6.0))
    frames.append(np.full(N, 0.4))
    a = np.full(N, 8.0); a[N // 2:] = 1.0 + rng.normal(0, 2.0, N // 2); frames.append(a)
    a = 1.0 + rng.normal(0, 2.0, N); a[N // 2:] = 8.0; frames.append(a)
    for shift in (1, 3, 17, 300, 2000):
        a = np.full(N, 5.0) + rng.normal(0, 1.0, N)
        a[N // 2 - shift: N // 2 - shift + 4] = -0.3
        frames.append(a)
    for sc in (2.0, 3.0, 4.0):
        frames.append(sc * (1.0 + rng.normal(0, 1.0, N)))
    llr = np.stack(frames).astype(np.float32)
    for max_iter in (1, 2, 40):
        exp = _oracle(fz, llr, max_iter)
        got = P.decode_batch(_code(fz), "csfg", llr, 0.9375, max_iter, ctx=ctx)
        _same(got, exp, f"max_iter {max_iter}")
    assert (exp["n_events"] > 0).all() and (exp["stop"] == 1).any() and (exp["stop"] == 0).any()


@pytest.mark.parametrize("k,snr", [(12288, 6.0), (16000, 6.0), (16000, 5.0)])
def test_pair_high_rate_completions(ctx, pair, k, snr):
    """High-rate codes at 6 dB: the frontier crosses at the frame's stages 1-2 and
    the second half completes the frame at the frame's stage 0 (the first half's
    whole sweep of that iteration is then not the reference's: it is uncounted)."""
    fz = O.construct(N, k, Z0)
    _, llr64 = O.trials(7, 0, 16, fz, snr, lib=O.C)
    llr = llr64.astype(np.float32)
    exp = _oracle(fz, llr, 40)
    got = P.decode_batch(_code(fz), "csfg", llr, 0.9375, 40, ctx=ctx)
    _same(got, exp, f"k={k} {snr} dB")
    if snr == 6.0:
        assert (exp["stop"] == 2).any()


@pytest.mark.parametrize("rate", [0.125, 0.25, 0.5, 0.875])
def test_pair_random_frozen_sets(ctx, pair, rate):
    rng = np.random.default_rng(int(1000 * rate) + 7)
    k = max(1, int(N * rate))
    fz = np.zeros(N, np.uint8)
    fz[rng.permutation(N)[:N - k]] = 1
    frames = 8
    scale = rng.choice([2.0, 4.0, 8.0, 16.0], size=(frames, 1))
    llr = (scale * (1.0 + rng.normal(0.0, 1.0, size=(frames, N)))).astype(np.float32)
    exp = _oracle(fz, llr, 30)
    got = P.decode_batch(_code(fz), "csfg", llr, 0.9375, 30, ctx=ctx)
    _same(got, exp, f"rate {rate}")


def test_pair_reroute_and_degenerate(ctx, pair):
    """A frame beyond the clamp-free bound is re-routed (the pair skips it together);
    max_iter 0; every row frozen but one."""
    fz = O.construct(N, N // 2, Z0)
    _, llr64 = O.trials(5, 0, 4, fz, 3.0, lib=O.C)
    llr = llr64.astype(np.float32)
    llr[1, 9000] = 1e30
    llr[2, :] *= 1e25
    exp = _oracle(fz, llr, 40)
    got = P.decode_batch(_code(fz), "csfg", llr, 0.9375, 40, ctx=ctx)
    assert ctx.last_launch_info()[1] == 2
    _same(got, exp, "reroute")
    got0 = P.decode_batch(_code(fz), "csfg", llr, 0.9375, 0, ctx=ctx)
    _same(got0, _oracle(fz, llr, 0), "max_iter 0")
    fz1 = np.ones(N, np.uint8); fz1[N - 1] = 0
    l1 = llr[[0, 3]]
    _same(P.decode_batch(_code(fz1), "csfg", l1, 0.9375, 40, ctx=ctx), _oracle(fz1, l1, 40), "k = 1")


def test_pair_equals_one_cta_per_frame(ctx, monkeypatch):
    """Both layouts on the same device-generated frames (config 4's code at 2.5 and
    4.5 dB, high-rate codes whose frames complete at 6 dB): identical per-frame results
    and identical counters."""
    for k, snr in ((N // 2, 2.5), (N // 2, 4.5), (12288, 6.0), (16000, 6.0)):
        code = P.PolarCode.construct(N, k, Z0)
        llr, _, _ = P.generate(code, 5, 0, 2000, snr, ctx=ctx)
        runs = []
        for on in ("1", "0"):
            monkeypatch.setenv("PBP_PAIR", on)
            runs.append(P.decode_batch(code, "csfg", llr, 0.9375, 40, ctx=ctx))
        _same_gpu(runs[0], runs[1], f"{snr} dB")
        cnts = []
        for on in ("1", "0"):
            monkeypatch.setenv("PBP_PAIR", on)
            cnts.append(P.simulate_point(code, "csfg", 5, 0, 2000, snr, 0.9375, 40, ctx=ctx))
        assert cnts[0] == cnts[1], snr


@pytest.mark.parametrize("snr", [2.5, 4.0, 6.0])
def test_pair_n4096_experiment(ctx, monkeypatch, snr):
    """The n = 4096 pair layout (PBP_PAIR=2, an A/B experiment: each CTA holds half of
    the frame in the n = 2048 layout, L(1) of the frame in registers) against the
    oracle and the default layout."""
    n = 4096
    monkeypatch.setenv("PBP_PAIR", "2")
    assert P.lib.pbp_kernel_cluster(n, 2) == 2
    k = n // 2 if snr < 6.0 else 3 * n // 4
    fz = O.construct(n, k, Z0)
    _, llr64 = O.trials(4, 0, 24, fz, snr, lib=O.C)
    llr = llr64.astype(np.float32)
    exp = O.decode_batch("csfg", fz, llr, 0.9375, 60, prec=32)
    got = P.decode_batch(P.PolarCode.from_frozen_mask(n, fz), "csfg", llr, 0.9375, 60, ctx=ctx)
    u = P.unpack_bits(got["u_hat_bits"], n)
    assert np.array_equal(u, exp["u_hat"])
    for f in ("iterations", "pe", "stop", "n_events"):
        assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), f


@pytest.mark.parametrize("kind", ["baseline", "gmatrix"])
def test_pair_gstop_and_fixed_iterations(ctx, pair, monkeypatch, kind):
    """G-stop and fixed-iteration decodes at n = 16384 on the cluster kernel: against
    the oracle on channel frames (2.5-6 dB: some frames stop on the G-check) and
    identical to one CTA per frame on 1000 device-generated frames."""
    fz = O.construct(N, N // 2, Z0)
    for snr in (2.5, 4.0, 6.0):
        _, llr64 = O.trials(5, 0, 4, fz, snr, lib=O.C)
        llr = llr64.astype(np.float32)
        exp = O.decode_batch(kind, fz, llr, 0.9375, 20, prec=32)
        got = P.decode_batch(_code(fz), kind, llr, 0.9375, 20, ctx=ctx)
        _same(got, exp, f"{kind} {snr} dB")
    code = P.PolarCode.construct(N, N // 2, Z0)
    llr, _, _ = P.generate(code, 5, 0, 1000, 4.5, ctx=ctx)
    runs = []
    for on in ("1", "0"):
        monkeypatch.setenv("PBP_PAIR", on)
        runs.append(P.decode_batch(code, kind, llr, 0.9375, 40, ctx=ctx))
    _same_gpu(runs[0], runs[1], kind)
