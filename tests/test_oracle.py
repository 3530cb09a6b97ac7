"""CPU: pin the oracle (C restatement) to the reference.

(a) against the golden fixtures produced by the reference compiled in place
    (tests/golden/make_golden.py), (b) against the compiled reference itself when
    oracle/_ref is present (dev container), (c) against the reference's own
    known-answer tests (/root/reference/proj/tests/*.cpp, cited per test).
"""
import math

import numpy as np
import pytest

import oracle as O
from conftest import load_manifest

Z0 = math.exp(-0.5)
MAN = load_manifest()
SMALL_CASES = [c for c in MAN["cases"] if c["n"] * c["frames"] * c["max_iter"] <= 1024 * 48 * 40]


def _unpack(a, n):
    return np.unpackbits(a, axis=1, bitorder="little")[:, :n]


def test_oracle_built():
    assert O.C is not None, "oracle/_build/liboracle.so missing: make -C oracle"


# ---- construction (test_polar_code.cpp) -------------------------------------

def test_construct_known_answers():
    # test_polar_code.cpp:27-38
    assert list(O.construct(2, 1, 0.5)) == [1, 0]
    assert list(np.flatnonzero(O.construct(8, 4, 0.5))) == [0, 1, 2, 4]
    assert O.construct(8, 8, 0.5).sum() == 0
    with pytest.raises(ValueError):
        O.construct(6, 3, 0.5)
    with pytest.raises(ValueError):
        O.construct(8, 4, 1.0)


def test_construct_matches_golden(golden):
    for key in golden.files:
        if not key.startswith("construct/"):
            continue
        n, k, z = key.split("/")[1].split("_")
        assert np.array_equal(O.construct(int(n), int(k), float(z)), golden[key]), key


def test_polar_transform_known_vectors():
    # test_polar_code.cpp:130-135
    v = np.array([1, 1, 1, 1], np.uint8)
    O.C.orc_polar_transform(v.ctypes.data_as(O._u8p), 4)
    assert list(v) == [0, 0, 0, 1]
    v = np.array([1, 0, 0, 0], np.uint8)
    O.C.orc_polar_transform(v.ctypes.data_as(O._u8p), 4)
    assert list(v) == [1, 0, 0, 0]


# ---- channel (channel.cpp, test_channel.cpp) ----------------------------------

def test_rng_first_draw_and_stream(golden):
    g = O.orc_mt64 = None
    import ctypes as C

    class MT(C.Structure):
        _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]
    O.C.orc_trial_rng.argtypes = [C.POINTER(MT), C.c_uint64, C.c_uint64]
    O.C.orc_mt64_next.argtypes = [C.POINTER(MT)]
    O.C.orc_mt64_next.restype = C.c_uint64
    O.C.orc_gaussian.argtypes = [C.POINTER(MT)]
    O.C.orc_gaussian.restype = C.c_double
    st = MT()
    O.C.orc_trial_rng(C.byref(st), 1, 0)
    assert O.C.orc_mt64_next(C.byref(st)) == 0x884FA46695B1825B
    for key in golden.files:
        if key.startswith("rng/") and key.endswith("/raw"):
            seed, trial = map(int, key.split("/")[1].split("_"))
            st = MT()
            O.C.orc_trial_rng(C.byref(st), seed, trial)
            raw = [O.C.orc_mt64_next(C.byref(st)) for _ in range(16)]
            assert raw == [int(x) for x in golden[key]], key
            st = MT()
            O.C.orc_trial_rng(C.byref(st), seed, trial)
            gs = np.array([O.C.orc_gaussian(C.byref(st)) for _ in range(16)])
            assert np.array_equal(gs, golden[key.replace("raw", "gauss")]), key


def test_noise_variance_reference_points():
    # test_channel.cpp:9-15
    assert O.C.orc_noise_variance(0.0, 0.5) == pytest.approx(1.0)
    assert O.C.orc_noise_variance(3.0, 0.5) == pytest.approx(1.0 / 10 ** 0.3)
    assert O.C.orc_noise_variance(0.0, 1.0) == pytest.approx(0.5)


@pytest.mark.parametrize("case", [c for c in MAN["cases"] if c["frames"] <= 64], ids=lambda c: c["name"])
def test_trial_frames_match_golden(golden, case):
    fz = golden[case["name"] + "/frozen"]
    head = golden[case["name"] + "/llr64_head"]
    info, llr = O.trials(case["seed"], case["first_trial"], head.shape[0], fz, case["ebn0_db"], lib=O.C)
    assert np.array_equal(llr, head)
    assert np.array_equal(info, golden[case["name"] + "/info"][: head.shape[0]])


# ---- decoders -------------------------------------------------------------------

@pytest.mark.parametrize("case", SMALL_CASES, ids=lambda c: c["name"])
def test_oracle_f32_matches_ref32_golden(golden, case):
    name = case["name"]
    fz = golden[name + "/frozen"]
    llr = golden[name + "/llr32"]
    r = O.decode_batch(case["decoder"], fz, llr, 0.9375, case["max_iter"], prec=32, lib=O.C)
    assert np.array_equal(np.packbits(r["u_hat"], axis=1, bitorder="little"), golden[name + "/ref32/u_hat"])
    for f in ("iterations", "pe", "stop", "n_events"):
        assert np.array_equal(r[f], golden[f"{name}/ref32/{f}"]), f


@pytest.mark.parametrize("case", SMALL_CASES[:6], ids=lambda c: c["name"])
def test_oracle_f64_matches_ref64_golden(golden, case):
    name = case["name"]
    fz = golden[name + "/frozen"]
    _, llr = O.trials(case["seed"], case["first_trial"], case["frames"], fz, case["ebn0_db"], lib=O.C)
    r = O.decode_batch(case["decoder"], fz, llr, 0.9375, case["max_iter"], prec=64, lib=O.C)
    assert np.array_equal(np.packbits(r["u_hat"], axis=1, bitorder="little"), golden[name + "/ref64/u_hat"])
    for f in ("iterations", "pe", "stop", "n_events"):
        assert np.array_equal(r[f], golden[f"{name}/ref64/{f}"]), f


def test_event_traces_match_golden(golden):
    for ec in MAN["event_cases"]:
        for i in range(ec["frames"]):
            p = f"{ec['name']}/{i}"
            r = O.decode("csfg", golden[p + "/frozen"], golden[p + "/llr32"], 0.9375, ec["max_iter"], prec=32)
            assert np.array_equal(r["events"], golden[p + "/events"].reshape(-1, 5)), p
            assert [r["iterations"], r["pe"], r["stop"], r["n_events"]] == list(golden[p + "/meta"])


def test_clean_8_4_trace():
    # test_csfg_freeze.cpp:222-246: one iteration, 7 PEs, events (0,0,4), (1,4,2), (2,6,1)
    fz = O.construct(8, 4, 0.5)
    r = O.decode("csfg", fz, np.full(8, 5.0), 0.9375, 40)
    assert r["stop"] == 1 and r["iterations"] == 1 and r["pe"] == 7
    assert [tuple(e[[1, 3, 4]]) for e in r["events"]] == [(0, 0, 4), (1, 4, 2), (2, 6, 1)]
    assert not r["u_hat"].any()


def test_baseline_gmatrix_known_answers():
    # test_bp_core.cpp:185-204
    fz = O.construct(8, 4, 0.5)
    r = O.decode("baseline", fz, np.full(8, 2.0), 0.9375, 40)
    assert (r["iterations"], r["pe"], r["stop"]) == (40, 480, 0)
    r = O.decode("gmatrix", fz, np.full(8, 2.0), 0.9375, 40)
    assert (r["iterations"], r["pe"], r["stop"]) == (1, 12, 1)


def test_pe_update_worked_example():
    # test_bp_core.cpp:23-37 and :93-100 (clamp)
    out = np.zeros(4)
    O.C.orc_pe_update_f64(np.array([2.0, -3.0, 1.0, 0.5]).ctypes.data_as(O._f64p), 0.9375,
                          out.ctypes.data_as(O._f64p))
    assert out[0] == pytest.approx(-1.875) and out[3] == pytest.approx(1.4375)
    assert out[1] == pytest.approx(-3.0 + 0.9375) and out[2] == pytest.approx(-0.9375)
    O.C.orc_pe_update_f64(np.full(4, 1e30).ctypes.data_as(O._f64p), 1.0, out.ctypes.data_as(O._f64p))
    assert out[1] == 1e30


@pytest.mark.skipif(O.REF is None, reason="reference build absent (GPU box)")
def test_oracle_vs_reference_random_llrs():
    rng = np.random.default_rng(123)
    for n in (8, 32, 256):
        fz = O.construct(n, n // 2, 0.5)
        llr = rng.normal(1.0, 2.0, size=(40, n))
        llr[:, ::7] = 0.0  # exact zeros (sgn(0) = +1 path)
        for kind in ("baseline", "gmatrix", "csfg"):
            for prec in (32, 64):
                a = O.decode_batch(kind, fz, llr, 0.9375, 20, prec=prec, lib=O.REF)
                b = O.decode_batch(kind, fz, llr, 0.9375, 20, prec=prec, lib=O.C)
                for f in a:
                    assert np.array_equal(a[f], b[f]), (n, kind, prec, f)
