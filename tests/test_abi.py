"""CPU: the C-ABI library loads, exports every symbol include/pbp.h declares, and its
host-side helpers agree with the oracle. No compute call needs a GPU here."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1505_04979_b200 as P
from paper_1505_04979_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "pbp.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pbp_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_abi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_abi.SIGNATURES), set(syms) ^ set(_abi.SIGNATURES)


def test_version_and_paths():
    assert P.lib.pbp_version() == 1
    assert P.lib.pbp_kernel_path(1024) == 1 and P.lib.pbp_kernel_path(128) == 1
    assert P.lib.pbp_kernel_path(4096) == 2 and P.lib.pbp_kernel_path(16384) == 2
    assert P.lib.pbp_kernel_path(64) == 0 and P.lib.pbp_kernel_path(32768) == 0


@pytest.mark.parametrize("n,k,z", [(2, 1, 0.5), (8, 4, 0.5), (64, 32, 0.5), (1024, 512, math.exp(-0.5)),
                                   (16384, 8192, math.exp(-0.5)), (128, 37, 0.3)])
def test_construct_matches_oracle(n, k, z):
    assert np.array_equal(P.PolarCode.construct(n, k, z).frozen, O.construct(n, k, z))


def test_construct_errors_match_reference_messages():
    # polar_code.cpp:54-55 and :31-32 messages, std::invalid_argument -> ValueError
    with pytest.raises(ValueError, match="construct: n must be a power of two"):
        P.PolarCode.construct(6, 3)
    with pytest.raises(ValueError, match="construct: k must satisfy 1 <= k <= n"):
        P.PolarCode.construct(8, 9)
    with pytest.raises(ValueError, match=r"design_z must be in \(0,1\)"):
        P.PolarCode.construct(8, 4, 1.0)


def test_transform_encode_vs_oracle():
    rng = np.random.default_rng(5)
    for m in range(0, 11):
        n = 1 << m
        v = rng.integers(0, 2, n).astype(np.uint8)
        a = P.polar_transform(v)
        b = v.copy()
        O.C.orc_polar_transform(b.ctypes.data_as(O._u8p), n)
        assert np.array_equal(a, b)
        assert np.array_equal(P.polar_transform(a), v)  # involution
    code = P.PolarCode.construct(8, 4, 0.5)
    cw = P.encode(code, [1, 0, 1, 1])
    assert list(cw.u) == [0, 0, 0, 1, 0, 0, 1, 1]  # test_polar_code.cpp:114-119
    assert list(P.extract_info_bits(code, cw.u)) == [1, 0, 1, 1]
    with pytest.raises(ValueError):
        P.encode(code, [1, 0, 1])
    with pytest.raises(ValueError):
        P.polar_transform([1, 0, 1])


def test_noise_variance():
    assert P.noise_variance(3.0, 0.5) == O.C.orc_noise_variance(3.0, 0.5)
    with pytest.raises(ValueError):
        P.noise_variance(0.0, 0.0)
    with pytest.raises(ValueError):
        P.noise_variance(float("inf"), 0.5)


def test_bit_packing_roundtrip():
    rng = np.random.default_rng(1)
    for n in (1, 8, 33, 1024):
        b = rng.integers(0, 2, (3, n)).astype(np.uint8)
        assert np.array_equal(P.unpack_bits(P.pack_bits(b), n), b)


@pytest.mark.skipif(P.device_count() > 0, reason="host has a GPU")
def test_no_cpu_fallback():
    with pytest.raises(Exception, match="no CUDA device"):
        P.Context()
