"""CPU: SASS-level guards on the built kernels (cuobjdump on libpbp.so).

The reference rounds every product and every sum separately (src/bp_core.cpp:21-30),
so no decoder kernel may contain a fused multiply-add with a live addend: ptxas fuses
mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under -fmad=false, which changed decisions
after ~20 iterations before products were written as fma(alpha, m, RZ)."""
import os
import re
import shutil
import subprocess

import pytest

from paper_1505_04979_b200 import _abi

CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"


def _sass():
    return subprocess.run([CUOBJDUMP, "-sass", _abi.LIB_PATH], capture_output=True, text=True, check=True).stdout


def _functions(sass):
    cur, out = None, {}
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = []
        elif cur:
            out[cur].append(line)
    return out


@pytest.mark.skipif(not os.path.exists(CUOBJDUMP), reason="cuobjdump absent")
def test_decoder_kernels_have_no_fused_multiply_add():
    fns = _functions(_sass())
    dec = {k: v for k, v in fns.items()
           if "bp_warp_kernel" in k or "bp_generic_kernel" in k or "bp_cta_kernel" in k or "bp_pair_kernel" in k}
    assert len(dec) >= 13 and any("bp_cta_kernel" in k for k in dec) and any("bp_pair_kernel" in k for k in dec)
    for name, lines in dec.items():
        for ln in lines:
            m = re.search(r"\bFFMA2?\b[^;]*;", ln)
            if m:
                ops = m.group(0).rstrip(";").split(",")
                assert ops[-1].strip().startswith("RZ"), f"{name}: fused multiply-add {m.group(0)}"


@pytest.mark.skipif(not os.path.exists(CUOBJDUMP), reason="cuobjdump absent")
def test_fast_kernel_uses_packed_fp32_and_xorsign_min():
    fns = _functions(_sass())
    k = [v for n, v in fns.items() if "bp_warp_kernelILi10ELi2E" in n][0]
    text = "\n".join(k)
    assert "FADD2" in text and "FFMA2" in text
    assert re.search(r"FMNMX[^;]*XORSIGN", text) or "FMNMX" in text


@pytest.mark.skipif(not os.path.exists(CUOBJDUMP), reason="cuobjdump absent")
def test_pair_kernel_uses_cluster_barrier_and_tmem():
    """The n = 16384 cluster kernel synchronises the pair with the cluster barrier
    (barrier.cluster -> UCGABAR_ARV / UCGABAR_WAIT; its DSMEM stores are generic
    ST.E to cluster-window addresses) and keeps its inner levels, R(0) and L(1) in
    tensor memory (STTM / LDTM)."""
    fns = _functions(_sass())
    k = [v for n, v in fns.items() if "bp_pair_kernelILi13ELi2E" in n]
    assert k, "bp_pair_kernel<13, 2> missing"
    text = "\n".join(k[0])
    assert "UCGABAR_ARV" in text and "UCGABAR_WAIT" in text
    assert "STTM" in text and "LDTM" in text
    assert re.search(r"\bST\.E\b", text)
