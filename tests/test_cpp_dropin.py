"""The C++ drop-in (include/polarbp/*.hpp over libpbp.so): compile the reference-style
test program against the headers and run it (host cases on CPU, all cases on GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1505_04979_b200", "_lib")


def _build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    subprocess.run(["g++", "-O1", "-std=c++20", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-L", LIBDIR, "-lpbp",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_dropin_host_cases(tmp_path):
    r = subprocess.run([_build(tmp_path), "--cpu-only"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_dropin_all_cases(tmp_path):
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
