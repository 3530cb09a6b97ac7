"""In-tree build of libpbp.so (CUDA kernels for sm_100a + C ABI + C++ host API).

Run as ``python paper_1505_04979_b200/build.py`` or via ``__graft_entry__.build()`` (not with
``-m``: importing the package loads the library it builds).
Objects go to build/, the shared library to paper_1505_04979_b200/_lib/ so it
travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", os.environ.get("PBP_OBJ_SUBDIR", "obj"))
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, os.environ.get("PBP_LIB_NAME", "libpbp.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: the reference rounds every product and sum separately
# (src/bp_core.cpp:21-30); ptxas would otherwise fuse mul.rn.f32x2 + add.rn.f32x2
# into FFMA2 (observed), changing decisions after ~20 iterations.
NVFLAGS = ARCH + os.environ.get("PBP_NVCC_EXTRA", "").split() + ["-O3", "-fmad=false", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
                  "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
                  "-I", os.path.join(ROOT, "include")]
CXXFLAGS = ["-O3", "-std=c++20", "-fPIC", "-I", os.path.join(ROOT, "include"),
            "-I", "/usr/local/cuda/include"]


def _sources():
    cu = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    cpp = sorted(f for f in os.listdir(CSRC) if f.endswith(".cpp"))
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".hpp"))]
    deps += [os.path.join(ROOT, "include", "pbp.h")]
    inc = os.path.join(ROOT, "include", "polarbp")
    if os.path.isdir(inc):
        deps += [os.path.join(inc, f) for f in os.listdir(inc)]
    return cu, cpp, deps


def _stale(obj, src, deps, flags):
    """Rebuild when a source or header is newer, or the compile command changed
    (a .flags stamp next to the object records the flags it was built with)."""
    stamp = obj + ".flags"
    if not os.path.exists(obj) or not os.path.exists(stamp):
        return True
    with open(stamp) as f:
        if f.read() != " ".join(flags):
            return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src] + deps)


def _stamp(cmd):
    obj = cmd[cmd.index("-o") + 1]
    flags = cmd[1:cmd.index("-c")]
    with open(obj + ".flags", "w") as f:
        f.write(" ".join(flags))


def build(verbose=False, jobs=None):
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    cu, cpp, deps = _sources()
    cmds, objs = [], []
    for f in cu:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        objs.append(obj)
        if _stale(obj, src, deps, NVFLAGS):
            cmds.append([NVCC] + NVFLAGS + ["-c", src, "-o", obj])
    for f in cpp:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        objs.append(obj)
        if _stale(obj, src, deps, CXXFLAGS):
            cmds.append(["g++"] + CXXFLAGS + ["-c", src, "-o", obj])
    procs = []
    for c in cmds:
        if verbose:
            print(" ".join(c), flush=True)
        procs.append((c, subprocess.Popen(c, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for c, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(out)
        else:
            _stamp(c)
            if verbose and out.strip():
                print(out)
    if failed:
        raise RuntimeError("libpbp build failed")
    if cmds or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        link = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs
        if verbose:
            print(" ".join(link), flush=True)
        subprocess.run(link, check=True)
    build_cli(verbose)
    return LIB


CLI_SRC = os.path.join(PKG, "cli", "polarbp_cli.cpp")
CLI = os.path.join(LIB_DIR, "polarbp")


def build_cli(verbose=False):
    """The `polarbp` command (reference tools/polarbp_main.cpp) linked to libpbp.so."""
    if os.environ.get("PBP_LIB_NAME"):  # experiment builds: library only
        return None
    deps = [CLI_SRC, LIB] + [os.path.join(ROOT, "include", "polarbp", f)
                             for f in os.listdir(os.path.join(ROOT, "include", "polarbp"))]
    if os.path.exists(CLI) and all(os.path.getmtime(d) <= os.path.getmtime(CLI) for d in deps):
        return CLI
    cmd = ["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"), CLI_SRC, "-L", LIB_DIR, "-lpbp",
           "-Wl,-rpath,$ORIGIN", "-o", CLI]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return CLI


if __name__ == "__main__":
    print(build(verbose=True))
