"""Profiling driver: decode one Eb/N0 point of config 2 through the device C ABI.
   python tools/prof_decode.py [--frames F] [--ebn0 X] [--kind csfg] [--reps R] [--n 1024]"""
import argparse, ctypes as C, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_04979_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=20000)
ap.add_argument("--ebn0", type=float, default=3.0)
ap.add_argument("--kind", default="csfg")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--generic", action="store_true", help="force the generic kernel")
a = ap.parse_args()
ctx = P.Context(0)
if a.generic:
    ctx.force_generic(True)
code = P.PolarCode.construct(a.n, a.n // 2, math.exp(-0.5))
cs = code.c_struct()
nw = max(1, a.n // 32)
llr = torch.empty((a.frames, a.n), dtype=torch.float32, device="cuda")
u = torch.empty((a.frames, nw), dtype=torch.int32, device="cuda")
cnt = torch.zeros(10, dtype=torch.int64, device="cuda")
P._check(P.lib.pbp_generate_device(ctx.handle, C.byref(cs), C.c_uint64(2), 0, a.frames, a.ebn0, 0,
                                   P._abi.f32p(llr.data_ptr()), None, P._abi.u32p(u.data_ptr()), None))
ctx.synchronize()
kind = P.DecoderKind.parse(a.kind)
_sm, _w = C.c_int32(), C.c_int32()
P.lib.pbp_kernel_info(a.n, kind, C.byref(_sm), C.byref(_w))
print(f"warp kernel: {_sm.value} B shared, {_w.value} warps/SM")
for r in range(a.reps):
    cnt.zero_()
    torch.cuda.synchronize()
    t = time.perf_counter()
    P._check(P.lib.pbp_decode_count_device(ctx.handle, C.byref(cs), kind, P._abi.f32p(llr.data_ptr()),
                                           P._abi.u32p(u.data_ptr()), a.frames, 0.9375, 40,
                                           P._abi.i64p(cnt.data_ptr()), None))
    ctx.synchronize()
    dt = time.perf_counter() - t
    c = cnt.cpu().tolist()
    print(f"rep {r}: {dt*1e3:.2f} ms  {a.frames/dt/1e6:.3f} Mframes/s  avg iters {c[3]/c[0]:.2f}  "
          f"PE/s {c[5]/dt:.3e}  ({c[5]*9/dt/1e12:.2f} TOP/s)")
if hasattr(P.lib, "pbp_prof_read") and os.environ.get("PBP_LIB"):
    # library built with -DPBP_PROF_SECTIONS: per-warp clock64 split of the last rep
    buf = (C.c_ulonglong * 16)()
    P.lib.pbp_prof_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    P.lib.pbp_prof_read(buf, 1)
    cnt.zero_()
    P._check(P.lib.pbp_decode_count_device(ctx.handle, C.byref(cs), kind, P._abi.f32p(llr.data_ptr()),
                                           P._abi.u32p(u.data_ptr()), a.frames, 0.9375, 40,
                                           P._abi.i64p(cnt.data_ptr()), None))
    ctx.synchronize()
    P.lib.pbp_prof_read(buf, 1)
    names = ["stage math", "snapshot", "walk0/resat", "walk", "commits", "gcheck", "frame load", "iter loop"]
    tot = buf[7] + buf[6]
    its = cnt.cpu().tolist()[3]
    for i, nm in enumerate(names):
        print(f"  {nm:12s} {buf[i]/tot*100:6.1f}%  {buf[i]/its:9.1f} clk/iter")
    if buf[15]:  # warp-specialised kernel: sweep-warp slots above (5 = wait for B, 4 = export), bookkeeping here
        for i, nm in enumerate(["wait C", "walk_tm", "apply_tm", "gcheck", "", "", "", "total"]):
            if nm:
                print(f"  bk {nm:9s} {buf[8 + i]/buf[15]*100:6.1f}%  {buf[8 + i]/its:9.1f} clk/iter")
