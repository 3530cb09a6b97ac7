"""Where does the host-API decode time go? python tools/e2e_probe.py [--frames F] [--n N]
Times (wall clock, after warm-up): the device decode alone, the pinned H2D copy alone,
and pbp_decode_batch (pipelined host call) on the same frames."""
import argparse, ctypes as C, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_04979_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=100000)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--ebn0", type=float, default=3.0)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
ctx = P.Context(0)
n, F = a.n, a.frames
code = P.PolarCode.construct(n, n // 2, math.exp(-0.5))
cs = code.c_struct()
nw = max(1, n // 32)
llr = torch.empty((F, n), dtype=torch.float32, device="cuda")
u = torch.empty((F, nw), dtype=torch.int32, device="cuda")
P._check(P.lib.pbp_generate_device(ctx.handle, C.byref(cs), C.c_uint64(2), 0, F, a.ebn0, 0,
                                   P._abi.f32p(llr.data_ptr()), None, P._abi.u32p(u.data_ptr()), None))
ctx.synchronize()
host = torch.empty((F, n), dtype=torch.float32, pin_memory=True)
host.copy_(llr)
outs = [torch.empty((F, nw), dtype=torch.int32, pin_memory=True), torch.empty(F, dtype=torch.int32, pin_memory=True),
        torch.empty(F, dtype=torch.int64, pin_memory=True), torch.empty(F, dtype=torch.uint8, pin_memory=True),
        torch.empty(F, dtype=torch.int32, pin_memory=True)]
fo = P._abi.PbpFrameOut(P._abi.u32p(outs[0].data_ptr()), P._abi.i32p(outs[1].data_ptr()),
                        P._abi.i64p(outs[2].data_ptr()), P._abi.u8p(outs[3].data_ptr()),
                        P._abi.i32p(outs[4].data_ptr()))
dout = [torch.empty((F, nw), dtype=torch.int32, device="cuda"), torch.empty(F, dtype=torch.int32, device="cuda"),
        torch.empty(F, dtype=torch.int64, device="cuda"), torch.empty(F, dtype=torch.uint8, device="cuda"),
        torch.empty(F, dtype=torch.int32, device="cuda")]
dfo = P._abi.PbpFrameOut(P._abi.u32p(dout[0].data_ptr()), P._abi.i32p(dout[1].data_ptr()),
                         P._abi.i64p(dout[2].data_ptr()), P._abi.u8p(dout[3].data_ptr()),
                         P._abi.i32p(dout[4].data_ptr()))
dst = torch.empty_like(llr)


def t(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3, sorted(ts)[len(ts) // 2] * 1e3


def dev():
    P._check(P.lib.pbp_decode_batch_device(ctx.handle, C.byref(cs), 2, P._abi.f32p(llr.data_ptr()), F, 0.9375, 40,
                                           C.byref(dfo), None))
    ctx.synchronize()


def h2d():
    dst.copy_(host, non_blocking=True)


def e2e():
    P._check(P.lib.pbp_decode_batch(ctx.handle, C.byref(cs), 2, P._abi.f32p(host.data_ptr()), F, 0.9375, 40,
                                    C.byref(fo)))


for name, fn in (("device decode", dev), ("pinned H2D", h2d), ("pbp_decode_batch", e2e)):
    mn, md = t(fn)
    print(f"{name:18s} min {mn:7.2f} ms  median {md:7.2f} ms  ({F * (n // 2) / (md / 1e3) / 1e9:.3f} Gbit/s info)")
