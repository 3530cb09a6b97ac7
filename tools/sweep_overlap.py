"""Config-2 sweep on the device: 7 Eb/N0 points decoded back to back on one stream vs
round-robin over three streams (tails of one point overlap the next).
   python tools/sweep_overlap.py [--frames F] [--streams 3]"""
import argparse, ctypes as C, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_04979_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=100000)
ap.add_argument("--streams", type=int, default=3)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
SNRS = [1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0]
ctx = P.Context(0)
dev = torch.device("cuda", 0)
code = P.PolarCode.construct(1024, 512, math.exp(-0.5))
cs = code.c_struct()
F = a.frames
llr = torch.empty((len(SNRS), F, 1024), dtype=torch.float32, device=dev)
u = torch.empty((len(SNRS), F, 32), dtype=torch.int32, device=dev)
for i, s in enumerate(SNRS):
    P._check(P.lib.pbp_generate_device(ctx.handle, C.byref(cs), C.c_uint64(2), 0, F, s, 0,
                                       P._abi.f32p(llr[i].data_ptr()), None, P._abi.u32p(u[i].data_ptr()), None))
ctx.synchronize()
cnt = torch.zeros((len(SNRS), 10), dtype=torch.int64, device=dev)
streams = [torch.cuda.Stream(dev) for _ in range(a.streams)]


def sweep(nst):
    cnt.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for st in streams[1:nst]:
        st.wait_event(e0)
    for i in range(len(SNRS)):
        st = streams[i % nst]
        P._check(P.lib.pbp_decode_count_device(ctx.handle, C.byref(cs), 2, P._abi.f32p(llr[i].data_ptr()),
                                               P._abi.u32p(u[i].data_ptr()), F, 0.9375, 40,
                                               P._abi.i64p(cnt[i].data_ptr()), C.c_void_p(st.cuda_stream)))
    for st in streams[1:nst]:
        ev = torch.cuda.Event()
        ev.record(st)
        streams[0].wait_event(ev)
    e1.record(streams[0])
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), cnt.sum(0).tolist()


for nst in (1, a.streams):
    sweep(nst)
    ts = []
    for _ in range(a.reps):
        t, c = sweep(nst)
        ts.append(t)
    print(f"{nst} stream(s): {min(ts):.2f} ms per sweep  frames {c[0]}  sum_pe {c[5]}  "
          f"{len(SNRS) * F * 512 / (min(ts) / 1e3) / 1e9:.3f} Gbit/s")
