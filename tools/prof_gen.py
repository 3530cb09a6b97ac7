"""Frame generation alone (decode_trial's channel, on the device): time per 10^5 frames.
   python tools/prof_gen.py [--n 1024] [--frames 100000] [--reps 3] [--ebn0 3.0]"""
import argparse, ctypes as C, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_04979_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--frames", type=int, default=100000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--ebn0", type=float, default=3.0)
a = ap.parse_args()
ctx = P.Context(0)
code = P.PolarCode.construct(a.n, a.n // 2, math.exp(-0.5))
cs = code.c_struct()
nw = max(1, a.n // 32)
llr = torch.empty((a.frames, a.n), dtype=torch.float32, device="cuda")
u = torch.empty((a.frames, nw), dtype=torch.int32, device="cuda")
st = torch.cuda.ExternalStream(ctx.stream())
for r in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    P._check(P.lib.pbp_generate_device(ctx.handle, C.byref(cs), C.c_uint64(2), 0, a.frames, a.ebn0, 0,
                                       P._abi.f32p(llr.data_ptr()), None, P._abi.u32p(u.data_ptr()), None))
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"rep {r}: {ms:.3f} ms for {a.frames} frames ({a.frames / ms / 1e3:.2f} Mframes/s)")
