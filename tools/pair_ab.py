"""A/B of the n = 16384 csfg layouts: 2-CTA cluster per frame (PBP_PAIR=1) against one
CTA per frame (PBP_PAIR=0), decode-only device time on the same device-generated frames
(config 4: seed 5, max_iter 40), counters compared.

   python tools/pair_ab.py [--frames 16384] [--snrs 2.5,4.5] [--reps 2]
"""
import argparse, ctypes as C, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_04979_b200 as P

ALPHA, Z0 = 0.9375, math.exp(-0.5)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--frames", type=int, default=16384)
    ap.add_argument("--snrs", default="2.5,4.5")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--max-iter", type=int, default=40)
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--on", default="1", help="PBP_PAIR value of the pair arm (2: also n = 4096)")
    a = ap.parse_args()
    n = a.n
    ctx = P.Context(0)
    dev = torch.device("cuda", 0)
    mhz = 1965.0
    peak_pe = torch.cuda.get_device_properties(0).multi_processor_count * 128 * mhz * 1e6 / 9.0
    stream = torch.cuda.Stream(dev)
    code = P.PolarCode.construct(n, n // 2, Z0)
    cs = code.c_struct()
    nw = n // 32
    llr = torch.empty((a.frames, n), dtype=torch.float32, device=dev)
    u = torch.empty((a.frames, nw), dtype=torch.int32, device=dev)
    for snr in [float(x) for x in a.snrs.split(",")]:
        P._check(P.lib.pbp_generate_device(ctx.handle, C.byref(cs), C.c_uint64(a.seed), 0, a.frames, snr, 0,
                                           P._abi.f32p(llr.data_ptr()), None, P._abi.u32p(u.data_ptr()),
                                           C.c_void_p(stream.cuda_stream)))
        stream.synchronize()
        res = {}
        for rep in range(a.reps):
            for on in (a.on, "0"):
                os.environ["PBP_PAIR"] = on
                cnt = torch.zeros(10, dtype=torch.int64, device=dev)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                P._check(P.lib.pbp_decode_count_device(ctx.handle, C.byref(cs), 2, P._abi.f32p(llr.data_ptr()),
                                                       P._abi.u32p(u.data_ptr()), a.frames, ALPHA, a.max_iter,
                                                       P._abi.i64p(cnt.data_ptr()), C.c_void_p(stream.cuda_stream)))
                e1.record(stream)
                e1.synchronize()
                ms = e0.elapsed_time(e1)
                c = cnt.tolist()
                if rep == a.reps - 1 or on not in res:
                    res[on] = (ms, c)
        (m1, c1), (m0, c0) = res[a.on], res["0"]
        print(json.dumps({"n": n, "ebn0_db": snr, "frames": a.frames, "pair_ms": round(m1, 3), "cta_ms": round(m0, 3),
                          "speedup": round(m0 / m1, 3), "counters_equal": c1 == c0,
                          "pair_roofline_frac": round(c1[5] / (m1 / 1e3) / peak_pe, 4),
                          "cta_roofline_frac": round(c0[5] / (m0 / 1e3) / peak_pe, 4),
                          "avg_iters": c1[3] / c1[0], "fer": c1[2] / c1[0],
                          "stops": c1[7:10], "cluster": P.lib.pbp_kernel_cluster(n, 2)}), flush=True)


if __name__ == "__main__":
    main()
