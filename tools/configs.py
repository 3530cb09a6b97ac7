"""Every workload of BASELINE.json / SURVEY.md 8(d) on one GPU, at its full frame count.

   python tools/configs.py [--configs 0,1,2,3,4] [--scale 1.0] > profiles/<tag>_configs.jsonl

One JSON line per (config, n, Eb/N0): decode-only device time (frames generated on the
device beforehand, chunked so no chunk exceeds 2^28 LLRs), decoded info bits/s, PE
activations/s and the fraction of the fp32 ALU roofline (9 ops per PE,
148 x 128 x sm_max_mhz), average iterations, FER/BER, freeze events per frame, and the
same point generated + decoded on the device (simulate_point_device) as gen_decode_bits_s,
and e2e_bits_per_s: pbp_decode_batch from pinned host LLRs (wall clock, copies included).
Config 4's multi-GPU sharding is bench.py's job; here it is the single-GPU rate per n."""
import argparse, ctypes as C, json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_04979_b200 as P

SNRS = [1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0]
CONFIGS = {  # decoder, n list, Eb/N0 list, max_iter, frames per point, seed
    0: ("baseline", [1024], [3.0], 40, 100_000, 1),
    1: ("gmatrix", [1024], SNRS, 40, 100_000, 2),
    2: ("csfg", [1024], SNRS, 40, 100_000, 2),
    3: ("csfg", [4096], [2.5], 60, 200_000, 4),
    4: ("csfg", [256, 1024, 4096, 16384], [2.5], 40, 1_000_000, 5),
}
ALPHA, Z0 = 0.9375, math.exp(-0.5)


def peaks():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,1,2,3,4")
    ap.add_argument("--scale", type=float, default=1.0, help="fraction of each point's frames")
    a = ap.parse_args()
    ctx = P.Context(0)
    dev = torch.device("cuda", 0)
    props = torch.cuda.get_device_properties(0)
    mhz = float(peaks().get("sm_max_mhz", 1965))
    peak_pe = props.multi_processor_count * 128 * mhz * 1e6 / 9.0
    stream = torch.cuda.Stream(dev)  # explicit: a null stream would select the context's own
    for cid in [int(x) for x in a.configs.split(",")]:
        kind_name, ns, snrs, max_iter, frames, seed = CONFIGS[cid]
        kind = P.DecoderKind.parse(kind_name)
        frames = max(1, int(frames * a.scale))
        for n in ns:
            code = P.PolarCode.construct(n, n // 2, Z0)
            cs = code.c_struct()
            nw = max(1, n // 32)
            chunk = min(frames, max(1, (1 << 28) // n))
            llr = torch.empty((chunk, n), dtype=torch.float32, device=dev)
            u = torch.empty((chunk, nw), dtype=torch.int32, device=dev)
            # untimed warm-up: the first decode of a code length sizes the context's buffers
            wcnt = torch.zeros(10, dtype=torch.int64, device=dev)
            P._check(P.lib.pbp_generate_device(ctx.handle, C.byref(cs), C.c_uint64(seed), 0, chunk, snrs[0], 0,
                                               P._abi.f32p(llr.data_ptr()), None, P._abi.u32p(u.data_ptr()),
                                               C.c_void_p(stream.cuda_stream)))
            P._check(P.lib.pbp_decode_count_device(ctx.handle, C.byref(cs), kind, P._abi.f32p(llr.data_ptr()),
                                                   P._abi.u32p(u.data_ptr()), chunk, ALPHA, max_iter,
                                                   P._abi.i64p(wcnt.data_ptr()), C.c_void_p(stream.cuda_stream)))
            for _ in range(3):  # simulate_point rotates over the context's three launch slots
                P._check(P.lib.pbp_simulate_point_device(ctx.handle, C.byref(cs), kind, C.c_uint64(seed), 0, chunk,
                                                         snrs[0], 0, ALPHA, max_iter, P._abi.i64p(wcnt.data_ptr()),
                                                         C.c_void_p(stream.cuda_stream)))
            stream.synchronize()
            for snr in snrs:
                cnt = torch.zeros(10, dtype=torch.int64, device=dev)
                torch.cuda.synchronize()
                ms = 0.0
                for first in range(0, frames, chunk):
                    cnt_f = min(chunk, frames - first)
                    P._check(P.lib.pbp_generate_device(ctx.handle, C.byref(cs), C.c_uint64(seed), first, cnt_f,
                                                       snr, 0, P._abi.f32p(llr.data_ptr()), None,
                                                       P._abi.u32p(u.data_ptr()), C.c_void_p(stream.cuda_stream)))
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    P._check(P.lib.pbp_decode_count_device(ctx.handle, C.byref(cs), kind,
                                                           P._abi.f32p(llr.data_ptr()), P._abi.u32p(u.data_ptr()),
                                                           cnt_f, ALPHA, max_iter, P._abi.i64p(cnt.data_ptr()),
                                                           C.c_void_p(stream.cuda_stream)))
                    e1.record(stream)
                    e1.synchronize()
                    ms += e0.elapsed_time(e1)
                stream.synchronize()
                c = cnt.tolist()
                # generation + decode on the device, one call per chunk
                cnt2 = torch.zeros(10, dtype=torch.int64, device=dev)
                torch.cuda.synchronize()
                g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                g0.record(stream)
                for first in range(0, frames, chunk):
                    P._check(P.lib.pbp_simulate_point_device(ctx.handle, C.byref(cs), kind, C.c_uint64(seed), first,
                                                             min(chunk, frames - first), snr, 0, ALPHA, max_iter,
                                                             P._abi.i64p(cnt2.data_ptr()),
                                                             C.c_void_p(stream.cuda_stream)))
                g1.record(stream)
                g1.synchronize()
                gms = g0.elapsed_time(g1)
                stream.synchronize()
                assert cnt2.tolist() == c, (c, cnt2.tolist())
                # end to end through the host C ABI: pinned host LLRs in, per-frame results
                # out (one staging chunk of generated frames; copies and decode pipelined
                # by the library)
                nf = min(chunk, frames)
                host = torch.empty((nf, n), dtype=torch.float32, pin_memory=True)
                host.copy_(llr[:nf])
                outs = [torch.empty(x, dtype=t, pin_memory=True) for x, t in
                        (((nf, nw), torch.int32), (nf, torch.int32), (nf, torch.int64), (nf, torch.uint8), (nf, torch.int32))]
                fo = P._abi.PbpFrameOut(P._abi.u32p(outs[0].data_ptr()), P._abi.i32p(outs[1].data_ptr()),
                                        P._abi.i64p(outs[2].data_ptr()), P._abi.u8p(outs[3].data_ptr()),
                                        P._abi.i32p(outs[4].data_ptr()))
                call = lambda: P._check(P.lib.pbp_decode_batch(ctx.handle, C.byref(cs), kind, P._abi.f32p(host.data_ptr()),
                                                               nf, ALPHA, max_iter, C.byref(fo)))
                call()
                t0 = time.perf_counter()
                call()
                e2e_s = time.perf_counter() - t0
                f = c[0]
                pe_s = c[5] / (ms / 1e3)
                print(json.dumps({
                    "config": cid, "decoder": kind_name, "n": n, "k": n // 2, "ebn0_db": snr,
                    "max_iter": max_iter, "seed": seed, "frames": f, "decode_ms": round(ms, 3),
                    "frames_per_s": round(f / (ms / 1e3), 1), "info_bits_per_s": round(f * (n // 2) / (ms / 1e3), 1),
                    "pe_per_s": round(pe_s, 1), "roofline_frac": round(pe_s / peak_pe, 4),
                    "avg_iters": round(c[3] / f, 4), "avg_pe": round(c[5] / f, 1),
                    "fer": c[2] / f, "ber": c[1] / (f * (n // 2)), "events_per_frame": round(c[6] / f, 3),
                    "stops": {"max_iter": c[7], "gmatrix": c[8], "complete": c[9]},
                    "gen_decode_ms": round(gms, 3),
                    "gen_decode_bits_per_s": round(f * (n // 2) / (gms / 1e3), 1),
                    "e2e_bits_per_s": round(nf * (n // 2) / e2e_s, 1), "e2e_frames": nf,
                    "kernel_path": P.lib.pbp_kernel_path(n),
                }), flush=True)


if __name__ == "__main__":
    main()
