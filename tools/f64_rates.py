"""fp64 decode throughput on the GPU (the reference's shipped double arithmetic, generic
kernel) for configs 0-2 at n = 1024, next to the fp32 fast path on the same frames.

   python tools/f64_rates.py [--frames 20000] > profiles/<tag>_f64_rates.jsonl

Frames: decode_trial's channel generated on the device (fp64 LLRs and their fp32 cast);
decode-only device time (CUDA events on the call's stream), outputs device-resident."""
import argparse, ctypes as C, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_04979_b200 as P

ALPHA, Z0 = 0.9375, math.exp(-0.5)
POINTS = [(0, "baseline", 3.0, 1), (1, "gmatrix", 1.0, 2), (1, "gmatrix", 3.0, 2), (2, "csfg", 1.0, 2), (2, "csfg", 3.0, 2)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=20000)
    a = ap.parse_args()
    n, k, F = 1024, 512, a.frames
    ctx = P.Context(0)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    code = P.PolarCode.construct(n, k, Z0)
    cs = code.c_struct()
    nw = n // 32
    l32 = torch.empty((F, n), dtype=torch.float32, device=dev)
    l64 = torch.empty((F, n), dtype=torch.float64, device=dev)
    u = torch.empty((F, nw), dtype=torch.int32, device=dev)
    outs = [torch.empty((F, nw), dtype=torch.int32, device=dev), torch.empty(F, dtype=torch.int32, device=dev),
            torch.empty(F, dtype=torch.int64, device=dev), torch.empty(F, dtype=torch.uint8, device=dev),
            torch.empty(F, dtype=torch.int32, device=dev)]
    fo = P._abi.PbpFrameOut(P._abi.u32p(outs[0].data_ptr()), P._abi.i32p(outs[1].data_ptr()),
                            P._abi.i64p(outs[2].data_ptr()), P._abi.u8p(outs[3].data_ptr()),
                            P._abi.i32p(outs[4].data_ptr()))
    for cfg, kind_name, ebn0, seed in POINTS:
        kind = P.DecoderKind.parse(kind_name)
        P._check(P.lib.pbp_generate_device(ctx.handle, C.byref(cs), C.c_uint64(seed), 0, F, ebn0, 0,
                                           P._abi.f32p(l32.data_ptr()), C.cast(l64.data_ptr(), C.POINTER(C.c_double)),
                                           P._abi.u32p(u.data_ptr()), C.c_void_p(st.cuda_stream)))
        st.synchronize()
        res = {}
        for prec in ("f64", "f32"):
            def call():
                if prec == "f64":
                    P._check(P.lib.pbp_decode_batch_f64_device(ctx.handle, C.byref(cs), kind,
                                                               C.cast(l64.data_ptr(), C.POINTER(C.c_double)), F,
                                                               ALPHA, 40, C.byref(fo), C.c_void_p(st.cuda_stream)))
                else:
                    P._check(P.lib.pbp_decode_batch_device(ctx.handle, C.byref(cs), kind, P._abi.f32p(l32.data_ptr()),
                                                           F, ALPHA, 40, C.byref(fo), C.c_void_p(st.cuda_stream)))
            call()  # warm-up (sizes the context's buffers)
            st.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            call()
            e1.record(st)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            pe = int(outs[2].sum().item())
            res[prec] = (ms, pe, float(outs[1].float().mean().item()))
        (m64, pe64, it64), (m32, pe32, it32) = res["f64"], res["f32"]
        print(json.dumps({"config": cfg, "decoder": kind_name, "n": n, "ebn0_db": ebn0, "frames": F,
                          "f64_ms": round(m64, 3), "f64_info_bits_per_s": round(F * k / (m64 / 1e3), 1),
                          "f64_pe_per_s": round(pe64 / (m64 / 1e3), 1), "f64_avg_iters": round(it64, 3),
                          "f32_ms": round(m32, 3), "f32_info_bits_per_s": round(F * k / (m32 / 1e3), 1),
                          "f32_over_f64": round(m64 / m32, 2)}), flush=True)


if __name__ == "__main__":
    main()
