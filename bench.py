"""Benchmark: decoded info bits/s of the csfg decoder (freeze + G-stop), N=1024 R=1/2.

Workload (BASELINE.json configs[2]): PolarCode(1024, 512) from the Bhattacharyya
construction at design z = e^-0.5 ("design Eb/N0 0 dB"), seed 2, Eb/N0 1.0..4.0 dB in
0.5 dB steps, 1e5 frames per point, alpha 0.9375, max 40 iterations. One "step" decodes
the whole sweep (7 x 1e5 frames). Frames are the reference's own seeded generator,
produced on the device (synthetic data; inputs 2.9 GB >> 126 MB L2, so no L2 reuse
between steps). Multi-GPU: one process per GPU, every rank decodes its own disjoint
trial range of the full sweep (weak scaling), counters combined with one NCCL int64
all-reduce per step; time = max over ranks of device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N, K, Z0, SEED, ALPHA, MAX_ITER = 1024, 512, math.exp(-0.5), 2, 0.9375, 40
SNRS = [1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0]
FRAMES_PER_POINT = 100_000
OPS_PER_PE = 9  # 3 min-with-sign, 3 alpha-multiplies, 3 adds
METRIC = "info bits/s decoded (N=1024 R=1/2, freeze+G-stop)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- CPU reference

def cpu_reference_run(seconds_per_step=8.0, steps=1, warmup=0, want_threads=None, with_ref32=True):
    """The reference's own CPU decoder (oracle/_ref = reference sources compiled in place,
    fp64 as shipped) over a bounded sample of the config-2 sweep, all host threads.
    Falls back to the C restatement (kind "port") when the reference build is absent.
    Like the stock decode_trial without --trace (sim_harness.cpp:84-90), no FreezeEvent
    list is recorded. with_ref32: the same sources compiled with double -> float (the
    GPU's arithmetic) timed on the same sample and reported beside it."""
    import oracle as O
    threads = want_threads or os.cpu_count() or 1
    kind = "reference" if O.REF is not None else "port"
    lib = O.REF if O.REF is not None else O.C
    fz = O.construct(N, K, Z0, lib=lib)
    # calibrate: frames per SNR point so one step takes ~seconds_per_step
    per_point = max(2, threads // 2)

    def make(per):
        out = []
        for snr in SNRS:
            _, llr = O.trials(SEED, 0, per, fz, snr, lib=lib, threads=threads)
            out.append(llr)
        return out

    def decode_all(llrs, prec):
        pe = 0
        for llr in llrs:
            r = O.decode_batch("csfg", fz, llr, ALPHA, MAX_ITER, prec=prec, lib=lib, threads=threads,
                               want_u=False, want_events=False)
            pe += int(r["pe"].sum())
        return pe

    llrs = make(per_point)
    t0 = time.perf_counter()
    decode_all(llrs, 64)
    dt = time.perf_counter() - t0
    per_point = max(per_point, int(per_point * seconds_per_step / max(dt, 1e-3)))
    llrs = make(per_point)
    frames = per_point * len(SNRS)

    def timed(prec):
        times, pe_total = [], 0
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            pe = decode_all(llrs, prec)
            dt = time.perf_counter() - t0
            if it >= warmup:
                times.append(dt)
                pe_total += pe
        tot = sum(times)
        return frames * K * len(times) / tot, tot, pe_total

    v64, tot, pe_total = timed(64)
    out = {"value": v64, "unit": "info bits/s", "cores": threads, "kind": kind,
           "frames_per_step": frames, "seconds": tot, "ms_per_step": 1e3 * tot / steps,
           "pe_per_s": pe_total / tot,
           "sample": f"{per_point} frames x {len(SNRS)} Eb/N0 points (trials 0..{per_point - 1}, seed {SEED}) "
                     f"of config 2, fp64 reference decode_csfg (no event list), {threads} threads, "
                     "LLRs pre-generated"}
    if with_ref32 and kind == "reference":
        v32, tot32, pe32 = timed(32)
        out["ref32"] = {"value": v32, "unit": "info bits/s", "pe_per_s": pe32 / tot32,
                        "what": "the same reference sources compiled with double -> float (the GPU's "
                                "operation order and precision), same sample and threads"}
    return out


def dram_traffic(frames_per_launch):
    """DRAM bytes (read + write) per decode launch, from the committed ncu capture
    (profiles/*_ncu_summary.json: dram__bytes_read.sum + dram__bytes_write.sum of
    bp_warp_kernel<10,2>, scaled per frame to this launch size); None if absent."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_summary.json")))
    for f in reversed(files):  # the newest summary of the headline kernel (other kernels' summaries skipped)
        try:
            return float(json.load(open(f))["csfg"]["dram_bytes_per_frame"]) * frames_per_launch
        except Exception:
            continue
    return None


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# --------------------------------------------------------------------------- launch

def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_command(argv, gpus, port):
    """torchrun command that runs this script on `gpus` ranks of one node (127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def relaunch_if_needed(args, argv):
    """`bench.py --gpus N` outside torchrun: start N ranks (one process per GPU) and exit
    with their status. Inside torchrun (WORLD_SIZE set) nothing happens."""
    if os.environ.get("WORLD_SIZE") or args.gpus <= 1:
        return
    cmd = launch_command(argv, args.gpus, free_port())
    log("bench: launching", " ".join(cmd))
    sys.exit(subprocess.call(cmd))


# --------------------------------------------------------------------------- GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=FRAMES_PER_POINT)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gen", action="store_true", help="skip the generate+decode figure")
    args = ap.parse_args()
    relaunch_if_needed(args, sys.argv[1:])

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        r = cpu_reference_run(seconds_per_step=6.0, steps=args.steps, warmup=min(args.warmup, 1))
        line = {"metric": METRIC, "value": r["value"], "unit": "info bits/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (reference TrialRng/encode/AWGN frames, seeded)",
                "impl": "reference",
                "config": {"workload": "config2 csfg N=1024 K=512 z=e^-0.5 seed 2 Eb/N0 1.0:4.0:0.5 "
                                       "(bounded CPU sample)", "decoder": "csfg", "max_iter": MAX_ITER,
                           "alpha": ALPHA, "cpu": cpu_model()},
                "cpu_baseline": {"value": r["value"], "unit": "info bits/s", "cores": r["cores"],
                                 "kind": r["kind"], "sample": r["sample"], "ref32": r.get("ref32")},
                "e2e": {"value": r["value"], "unit": "info bits/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_1505_04979_b200 as P

    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    dist = None
    if world > 1 or os.environ.get("TORCHELASTIC_RUN_ID"):  # every torchrun launch, even 1 rank
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = P.Context(local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)
    code = P.PolarCode.construct(N, K, Z0)
    cs = code.c_struct()
    frames = args.frames
    nw = N // 32
    first = rank * frames  # disjoint trial range per rank (weak scaling)

    # ---- inputs resident in HBM: the full sweep, generated on the device ----
    llr = torch.empty((len(SNRS), frames, N), dtype=torch.float32, device=dev)
    truth = torch.empty((len(SNRS), frames, nw), dtype=torch.int32, device=dev)
    for i, snr in enumerate(SNRS):
        P._check(P.lib.pbp_generate_device(ctx.handle, C.byref(cs), C.c_uint64(SEED), first, frames, snr, 0,
                                           P._abi.f32p(llr[i].data_ptr()), None,
                                           P._abi.u32p(truth[i].data_ptr()), None))
    ctx.synchronize()
    counters = torch.zeros((len(SNRS), 10), dtype=torch.int64, device=dev)
    ubits = torch.empty((frames, nw), dtype=torch.int32, device=dev)
    iters = torch.empty(frames, dtype=torch.int32, device=dev)
    pe = torch.empty(frames, dtype=torch.int64, device=dev)
    stopv = torch.empty(frames, dtype=torch.uint8, device=dev)
    nev = torch.empty(frames, dtype=torch.int32, device=dev)

    # the whole sweep in ONE decode launch: the points are stored one after the other
    # and the kernel keeps one counter set per point (cnt_batch = frames)
    def decode_sweep():
        P._check(P.lib.pbp_decode_count_batches_device(ctx.handle, C.byref(cs), 2, P._abi.f32p(llr.data_ptr()),
                                                       P._abi.u32p(truth.data_ptr()), len(SNRS) * frames, frames,
                                                       ALPHA, MAX_ITER, P._abi.i64p(counters.data_ptr()), None))

    def step():
        counters.zero_()
        decode_sweep()

    # kernel-level timing of the dominant kernel: the sweep's decode launch
    def timed_sweep():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        decode_sweep()
        e1.record(stream)
        return e0, e1

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        sampler = ClockSampler(local_rank)
        sampler.start()
        time.sleep(0.3)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        per_point_events = []
        for s in range(args.steps):
            counters.zero_()
            per_point_events.append(timed_sweep())
            if dist:
                dist.all_reduce(counters)  # NCCL int64 sum of the Accumulator fields
        t1.record(stream)
        torch.cuda.synchronize()
        clocks = sampler.stop()
        elapsed_ms = t0.elapsed_time(t1)
        launch_ms = [a.elapsed_time(b) for a, b in per_point_events]
    if dist:
        tt = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = float(tt.item())
    tot = counters.cpu().numpy()
    total_frames = int(tot[:, 0].sum())
    total_pe = int(tot[:, 5].sum())
    steps = args.steps
    assert total_frames == len(SNRS) * frames * world, total_frames
    value = total_frames * K * steps / (elapsed_ms / 1e3)

    # ---- roofline: 9 fp32 ops per PE activation vs 148 SMs x 128 lanes x f_clk ----
    peaks = measured_peaks()
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    fclk = (peaks.get("sm_max_mhz") or 1965.0) * 1e6
    peak_tops = sm_count * 128 * fclk / 1e12
    # per-launch algorithmic ops: PE activations of one sweep decode (this rank)
    pe_per_launch = tot[:, 5].sum() / max(1, world)  # counters summed over ranks
    ms_mean = float(np.mean(launch_ms))
    achieved = float(pe_per_launch * OPS_PER_PE / (ms_mean / 1e3) / 1e12)

    line = {"metric": METRIC, "value": value, "unit": "info bits/s", "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference TrialRng/encode/AWGN frames generated on device, seeded)",
            "config": {"workload": "config2: csfg N=1024 K=512 design z=e^-0.5 seed 2, Eb/N0 1.0:4.0:0.5, "
                                   f"{frames} frames/point/GPU, alpha 0.9375, max_iter 40",
                       "decoder": "csfg (freeze + G-stop)", "frames_per_step": len(SNRS) * frames * world,
                       "l2": "inputs 2.9 GB/GPU > 126 MB L2, no flush needed", "parallelism": f"dp{world}"},
            "frames_per_s": len(SNRS) * frames * world * steps / (elapsed_ms / 1e3),
            "pe_per_s": total_pe * steps / (elapsed_ms / 1e3),
            "avg_iters_per_point": [round(float(t[3] / max(t[0], 1)), 4) for t in tot],
            "fer_per_point": [float(t[2] / max(t[0], 1)) for t in tot],
            "gpu_launches": steps * 2,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_tops, "unit": "TOP/s (fp32 ops)",
                         "frac": achieved / peak_tops, "traffic": dram_traffic(frames),
                         "note": f"9 fp32 ops per PE activation (reference pe_activations counter); peak = "
                                 f"{sm_count} SMs x 128 lanes x {fclk / 1e6:.0f} MHz (sm_max_mhz of "
                                 "MEASURED_PEAKS.json); achieved from CUDA-event launch times"},
            "clocks": clocks}

    # ---- generation + decode: the same trials generated on the device inside the timed
    #      region (pbp_simulate_point_device: decode_trial's channel + decode, counters) ----
    if not args.no_gen:
        gcnt = torch.zeros((len(SNRS), 10), dtype=torch.int64, device=dev)

        def gen_step():
            gcnt.zero_()
            for i, snr in enumerate(SNRS):
                P._check(P.lib.pbp_simulate_point_device(ctx.handle, C.byref(cs), 2, C.c_uint64(SEED), first,
                                                         frames, snr, 0, ALPHA, MAX_ITER,
                                                         P._abi.i64p(gcnt[i].data_ptr()), None))
            if dist:
                dist.all_reduce(gcnt)

        with torch.cuda.stream(stream):
            gen_step()  # staging allocation, warm
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(args.steps):
                gen_step()
            g1.record(stream)
            torch.cuda.synchronize()
            gen_ms = g0.elapsed_time(g1)
        if dist:
            tt = torch.tensor([gen_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            gen_ms = float(tt.item())
        same = bool(torch.equal(gcnt.cpu(), torch.from_numpy(tot)))
        line["gen_decode"] = {"value": total_frames * K * steps / (gen_ms / 1e3), "unit": "info bits/s",
                              "ms_per_step": gen_ms / steps, "counters_equal_decode_only": same,
                              "what": "pbp_simulate_point_device per Eb/N0 point: the reference's seeded "
                                      "TrialRng/encode/AWGN frames generated on the device and decoded, "
                                      "both inside the timed region (device time, max over ranks)"}

    # ---- e2e through the host-buffer C ABI (pinned host LLRs in, results out) ----
    if not args.no_e2e and rank == 0 or (not args.no_e2e and world > 1):
        # the whole sweep (every Eb/N0 point's frames) in one host-buffer call;
        # if that much host memory cannot be pinned, the 3 dB point alone
        try:
            host_llr = torch.empty((len(SNRS) * frames, N), dtype=torch.float32, pin_memory=True)
            whole = 1
        except RuntimeError:
            host_llr, whole = None, 0
        if dist:  # every rank times the same scope
            flag = torch.tensor([whole], device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            whole = int(flag.item())
        if whole:
            nb = len(SNRS) * frames
            host_llr.copy_(llr.reshape(nb, N))
            e2e_scope = f"the sweep's {nb} frames/GPU"
        else:
            del host_llr
            nb = frames
            host_llr = torch.empty((nb, N), dtype=torch.float32, pin_memory=True)
            host_llr.copy_(llr[SNRS.index(3.0)])
            e2e_scope = f"the 3.0 dB point's {nb} frames/GPU (pinning the sweep failed)"
        outs = {"u": torch.empty((nb, nw), dtype=torch.int32, pin_memory=True),
                "it": torch.empty(nb, dtype=torch.int32, pin_memory=True),
                "pe": torch.empty(nb, dtype=torch.int64, pin_memory=True),
                "st": torch.empty(nb, dtype=torch.uint8, pin_memory=True),
                "ne": torch.empty(nb, dtype=torch.int32, pin_memory=True)}
        fo = P._abi.PbpFrameOut(P._abi.u32p(outs["u"].data_ptr()), P._abi.i32p(outs["it"].data_ptr()),
                                P._abi.i64p(outs["pe"].data_ptr()), P._abi.u8p(outs["st"].data_ptr()),
                                P._abi.i32p(outs["ne"].data_ptr()))

        def e2e_once():
            P._check(P.lib.pbp_decode_batch(ctx.handle, C.byref(cs), 2,
                                            P._abi.f32p(host_llr.data_ptr()), nb, ALPHA, MAX_ITER, C.byref(fo)))
        e2e_once()
        reps = max(1, steps)
        if dist:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(reps):
            e2e_once()
        dt = time.perf_counter() - t
        if dist:
            tt = torch.tensor([dt], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        line["e2e"] = {"value": nb * world * K * reps / dt, "unit": "info bits/s",
                       "h2d_bytes_per_step": nb * N * 4, "d2h_bytes_per_step": nb * (nw * 4 + 4 + 8 + 1 + 4),
                       "what": f"pbp_decode_batch (host C ABI), one call over {e2e_scope}: pinned host "
                               "LLRs -> device -> decode -> host results (copies pipelined with the decode), "
                               "wall clock"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference_run(seconds_per_step=8.0, steps=1, warmup=0)
            line["cpu_baseline"] = {"value": r["value"], "unit": "info bits/s", "cores": r["cores"],
                                    "kind": r["kind"], "sample": r["sample"], "cpu": cpu_model(),
                                    "ref32": r.get("ref32")}
        except Exception as e:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
