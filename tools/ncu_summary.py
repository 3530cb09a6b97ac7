"""Summarise the full ncu captures of refresh_profiles.sh into profiles/<TAG>_ncu_summary.json.

   python tools/ncu_summary.py TAG [--frames 20000] [--iters-csfg 25.66] [--iters-base 40]

Reads gpurun_out/<TAG>_prof_csfg.ncu-rep and <TAG>_prof_base.ncu-rep (one launch each of
bp_warp_kernel<10,2> / <10,0>, 20 000 frames of config 2 at 3 dB); DRAM bytes are
converted to bytes whatever unit ncu prints. bench.py's roofline.traffic reads the newest
profiles/*_ncu_summary.json."""
import csv, io, json, subprocess, sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[2]
    m = {}
    for i, n in enumerate(h):
        try:
            m[n] = float(v[i]) * SCALE.get(u[i], 1)
        except ValueError:
            m[n] = v[i]
    return m


def kernel(rep, frames, iters):
    m = raw(rep)
    ins = m["smsp__inst_executed.sum"]
    return {
        "kernel": m.get("Kernel Name", ""),
        "duration_ms_under_ncu": m["gpu__time_duration.sum"],
        "dram_read_bytes": m["dram__bytes_read.sum"],
        "dram_write_bytes": m["dram__bytes_write.sum"],
        "dram_bytes_per_frame": (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / frames,
        "warp_instructions": ins,
        "warp_instr_per_frame_iteration": ins / (frames * iters),
        "warps_active_per_sm": m["sm__warps_active.avg.per_cycle_active"],
        "issue_active_pct": m["smsp__issue_active.avg.pct_of_peak_sustained_active"],
        "registers": m["launch__registers_per_thread"],
        "occupancy_limit_smem_blocks": m["launch__occupancy_limit_shared_mem"],
        "no_instruction_stall_per_issue": m["smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio"],
        "stalls_per_issue": {k.split("stalled_")[1].replace("_per_issue_active.ratio", ""): round(v, 3)
                             for k, v in m.items() if k.startswith("smsp__average_warps_issue_stalled_")
                             and k.endswith("_per_issue_active.ratio") and isinstance(v, float) and v > 0.01},
    }


def main():
    tag = sys.argv[1]
    arg = lambda k, d: float(sys.argv[sys.argv.index(k) + 1]) if k in sys.argv else d
    frames = int(arg("--frames", 20000))
    out = {
        "source": "ncu --set full --clock-control none -k regex:bp_warp_kernel -c 1, python tools/prof_decode.py "
                  "--n 1024 --frames 20000 --reps 1 (config 2, 3 dB; baseline: --kind baseline); reports "
                  f"gpurun_out/{tag}_prof_*.ncu-rep (not committed); tools/ncu_summary.py",
        "frames_per_launch": frames,
        "csfg": kernel(f"gpurun_out/{tag}_prof_csfg.ncu-rep", frames, arg("--iters-csfg", 25.659)),
    }
    import os
    if os.path.exists(f"gpurun_out/{tag}_prof_base.ncu-rep"):
        out["baseline"] = kernel(f"gpurun_out/{tag}_prof_base.ncu-rep", frames, arg("--iters-base", 40.0))
    with open(f"profiles/{tag}_ncu_summary.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
