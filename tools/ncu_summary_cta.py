"""Summarise the full ncu captures of tools/r2_cta_captures.sh into profiles/<TAG>_cta_ncu_summary.json.

   python tools/ncu_summary_cta.py TAG

bp_cta_kernel<12,2> (n = 4096, 4440 frames) and bp_pair_kernel<13,2> (n = 16384 on 2-CTA
clusters, 740 frames), csfg at 2.5 dB, max_iter 40; per-frame DRAM bytes, warp-instructions
per PE slot (n/2 x log2 n PE slots per iteration), issue/pipe utilisation, stall reasons and
the top source lines by stall samples (tools/ncu_lines.py)."""
import json, re, subprocess, sys
sys.path.insert(0, "tools")
from ncu_summary import raw  # noqa: E402


def one(rep, log, n, frames):
    m = raw(rep)
    it = 40.0
    try:
        mm = re.search(r"avg iters ([0-9.]+)", open(log).read())
        it = float(mm.group(1)) if mm else it
    except OSError:
        pass
    ins = m["smsp__inst_executed.sum"]
    slots = (n // 2) * (n.bit_length() - 1)
    lines = subprocess.run(["python", "tools/ncu_lines.py", rep, "paper_1505_04979_b200/csrc/bp_cta.cu", "--top", "12"],
                           capture_output=True, text=True).stdout.splitlines()
    top = [l.strip() for l in lines if re.match(r"\s*\d+\s+\d+\s+[0-9.]+%", l)][:12]
    return {
        "kernel": m.get("Kernel Name", ""),
        "frames": frames, "avg_iters": it,
        "duration_ms_under_ncu": m["gpu__time_duration.sum"],
        "dram_bytes_per_frame": (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / frames,
        "l2_hit_pct": m.get("lts__t_sector_hit_rate.pct"),
        "warp_instr_per_frame_iteration": ins / (frames * it),
        "warp_instr_per_pe_slot": ins / (frames * it * slots),
        "issue_active_pct": m["smsp__issue_active.avg.pct_of_peak_sustained_active"],
        "warps_active_per_sm": m["sm__warps_active.avg.per_cycle_active"],
        "registers": m["launch__registers_per_thread"],
        "stalls_per_issue": {k.split("stalled_")[1].replace("_per_issue_active.ratio", ""): round(v, 3)
                             for k, v in m.items() if k.startswith("smsp__average_warps_issue_stalled_")
                             and k.endswith("_per_issue_active.ratio") and isinstance(v, float) and v > 0.01},
        "top_lines_by_stall_samples": top,
    }


def main():
    tag = sys.argv[1]
    out = {
        "source": f"ncu --set full --import-source on --clock-control none -c 1, python tools/prof_decode.py --ebn0 2.5 "
                  f"(csfg, max_iter 40); tools/r2_cta_captures.sh {tag}; reports gpurun_out/{tag}_prof_*.ncu-rep (not "
                  "committed); tools/ncu_summary_cta.py",
        "n4096_bp_cta_kernel": one(f"gpurun_out/{tag}_prof_cta4096.ncu-rep", f"gpurun_out/{tag}_ncu_cta4096.log", 4096, 4440),
        "n16384_bp_pair_kernel": one(f"gpurun_out/{tag}_prof_pair16384.ncu-rep", f"gpurun_out/{tag}_ncu_pair.log", 16384, 740),
    }
    with open(f"profiles/{tag}_cta_ncu_summary.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
