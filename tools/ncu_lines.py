"""Aggregate ncu warp-stall samples of one kernel by source line and enclosing function.
   python tools/ncu_lines.py report.ncu-rep [source.cu] [--top 30] [--by-inst]
The report must be captured with -lineinfo builds and --import-source on. Samples are
attributed to the innermost inlined line; functions are found by scanning the source for
definitions, so helpers shared by several callers show up under their own name."""
import csv, io, re, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
by_inst = "--by-inst" in sys.argv  # rank lines by executed warp instructions
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
lines = {}
path = None
for r in rows:
    if r and r[0] == "File Path":
        path = r[1]
    if len(r) != len(hdr) or not r[0].isdigit() or r[2] != "-":
        continue
    ln = int(r[0])
    lines[(path, ln)] = (r[1], int(r[ix["# Samples"]] or 0), int(r[ix["Instructions Executed"]] or 0),
                         {c: int(r[ix[c]] or 0) for c in stall_cols})

fn_re = re.compile(r"__device__[^;{]*?\b(\w+)\s*\(")
def func_map(p):
    try:
        text = open(src or p).read().splitlines()
    except OSError:
        return {}
    m, cur = {}, "?"
    for i, t in enumerate(text, 1):
        mm = fn_re.search(t)
        if mm and "__forceinline__" in t or (mm and "__global__" in t):
            cur = mm.group(1)
        elif "__global__" in t:
            cur = "kernel"
        m[i] = cur
    return m

fmaps = {}
byfn = defaultdict(lambda: [0, 0, defaultdict(int)])
tot = sum(v[1] for v in lines.values())
for (p, ln), (s, n, ins, st) in lines.items():
    fm = fmaps.setdefault(p, func_map(p))
    f = fm.get(ln, "?") if p and p.endswith("bp_warp.cu") else (p or "?").split("/")[-1]
    e = byfn[f]
    e[0] += n
    e[1] += ins
    for c, v in st.items():
        e[2][c] += v
print(f"total samples {tot}")
print(f"{'function':24s} {'samples':>8s} {'%':>6s} {'warp-inst':>12s}  top stalls")
for f, (n, ins, st) in sorted(byfn.items(), key=lambda kv: -kv[1][0]):
    tops = sorted(st.items(), key=lambda kv: -kv[1])[:4]
    print(f"{f:24s} {n:8d} {100*n/max(tot,1):6.1f} {ins:12d}  " +
          " ".join(f"{c[6:]}={100*v/max(n,1):.0f}%" for c, v in tops))
print()
tot_ins = sum(v[2] for v in lines.values())
for (p, ln), (s, n, ins, st) in sorted(lines.items(), key=lambda kv: -kv[1][2 if by_inst else 1])[:top]:
    tops = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    if by_inst:
        print(f"{ln:5d} {ins:11d} {100*ins/max(tot_ins,1):5.1f}% {s.strip()[:90]}")
        continue
    print(f"{ln:5d} {n:7d} {100*n/max(tot,1):5.1f}% {s.strip()[:70]:70s} " +
          " ".join(f"{c[6:]}={v}" for c, v in tops))
