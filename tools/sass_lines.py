"""Static SASS size of one kernel broken down by (inlined) source function.
   python tools/sass_lines.py <cubin> <kernel-substring> [source.cu]
Uses nvdisasm -gi (line info with inlining chains; build with -lineinfo). Prints the
inclusive instruction count per function: an instruction counts for every function on
its inline chain."""
import re, subprocess, sys
from collections import Counter

cubin, kern = sys.argv[1], sys.argv[2]
src = sys.argv[3] if len(sys.argv) > 3 else None
txt = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout.splitlines()
fn_re = re.compile(r"__device__[^;{]*?\b(\w+)\s*\(")


def func_map(path):
    m, cur = {}, "?"
    for i, t in enumerate(open(path).read().splitlines(), 1):
        mm = fn_re.search(t)
        if mm and ("__forceinline__" in t or "__global__" in t):
            cur = mm.group(1)
        m[i] = cur
    return m


fmaps = {}
inside, chain, pending = False, [], []
incl, leaf = Counter(), Counter()
loc_re = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
for t in txt:
    if t.startswith("//---------------------"):
        inside = kern in t
        continue
    if not inside:
        continue
    mm = loc_re.search(t)
    if mm:
        pending.append((mm.group(1), int(mm.group(2))))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", t):
        if pending:
            chain, pending = pending, []
        names = []
        for path, ln in chain:
            fm = fmaps.setdefault(path, func_map(src if (src and path.endswith(src.split("/")[-1])) else path)
                                  if path.endswith(".cu") or path.endswith(".cuh") else {})
            names.append(fm.get(ln, path.split("/")[-1]))
        for nm in set(names):
            incl[nm] += 1
        if names:
            leaf[names[0]] += 1
total = sum(leaf.values())
print(f"{total} instructions ({total * 16 / 1024:.1f} KB)")
print(f"{'function':28s} {'inclusive':>9s} {'leaf':>6s}")
for nm, c in incl.most_common():
    print(f"{nm:28s} {c:9d} {leaf[nm]:6d}")
