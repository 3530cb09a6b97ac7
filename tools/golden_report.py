"""Per-case mismatch report of the CUDA decoders vs the golden ref32 fixtures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_1505_04979_b200 as P
from conftest import load_manifest
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/golden.npz"))
ctx = P.Context(0)
for generic in (False, True):
    ctx.force_generic(generic)
    for c in load_manifest()["cases"]:
        name = c["name"]
        code = P.PolarCode.from_frozen_mask(c["n"], g[name + "/frozen"])
        r = P.decode_batch(code, c["decoder"], g[name + "/llr32"], 0.9375, c["max_iter"], ctx=ctx)
        n = c["n"]
        gu = P.unpack_bits(r["u_hat_bits"], n)
        eu = np.unpackbits(g[name + "/ref32/u_hat"], axis=1, bitorder="little")[:, :n]
        bad = {"u": int((gu != eu).any(1).sum())}
        for f in ("iterations", "pe", "stop", "n_events"):
            bad[f] = int((r[f].astype(np.int64) != g[f"{name}/ref32/{f}"].astype(np.int64)).sum())
        flag = "OK " if not any(bad.values()) else "BAD"
        print(flag, "generic" if generic else "auto   ", f"{name:28s}", bad, flush=True)
        if flag == "BAD":
            idx = np.flatnonzero((gu != eu).any(1))[:3]
            for i in idx:
                print("    frame", i, "it", r["iterations"][i], g[f"{name}/ref32/iterations"][i], "pe", r["pe"][i],
                      g[f"{name}/ref32/pe"][i], "bits differ", int((gu[i] != eu[i]).sum()), "first", int(np.flatnonzero(gu[i] != eu[i])[0]))
