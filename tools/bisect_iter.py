"""Find the first max_iter at which the GPU decode diverges from the oracle (debug aid)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_1505_04979_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ebn0 = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ctx = P.Context(0)
fz = O.construct(n, n // 2, math.exp(-0.5))
code = P.PolarCode.from_frozen_mask(n, fz)
_, llr = O.trials(seed, 0, 64, fz, ebn0, lib=O.C)
llr = llr.astype(np.float32)
for kind in ("baseline", "gmatrix", "csfg"):
    first = None
    for mi in range(1, 41):
        exp = O.decode_batch(kind, fz, llr, 0.9375, mi, prec=32)
        got = P.decode_batch(code, kind, llr, 0.9375, mi, ctx=ctx)
        gu = P.unpack_bits(got["u_hat_bits"], n)
        bad = np.flatnonzero((gu != exp["u_hat"]).any(1) | (got["iterations"] != exp["iterations"]) | (got["pe"] != exp["pe"]))
        if bad.size:
            first = mi
            print(kind, "first divergence at max_iter", mi, "frames", bad[:8], "nbits", [(int((gu[b] != exp["u_hat"][b]).sum())) for b in bad[:8]])
            break
    if first is None:
        print(kind, "no divergence up to 40")
