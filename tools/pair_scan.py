import math, os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1505_04979_b200 as P
import oracle as O
N = 16384; Z0 = math.exp(-0.5)
ctx = P.Context(0)
rng = np.random.default_rng(5)
for k in (16, 256, 2048, 8192, 12288, 16000):
    for mode in ("construct", "random"):
        if mode == "construct":
            code = P.PolarCode.construct(N, k, Z0); fz = code.frozen
        else:
            fz = np.ones(N, np.uint8); fz[rng.permutation(N)[:k]] = 0; code = P.PolarCode.from_frozen_mask(N, fz)
        for snr in (0.0, 1.0, 2.0, 3.0, 4.0, 6.0):
            llr, _, _ = P.generate(code, 7, 0, 4096, snr, ctx=ctx)
            res = {}
            for on in ("1", "0"):
                os.environ["PBP_PAIR"] = on
                res[on] = P.decode_batch(code, "csfg", llr, 0.9375, 40, ctx=ctx)
            same = all(np.array_equal(res["1"][f], res["0"][f]) for f in ("u_hat_bits", "iterations", "pe", "stop", "n_events"))
            st = np.bincount(res["0"]["stop"].astype(np.int64), minlength=3)
            print(k, mode, snr, "stops", st.tolist(), "same", same, flush=True)
