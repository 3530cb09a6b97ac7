"""Generate the golden fixtures from the REFERENCE compiled in place (oracle/_ref).

Run in the dev container (needs /root/reference):  python tests/golden/make_golden.py
Writes tests/golden/golden.npz and tests/golden/manifest.json (committed).

Every expected value comes from the unmodified reference core
(/root/reference/proj/src/{polar_code,channel,bp_core,csfg_freeze}.cpp) through
oracle/ref_wrap.cpp:
  * frames: ref64_trials = TrialRng + encode + modulate_bpsk + transmit_awgn
    (the decode_trial generation, sim_harness.cpp:67-73), fp64 LLRs;
  * "ref32" outcomes: the reference sources compiled with `double` -> `float`,
    fed (float)LLR: the bit-exact target of the CUDA kernels;
  * "ref64" outcomes: the shipped double-precision reference.
The design point "Eb/N0 0 dB" of BASELINE.json is declared as z = exp(-R) = e^-0.5
(SURVEY.md 8d); the reference's own default z = 0.5 is used for its test cases.
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

Z0 = math.exp(-0.5)

# name, n, k, z, seed, ebn0, kind, max_iter, frames, first_trial
CASES = [
    ("c0_base_1024_3.0", 1024, 512, Z0, 1, 3.0, "baseline", 40, 24, 0),
    ("c1_gm_1024_1.0", 1024, 512, Z0, 2, 1.0, "gmatrix", 40, 16, 0),
    ("c1_gm_1024_2.5", 1024, 512, Z0, 2, 2.5, "gmatrix", 40, 24, 0),
    ("c1_gm_1024_4.0", 1024, 512, Z0, 2, 4.0, "gmatrix", 40, 24, 0),
    ("c2_csfg_1024_1.0", 1024, 512, Z0, 2, 1.0, "csfg", 40, 16, 0),
    ("c2_csfg_1024_2.0", 1024, 512, Z0, 2, 2.0, "csfg", 40, 32, 0),
    ("c2_csfg_1024_2.5", 1024, 512, Z0, 2, 2.5, "csfg", 40, 48, 0),
    ("c2_csfg_1024_3.0", 1024, 512, Z0, 2, 3.0, "csfg", 40, 48, 0),
    ("c2_csfg_1024_4.0", 1024, 512, Z0, 2, 4.0, "csfg", 40, 32, 0),
    ("c3_csfg_4096_2.5", 4096, 2048, Z0, 4, 2.5, "csfg", 60, 6, 0),
    ("c4_csfg_256_2.5", 256, 128, Z0, 5, 2.5, "csfg", 40, 64, 0),
    ("c4_csfg_16384_2.5", 16384, 8192, Z0, 5, 2.5, "csfg", 40, 2, 0),
    ("c4_csfg_1024_2.5", 1024, 512, Z0, 5, 2.5, "csfg", 40, 32, 0),
    ("c4_csfg_4096_2.5", 4096, 2048, Z0, 5, 2.5, "csfg", 40, 4, 0),
    # the reference's own test settings (design z = 0.5)
    ("t_csfg_64_2.0_s4242", 64, 32, 0.5, 4242, 2.0, "csfg", 40, 300, 0),
    ("t_gm_64_6.0_s99", 64, 32, 0.5, 99, 6.0, "gmatrix", 40, 50, 0),
    ("t_csfg_1024_3.0_s61803", 1024, 512, 0.5, 61803, 3.0, "csfg", 40, 32, 0),
    ("t_gm_1024_2.0_s61803", 1024, 512, 0.5, 61803, 2.0, "gmatrix", 40, 16, 100),
    ("t_csfg_128_1.5", 128, 64, Z0, 7, 1.5, "csfg", 40, 64, 0),
    ("t_csfg_512_2.5", 512, 256, Z0, 8, 2.5, "csfg", 40, 32, 0),
    ("t_base_256_2.0", 256, 128, Z0, 9, 2.0, "baseline", 12, 32, 0),
    ("t_csfg_32_3.0", 32, 16, 0.5, 10, 3.0, "csfg", 40, 64, 0),
    ("t_csfg_1024_0.0_it2", 1024, 512, Z0, 11, 0.0, "csfg", 2, 16, 0),
]


def main():
    if O.REF is None:
        raise SystemExit("oracle/_ref/libpbp_ref.so missing: run `make -C oracle` with /root/reference present")
    arrays = {}
    manifest = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (reference compiled in place)",
                "cases": []}
    codes = {}
    for name, n, k, z, seed, ebn0, kind, max_iter, frames, first in CASES:
        key = (n, k, z)
        if key not in codes:
            codes[key] = O.construct(n, k, z, lib=O.REF)
        fz = codes[key]
        info, llr64 = O.trials(seed, first, frames, fz, ebn0, lib=O.REF)
        llr32 = llr64.astype(np.float32)
        r32 = O.decode_batch(kind, fz, llr32, 0.9375, max_iter, prec=32, lib=O.REF)
        r64 = O.decode_batch(kind, fz, llr64, 0.9375, max_iter, prec=64, lib=O.REF)
        arrays[f"{name}/frozen"] = fz
        arrays[f"{name}/info"] = info
        arrays[f"{name}/llr32"] = llr32
        arrays[f"{name}/llr64_head"] = llr64[:2]
        for tag, r in (("ref32", r32), ("ref64", r64)):
            arrays[f"{name}/{tag}/u_hat"] = np.packbits(r["u_hat"], axis=1, bitorder="little")
            arrays[f"{name}/{tag}/iterations"] = r["iterations"]
            arrays[f"{name}/{tag}/pe"] = r["pe"]
            arrays[f"{name}/{tag}/stop"] = r["stop"].astype(np.uint8)
            arrays[f"{name}/{tag}/n_events"] = r["n_events"]
        manifest["cases"].append({"name": name, "n": n, "k": k, "design_z": z, "seed": seed,
                                  "ebn0_db": ebn0, "decoder": kind, "max_iter": max_iter,
                                  "frames": frames, "first_trial": first,
                                  "ref32_fer": float((r32["u_hat"][:, fz == 0] != info).any(1).mean()),
                                  "ref32_avg_iters": float(r32["iterations"].mean()),
                                  "ref32_avg_pe": float(r32["pe"].mean())})
        print(name, manifest["cases"][-1]["ref32_fer"], manifest["cases"][-1]["ref32_avg_iters"], flush=True)

    # single-frame traces with the freeze-event log
    ev_cases = [("ev_8_clean", 8, 4, 0.5, None), ("ev_64_2.0", 64, 32, 0.5, (4242, 2.0, 40)),
                ("ev_1024_2.5", 1024, 512, Z0, (2, 2.5, 40)), ("ev_256_2.5", 256, 128, Z0, (5, 2.5, 40))]
    for name, n, k, z, gen in ev_cases:
        fz = O.construct(n, k, z, lib=O.REF)
        if gen is None:
            llrs = np.full((1, n), 5.0)
            max_iter = 40
        else:
            seed, ebn0, max_iter = gen
            _, llrs = O.trials(seed, 0, 8, fz, ebn0, lib=O.REF)
        for i in range(llrs.shape[0]):
            r = O.decode("csfg", fz, llrs[i].astype(np.float32), 0.9375, max_iter, prec=32, lib=O.REF)
            arrays[f"{name}/{i}/frozen"] = fz
            arrays[f"{name}/{i}/llr32"] = llrs[i].astype(np.float32)
            arrays[f"{name}/{i}/events"] = r["events"]
            arrays[f"{name}/{i}/u_hat"] = r["u_hat"]
            arrays[f"{name}/{i}/meta"] = np.array([r["iterations"], r["pe"], r["stop"], r["n_events"]], np.int64)
        manifest.setdefault("event_cases", []).append({"name": name, "frames": int(llrs.shape[0]),
                                                       "max_iter": max_iter})

    # RNG stream pins: raw draws and Gaussians of TrialRng (channel.cpp:31-39)
    for seed, trial in ((1, 0), (42, 7), (61803, 5), (2, 99999)):
        raw = np.zeros(16, np.uint64)
        O.REF.ref64_rng_raw(seed, trial, 16, raw.ctypes.data_as(O._u64p))
        g = np.zeros(16, np.float64)
        O.REF.ref64_rng_gaussian(seed, trial, 16, g.ctypes.data_as(O._f64p))
        arrays[f"rng/{seed}_{trial}/raw"] = raw
        arrays[f"rng/{seed}_{trial}/gauss"] = g
    # construction pins
    for n, k, z in ((2, 1, 0.5), (8, 4, 0.5), (8, 8, 0.5), (64, 32, 0.5), (1024, 512, 0.5), (256, 128, Z0),
                    (1024, 512, Z0), (4096, 2048, Z0), (16384, 8192, Z0), (128, 37, 0.3)):
        arrays[f"construct/{n}_{k}_{z:.17g}"] = O.construct(n, k, z, lib=O.REF)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()
