"""Generate the exhaustive-sweep golden data with the CPU oracle (test data).

For every function and every one of the 4096 chunks of 2^20 binary32 bit
patterns, store the per-mode commutative hash
    H[c, m] = sum_{p in chunk c} mix64((oracle_m(p) << 32) | p)  mod 2^64
(see oracle/crvec_oracle.c: crvec_oracle_sweep_hashes). The GPU sweep computes
the same hash from the kernel outputs; equal hashes per chunk and mode = the
kernel matches the oracle on all 2^32 inputs of that chunk (up to a 2^-64
collision probability per chunk; any mismatching chunk is re-checked element
by element on the CPU).

Usage: python tools/gen_golden.py [fn ...]   (default: all 18 oracle functions)
Output: tests/golden/sweep/<fn>.npy (uint64[4096, 4]) + <fn>.json (provenance).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "sweep")
ORDER = ["exp", "log", "log2", "log10", "log1p", "exp2", "sin", "cos", "tan", "exp10",
         "expm1", "rsqrt", "atan", "asin", "acos", "sinh", "cosh", "tanh"]


def main():
    fns = sys.argv[1:] or ORDER
    os.makedirs(OUT, exist_ok=True)
    for fn in fns:
        path = os.path.join(OUT, fn + ".npy")
        if os.path.exists(path):
            print(fn, "exists, skipping", flush=True)
            continue
        t0 = time.time()
        O.lib().crvec_oracle_reset_counters()
        parts = []
        for lo in range(0, 4096, 256):
            parts.append(O.sweep_hashes(fn, lo, lo + 256))
        h = np.concatenate(parts)
        dt = time.time() - t0
        if O.lib().crvec_oracle_cap_failures():
            raise SystemExit(f"{fn}: oracle precision cap hit")
        np.save(path + ".tmp.npy", h)
        os.replace(path + ".tmp.npy", path)
        meta = {"fn": fn, "chunks": 4096, "chunk_bits": 20, "modes": ["rne", "rz", "ru", "rd"],
                "seconds": round(dt, 1), "threads": os.cpu_count(),
                "mpfr_calls": int(O.lib().crvec_oracle_mpfr_calls()),
                "ld_rung_decided": int(O.lib().crvec_oracle_ld_decided()),
                "total_hash": [int(v) for v in (h.sum(axis=0, dtype=np.uint64))]}
        with open(os.path.join(OUT, fn + ".json"), "w") as f:
            json.dump(meta, f, indent=1)
        print(fn, f"{dt:.0f}s", meta["mpfr_calls"], "mpfr calls", flush=True)


if __name__ == "__main__":
    main()
