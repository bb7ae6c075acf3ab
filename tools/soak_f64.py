"""Developer soak test: binary64 exp2 / log on the GPU vs the CPU oracle over
2^N random inputs per range (paper range, wide range, random bit patterns) in
all four modes. Prints mismatch counts and the fast-path undecided rate.
usage: python tools/soak_f64.py [log2n=23] [seed=2026]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_15547_b200 as crvec  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    import torch
    n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 23)
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 2026
    rng = np.random.default_rng(seed)
    sets = {
        "exp2": [rng.uniform(-20, 20, n), rng.uniform(-1075, 1024, n // 4),
                 rng.integers(0, 2 ** 64, n // 4, dtype=np.uint64).view(np.float64)],
        "log": [rng.uniform(0.125, 8, n), rng.uniform(0.5, 2, n // 4),
                rng.integers(0, 2 ** 63, n // 4, dtype=np.uint64).view(np.float64)],
    }
    for name, parts in sets.items():
        x = np.concatenate(parts)
        t = time.time()
        want = O.f64(name, x.view(np.uint64), None)
        to = time.time() - t
        xt = torch.from_numpy(x).cuda()
        bad = 0
        for mode in range(4):
            st = crvec.Stats() if hasattr(crvec, "Stats") else None
            got = crvec._f64(name, xt, mode, None).cpu().numpy().view(np.uint64)
            bad += int((got != want[:, mode]).sum())
        print(f"{name}: {x.size} inputs x 4 modes, mismatches {bad} (oracle {to:.0f} s)", flush=True)


if __name__ == "__main__":
    main()
