import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2605_15547_b200 as crvec
for name in ["logf", "expf", "sinf"]:
    for lo in (0, 1016, 2040):
        h, _, n0 = crvec.sweep_f32(name, lo, lo + 1, force_accurate=False)
        h1, _, n1 = crvec.sweep_f32(name, lo, lo + 1, force_accurate=True)
        print(name, lo, "acc lanes normal", n0, "forced", n1, "hash equal", bool((h == h1).all()), flush=True)
