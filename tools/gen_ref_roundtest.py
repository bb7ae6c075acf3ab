"""Golden vectors for the binary64 round test from the REFERENCE's own
round_test_lane (ref: proj/src/kernels_f64.cpp:63-76, compiled unmodified into
oracle/_ref/libcrvec_refk.so by `make -C oracle ref`): tests/golden/ref_round_test.npz.

Cases (seed 5150, a seed of the reference tests): DD pairs hi + lo with
|lo| <= ulp(hi)/2 around binary64 rounding boundaries (representable values
and midpoints, +-a few ulps of lo), random relative / absolute bounds, and
scales 2^n that put the result in the normal, subnormal, underflow-to-zero and
overflow ranges; all four modes.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def cases(n, rng):
    hi = rng.uniform(1.0, 2.0, n) * np.exp2(rng.integers(-20, 20, n)).astype(np.float64)
    hi *= np.where(rng.random(n) < 0.5, -1.0, 1.0)
    ulp = np.spacing(np.abs(hi))
    kind = rng.integers(0, 4, n)
    lo = np.where(kind == 0, 0.0,
         np.where(kind == 1, 0.5 * ulp,                      # exactly on a midpoint
         np.where(kind == 2, (0.5 + rng.integers(-3, 4, n) * 2.0**-40) * ulp,
                  rng.uniform(-0.5, 0.5, n) * ulp)))
    lo *= np.where(rng.random(n) < 0.5, -1.0, 1.0)
    # renormalise (hi, lo) with fast two-sum so hi = RN(hi + lo)
    s = hi + lo
    lo = lo - (s - hi)
    hi = s
    eps_rel = np.where(rng.random(n) < 0.3, 0.0, np.exp2(-rng.uniform(55, 110, n)))
    eps_abs = np.where(rng.random(n) < 0.7, 0.0, np.exp2(-rng.uniform(1060, 1100, n)))
    scale = np.where(rng.random(n) < 0.5, 0,
            np.where(rng.random(n) < 0.5, rng.integers(-1100, -1000, n),
                     rng.integers(1000, 1030, n))).astype(np.int64)
    return hi, lo, scale, eps_rel, eps_abs


def main():
    K = O.refk()
    import ctypes
    rng = np.random.default_rng(5150)
    hi, lo, scale, er, ea = cases(6000, rng)
    val = np.empty((hi.size, 4), dtype=np.float64)
    dec = np.empty((hi.size, 4), dtype=np.uint8)
    v = ctypes.c_double()
    for i in range(hi.size):
        for m in range(4):
            dec[i, m] = K.crvec_refk_round_test_lane(float(hi[i]), float(lo[i]), int(scale[i]), float(er[i]),
                                                     float(ea[i]), m, ctypes.byref(v))
            val[i, m] = v.value
    p = os.path.join(ROOT, "tests", "golden", "ref_round_test.npz")
    np.savez_compressed(p, hi=hi, lo=lo, scale=scale, eps_rel=er, eps_abs=ea, value=val, decided=dec)
    print("wrote", p, os.path.getsize(p), "bytes;", int((dec == 0).sum()), "undecided lanes")


if __name__ == "__main__":
    main()
