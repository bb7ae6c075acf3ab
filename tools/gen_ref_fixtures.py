"""Golden vectors from the REFERENCE's own oracle (compiled from
/root/reference by `make -C oracle ref`), committed as tests/golden/ref_oracle.npz
so the oracle restatement stays pinned where /root/reference is absent.

Seeds follow the reference tests (ref: proj/tests/test_oracle.cpp uses 11, 2024,
5, 99): f32 inputs are uniform bit patterns + uniform reals; f64 inputs are
uniform reals on the paper's ranges plus bit patterns.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def main():
    assert O.ref_available(), "build the reference oracle first: make -C oracle ref"
    out = {}
    rng = np.random.default_rng(2024)
    x32 = np.concatenate([rng.integers(0, 2**32, 6000, dtype=np.uint64).astype(np.uint32),
                          rng.uniform(-80, 80, 3000).astype(np.float32).view(np.uint32),
                          (np.abs(rng.uniform(-80, 80, 3000)) + 0.0078125).astype(np.float32).view(np.uint32)])
    out["x32"] = x32
    for fn in O.REF_FNS:
        out[f"f32_{fn}"] = np.stack([O.ref_f32(fn, x32, m) for m in range(4)], axis=1)
    rng = np.random.default_rng(99)
    x64 = np.concatenate([rng.uniform(-20, 20, 2000), rng.uniform(0.125, 8, 2000),
                          rng.uniform(-1075, 1024, 1000),
                          rng.integers(0, 2**64, 1000, dtype=np.uint64).view(np.float64)]).view(np.uint64)
    out["x64"] = x64
    for fn in ("exp2", "log"):
        out[f"f64_{fn}"] = np.stack([O.ref_f64(fn, x64, m) for m in range(4)], axis=1)
    # reference software conversion (ref: proj/src/fpbits.cpp:164-187)
    rng = np.random.default_rng(12345)
    c = rng.integers(0, 2**64, 20000, dtype=np.uint64)
    out["cvt_in"] = c
    out["cvt_out"] = np.array([[O.ref().crvec_ref_convert_f64_to_f32(int(v), m) for m in range(4)]
                               for v in c], dtype=np.uint32)
    p = os.path.join(ROOT, "tests", "golden", "ref_oracle.npz")
    np.savez_compressed(p, **out)
    print("wrote", p, os.path.getsize(p), "bytes")


if __name__ == "__main__":
    main()
