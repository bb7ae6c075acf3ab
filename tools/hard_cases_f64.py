"""Seeded binary64 hard-to-round set for exp2 / log (config C5 (iii); SURVEY
8d): a GPU screen, re-ranked by the REFERENCE's boundary distance.

1. crvec_hardcase_scan_f64 evaluates the fast path of 2^SCREEN seeded inputs
   per function (seed 5; the paper ranges exp2 U[-20, 20], log U[0.125, 8],
   plus wide ranges) and returns the inputs whose double-double value lies
   within 2^-THR (relative) of a binary64 rounding boundary;
2. every candidate is re-measured with the reference's own
   boundary_distance_f64 (ref: proj/src/oracle.cpp:502-563, compiled
   unmodified into oracle/_ref/libcrvec_ref.so; an ABSOLUTE distance x 2^160),
   normalised by ulp(f(x)) so exp2's tiny results do not dominate, and the TOP
   closest are kept;
3. expected outputs in all four modes come from the reference's
   ziv_correctly_round_f64 (ref: proj/src/oracle.cpp:326-345) and are checked
   equal to the oracle restatement's.

Output: tests/golden/hardcases_f64/<fn>.npz {x (uint64 bits), dist (x 2^160),
want (uint64 [n, 4])} + <fn>.json provenance. Run on a GPU box:
    python tools/hard_cases_f64.py [--screen 28] [--thr 72] [--top 512] [--out DIR]
"""
import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_15547_b200 as crvec  # noqa: E402
from oracle import oracle as O  # noqa: E402

# (lo, hi, fraction of the screen); "bits": random positive normal patterns.
# Near 1 (log) / near 0 (exp2) the value is r-dominated: the regime where the
# fast path's r^3-term rounding errors matter most.
RANGES = {"exp2": [(-20.0, 20.0, 0.625), (-1022.0, 1024.0, 0.25), (-2.0 ** -10, 2.0 ** -10, 0.125)],
          "log": [(0.125, 8.0, 0.5), ("bits", None, 0.125), (1 - 2.0 ** -8, 1 + 2.0 ** -8, 0.375)]}


def screen_inputs(name, n, gen):
    parts = []
    for lo, hi, frac in RANGES[name]:
        m = int(n * frac)
        if lo == "bits":  # random positive normal patterns
            b = torch.randint(0x0010000000000000, 0x7FEFFFFFFFFFFFFF, (m,), generator=gen, device="cuda",
                              dtype=torch.int64)
            parts.append(b.view(torch.float64))
        else:
            parts.append(torch.rand(m, generator=gen, device="cuda", dtype=torch.float64) * (hi - lo) + lo)
    return torch.cat(parts)


def scan(fn_id, x, thr, cap):
    L = crvec.lib()
    L.crvec_hardcase_scan_f64.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_double,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                          ctypes.c_void_p]
    ox = torch.zeros(cap, dtype=torch.float64, device="cuda")
    od = torch.zeros(cap, dtype=torch.float64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    rc = L.crvec_hardcase_scan_f64(fn_id, x.data_ptr(), x.numel(), thr, ox.data_ptr(), od.data_ptr(), cap,
                                   cnt.data_ptr(), ctypes.c_void_p(s.cuda_stream))
    assert rc == 0, rc
    torch.cuda.synchronize()
    k = min(int(cnt.item()), cap)
    return ox[:k].cpu().numpy(), od[:k].cpu().numpy(), int(cnt.item())


def ref_boundary_distance(name, xs):
    R = O.ref()
    R.crvec_ref_boundary_distance_f64.argtypes = [ctypes.c_int, ctypes.c_uint64] + [ctypes.c_void_p] * 3
    out = []
    for b in xs.view(np.uint64):
        d, ex, dom = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
        R.crvec_ref_boundary_distance_f64(O.FN[name], int(b), ctypes.byref(d), ctypes.byref(ex), ctypes.byref(dom))
        out.append((d.value, bool(ex.value), bool(dom.value)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--screen", type=int, default=28)
    ap.add_argument("--thr", type=float, default=72.0)
    ap.add_argument("--top", type=int, default=512)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "hardcases_f64"))
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    for fid, name in enumerate(("exp2", "log")):
        gen = torch.Generator(device="cuda")
        gen.manual_seed(5 + fid)
        t0 = time.time()
        cx, cd, total = [], [], 0
        for part in range(max(1, (1 << a.screen) >> 26)):  # 2^26 inputs per pass
            x = screen_inputs(name, min(1 << 26, 1 << a.screen), gen)
            ox, od, cnt = scan(fid, x, 2.0 ** -a.thr, 1 << 20)
            cx.append(ox)
            cd.append(od)
            total += cnt
            del x
        cx, cd = np.concatenate(cx), np.concatenate(cd)
        t_scan = time.time() - t0
        cx = np.unique(cx)
        bd = ref_boundary_distance(name, cx)
        keep = np.array([dom and not ex for d, ex, dom in bd], dtype=bool)
        cx = cx[keep]
        dabs = np.array([d for d, ex, dom in bd], dtype=np.float64)[keep]
        yrn = O.ref_f64(name, cx.view(np.uint64), 0).view(np.float64)
        ulp = np.spacing(np.abs(yrn))
        dulp = (dabs / ulp) * 2.0 ** -160  # reference distance in ulps of the result (divide first: no underflow)
        order = np.argsort(dulp, kind="stable")[: a.top]
        top = [(float(dulp[i]), float(cx[i]), float(dabs[i])) for i in order]
        xs = np.array([x for _, x, _ in top], dtype=np.float64)
        want = np.stack([O.ref_f64(name, xs.view(np.uint64), m) for m in range(4)], axis=1)
        mine = O.f64(name, xs.view(np.uint64), None)
        assert (mine == want).all(), "oracle restatement disagrees with the reference on the hard set"
        np.savez_compressed(os.path.join(a.out, f"{name}.npz"), x=xs.view(np.uint64),
                            dist=np.array([d for _, _, d in top]), dist_ulp=np.array([u for u, _, _ in top]),
                            want=want)
        meta = {"fn": name, "screen_inputs": 1 << a.screen, "ranges": [list(map(str, r)) for r in RANGES[name]],
                "seed": 5 + fid, "rng": f"torch {torch.__version__} cuda Generator",
                "fast_path_threshold": f"2^-{a.thr:g} relative", "candidates": total,
                "kept": len(top), "rank": "reference boundary_distance_f64 (x 2^160, ref: proj/src/oracle.cpp:502-563) "
                                          "/ ulp(f(x)), ascending",
                "expected": "reference ziv_correctly_round_f64, 4 modes (== oracle restatement)",
                "hardest_dist_ulps": top[0][0] if top else None,
                "kept_dist_ulps_max": top[-1][0] if top else None, "screen_seconds": round(t_scan, 2)}
        with open(os.path.join(a.out, f"{name}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        print(f"{name}: screen {t_scan:.1f}s, {total} candidates, kept {len(top)}, "
              f"hardest {meta['hardest_dist_ulps']:.3g} ulp, 512th {meta['kept_dist_ulps_max']:.3g} ulp", flush=True)


if __name__ == "__main__":
    main()
