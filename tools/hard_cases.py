"""Find the hardest-to-round binary32 inputs of every function (GPU screen +
oracle confirmation) and write a corpus under tests/golden/hardcases/.

1. crvec_hardcase_scan_f32 evaluates all 2^32 patterns on the double-double
   path and returns those within 2^-THR (relative) of a rounding boundary;
2. the candidates are ranked by that distance, and the top N are re-measured
   with the oracle's MPFR boundary distance (restating ref:
   proj/src/oracle.cpp:443-500) and correctly rounded in all four modes by the
   oracle;
3. corpus lines: `<bits> <hex-float x> <distance*2^160> <rne> <rz> <ru> <rd>`
   (the SPEC corpus format, ref: SPEC.md verify "HardCaseRecord", extended
   with per-mode expected outputs).

Usage (on a GPU box): python tools/hard_cases.py [--thr 46] [--top 64] [fn ...]
"""
import argparse
import ctypes
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_15547_b200 as crvec  # noqa: E402
from oracle import oracle as O  # noqa: E402

OUT = os.environ.get("CRVEC_HARDCASE_OUT", os.path.join(ROOT, "tests", "golden", "hardcases"))


def scan(name, thr, cap=1 << 20):
    L = crvec.lib()
    L.crvec_hardcase_scan_f32.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                          ctypes.c_void_p]
    bits = torch.zeros(cap, dtype=torch.int32, device="cuda")
    dist = torch.zeros(cap, dtype=torch.float64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    for lo in range(0, 4096, 512):
        rc = L.crvec_hardcase_scan_f32(crvec.FN_IDS[name], lo, lo + 512, 2.0 ** -thr, bits.data_ptr(),
                                       dist.data_ptr(), cap, cnt.data_ptr(), ctypes.c_void_p(s.cuda_stream))
        assert rc == 0, rc
    torch.cuda.synchronize()
    n = min(int(cnt.item()), cap)
    return bits[:n].cpu().numpy().view(np.uint32), dist[:n].cpu().numpy(), int(cnt.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--thr", type=float, default=46.0)
    ap.add_argument("--top", type=int, default=64)
    ap.add_argument("fns", nargs="*")
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    L = O.lib()
    L.crvec_oracle_boundary_distance_f32.argtypes = [ctypes.c_int, ctypes.c_uint32] + [ctypes.c_void_p] * 3
    for name in a.fns or crvec.F32_FUNCS:
        t0 = time.time()
        bits, dist, total = scan(name, a.thr)
        t1 = time.time() - t0
        keep = dist > 0  # distance 0: algebraically exact results (2^k, log2(2^k)), not hard cases
        bits, dist = bits[keep], dist[keep]
        order = np.argsort(dist, kind="stable")[: 4 * a.top]
        cand = bits[order]
        ofn = crvec.ORACLE_NAME[name]
        exact = []
        for b in cand:
            d, ex, dom = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
            L.crvec_oracle_boundary_distance_f32(O.FN[ofn], int(b), ctypes.byref(d), ctypes.byref(ex),
                                                 ctypes.byref(dom))
            if dom.value and not ex.value:
                exact.append((d.value, int(b)))
        exact.sort()
        top = exact[: a.top]
        xs = np.array([b for _, b in top], dtype=np.uint32)
        want = O.f32(ofn, xs, None) if len(xs) else np.zeros((0, 4), np.uint32)
        path = os.path.join(OUT, f"{name}.txt")
        with open(path, "w") as f:
            f.write(f"# {name}: hardest binary32 inputs (GPU double-double screen over all 2^32 patterns,\n"
                    f"# {total} within 2^-{a.thr:g} of a rounding boundary; top {len(top)} re-ranked by the\n"
                    f"# oracle's MPFR boundary distance). bits hexfloat dist*2^160 rne rz ru rd\n")
            for (d, b), w in zip(top, want):
                x = float(np.array([b], np.uint32).view(np.float32)[0])
                f.write(f"{b:08x} {x.hex()} {d:.6g} {w[0]:08x} {w[1]:08x} {w[2]:08x} {w[3]:08x}\n")
        print(f"{name}: scan {t1:.2f}s, {total} candidates, {len(top)} kept, "
              f"hardest d*2^160 = {top[0][0] if top else float('nan'):.4g}", flush=True)


if __name__ == "__main__":
    main()
