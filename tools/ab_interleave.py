"""Developer A/B: several libcrvec builds loaded side by side in ONE process
(ctypes handles on distinct paths), each function's 2^28 input generated
once, then R rounds in which every variant runs K event-timed launches in
turn (ABCABC...). Reports, per function and variant, the median over rounds
of the per-round median launch time, and the ratio to the first variant, so
box-level drift (clocks, power) hits every variant alike.

usage: python tools/ab_interleave.py [--fn f ...] [--dist config|uniform]
           [--rounds R] [--reps K] base var1 var2 ...
       (base = the product libcrvec.so; other names = variants/libcrvec_<v>.so)"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_15547_b200 as crvec  # noqa: E402
from tests.inputs import device_input  # noqa: E402


def load(v):
    p = os.path.join(ROOT, "paper_2605_15547_b200",
                     "libcrvec.so" if v == "base" else os.path.join("variants", f"libcrvec_{v}.so"))
    L = ctypes.CDLL(p)
    L.crvec_eval_f32_dev.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    for f in ("crvec_exp2_dev", "crvec_log_dev"):
        getattr(L, f).argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--fn", nargs="*")
    ap.add_argument("--dist", default="config")
    ap.add_argument("--rounds", type=int, default=7)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--mode", type=int, default=0)
    a = ap.parse_args()
    n = 1 << 28
    libs = [load(v) for v in a.variants]
    s = torch.cuda.current_stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    print(f"-- variants: {a.variants}")
    names = a.fn or (crvec.F32_FUNCS + ["sincosf"])
    if "f64" in names:  # binary64 pair: 2^26 uniform inputs as in tools/perf.py
        names = [m for m in names if m != "f64"]
        n64 = 1 << 26
        rng = np.random.default_rng(5)
        for nm, xs in (("exp2", rng.uniform(-20, 20, n64)), ("log", rng.uniform(0.125, 8, n64))):
            x = torch.from_numpy(xs).cuda()
            yy = torch.empty_like(x)
            fns = [getattr(L, f"crvec_{nm}_dev") for L in libs]
            for fn in fns:
                for _ in range(2):
                    fn(x.data_ptr(), yy.data_ptr(), n64, a.mode, sp)
            torch.cuda.synchronize()
            per = [[] for _ in libs]
            for _ in range(a.rounds):
                for i, fn in enumerate(fns):
                    ts = []
                    for _ in range(a.reps):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(s)
                        fn(x.data_ptr(), yy.data_ptr(), n64, a.mode, sp)
                        e1.record(s)
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1))
                    per[i].append(float(np.median(ts)))
            g = [n64 / (float(np.median(p)) * 1e-3) / 1e9 for p in per]
            print(f"{nm + '(f64)':8s} " + " ".join(f"{v:9.1f}" for v in g) + "   " +
                  " ".join(f"{v / g[0]:7.3f}" for v in g[1:]), flush=True)
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    y2 = torch.empty(n, dtype=torch.float32, device="cuda")
    print(f"-- {a.dist}, 2^28, mode {a.mode}: Gelem/s (median of {a.rounds} interleaved rounds x "
          f"{a.reps} launches); ratio to {a.variants[0]}")
    print("fn       " + " ".join(f"{v:>9s}" for v in a.variants) + "   " +
          " ".join(f"{v:>7s}" for v in a.variants[1:]))
    for name in names:
        x = device_input(name, n, a.dist)
        fid = crvec.FN_IDS[name]
        for L in libs:  # warm-up (module load, first-launch costs)
            for _ in range(2):
                L.crvec_eval_f32_dev(fid, x.data_ptr(), y.data_ptr(), y2.data_ptr(), n, a.mode, sp)
        torch.cuda.synchronize()
        per = [[] for _ in libs]
        for _ in range(a.rounds):
            for i, L in enumerate(libs):
                ts = []
                for _ in range(a.reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    L.crvec_eval_f32_dev(fid, x.data_ptr(), y.data_ptr(), y2.data_ptr(), n, a.mode, sp)
                    e1.record(s)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                per[i].append(float(np.median(ts)))
        g = [n / (float(np.median(p)) * 1e-3) / 1e9 for p in per]
        print(f"{name:8s} " + " ".join(f"{v:9.1f}" for v in g) + "   " +
              " ".join(f"{v / g[0]:7.3f}" for v in g[1:]), flush=True)
        print(json.dumps({"fn": name, "dist": a.dist, "gelem_s": dict(zip(a.variants, g))}), file=sys.stderr)
        del x


if __name__ == "__main__":
    main()
