"""Per-function device throughput at 2^28 elements (CUDA events), all 19
binary32 functions + the binary64 pair; prints one JSON line per function and
a summary table. Usage: python tools/perf.py [--n LOG2N] [--fn name ...]"""
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
from tests.inputs import device_input, log_family_input, mixed_f32, trig_input  # noqa: E402


def inputs(name, n, dist="config"):
    if dist == "uniform":
        rng = np.random.default_rng(7)
        lo, hi = __import__("tests.inputs", fromlist=["RANGES"]).RANGES[name]
        return rng.uniform(lo, hi, n).astype(np.float32).view(np.uint32)
    if name in ("logf", "log2f", "log10f", "log1pf"):
        return log_family_input(name, n)
    if name in ("sinf", "cosf", "tanf", "sincosf"):
        return trig_input(n)
    rng = np.random.default_rng(7)
    lo, hi = __import__("tests.inputs", fromlist=["RANGES"]).RANGES[name]
    return rng.uniform(lo, hi, n).astype(np.float32).view(np.uint32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--fn", nargs="*")
    ap.add_argument("--mode", type=int, default=0)
    ap.add_argument("--dist", default="config", choices=["config", "uniform", "nospecial"])
    ap.add_argument("--no-f64", action="store_true")
    a = ap.parse_args()
    n = 1 << a.n
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    L = crvec.lib()
    s = torch.cuda.current_stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    names = a.fn or (crvec.F32_FUNCS + ["sincosf"])
    want64 = (not a.fn and not a.no_f64) or (a.fn and "f64" in a.fn)
    names = [nm for nm in names if nm != "f64"]
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    y2 = torch.empty(n, dtype=torch.float32, device="cuda")
    rows = []
    for name in names:
        x = device_input(name, n, "config" if a.dist == "nospecial" else a.dist,
                         specials=a.dist != "nospecial")
        fid = crvec.FN_IDS[name]
        for _ in range(3):
            L.crvec_eval_f32_dev(fid, x.data_ptr(), y.data_ptr(), y2.data_ptr(), n, a.mode, sp)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            L.crvec_eval_f32_dev(fid, x.data_ptr(), y.data_ptr(), y2.data_ptr(), n, a.mode, sp)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = float(np.median(ts))
        bpe = 12 if name == "sincosf" else 8
        r = {"fn": name, "n": n, "ms": t * 1e3, "gelem_s": n / t / 1e9, "gb_s": bpe * n / t / 1e9,
             "frac_hbm": bpe * n / t / 1e9 / peak}
        rows.append(r)
        print(json.dumps(r), flush=True)
        del x
    # binary64
    if hasattr(L, "crvec_exp2_dev") and want64:
        rng = np.random.default_rng(5)
        n64 = 1 << 26
        for name, xs in (("exp2", rng.uniform(-20, 20, n64)), ("log", rng.uniform(0.125, 8, n64))):
            x = torch.from_numpy(xs).cuda()
            yy = torch.empty_like(x)
            fn = getattr(L, f"crvec_{name}_dev")
            for _ in range(3):
                fn(x.data_ptr(), yy.data_ptr(), n64, a.mode, sp)
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                fn(x.data_ptr(), yy.data_ptr(), n64, a.mode, sp)
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
            t = float(np.median(ts))
            r = {"fn": name + "(f64)", "n": n64, "ms": t * 1e3, "gelem_s": n64 / t / 1e9,
                 "gb_s": 16 * n64 / t / 1e9, "frac_hbm": 16 * n64 / t / 1e9 / peak}
            rows.append(r)
            print(json.dumps(r), flush=True)
    print("\n%-10s %8s %9s %8s" % ("fn", "ms", "Gelem/s", "%HBM"))
    for r in rows:
        print("%-10s %8.3f %9.1f %7.1f%%" % (r["fn"], r["ms"], r["gelem_s"], 100 * r["frac_hbm"]))


if __name__ == "__main__":
    main()
