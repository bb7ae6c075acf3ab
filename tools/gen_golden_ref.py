"""Regenerate the exhaustive-sweep golden hashes of the three functions the
reference implements (exp2, log, log2 — FuncId order of
ref: proj/include/crvec/oracle.hpp:21) with the REFERENCE's OWN oracle
(oracle_all_modes_f32, ref: proj/src/oracle.cpp:347-388, compiled unmodified
into oracle/_ref/libcrvec_ref.so by `make -C oracle ref`). Test-data tool.

The result replaces tests/golden/sweep/<fn>.npy only if it equals the
restatement's hashes chunk for chunk (otherwise it stops and reports the
differing chunks); the provenance JSON then records "source": "reference build".
Progress is checkpointed to oracle/_ref/golden_partial/<fn>.ref.partial.npy
(git-ignored, outside the fixture directory), so an interrupted run resumes.

Usage: python tools/gen_golden_ref.py [exp2 log log2] [--threads T] [--step CHUNKS]
"""
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "sweep")
PARTIAL = os.path.join(ROOT, "oracle", "_ref", "golden_partial")


def ref_lib():
    L = ctypes.CDLL(O.REF_PATH)
    L.crvec_ref_sweep_hashes.restype = ctypes.c_uint64
    L.crvec_ref_sweep_hashes.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                         ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    return L


def ref_hashes(L, fn, lo, hi, threads):
    h = np.zeros((hi - lo, 4), dtype=np.uint64)
    fails = L.crvec_ref_sweep_hashes(O.FN[fn], lo, hi, h.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                     threads)
    if fails:
        raise SystemExit(f"{fn}: reference oracle threw on {fails} patterns in chunks {lo}..{hi}")
    return h


def main():
    args = [a for a in sys.argv[1:]]
    threads, step = 0, 32
    if "--threads" in args:
        i = args.index("--threads"); threads = int(args[i + 1]); del args[i:i + 2]
    if "--step" in args:
        i = args.index("--step"); step = int(args[i + 1]); del args[i:i + 2]
    fns = args or ["exp2", "log", "log2"]
    L = ref_lib()
    for fn in fns:
        os.makedirs(PARTIAL, exist_ok=True)
        part = os.path.join(PARTIAL, f"{fn}.ref.partial.npy")
        h = np.load(part) if os.path.exists(part) else np.zeros((4096, 4), dtype=np.uint64)
        done = np.load(part + ".done.npy") if os.path.exists(part + ".done.npy") else np.zeros(4096, bool)
        t0 = time.time()
        for lo in range(0, 4096, step):
            if done[lo:lo + step].all():
                continue
            h[lo:lo + step] = ref_hashes(L, fn, lo, lo + step, threads)
            done[lo:lo + step] = True
            np.save(part, h)
            np.save(part + ".done.npy", done)
            print(fn, lo + step, "/ 4096", f"{time.time() - t0:.0f}s", flush=True)
        gold = np.load(os.path.join(OUT, fn + ".npy"))
        diff = np.nonzero((gold != h).any(axis=1))[0]
        if len(diff):
            raise SystemExit(f"{fn}: reference hashes differ from the restatement in chunks {diff[:20]}")
        np.save(os.path.join(OUT, fn + ".npy"), h)
        jp = os.path.join(OUT, fn + ".json")
        meta = json.load(open(jp)) if os.path.exists(jp) else {}
        meta.update({"source": "reference build",
                     "generator": "tools/gen_golden_ref.py -> oracle/_ref/libcrvec_ref.so "
                                  "crvec_ref_sweep_hashes (oracle_all_modes_f32, ref: proj/src/oracle.cpp:347-388)",
                     "restatement_agrees": True,
                     "reference_seconds": round(time.time() - t0, 1)})
        json.dump(meta, open(jp, "w"), indent=1)
        os.remove(part)
        os.remove(part + ".done.npy")
        print(fn, "done: reference build == restatement on all 4096 chunks x 4 modes", flush=True)


if __name__ == "__main__":
    main()
