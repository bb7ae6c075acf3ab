"""DEVELOPER TOOL: g++ build of the binary64 device math vs the oracle."""
import ctypes, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O
E = ctypes.CDLL(os.path.join(ROOT, "tools/emu/libemu64.so"))
for nm in ("emu64",):
    getattr(E, nm).argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), ctypes.c_uint64, ctypes.c_int, O._u64p]
E.emu64_acc.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), ctypes.c_uint64, O._u64p]
dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
def run(fn, x, force=0, acc=False):
    x = np.ascontiguousarray(x, np.float64); y = np.empty((x.size, 4)); st = np.zeros(4, np.uint64)
    if acc: E.emu64_acc(fn, dp(x), dp(y), x.size, O._p64(st))
    else: E.emu64(fn, dp(x), dp(y), x.size, force, O._p64(st))
    return y.view(np.uint64), st
rng = np.random.default_rng(5)
for fn, name in ((0, "exp2"), (1, "log")):
    if fn == 0:
        xs = np.concatenate([rng.uniform(-20, 20, 40000), rng.uniform(-1075, 1024, 20000),
                             rng.integers(0, 2**64, 20000, dtype=np.uint64).view(np.float64),
                             np.array([0.0, -0.0, 1.0, -1.0, 1023.5, -1074.5, -1075.0, -1074.9, -1022.5, 2.0**-60, -2.0**-60, 0.5, np.inf, -np.inf, np.nan, 1023.999999])])
    else:
        xs = np.concatenate([rng.uniform(0.125, 8, 40000), rng.uniform(0.5, 2, 20000),
                             rng.integers(0, 2**63, 20000, dtype=np.uint64).view(np.float64),
                             1 + 2.0 ** -np.arange(1, 53), 1 - 2.0 ** -np.arange(1, 54),
                             np.array([0.0, -0.0, 1.0, -1.0, 5e-324, 2.2e-308, np.inf, -np.inf, np.nan, 2.0, 10.0])])
    t = time.time(); want = O.f64(name, xs.view(np.uint64), None); t1 = time.time() - t
    got, st = run(fn, xs)
    bad = np.nonzero((got != want).any(1))[0]
    print(f"{name}: fast+acc mismatches {len(bad)}  accurate lanes {st[0]} undecided {st[1]}  (oracle {t1:.1f}s)")
    for i in bad[:4]:
        print("   x=%r want %s got %s" % (xs[i], [hex(v) for v in want[i]], [hex(v) for v in got[i]]))
    sel = np.nonzero(np.isfinite(xs) & ((xs > 0) | (fn == 0)))[0][:3000]
    gota, sta = run(fn, xs[sel], acc=True)
    bada = np.nonzero((gota != want[sel]).any(1))[0]
    print(f"{name}: accurate-path-only mismatches {len(bada)} / {len(sel)}  undecided {sta[1]}")
    for i in bada[:4]:
        j = sel[i]; print("   x=%r want %s got %s" % (xs[j], [hex(v) for v in want[j]], [hex(v) for v in gota[i]]))
