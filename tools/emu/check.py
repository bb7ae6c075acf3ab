"""DEVELOPER TOOL: compare the g++ build of the device math with the oracle."""
import ctypes, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O

E = ctypes.CDLL(os.path.join(ROOT, "tools/emu/libemu.so"))
E.emu_eval.argtypes = [ctypes.c_int, O._u32p, O._u32p, ctypes.c_uint64, ctypes.c_int,
                       ctypes.POINTER(ctypes.c_uint64)]

def emu(fn, x, force=0):
    x = np.ascontiguousarray(x, np.uint32); y = np.empty((x.size, 4), np.uint32)
    s = ctypes.c_uint64(0)
    E.emu_eval(O.FN[fn], O._p32(x), O._p32(y), x.size, force, ctypes.byref(s))
    return y, s.value

def inputs(fn, n, seed=1):
    rng = np.random.default_rng(seed)
    parts = [rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)]
    lo, hi = {"exp": (-110, 95), "exp2": (-155, 135), "exp10": (-50, 45), "expm1": (-20, 95),
              "sinh": (-95, 95), "cosh": (-95, 95), "tanh": (-12, 12), "log": (0, 10),
              "log2": (0, 10), "log10": (0, 10), "log1p": (-1, 5), "sin": (-100, 100),
              "cos": (-100, 100), "tan": (-100, 100), "asin": (-1, 1), "acos": (-1, 1),
              "atan": (-50, 50), "rsqrt": (0, 100)}[fn]
    parts.append(rng.uniform(lo, hi, n).astype(np.float32).view(np.uint32))
    parts.append(rng.uniform(-1, 1, n // 4).astype(np.float32).view(np.uint32))
    return np.concatenate(parts)

fns = sys.argv[1:] or list(O.FN)
for fn in fns:
    x = inputs(fn, 100000)
    t = time.time()
    want = O.f32(fn, x, None)
    got, slow = emu(fn, x)
    got2, slow2 = emu(fn, x, 1)
    bad = np.nonzero((got != want).any(1))[0]
    bad2 = np.nonzero((got2 != want).any(1))[0]
    print(f"{fn:6s} fast-mismatch {len(bad):6d} (slow lanes {slow:6d})  forced-accurate mismatch {len(bad2):6d}  {time.time()-t:.1f}s")
    for i in list(bad[:3]) + list(bad2[:2]):
        xv = x[i].view(np.float32)
        print("    x=%r (0x%08x) want %s got %s acc %s" % (float(xv), x[i], [hex(v) for v in want[i]], [hex(v) for v in got[i]], [hex(v) for v in got2[i]]))
