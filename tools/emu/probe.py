"""DEVELOPER TOOL: max observed fast-path error (double ulps) vs tolerance E."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O
from tests.inputs import RANGES
import paper_2605_15547_b200 as crvec
E = ctypes.CDLL(os.path.join(ROOT, "tools/emu/libemu.so"))
E.emu_probe.restype = ctypes.c_double
E.emu_probe.argtypes = [ctypes.c_int, O._u32p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint32)]
rng = np.random.default_rng(11)
for name in crvec.F32_FUNCS:
    lo, hi = RANGES[name]
    x = np.concatenate([rng.integers(0, 2**32, 400000, dtype=np.uint64).astype(np.uint32),
                        rng.uniform(lo, hi, 400000).astype(np.float32).view(np.uint32)])
    e = ctypes.c_uint32()
    w = E.emu_probe(O.FN[crvec.ORACLE_NAME[name]], O._p32(x), x.size, ctypes.byref(e))
    print(f"{name:8s} max err {w:8.2f} ulp   tolerance E = {e.value:5d}   margin x{e.value / max(w, 1e-9):.1f}")
