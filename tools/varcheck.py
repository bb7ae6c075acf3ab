"""Developer: bit-compare variant builds against the product library on the
config and uniform inputs of a function subset (all four modes, 2^24 elements
each). The product library is itself checked against the oracle by the tests.
usage: python tools/varcheck.py "fn1 fn2" var1 var2 ..."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_15547_b200 as crvec  # noqa: E402
from tests.inputs import device_input  # noqa: E402


def load(path):
    L = ctypes.CDLL(path)
    L.crvec_eval_f32_dev.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    return L


def main():
    fns = sys.argv[1].split()
    base = crvec.lib()
    n = 1 << 24
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for v in sys.argv[2:]:
        L = load(os.path.join(ROOT, "paper_2605_15547_b200", "variants", f"libcrvec_{v}.so"))
        bad = 0
        for name in [f for f in fns if f in ("exp2d", "logd")]:  # binary64 pair
            g = torch.Generator(device="cuda")
            g.manual_seed(13)
            lo, hi = (-20.0, 20.0) if name == "exp2d" else (0.125, 8.0)
            xs = [torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * (hi - lo) + lo,
                  torch.randint(-2**63, 2**63 - 1, (n,), generator=g, device="cuda", dtype=torch.int64).view(torch.float64)]
            for x in xs:
                for m in range(4):
                    outs = []
                    for lib in (base, L):
                        y = torch.empty_like(x)
                        f = getattr(lib, "crvec_exp2_dev" if name == "exp2d" else "crvec_log_dev")
                        assert f(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), ctypes.c_size_t(n), m, s) == 0
                        outs.append(y.view(torch.int64))
                    torch.cuda.synchronize()
                    d = int((outs[0] != outs[1]).sum())
                    if d:
                        print(f"{v} {name} mode {m}: {d} differing outputs", flush=True)
                    bad += d
        fns32 = [f for f in fns if f not in ("exp2d", "logd")]
        for fn in fns32:
            for dist in ("config", "uniform", "bits"):
                if dist == "bits":  # every bit pattern class: NaN payloads, Inf, zeros, subnormals
                    x = torch.randint(-2**31, 2**31, (n,), device="cuda", dtype=torch.int64).to(torch.int32).view(torch.float32)
                else:
                    x = device_input(fn, n, dist, seed=11)
                for m in range(4):
                    outs = []
                    for lib in (base, L):
                        y = torch.empty_like(x)
                        y2 = torch.empty_like(x)
                        rc = lib.crvec_eval_f32_dev(crvec.FN_IDS[fn], x.data_ptr(), y.data_ptr(), y2.data_ptr(), n, m, s)
                        assert rc == 0, rc
                        outs.append((y.view(torch.int32), y2.view(torch.int32)))
                    torch.cuda.synchronize()
                    d = int((outs[0][0] != outs[1][0]).sum())
                    if fn == "sincosf":
                        d += int((outs[0][1] != outs[1][1]).sum())
                    if d:
                        print(f"{v} {fn} {dist} mode {m}: {d} differing outputs", flush=True)
                    bad += d
        print(f"{v}: {'OK' if bad == 0 else 'MISMATCH ' + str(bad)}", flush=True)


if __name__ == "__main__":
    main()
