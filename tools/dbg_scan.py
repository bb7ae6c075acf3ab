import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tools.hard_cases as H
for thr in (20, 30, 40, 46):
    b, d, tot = H.scan("exp2f", thr, cap=1 << 16)
    print("thr", thr, "total", tot, "first", [hex(int(v)) for v in b[:3]], d[:3], flush=True)
