"""Developer: per-function time of the exhaustive 2^32 x 4-mode sweep on one GPU."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_15547_b200 as crvec  # noqa: E402
from paper_2605_15547_b200 import sweep  # noqa: E402

fns = crvec.F32_FUNCS + ["sincosf"]
sweep.run_device(fns, 0, sweep.CHUNKS, reduce=False)
torch.cuda.synchronize()
for fn in fns:
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sweep.run_device([fn], 0, 1)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"{fn:8s} {best:7.2f} ms", flush=True)
