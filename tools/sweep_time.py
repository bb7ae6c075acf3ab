"""Developer: time the exhaustive 2^32 x 4-mode sweep of all 19 functions on
one GPU (device events; warm-up excluded) and compare with the golden hashes.
usage: [CRVEC_LIB=...] python tools/sweep_time.py [reps]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_15547_b200 as crvec  # noqa: E402
from paper_2605_15547_b200 import sweep  # noqa: E402

fns = crvec.F32_FUNCS + ["sincosf"]
sweep.run_device(fns, 0, sweep.CHUNKS, reduce=False)  # warm-up (module loading)
torch.cuda.synchronize()
ts = []
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    rows, table, _ = sweep.run_device(fns, 0, 1)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 1e3)
res = sweep.compare(rows, table.cpu().numpy().view(np.uint64), ROOT, crvec.ORACLE_NAME)
bad = sum(len(v) for v in res.values() if v is not None)
print(f"{os.environ.get('CRVEC_LIB', 'product')}: sweep {min(ts):.3f} s (best of {len(ts)}), "
      f"mismatching chunks {bad}", flush=True)
