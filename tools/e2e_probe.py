"""Developer probe: host-pointer (e2e) throughput of logf at 2^28 through the
C ABI with pinned buffers, and the raw pinned H2D / D2H copy rates."""
import ctypes, os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2605_15547_b200 as crvec
L = crvec.lib(); n = 1 << 28
x = torch.rand(n).pin_memory(); y = torch.empty(n).pin_memory()
fid = crvec.FN_IDS["logf"]
L.crvec_eval_f32(fid, x.data_ptr(), y.data_ptr(), None, n, 0)
t = time.perf_counter()
for _ in range(4): L.crvec_eval_f32(fid, x.data_ptr(), y.data_ptr(), None, n, 0)
dt = (time.perf_counter() - t) / 4
print(os.environ.get("CRVEC_LIB", "product"), f"e2e {n/dt/1e9:.2f} Gelem/s")
xd = torch.empty(n, device="cuda"); torch.cuda.synchronize()
t = time.perf_counter(); xd.copy_(x, non_blocking=True); torch.cuda.synchronize(); h2d = 4*n/(time.perf_counter()-t)/1e9
t = time.perf_counter(); y.copy_(xd, non_blocking=True); torch.cuda.synchronize(); d2h = 4*n/(time.perf_counter()-t)/1e9
print(f"h2d {h2d:.1f} GB/s d2h {d2h:.1f} GB/s", flush=True)
# duplex: H2D of x and D2H of y at the same time on two streams
yd = torch.empty(n, device="cuda"); s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(); torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1): xd.copy_(x, non_blocking=True)
with torch.cuda.stream(s2): y.copy_(yd, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"duplex h2d+d2h {4*n/dt/1e9:.1f} GB/s each way -> e2e ceiling {n/dt/1e9:.2f} Gelem/s (4 B in + 4 B out)", flush=True)
