"""bench.py — headline benchmark (BASELINE.json metric) for crvec-b200.

Metric: "CR Gelem/s per function at 2^28 fp32 (% HBM roofline); 2^32 sweep s @1-8 GPU".

Workload at N=1 (BASELINE.json configs[1]): the log family — logf, log2f,
log10f, log1pf — each over 2^28 binary32 inputs including denormals / Inf /
NaN (tests/inputs.py:log_family_input), RNE. One step = one pass of the four
kernels over their 2^28 inputs (4 * 2^28 elements, 8 GiB of HBM traffic).
Inputs are 1 GiB per function (> 126 MB L2), so no L2 flush is needed.

  value      device-resident throughput (Gelem/s, all ranks), CUDA events on
             the launch stream, barrier + synchronize around the K timed steps,
             max over ranks.
  e2e        same metric through the C ABI host-pointer entry points
             (crvec_logf ... with pinned host buffers): every step includes the
             H2D copy of the inputs and the D2H copy of the results.
  roofline   the dominant kernel (the slowest of the four k_map_vec launches): 8 algorithmic bytes per
             element x 2^28 / its average event-timed duration vs the measured
             HBM copy bandwidth of MEASURED_PEAKS.json.
  cpu_baseline  the reference's own CPU kernel on the path, cr_log2f<16>
             (Backend::vector; compiled unmodified from the reference's sources
             with generated tables by `make -C oracle ref`), on a bounded sample
             of the config-2 log2f input, all host threads, rank 0; its 1-core
             rate and the reference oracle's rate beside it.
  sweep      exhaustive 2^32 x 4-mode sweep of all 19 functions, sharded by
             chunk range across ranks, one NCCL all_reduce of the per-chunk
             hashes; seconds (max over ranks) and mismatching chunks vs golden.

--impl reference times the reference's cr_log2f<16> alone on the host cores
(rank 0; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CR Gelem/s per function at 2^28 fp32 (% HBM roofline); 2^32 sweep s @1-8 GPU"
LOG_FAMILY = ["logf", "log2f", "log10f", "log1pf"]
N_ELEM = 1 << 28


def ncu_traffic(fn: str):
    """DRAM bytes (read + write) per launch of k_map_vec<fn> from the committed
    `ncu --set full` capture (profiles/rNN/ncu_full_<fn>.csv, latest round), or None."""
    import csv
    p = None
    for rnd in ("r02", "r01"):
        c = os.path.join(ROOT, "profiles", rnd, f"ncu_full_{fn}.csv")
        if os.path.exists(c):
            p = c
            break
    if p is None:
        return None
    try:
        rows = list(csv.reader(open(p)))
        hdr, units, vals = rows[0], rows[1], rows[2]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            tot += float(vals[i].replace(",", "")) * scale[units[i]]
        return tot
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region (NVML every
    5 ms; falls back to nvidia-smi polling when NVML is unavailable)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, mx, rs))
                self._stop.wait(0.005)
            return
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                v = [t.strip() for t in out.split(",")]
                bits = sum(b for b, on in zip((0x8, 0x40, 0x20, 0x4), v[2:6]) if on.lower() == "active")
                self.samples.append((float(v[0]), float(v[1]), bits))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        # the sampler is live (NVML initialised, one sample taken) before the
        # timed region starts, so even a short region is sampled
        t0 = time.time()
        while not self.samples and time.time() - t0 < 10 and self._t.is_alive():
            time.sleep(0.001)
        self._n0 = len(self.samples)
        return self

    def sample_now(self):
        """One synchronous sample (taken at the end of the timed region)."""
        try:
            import pynvml
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                 pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM),
                                 pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        except Exception:
            pass

    def __exit__(self, *a):
        self.sample_now()
        self._stop.set()
        self._t.join(timeout=10)
        # keep the samples taken during the region (plus the one at its end)
        if len(self.samples) > self._n0:
            self.samples = self.samples[self._n0:]

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for s in self.samples for bit, name in self.REASONS.items() if s[2] & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(s[1] for s in self.samples)),
                "reasons": reasons, "samples": len(self.samples), "source": "nvml 5 ms"}


def dist_init(backend: str = "nccl"):
    """One process per GPU (torchrun env). NCCL over NVLink on GPUs; gloo for
    the CPU self-test of the launch / shard / reduce path."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            # create the communicator now (untimed): one tiny collective
            t = torch.ones(1, device="cuda")
            dist.all_reduce(t)
            torch.cuda.synchronize()
        else:
            dist.init_process_group("gloo")
        dist.barrier()
    elif backend == "nccl" and torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def self_launch(argv, n: int) -> int:
    """`bench.py --gpus N` run as a plain process (no torchrun environment):
    re-exec under torch.distributed.run with N ranks on this node, rendezvous on
    127.0.0.1, and return the launcher's exit status."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")         # communicator lines (nranks) for the record
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + argv
    return subprocess.run(cmd, env=env).returncode


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------ reference arm --
REF_WORKLOAD = ("log2f over the config-2 log-family input distribution (tests/inputs.py log_family_input, "
                "seed 4), RNE, through the reference's cr_log2f<16> (Backend::vector) -- log2f is the "
                "only log-family function the reference implements (ref: proj/src/kernels_f32.cpp:119-191); "
                "std::thread over 16K-element chunks, all host cores")


_REF_INPUT = {}


def cpu_reference_kernel(sample: int, threads: int = 0, vector: bool = True, reps: int = 1):
    """The reference's own CPU kernel on the path: cr_log2f<16> (Backend::vector,
    compiled unmodified from /root/reference with generated tables into
    oracle/_ref/libcrvec_refk*.so), `reps` passes over a sample of the config-2
    log2f input (generated once per size). Returns (Gelem/s, seconds)."""
    from oracle import oracle as O
    from tests.inputs import log_family_input
    if sample not in _REF_INPUT:
        _REF_INPUT[sample] = log_family_input("log2f", sample, seed=4)
    x = _REF_INPUT[sample]
    O.refk_f32("log2", x[:4096], 0, threads, vector)  # warm the thread pool / tables
    t0 = time.perf_counter()
    for _ in range(reps):
        O.refk_f32("log2", x, 0, threads, vector)
    dt = time.perf_counter() - t0
    return sample * reps / dt / 1e9, dt


def cpu_reference_oracle(sample: int, threads: int = 0):
    """The reference's Ziv oracle (ziv_correctly_round_f32, FuncId::log), the
    only reference CPU path for logf. Returns (Gelem/s, seconds)."""
    from oracle import oracle as O
    from tests.inputs import log_family_input
    x = log_family_input("logf", sample, seed=3)
    t0 = time.perf_counter()
    O.ref_f32("log", x, 0, threads)
    dt = time.perf_counter() - t0
    return sample / dt / 1e9, dt


def cpu_baseline_record(sample: int):
    """cpu_baseline: the reference's vector kernel on all host cores (value),
    with its 1-thread rate and the reference oracle's rate beside it."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    if not O.refk_available():
        v, dt = cpu_reference_oracle(min(sample, 1 << 21))
        return {"value": v, "unit": "Gelem/s", "cores": cores, "kind": "reference",
                "sample": f"reference oracle ziv_correctly_round_f32(log), {min(sample, 1 << 21)} elements, {dt:.2f} s"}
    v, dt = cpu_reference_kernel(sample, reps=4)  # ~10 core-seconds of the reference kernel
    v1, dt1 = cpu_reference_kernel(sample // 16, threads=1)
    vo, dto = cpu_reference_oracle(1 << 20)
    return {"value": v, "unit": "Gelem/s", "cores": cores, "kind": "reference",
            "sample": f"4 passes over {sample} elements of the config-2 log2f input through cr_log2f<16> "
                      f"(Backend::vector), {dt:.2f} s on {cores} threads ({dt * cores:.1f} core-s)",
            "paths": {"cr_log2f<16> vector, all cores": {"gelem_s": v, "cores": cores},
                      "cr_log2f<16> vector, 1 core": {"gelem_s": v1, "cores": 1},
                      "ziv_correctly_round_f32(log) oracle, all cores": {"gelem_s": vo, "cores": cores}},
            "isa": os.path.basename(O.refk_path() or "")}


def run_reference(args, rank, world):
    """Reference arm: the reference's own CPU implementation of the path on the
    box's host cores (rank 0 only; other ranks exit 0 without work). One step =
    one bounded sample of the workload through cr_log2f<16>."""
    if rank != 0:
        return
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    sample = args.ref_sample
    if not O.refk_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libcrvec_refk*.so not built "
                          "(make -C oracle ref with /root/reference present)"}), flush=True)
        return
    for _ in range(args.warmup):
        cpu_reference_kernel(sample)
    ts = []
    for _ in range(args.steps):
        _, dt = cpu_reference_kernel(sample)
        ts.append(dt)
    secs = float(np.sum(ts))
    value = sample * args.steps / secs / 1e9
    v1, _ = cpu_reference_kernel(max(1 << 16, sample // 16), threads=1)
    vo, dto = cpu_reference_oracle(1 << 20)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gelem/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": REF_WORKLOAD, "sample_elems_per_step": sample},
        "cpu_baseline": {"value": value, "unit": "Gelem/s", "cores": cores, "kind": "reference",
                         "sample": f"{sample} elements of the config-2 log2f input per step",
                         "paths": {"cr_log2f<16> vector, all cores": {"gelem_s": value, "cores": cores},
                                   "cr_log2f<16> vector, 1 core": {"gelem_s": v1, "cores": 1},
                                   "ziv_correctly_round_f32(log) oracle, all cores": {"gelem_s": vo,
                                                                                       "cores": cores}},
                         "isa": os.path.basename(O.refk_path() or "")},
        "e2e": {"value": value, "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ sweep ----
def run_sweep(rank, world, fns):
    """Exhaustive 2^32 x 4-mode sweep of `fns`: chunk ranges sharded across
    ranks (paper_2605_15547_b200/sweep.py run_device): the sweep kernels
    accumulate every function's chunk hashes into ONE device table, then ONE
    NCCL all_reduce; no host round trip or per-function synchronisation inside
    the timed region. Seconds = max over ranks of the device time from the
    first sweep launch to the end of the all_reduce (communicator created
    before, untimed); one D2H copy of the table after the region."""
    import torch
    import paper_2605_15547_b200 as crvec
    from paper_2605_15547_b200 import sweep
    # untimed warm-up: one chunk per function (shard 0 of 4096, no collective) so the
    # sweep kernels are loaded (CUDA lazy module loading) before the timed region
    sweep.run_device(fns, 0, sweep.CHUNKS, reduce=False)
    barrier(world)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(s)
    rows, table, _ = sweep.run_device(fns, rank, world)
    ev1.record(s)
    torch.cuda.synchronize()
    secs = max_over_ranks(ev0.elapsed_time(ev1) / 1e3, world)
    host = table.cpu().numpy().view(np.uint64)
    res = sweep.compare(rows, host, ROOT, crvec.ORACLE_NAME) if rank == 0 else {}
    mism = sum(len(v) for v in res.values() if v is not None)
    checked = sum(1 for v in res.values() if v is not None)
    return secs, mism, checked, len(rows)


def run_selftest(args, rank, world):
    """CPU self-test of the multi-rank plumbing bench.py uses on GPUs (gloo):
    self-launch, chunk sharding, one all_reduce of the hash table, max-over-
    ranks timing. Each rank fills its shard with a deterministic stand-in hash
    (no kernels, no oracle), rank 0 checks the reduced table equals the full
    single-rank table. Prints one JSON line."""
    import torch
    from paper_2605_15547_b200 import sweep

    def fill(names, lo, hi):
        c = np.arange(lo, hi, dtype=np.uint64)[:, None] * np.uint64(4) + np.arange(4, dtype=np.uint64)[None]
        return [torch.from_numpy((c * np.uint64(0x9E3779B97F4A7C15 + k)).view(np.int64)) for k in range(len(names))]

    names = ["logf", "log2f", "sincosf"]
    rows = sweep.rows_for(names)
    t0 = time.perf_counter()
    table = torch.zeros((len(rows), sweep.CHUNKS, 4), dtype=torch.int64)
    lo, hi = sweep.shard(rank, world)
    for i, part in enumerate(fill(rows, lo, hi)):
        table[i, lo:hi] = part
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(table)
    secs = max_over_ranks_cpu(time.perf_counter() - t0, world)
    if rank == 0:
        full = torch.stack([p for p in fill(rows, 0, sweep.CHUNKS)])
        mism = int((table != full).any(dim=2).sum())
        print(json.dumps({"metric": METRIC, "value": None, "selftest": True, "n_gpus": world,
                          "backend": "gloo", "sweep": {"seconds": secs, "ranks": world, "rows": len(rows),
                                                       "mismatching_chunks": mism,
                                                       "collective": "one all_reduce of the hash table"}}),
              flush=True)


def max_over_ranks_cpu(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _libm_ops():
    import torch
    return {"expf": torch.exp, "exp2f": torch.exp2, "expm1f": torch.expm1, "logf": torch.log,
            "log2f": torch.log2, "log10f": torch.log10, "log1pf": torch.log1p, "sinf": torch.sin,
            "cosf": torch.cos, "tanf": torch.tan, "asinf": torch.asin, "acosf": torch.acos,
            "atanf": torch.atan, "sinhf": torch.sinh, "coshf": torch.cosh, "tanhf": torch.tanh,
            "rsqrtf": torch.rsqrt}


LIBM_OPS = {}

# Fast-path lookup tables + polynomial coefficients read per element, bytes
# (csrc/crvec_tables.inc; shared-memory pair tables counted at their 16-byte
# entries). The paper reports its table footprint beside the timings
# (ref: SPEC.md:629-634); the reference's own sizes are in REF_TABLE_BYTES.
TABLE_BYTES = {
    "expf": 160, "exp2f": 160, "exp10f": 160, "expm1f": 168, "sinhf": 160, "coshf": 160,
    "tanhf": 168, "logf": 304, "log2f": 304, "log10f": 304, "log1pf": 304,
    "sinf": 304, "cosf": 304, "tanf": 304, "sincosf": 304, "asinf": 544, "acosf": 544,
    "atanf": 352, "rsqrtf": 0, "exp2(f64)": 2080, "log(f64)": 12344,
}
PH_TABLE_BYTES = 3712  # Payne-Hanek 16/pi chunk table (trig big-argument path only)
REF_TABLE_BYTES = {"exp2f": 120, "log2f": 640, "exp2(f64)": 816, "log(f64)": 1104}  # ref: proj/src/tables.cpp:228-231


def all_functions_table(n=1 << 28, reps=9):
    """Device throughput of every binary32 function (and the binary64 pair) at
    2^28 (2^26 for binary64), inputs generated on the device: the configs'
    distributions for the log and trig families, uniform over each function's
    interesting range otherwise. Median of `reps` event-timed launches; next to
    it, PyTorch's non-CR CUDA libm kernel on the same array (the cost of CR)."""
    import ctypes
    import torch
    import paper_2605_15547_b200 as crvec
    from tests.inputs import device_input
    peak, _ = peaks()
    L = crvec.lib()
    LIBM_OPS.update(_libm_ops())
    s = torch.cuda.current_stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    y2 = torch.empty(n, dtype=torch.float32, device="cuda")
    out = {}

    def timed(fn):
        for _ in range(2):
            fn()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        return float(np.median(ts))

    for name in crvec.F32_FUNCS + ["sincosf"]:
        # config C2 (log family: specials injected) / C3 (trig: 1/8 large-argument
        # tail) distributions, uniform over the function's range otherwise
        x = device_input(name, n, "config")
        fid = crvec.FN_IDS[name]
        t = timed(lambda: L.crvec_eval_f32_dev(fid, x.data_ptr(), y.data_ptr(), y2.data_ptr(), n, 0, sp))
        bpe = 12 if name == "sincosf" else 8
        out[name] = {"gelem_s": round(n / t / 1e9, 1), "frac_hbm": round(bpe * n / t / 1e9 / peak, 3)}
        # the paper's Table III analogue: the same array through PyTorch's
        # (non-CR, ~1-ulp CUDA libm) elementwise kernel, for the cost of CR
        op = LIBM_OPS.get(name)
        if op is not None:
            tl = timed(lambda: op(x, out=y))
            out[name]["torch_libm_gelem_s"] = round(n / tl / 1e9, 1)
        elif name == "exp10f":  # no torch exp10: CUDA powf(10, x), the library's 1-ulp path
            tl = timed(lambda: torch.pow(10.0, x, out=y))
            out[name]["torch_libm_gelem_s"] = round(n / tl / 1e9, 1)
            out[name]["torch_libm_op"] = "torch.pow(10, x)"
        elif name == "sincosf":  # two library launches (sin, cos) for the two outputs
            tl = timed(lambda: (torch.sin(x, out=y), torch.cos(x, out=y2)))
            out[name]["torch_libm_gelem_s"] = round(n / tl / 1e9, 1)
            out[name]["torch_libm_op"] = "torch.sin + torch.cos"
        out[name]["table_bytes"] = TABLE_BYTES[name] + (PH_TABLE_BYTES if name in ("sinf", "cosf", "tanf", "sincosf") else 0)
        if name in REF_TABLE_BYTES:
            out[name]["ref_table_bytes"] = REF_TABLE_BYTES[name]
        del x
    n64 = 1 << 26
    for name, lo, hi in (("exp2", -20.0, 20.0), ("log", 0.125, 8.0)):
        x = torch.rand(n64, device="cuda", generator=g, dtype=torch.float64) * (hi - lo) + lo
        yy = torch.empty_like(x)
        f = getattr(L, f"crvec_{name}_dev")
        t = timed(lambda: f(x.data_ptr(), yy.data_ptr(), n64, 0, sp))
        k = name + "(f64)"
        out[k] = {"gelem_s": round(n64 / t / 1e9, 1), "frac_hbm": round(16 * n64 / t / 1e9 / peak, 3)}
        # Table IV analogue (ref: PAPER.md:229-234): the library's 1-ulp float64 kernel on the same array
        op = torch.exp2 if name == "exp2" else torch.log
        tl = timed(lambda: op(x, out=yy))
        out[k]["torch_libm_gelem_s"] = round(n64 / tl / 1e9, 1)
        out[k]["cr_over_libm_time"] = round(t / tl, 2)
        out[k]["table_bytes"] = TABLE_BYTES[k]
        out[k]["ref_table_bytes"] = REF_TABLE_BYTES[k]
    for v in out.values():  # the paper's "cost of CR" column: CR time / library time
        if "torch_libm_gelem_s" in v:
            v["cr_over_libm_time"] = round(v["torch_libm_gelem_s"] / v["gelem_s"], 2)
    return out


# --------------------------------------------------------------- our arm -----
def run_crvec(args, rank, world, local):
    import ctypes
    import torch
    import paper_2605_15547_b200 as crvec
    from paper_2605_15547_b200.sweep import shard
    from tests.inputs import log_family_input

    L = crvec.lib()
    n = N_ELEM
    fns = LOG_FAMILY
    # synthetic inputs generated once on the host (pinned for the e2e leg) and
    # made resident in HBM before timing
    hx = {f: torch.from_numpy(log_family_input(f, n, seed=3 + i).view(np.float32)).pin_memory()
          for i, f in enumerate(fns)}
    xs = {f: hx[f].cuda() for f in fns}
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)

    def step(evs=None):
        for i, f in enumerate(fns):
            if evs is not None:
                evs[f][0].record(stream)
            rc = L.crvec_eval_f32_dev(crvec.FN_IDS[f], xs[f].data_ptr(), y.data_ptr(), None, n, 0, sp)
            if evs is not None:
                evs[f][1].record(stream)
            assert rc == 0, rc

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    per_fn = {f: [] for f in fns}
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            evs = {f: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for f in fns}
            step(evs)
            per_fn_events = evs
            for f in fns:
                per_fn[f].append(per_fn_events[f])
        t1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    secs = max_over_ranks(t0.elapsed_time(t1) / 1e3, world)
    elems_step = n * len(fns) * world
    value = elems_step * args.steps / secs / 1e9
    fn_ms = {f: float(np.mean([a.elapsed_time(b) for a, b in per_fn[f]])) for f in fns}
    peak, peak_kind = peaks()
    dom = max(fns, key=lambda f: fn_ms[f])
    achieved = 8.0 * n / (fn_ms[dom] / 1e3) / 1e9
    per_fn_gelem = {f: n / (fn_ms[f] / 1e3) / 1e9 for f in fns}

    # ---- e2e: C ABI host-pointer path, pinned host buffers, copies in region
    hy = torch.empty(n, dtype=torch.float32).pin_memory()
    e2e_steps = max(1, min(args.steps, 3))

    def e2e_step():
        for f in fns:
            rc = L.crvec_eval_f32(crvec.FN_IDS[f], hx[f].data_ptr(), hy.data_ptr(), None, n, 0)
            assert rc == 0, rc

    e2e_step()
    barrier(world)
    t = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_secs = max_over_ranks(time.perf_counter() - t, world)
    e2e_value = elems_step * e2e_steps / e2e_secs / 1e9

    # ---- exhaustive sweep (sharded across ranks)
    sweep = None
    if not args.no_sweep:
        secs_sw, mism, checked, nrows = run_sweep(rank, world, crvec.F32_FUNCS + ["sincosf"])
        sweep = {"seconds": secs_sw, "functions": 19, "modes": 4, "patterns": 2 ** 32,
                 "mismatching_chunks": mism, "golden_sets_checked": checked, "ranks": world,
                 "chunks_per_rank": [b - a for a, b in (shard(r, world) for r in range(world))],
                 "collective": (f"one NCCL all_reduce of the {nrows}x4096x4 u64 chunk-hash table"
                                if world > 1 else None),
                 "timed": "first sweep launch .. end of the all_reduce, device events, max over ranks"}

    table = all_functions_table() if (rank == 0 and not args.no_table) else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_record(args.ref_sample)

    launches = len(fns) * args.steps
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gelem/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "log family (logf, log2f, log10f, log1pf) x 2^28 fp32 each, "
                                   "config-2 inputs incl. denormals/Inf/NaN, RNE, HBM-resident",
                       "elements_per_step_per_gpu": n * len(fns), "l2": "inputs 1 GiB > L2, no flush",
                       "per_function_gelem_s": per_fn_gelem, "per_function_ms": fn_ms},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(dom),
                         "traffic_note": "dram read+write bytes per launch from the latest profiles/rNN/ncu_full_<fn>.csv "
                                         f"(algorithmic {8 * n} B)",
                         "kernel": f"k_map_vec<{dom}> (8 B/elem x 2^28)", "peak_source": peak_kind},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "Gelem/s",
                    "h2d_bytes_per_step": 4 * n * len(fns), "d2h_bytes_per_step": 4 * n * len(fns)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "sweep": sweep,
            "functions": table,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="crvec", choices=["crvec", "reference"])
    ap.add_argument("--ref-sample", type=int, default=1 << 26,
                    help="elements per reference-arm step (cr_log2f<16> on the host cores)")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-table", action="store_true")
    ap.add_argument("--selftest", action="store_true",
                    help="CPU (gloo) self-test of the multi-rank launch / shard / reduce path")
    args = ap.parse_args()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, rank, int(os.environ.get("WORLD_SIZE", "1")))
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(sys.argv[1:], args.gpus))
    rank, world, local = dist_init("gloo" if args.selftest else "nccl")
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.selftest:
        run_selftest(args, rank, world)
    else:
        run_crvec(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
