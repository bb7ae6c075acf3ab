"""Exhaustive binary32 sweep, sharded across ranks (the verify module's
exhaustive_f32, ref: SPEC.md:250-258 / chunking :289-290; the reference's
proj/src/verify.cpp is a stub).

The 2^32 input patterns are 4096 chunks of 2^20. Rank r of W evaluates the
contiguous chunk range shard(r, W) for every function and writes per-chunk,
per-mode commutative hashes into a zero-initialised [F, 4096, 4] tensor; ONE
all_reduce(sum) (NCCL over NVLink on GPUs, gloo in the CPU tests) then gives
every rank the full table, which rank 0 compares with the golden hashes.
There is no other data-path collective: the sweep partitions the input space.
"""
from __future__ import annotations

import os
import time
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

CHUNKS = 4096


def shard(rank: int, world: int, chunks: int = CHUNKS) -> tuple[int, int]:
    """Contiguous, balanced chunk range of `rank` (world need not divide chunks)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(chunks, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


# evaluator(name, lo, hi) -> uint64 array [hi - lo, 4] (and [hi-lo, 4] cos for sincosf)
Evaluator = Callable[[str, int, int], np.ndarray]


def run(names: Sequence[str], evaluator: Evaluator, rank: int = 0, world: int = 1,
        chunks: int = CHUNKS, device: str = "cpu", reduce: bool = True):
    """Evaluate this rank's shard for every function and all_reduce the table.

    Returns (table: uint64 [len(names) (+1 if sincosf), chunks, 4], seconds
    measured around compute + collective on this rank)."""
    import torch
    rows = rows_for(names)
    table = torch.zeros((len(rows), chunks, 4), dtype=torch.int64, device=device)
    lo, hi = shard(rank, world, chunks)
    t0 = time.perf_counter()
    if hi > lo:
        for i, name in enumerate(names):
            out = evaluator(name, lo, hi)
            if name == "sincosf":
                s, c = out
                table[i, lo:hi] = torch.from_numpy(np.ascontiguousarray(s).view(np.int64)).to(device)
                table[rows.index("sincosf:cos"), lo:hi] = torch.from_numpy(
                    np.ascontiguousarray(c).view(np.int64)).to(device)
            else:
                table[i, lo:hi] = torch.from_numpy(np.ascontiguousarray(out).view(np.int64)).to(device)
    if reduce and world > 1:
        import torch.distributed as dist
        dist.all_reduce(table)  # sum mod 2^64: chunk hashes are disjoint per rank
    if device != "cpu":
        torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    return rows, table.cpu().numpy().view(np.uint64), secs


def rows_for(names: Sequence[str]) -> List[str]:
    """Table rows: one per function, plus the cos half of sincosf."""
    return list(names) + (["sincosf:cos"] if "sincosf" in names else [])


def run_device(names: Sequence[str], rank: int = 0, world: int = 1, chunks: int = CHUNKS,
               force_accurate: int = 0, reduce: bool = True, stream=None):
    """Device-resident sweep (the GPU path bench.py times): every function's
    chunk hashes are accumulated by the crvec_sweep_f32 kernels straight into
    one zeroed [rows, chunks, 4] int64 tensor on this rank's GPU (no host round
    trip, no per-function synchronisation), then ONE all_reduce(sum) over NCCL.

    force_accurate: 0 = the sweep kernels (fast path + accurate fallback),
    1 = every main-range lane through the accurate path, 3 = the product map
    kernels (crvec_<fn>f_dev) over every pattern in all four modes.

    Returns (rows, table tensor on the device, accurate-lane counter tensor).
    The caller copies the table to the host once, after its timing events."""
    import ctypes

    import torch
    import paper_2605_15547_b200 as crvec

    dev = torch.device("cuda", torch.cuda.current_device())
    rows = rows_for(names)
    table = torch.zeros((len(rows), chunks, 4), dtype=torch.int64, device=dev)
    ctr = torch.zeros(4, dtype=torch.int64, device=dev)
    lo, hi = shard(rank, world, chunks)
    s = torch.cuda.current_stream(dev) if stream is None else stream
    sp = ctypes.c_void_p(s.cuda_stream)
    L = crvec.lib()
    if hi > lo:
        for i, name in enumerate(names):
            h2 = table[rows.index("sincosf:cos"), lo].data_ptr() if name == "sincosf" else None
            rc = L.crvec_sweep_f32(crvec.FN_IDS[name], lo, hi, table[i, lo].data_ptr(), h2, ctr.data_ptr(),
                                   int(force_accurate), sp)
            if rc != 0:
                raise crvec.CrvecError(f"crvec_sweep_f32({name}) failed: {rc}")
    if reduce and world > 1:
        import torch.distributed as dist
        dist.all_reduce(table)  # sum mod 2^64: chunk hashes are disjoint per rank
    return rows, table, ctr


def golden_path(root: str, name: str) -> str:
    return os.path.join(root, "tests", "golden", "sweep", name + ".npy")


def compare(rows: List[str], table: np.ndarray, golden_dir_root: str,
            oracle_name: Dict[str, str]) -> Dict[str, Optional[List[int]]]:
    """Mismatching chunk indices per row (None when no golden is available)."""
    res = {}
    for i, row in enumerate(rows):
        if row == "sincosf":
            g = "sin"
        elif row == "sincosf:cos":
            g = "cos"
        else:
            g = oracle_name.get(row, row)
        p = golden_path(golden_dir_root, g)
        if not os.path.exists(p):
            res[row] = None
            continue
        gold = np.load(p)
        res[row] = [int(c) for c in np.nonzero((gold != table[i]).any(axis=1))[0]]
    return res


def gpu_evaluator(force_accurate: bool = False) -> Evaluator:
    """Evaluator backed by the crvec_sweep_f32 C-ABI kernel on the current device."""
    import paper_2605_15547_b200 as crvec

    def ev(name: str, lo: int, hi: int):
        h, h2, _ = crvec.sweep_f32(name, lo, hi, force_accurate=force_accurate)
        return (h, h2) if name == "sincosf" else h

    return ev
