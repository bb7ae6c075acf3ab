"""Multi-rank exhaustive-sweep host logic on CPU (gloo, world_size 2).

The sweep partitions the 2^32 input space into contiguous chunk ranges per
rank and reduces the per-chunk hash table with ONE all_reduce. Here the
per-chunk evaluator is the CPU oracle (the checker) on a reduced chunk grid,
so the sharding + reduction + golden comparison path is exercised exactly as
bench.py runs it over NCCL on GPUs."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2605_15547_b200 import sweep

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_partition_covers_exactly():
    for world in (1, 2, 3, 4, 8, 7):
        spans = [sweep.shard(r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 4096
        for (a, b), (c, d) in zip(spans, spans[1:]):
            assert b == c
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CHUNK_BASE = 1000   # evaluate 4 real chunks [1000, 1004) mapped onto a 4-chunk grid


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O

    def ev(name, lo, hi):
        return O.sweep_hashes(name, CHUNK_BASE + lo, CHUNK_BASE + hi, threads=2)

    rows, table, _ = sweep.run(["exp", "log"], ev, rank, world, chunks=4)
    q.put((rank, rows, table))
    dist.destroy_process_group()


def test_gloo_two_ranks_match_single_rank_and_golden(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, rows0, t0), (_, rows1, t1) = sorted(res, key=lambda r: r[0])
    assert rows0 == rows1 == ["exp", "log"]
    assert (t0 == t1).all(), "all_reduce must give every rank the full table"
    for i, fn in enumerate(rows0):
        g = np.load(os.path.join(ROOT, "tests", "golden", "sweep", fn + ".npy"))
        assert (t0[i] == g[CHUNK_BASE:CHUNK_BASE + 4]).all(), fn
