"""The sharded device sweep on real kernels: two ranks (processes) share the
one B200 of the test box, each runs `sweep.run_device` over its half of the
4096 chunks for a few functions (the sweep kernels, and mode 3 = the product
map kernels), the [rows, chunks, 4] hash table is reduced with ONE
all_reduce, and the result must equal the golden hashes chunk for chunk.
bench.py does the same over NCCL with one GPU per rank; NCCL refuses two
ranks on one device, so the collective here is gloo (CUDA tensors staged
through the host) - the sharding, the device-resident accumulation and the
single reduction are the ones bench.py runs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_2605_15547_b200 as crvec
from paper_2605_15547_b200 import sweep

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["expf", "log1pf", "sincosf"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows, table, _ = sweep.run_device(NAMES, rank, world, force_accurate=mode)
    torch.cuda.synchronize()
    if rank == 0:
        q.put((rows, table.cpu().numpy().view(np.uint64)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [crvec.SWEEP_KERNELS, crvec.SWEEP_MAP_KERNELS])
def test_two_rank_sharded_sweep_equals_golden(cuda, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, int(mode), q)) for r in range(2)]
    for p in procs:
        p.start()
    rows, table = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    bad = sweep.compare(rows, table, ROOT, crvec.ORACLE_NAME)
    assert set(bad) == set(sweep.rows_for(NAMES))
    for row, chunks in bad.items():
        assert chunks == [], f"{row}: {len(chunks)} chunks differ after the 2-rank reduction"
