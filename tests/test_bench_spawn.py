"""bench.py's multi-rank path on CPU (gloo): `python bench.py --gpus 2` run as a
plain process re-launches itself under torch.distributed.run with 2 ranks,
shards the sweep's 4096 chunks, reduces the hash table with ONE all_reduce and
reports n_gpus / sweep.ranks = 2."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(n):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--selftest",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300,
                       env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [1, 2])
def test_bench_self_launch_gloo(n):
    d = _run(n)
    assert d["n_gpus"] == n and d["sweep"]["ranks"] == n
    assert d["sweep"]["mismatching_chunks"] == 0
