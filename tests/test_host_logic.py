"""CPU tests of host-side logic that needs no GPU: the verify CLI's pure
helpers (ulp distance, corpus parsing, argument surface), the sweep sharding
and golden comparison, and the bench's table-byte bookkeeping."""
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ulp32_distance():
    from tests.verify_cli import ulp32_distance
    one = np.float32(1.0).view(np.uint32)
    a = np.array([one, one, 0x00000000, 0x80000000, 0x7FC00000], np.uint32)
    b = np.array([one + 1, one - 3, 0x80000000, 0x00000001, one], np.uint32)
    d = ulp32_distance(a, b)
    assert list(d[:4]) == [1, 3, 1, 2] and d[4] == -1  # +-0 are one ordered step apart; NaN -> -1


def test_corpus_parser_diagnostics(tmp_path):
    """Corpus format of the SPEC verify module: `<hex-float>[,<hex-float-expected>]`,
    '#' comments, per-line diagnostics that do not stop the run."""
    from tests.verify_cli import parse_corpus
    p = tmp_path / "c.txt"
    p.write_text("# header\n0x1p+0\n0x1.8p+1, 0x1.193ea7aad030bp+0\nnot-a-number\n\n0x1p-1074 # tiny\n")
    recs, diags = parse_corpus(str(p))
    assert [r[0] for r in recs] == [2, 3, 6]
    assert recs[1][2] == float.fromhex("0x1.193ea7aad030bp+0") and recs[0][2] is None
    assert len(diags) == 1 and diags[0]["line"] == 4


def test_cli_surface():
    """Every SPEC command parses (verify --jobs, corpus, callouts, consistency, exactness)."""
    from tests import verify_cli
    seen = {}

    def fake(a):
        seen[a.cmd] = a
        return 0
    # parse only: intercept the dispatch
    orig = {k: getattr(verify_cli, k) for k in ("cmd_verify", "cmd_corpus", "cmd_callouts",
                                                "cmd_consistency", "cmd_exactness")}
    try:
        for k in orig:
            setattr(verify_cli, k, fake)
        assert verify_cli.main(["verify", "--fn", "expf", "--mode", "rd", "--stride", "256", "--jobs", "3"]) == 0
        assert seen["verify"].jobs == 3 and verify_cli.JOBS == 3
        assert verify_cli.main(["corpus", "--fn", "log", "--file", "x", "--all-modes"]) == 0
        assert verify_cli.main(["callouts", "--fn", "exp2", "--uniform=-20:20", "--n", "10"]) == 0
        assert verify_cli.main(["consistency", "--fn", "sincosf", "--n", "1000"]) == 0
        assert verify_cli.main(["exactness"]) == 0
        with pytest.raises(SystemExit):
            verify_cli.main(["verify", "--fn", "nosuchf"])
    finally:
        for k, v in orig.items():
            setattr(verify_cli, k, v)
        verify_cli.JOBS = 0


def test_sweep_shard_covers_every_chunk_once():
    from paper_2605_15547_b200.sweep import CHUNKS, shard
    for world in (1, 2, 3, 4, 5, 8, 4096):
        spans = [shard(r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == CHUNKS
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(2, 2)


def test_sweep_compare_reports_mismatching_chunks(tmp_path):
    from paper_2605_15547_b200 import sweep
    gdir = tmp_path / "tests" / "golden" / "sweep"
    gdir.mkdir(parents=True)
    g = np.arange(4096 * 4, dtype=np.uint64).reshape(4096, 4)
    np.save(gdir / "exp.npy", g)
    t = g.copy()[None]
    t[0, 17, 2] ^= np.uint64(1)
    res = sweep.compare(["expf"], t, str(tmp_path), {"expf": "exp"})
    assert res == {"expf": [17]}
    assert sweep.compare(["logf"], t, str(tmp_path), {"logf": "log"}) == {"logf": None}


def test_bench_table_bytes_cover_every_function():
    import bench
    import paper_2605_15547_b200 as crvec
    names = crvec.F32_FUNCS + ["sincosf", "exp2(f64)", "log(f64)"]
    assert set(bench.TABLE_BYTES) == set(names)
    # binary32: <= 16 table entries of <= 32 B plus a few coefficients
    assert all(v <= 16 * 32 + 64 for k, v in bench.TABLE_BYTES.items() if "f64" not in k)
    assert set(bench.REF_TABLE_BYTES) <= set(names)


def test_golden_provenance_names_the_reference_for_its_functions():
    """The exhaustive golden of the three functions the reference implements
    comes from the reference's own oracle (tools/gen_golden_ref.py)."""
    for fn in ("exp2", "log", "log2"):
        meta = json.load(open(os.path.join(ROOT, "tests", "golden", "sweep", fn + ".json")))
        assert meta.get("source") == "reference build" and meta.get("restatement_agrees") is True, fn
