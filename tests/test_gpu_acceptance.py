"""SPEC acceptance criteria (ref: SPEC.md:358-368) on the GPU kernels, beyond
the exhaustive sweep: the verify CLI, exactness suite (#5), consistency
between the vectorized and the scalar kernels (#6), monotonicity ladders
(#7), fp64 round-test statistics (#4) and corpus replay (#3)."""
import os

import numpy as np
import pytest

import paper_2605_15547_b200 as crvec
from tests import verify_cli

pytestmark = pytest.mark.gpu


def test_verify_cli_exhaustive_and_strided(cuda, tmp_path):
    rep = tmp_path / "r.json"
    assert verify_cli.main(["verify", "--fn", "exp2f", "--mode", "all", "--report", str(rep)]) == 0
    assert verify_cli.main(["verify", "--fn", "log2f", "--mode", "all", "--stride", "256",
                            "--range", "0x3f000000:0x3fffffff"]) == 0


def test_exactness_suite(cuda):
    """exp2f/exp2 exact on integers, log2f on powers of two, log(1) = +0, all modes."""
    ints = np.arange(-149, 128, dtype=np.float32)
    p2 = np.array([2.0 ** k for k in range(-149, 128)], dtype=np.float32)
    for m in range(4):
        assert (crvec.cr_exp2f(ints, m) == np.ldexp(np.float32(1), ints.astype(int))).all()
        assert (crvec.cr_log2f(p2, m) == np.arange(-149, 128, dtype=np.float32)).all()
        i64 = np.arange(-1074, 1024, dtype=np.float64)
        assert (crvec.cr_exp2(i64, m) == np.ldexp(1.0, i64.astype(int))).all()
        r = crvec.cr_log(np.array([1.0]), m)
        assert r[0] == 0.0 and not np.signbit(r[0])


def test_vector_and_scalar_kernels_agree(cuda):
    """Aligned (float4 kernel) vs misaligned (scalar kernel) paths: bit-identical."""
    rng = np.random.default_rng(3)
    n = 1 << 22
    x = rng.integers(0, 2 ** 32, n + 1, dtype=np.uint64).astype(np.uint32)
    for name in crvec.F32_FUNCS:
        t = cuda.from_numpy(x.view(np.float32)).cuda()
        a = crvec.eval_f32(name, t[1:].clone(), 0)          # aligned copy -> vector kernel
        b = crvec.eval_f32(name, t[1:], 0)                  # offset by 4 bytes -> scalar kernel
        assert (a.cpu().numpy().view(np.uint32) == b.cpu().numpy().view(np.uint32)).all(), name


@pytest.mark.parametrize("name,lo,inc", [("expf", -20.0, True), ("exp2f", 0.5, True), ("logf", 0.25, True),
                                         ("log1pf", -0.5, True), ("atanf", -3.0, True), ("tanhf", -2.0, True),
                                         ("rsqrtf", 0.5, False), ("acosf", -0.9, False), ("sinhf", -5.0, True)])
def test_monotonicity_ladders(cuda, name, lo, inc):
    """10^6 consecutive binary32 inputs in a monotone domain, every mode."""
    b0 = int(np.array([lo], np.float32).view(np.uint32)[0])
    if lo < 0:  # walk towards zero then through positives: use increasing values
        x = np.sort(np.concatenate([
            np.arange(b0 - 500000, b0, dtype=np.uint64).astype(np.uint32).view(np.float32),
            np.arange(b0, b0 + 500000, dtype=np.uint64).astype(np.uint32).view(np.float32)]))
    else:
        x = np.arange(b0, b0 + 1000000, dtype=np.uint64).astype(np.uint32).view(np.float32)
    for m in range(4):
        y = crvec.eval_f32(name, x, m).astype(np.float64)
        d = np.diff(y)
        assert ((d >= 0) if inc else (d <= 0)).all(), (name, m)


def test_fp64_callout_rate_cli(cuda, capsys):
    for fn, rng_ in (("exp2", "-20:20"), ("log", "0.125:8"), ("log", "0.5:2")):
        assert verify_cli.main(["callouts", "--fn", fn, f"--uniform={rng_}", "--n", "4000000"]) == 0
        import json
        rep = json.loads(capsys.readouterr().out)
        assert rep["rate"] < 2.0 ** -15 and rep["accurate_undecided"] == 0 and rep["host_callouts"] == 0


def test_corpus_replay_fp64(cuda, tmp_path):
    """SPEC corpus format `<hex-float>[,<expected>]` through the full fp64 kernels."""
    from tests.test_gpu_f64 import hard_exp2, hard_log
    p = tmp_path / "log.txt"
    p.write_text("# hard log\n" + "\n".join(v.hex() for v in hard_log()) + "\n0x1p+0,0x0p+0\n")
    assert verify_cli.main(["corpus", "--fn", "log", "--file", str(p), "--all-modes"]) == 0
    p = tmp_path / "exp2.txt"
    p.write_text("\n".join(v.hex() for v in hard_exp2()) + "\n")
    assert verify_cli.main(["corpus", "--fn", "exp2", "--file", str(p), "--all-modes"]) == 0


@pytest.mark.parametrize("fn", ["expf", "logf", "log1pf", "sinf", "sincosf", "acosf", "rsqrtf"])
def test_verify_cli_consistency(cuda, fn):
    """SPEC consistency_check through the CLI: device vs host path, alignment /
    split independence, array vs scalar entry point, oracle subset; all modes."""
    assert verify_cli.main(["consistency", "--fn", fn, "--n", "300000", "--seed", "7"]) == 0


def test_verify_cli_exactness_and_jobs(cuda):
    assert verify_cli.main(["exactness"]) == 0
    assert verify_cli.main(["verify", "--fn", "expm1f", "--mode", "rd", "--stride", "4096", "--jobs", "2"]) == 0
