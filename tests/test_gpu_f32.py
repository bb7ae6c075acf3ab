"""GPU parity tests for the 19 binary32 CR functions (through the C ABI).

Bit-exact against the CPU oracle (oracle/, a restatement of the reference's
Ziv oracle, ref: proj/src/oracle.cpp:302-388) in all four rounding modes, on
seeded random + special inputs, on the configs' input distributions, and —
exhaustively over all 2^32 patterns — against the committed golden chunk
hashes (tests/golden/sweep/) that the same oracle produced.
"""
import os

import numpy as np
import pytest

import paper_2605_15547_b200 as crvec
from tests.inputs import log_family_input, mixed_f32, trig_input

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "sweep")


def _mismatch_report(x, got, want):
    bad = np.nonzero(got != want)[0]
    return [(hex(int(x[i])), hex(int(got[i])), hex(int(want[i]))) for i in bad[:5]], len(bad)


@pytest.mark.parametrize("name", crvec.F32_FUNCS)
def test_random_and_specials_all_modes(cuda, oracle, name):
    x = mixed_f32(name, 1 << 17, seed=11)
    want = oracle.f32(crvec.ORACLE_NAME[name], x, None)
    xt = cuda.from_numpy(x.view(np.float32)).cuda()
    for mode in range(4):
        got = crvec.eval_f32(name, xt, mode).cpu().numpy().view(np.uint32)
        ex, nbad = _mismatch_report(x, got, want[:, mode])
        assert nbad == 0, f"{name} mode {mode}: {nbad} mismatches, e.g. {ex}"


@pytest.mark.parametrize("name", ["logf", "log2f", "log10f", "log1pf"])
def test_log_family_config_inputs(cuda, oracle, name):
    """Config C2 distribution (denormals / Inf / NaN / negatives injected)."""
    x = log_family_input(name, 1 << 18)
    for mode in range(4):
        want = oracle.f32(crvec.ORACLE_NAME[name], x, mode)
        got = crvec.eval_f32(name, x.view(np.float32), mode).view(np.uint32)  # host path
        ex, nbad = _mismatch_report(x, got, want)
        assert nbad == 0, f"{name} mode {mode}: {ex}"


@pytest.mark.parametrize("name", ["sinf", "cosf", "tanf"])
def test_trig_config_inputs_big_args(cuda, oracle, name):
    """Config C3: 1/8 large-argument tail, randomly interleaved (Payne-Hanek path)."""
    x = trig_input(1 << 18)
    xt = cuda.from_numpy(x.view(np.float32)).cuda()
    for mode in range(4):
        want = oracle.f32(crvec.ORACLE_NAME[name], x, mode)
        got = crvec.eval_f32(name, xt, mode).cpu().numpy().view(np.uint32)
        ex, nbad = _mismatch_report(x, got, want)
        assert nbad == 0, f"{name} mode {mode}: {ex}"


def test_sincosf_matches_sin_and_cos(cuda, oracle):
    x = np.concatenate([trig_input(1 << 16), mixed_f32("sincosf", 1 << 16)])
    xt = cuda.from_numpy(x.view(np.float32)).cuda()
    for mode in range(4):
        s, c = crvec.cr_sincosf(xt, mode)
        assert (s.cpu().numpy().view(np.uint32) == oracle.f32("sin", x, mode)).all()
        assert (c.cpu().numpy().view(np.uint32) == oracle.f32("cos", x, mode)).all()


def test_expf_config1_full_2p24(cuda, oracle):
    """Config C1: expf over 2^24 uniform-random inputs, all four modes, bit-exact."""
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.integers(0, 2**32, 1 << 23, dtype=np.uint64).astype(np.uint32),
                        rng.uniform(-104, 89, 1 << 23).astype(np.float32).view(np.uint32)])
    want = oracle.f32("exp", x, None)
    xt = cuda.from_numpy(x.view(np.float32)).cuda()
    for mode in range(4):
        got = crvec.cr_expf(xt, mode).cpu().numpy().view(np.uint32)
        ex, nbad = _mismatch_report(x, got, want[:, mode])
        assert nbad == 0, f"mode {mode}: {ex}"


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 31, 33, 127, 129, 1000])
def test_sizes_alignment_inplace(cuda, oracle, n):
    x = mixed_f32("logf", max(n, 1), seed=n)[:n]
    want = oracle.f32("log", x, 0) if n else np.zeros(0, np.uint32)
    got = crvec.cr_logf(x.view(np.float32)).view(np.uint32)
    assert (got == want).all()
    # unaligned device pointers (offset by one element) and in-place
    buf = cuda.zeros(n + 1, dtype=cuda.float32, device="cuda")
    buf[1:] = cuda.from_numpy(x.view(np.float32)).cuda()
    v = buf[1:]
    crvec.eval_f32("logf", v, 0, out=v)
    assert (v.cpu().numpy().view(np.uint32) == want).all()


def test_scalar_api_and_reference_examples(cuda):
    """SPEC examples for cr_exp2f / cr_log2f (ref: SPEC.md kernels_f32 examples)."""
    RM = crvec.RoundingMode
    for m in RM:
        assert crvec.cr_exp2f_scalar(0.0, m) == 1.0
        assert crvec.cr_exp2f_scalar(127.0, m) == 2.0 ** 127
        assert crvec.cr_log2f_scalar(1.0, m) == 0.0
        assert crvec.cr_log2f_scalar(8.0, m) == 3.0
        assert crvec.cr_log2f_scalar(2.0 ** -149, m) == -149.0
    assert crvec.cr_exp2f_scalar(float("-inf")) == 0.0
    assert np.isinf(crvec.cr_exp2f_scalar(128.0, RM.NearestEven))
    assert crvec.cr_exp2f_scalar(128.0, RM.TowardZero) == np.finfo(np.float32).max
    assert crvec.cr_exp2f_scalar(128.0, RM.TowardNegative) == np.finfo(np.float32).max
    assert np.isneginf(crvec.cr_log2f_scalar(0.0))
    nan = np.array([0xFF912345], np.uint32).view(np.float32)
    assert crvec.cr_exp2f(nan).view(np.uint32)[0] == 0xFFD12345
    assert crvec.cr_log2f(np.array([-1.0], np.float32)).view(np.uint32)[0] == 0x7FC00000


def _golden(name):
    p = os.path.join(GOLDEN, name + ".npy")
    if not os.path.exists(p):
        pytest.fail(f"golden sweep data missing: {p} (python tools/gen_golden.py {name})")
    return np.load(p)


@pytest.mark.parametrize("name", crvec.F32_FUNCS + ["sincosf"])
def test_exhaustive_sweep_vs_golden(cuda, name):
    """All 2^32 inputs x 4 modes: per-chunk hashes equal the oracle's golden."""
    h, h2, _ = crvec.sweep_f32(name)
    if name == "sincosf":
        gs, gc = _golden("sin"), _golden("cos")
        assert (h == gs).all(), f"sin chunks differ: {np.nonzero((h != gs).any(1))[0][:10]}"
        assert (h2 == gc).all(), f"cos chunks differ: {np.nonzero((h2 != gc).any(1))[0][:10]}"
        return
    g = _golden(crvec.ORACLE_NAME[name])
    bad = np.nonzero((h != g).any(1))[0]
    assert len(bad) == 0, f"{name}: {len(bad)} chunks differ, first {bad[:10]}"


@pytest.mark.parametrize("name", crvec.F32_FUNCS + ["sincosf"])
def test_map_kernels_exhaustive_vs_golden(cuda, name):
    """The PRODUCT map kernels (crvec_<fn>f_dev: streaming template, rare-path
    form, kernel shape) over all 2^32 inputs x 4 modes, hashed per 2^20 chunk
    like the sweep: equal to the oracle's golden (sweep force mode 3)."""
    h, h2, _ = crvec.sweep_f32(name, force_accurate=crvec.SWEEP_MAP_KERNELS)
    if name == "sincosf":
        gs, gc = _golden("sin"), _golden("cos")
        assert (h == gs).all(), f"sin chunks differ: {np.nonzero((h != gs).any(1))[0][:10]}"
        assert (h2 == gc).all(), f"cos chunks differ: {np.nonzero((h2 != gc).any(1))[0][:10]}"
        return
    g = _golden(crvec.ORACLE_NAME[name])
    bad = np.nonzero((h != g).any(1))[0]
    assert len(bad) == 0, f"{name}: {len(bad)} chunks differ, first {bad[:10]}"


@pytest.mark.parametrize("name", crvec.F32_FUNCS + ["sincosf"])
def test_element_kernels_exhaustive_vs_golden(cuda, name):
    """The element kernel (k_map_scalar: relatively misaligned arrays, one
    element per lane, register-form rare path) over all 2^32 inputs x 4 modes:
    equal to the golden (sweep mode 4)."""
    h, h2, _ = crvec.sweep_f32(name, force_accurate=crvec.SWEEP_ELEMENT_KERNELS)
    if name == "sincosf":
        assert (h == _golden("sin")).all() and (h2 == _golden("cos")).all()
        return
    g = _golden(crvec.ORACLE_NAME[name])
    bad = np.nonzero((h != g).any(1))[0]
    assert len(bad) == 0, f"{name}: {len(bad)} chunks differ, first {bad[:10]}"


@pytest.mark.parametrize("name", crvec.F32_FUNCS)
def test_accurate_path_self_check(cuda, name):
    """Route EVERY non-special lane through the double-double accurate path
    (the rarely-taken fallback) over 64 spread chunks: must still match."""
    g = _golden(crvec.ORACLE_NAME[name])
    total = 0
    for lo in list(range(0, 4096, 512)) + [1008, 1016, 3056]:
        h, _, n_acc = crvec.sweep_f32(name, lo, lo + 8, force_accurate=True)
        total += n_acc
        assert (h == g[lo:lo + 8]).all(), f"{name}: forced-accurate chunk mismatch at {lo}"
    assert total > 1 << 20, total  # millions of lanes really went through the accurate path


@pytest.mark.parametrize("name", crvec.F32_FUNCS)
def test_inplace_vector_path_with_rare_lanes(cuda, oracle, name):
    """Aligned in-place call large enough for the vector kernel (several grid
    strides, ragged last step), inputs full of specials and hard lanes: the
    rare path must resolve lanes before the in-place store overwrites them."""
    n = (1 << 16) + 7
    x = mixed_f32(name, n, seed=21)[:n]
    for mode in (0, 3):
        want = oracle.f32(crvec.ORACLE_NAME[name], x, mode)
        v = cuda.from_numpy(x.view(np.float32).copy()).cuda()
        crvec.eval_f32(name, v, mode, out=v)
        ex, nbad = _mismatch_report(x, v.cpu().numpy().view(np.uint32), want)
        assert nbad == 0, f"{name} mode {mode}: {ex}"


@pytest.mark.parametrize("name", ["expf", "sinf", "sincosf"])
def test_host_pipeline_multichunk(cuda, name):
    """Host-pointer entry point over several staging chunks rotating through
    the staging streams equals the device entry point (validated above)."""
    import ctypes
    n = 2 * (1 << 24) + 5  # three 2^24-element chunks
    rng = np.random.default_rng(5)
    x = rng.uniform(-80, 80, n).astype(np.float32)
    L = crvec.lib()
    fid = crvec.FN_IDS[name]
    hy = np.empty(n, np.float32)
    hy2 = np.empty(n, np.float32)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    assert L.crvec_eval_f32(fid, p(x), p(hy), p(hy2) if name == "sincosf" else None, n, 1) == 0
    xd = cuda.from_numpy(x).cuda()
    yd = cuda.empty_like(xd)
    yd2 = cuda.empty_like(xd)
    s = ctypes.c_void_p(cuda.cuda.current_stream().cuda_stream)
    assert L.crvec_eval_f32_dev(fid, xd.data_ptr(), yd.data_ptr(), yd2.data_ptr(), n, 1, s) == 0
    assert (yd.cpu().numpy().view(np.uint32) == hy.view(np.uint32)).all()
    if name == "sincosf":
        assert (yd2.cpu().numpy().view(np.uint32) == hy2.view(np.uint32)).all()


@pytest.mark.parametrize("name", ["logf", "expf", "sinf"])
@pytest.mark.parametrize("ox,oy", [(4, 4), (1, 1), (4, 0), (0, 3)])
def test_offset_pointers_head_peel(cuda, oracle, name, ox, oy):
    """Device pointers offset by ox / oy floats from a 256-byte boundary: equal
    offsets peel a scalar head up to the 128/256-bit vector boundary, unequal
    ones take the element kernel; results are identical either way."""
    n = (1 << 18) + 3
    x = mixed_f32(name, n, seed=31 + ox)[:n]
    want = oracle.f32(crvec.ORACLE_NAME[name], x, 0)
    bx = cuda.zeros(n + 8, dtype=cuda.float32, device="cuda")
    by = cuda.zeros(n + 8, dtype=cuda.float32, device="cuda")
    bx[ox:ox + n] = cuda.from_numpy(x.view(np.float32)).cuda()
    crvec.eval_f32(name, bx[ox:ox + n], 0, out=by[oy:oy + n])
    ex, nbad = _mismatch_report(x, by[oy:oy + n].cpu().numpy().view(np.uint32), want)
    assert nbad == 0, f"{name} ({ox},{oy}): {ex}"


@pytest.mark.gpu
@pytest.mark.parametrize("ox,oy,oc", [(0, 0, 0), (1, 1, 1), (3, 3, 3), (5, 5, 5), (1, 0, 1), (2, 2, 0)])
def test_sincosf_offset_pointers_head_peel(cuda, oracle, ox, oy, oc):
    """sincosf with its three arrays offset from a 256-byte boundary: equal
    offsets peel a scalar head to the 256-bit boundary, any unequal offset
    takes the element kernel; both outputs match sinf / cosf of the oracle."""
    n = (1 << 18) + 5
    x = np.concatenate([trig_input(n // 2), mixed_f32("sincosf", n)])[:n]
    want_s = oracle.f32(crvec.ORACLE_NAME["sinf"], x, 0)
    want_c = oracle.f32(crvec.ORACLE_NAME["cosf"], x, 0)
    bx = cuda.zeros(n + 8, dtype=cuda.float32, device="cuda")
    bs = cuda.zeros(n + 8, dtype=cuda.float32, device="cuda")
    bc = cuda.zeros(n + 8, dtype=cuda.float32, device="cuda")
    bx[ox:ox + n] = cuda.from_numpy(x.view(np.float32)).cuda()
    crvec.eval_f32("sincosf", bx[ox:ox + n], 0, out=bs[oy:oy + n], out2=bc[oc:oc + n])
    for got, want, what in ((bs[oy:oy + n], want_s, "sin"), (bc[oc:oc + n], want_c, "cos")):
        ex, nbad = _mismatch_report(x, got.cpu().numpy().view(np.uint32), want)
        assert nbad == 0, f"sincosf {what} ({ox},{oy},{oc}): {ex}"
