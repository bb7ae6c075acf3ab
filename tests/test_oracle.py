"""CPU tests pinning the oracle (the parity checker) to the reference.

1. Known-answer tests of ref: proj/tests/test_oracle.cpp:52-110 and
   ref: proj/tests/test_fpbits.cpp:69-93, run through our C restatement.
2. Bit equality with the reference's OWN oracle: the committed golden vectors
   tests/golden/ref_oracle.npz (tools/gen_ref_fixtures.py) and, when
   /root/reference is present, the live reference build oracle/_ref/.
3. The reference's own unit-test binaries (compiled from /root/reference) pass.
4. Extension functions: equality with MPFR-direct rounding under an emulated
   binary32 exponent range (ref: proj/tests/test_oracle.cpp:193-217 idiom) on
   random + threshold-neighbourhood inputs.
5. The 64-bit extended-precision rung never changes a result (vs MPFR-only).
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "ref_oracle.npz")
HAVE_REF_SRC = os.path.isdir("/root/reference/proj")

f2u = lambda v: int(np.array([v], np.float32).view(np.uint32)[0])  # noqa: E731
d2u = lambda v: int(np.array([v], np.float64).view(np.uint64)[0])  # noqa: E731
RNE, RZ, RU, RD = range(4)


def z32(O, fn, xbits, mode, start=96):
    return O.lib().crvec_oracle_f32(O.FN[fn], xbits, mode, start, None, None)


def z64(O, fn, xbits, mode, start=96):
    return O.lib().crvec_oracle_f64(O.FN[fn], xbits, mode, start, None)


def test_known_answers_exact(oracle):
    O = oracle
    assert z32(O, "exp2", f2u(127.0), RNE) == f2u(2.0 ** 127)
    assert z32(O, "log2", f2u(8.0), RD) == f2u(3.0)
    assert z64(O, "log", d2u(1.0), RZ) == 0  # +0
    assert z32(O, "log2", 0x00000001, RNE) == f2u(-149.0)
    assert z64(O, "exp2", d2u(-1075.0), RNE) == 0
    assert z64(O, "exp2", d2u(-1075.0), RU) == 1


def test_known_answers_specials(oracle):
    O = oracle
    assert z32(O, "exp2", 0x7F800000, RNE) == 0x7F800000
    assert z32(O, "exp2", 0xFF800000, RNE) == 0
    assert z32(O, "log", 0, RZ) == 0xFF800000
    assert z32(O, "log", 0x80000000, RZ) == 0xFF800000
    assert z32(O, "log2", f2u(-1.0), RNE) == 0x7FC00000
    assert z32(O, "exp2", 0xFF912345, RNE) == 0xFFD12345
    assert z64(O, "exp2", d2u(128000.5), RZ) == 0x7FEFFFFFFFFFFFFF
    assert z64(O, "exp2", d2u(-4e9), RU) == 1
    assert z64(O, "exp2", d2u(1e300), RNE) == 0x7FF0000000000000


def test_conversion_known_answers(oracle):
    """ref: proj/tests/test_fpbits.cpp:69-93."""
    cv = oracle.lib().crvec_oracle_convert_f64_to_f32
    for m in range(4):
        assert cv(d2u(1.5), m) == f2u(1.5)
    assert cv(d2u(2.0 ** -150), RNE) == 0
    assert cv(d2u(2.0 ** -150), RU) == 1
    assert cv(d2u(2.0 ** 128 * (1 - 2.0 ** -30)), RZ) == 0x7F7FFFFF
    assert cv(d2u(-0.0), RNE) == 0x80000000
    assert cv(0x7FF8000000000001, RNE) & 0x7FC00000 == 0x7FC00000


def test_matches_reference_golden_vectors(oracle):
    """Bit equality with vectors produced by the reference's own oracle."""
    g = np.load(FIX)
    x32 = g["x32"]
    for fn in oracle.REF_FNS:
        got = oracle.f32(fn, x32, None, use_ld=False)
        assert (got == g[f"f32_{fn}"]).all(), fn
        got = oracle.f32(fn, x32, None, use_ld=True)
        assert (got == g[f"f32_{fn}"]).all(), fn + " (extended rung)"
    x64 = g["x64"]
    for fn in ("exp2", "log"):
        assert (oracle.f64(fn, x64, None) == g[f"f64_{fn}"]).all(), fn
    cv = oracle.lib().crvec_oracle_convert_f64_to_f32
    cin, cout = g["cvt_in"], g["cvt_out"]
    for i in range(0, len(cin), 7):
        for m in range(4):
            assert cv(int(cin[i]), m) == cout[i, m]


@pytest.fixture(scope="module")
def ref_oracle(oracle):
    if not oracle.ref_available():
        if not HAVE_REF_SRC:
            pytest.skip("reference sources absent (golden vectors cover this box)")
        oracle.build(ref=True)
    return oracle


def test_matches_live_reference_build(ref_oracle):
    O = ref_oracle
    rng = np.random.default_rng(31337)
    x = rng.integers(0, 2**32, 50000, dtype=np.uint64).astype(np.uint32)
    for fn in O.REF_FNS:
        mine = O.f32(fn, x, None, use_ld=True)
        for m in range(4):
            assert (mine[:, m] == O.ref_f32(fn, x, m)).all(), (fn, m)
    x64 = rng.integers(0, 2**64, 4000, dtype=np.uint64)
    for fn in ("exp2", "log"):
        mine = O.f64(fn, x64, None)
        for m in range(4):
            assert (mine[:, m] == O.ref_f64(fn, x64, m)).all(), (fn, m)


def test_reference_unit_tests_pass(ref_oracle):
    """The reference's own test_oracle / test_fpbits, compiled from its sources."""
    for t in ("test_oracle", "test_fpbits"):
        exe = os.path.join(ROOT, "oracle", "_ref", t)
        if not os.path.exists(exe):
            pytest.skip("reference test binaries not built")
        r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "failed: 0" in r.stdout


def _direct(O, fn, x):
    L = O.lib()
    L.crvec_oracle_direct_f32_batch.argtypes = [ctypes.c_int, O._u32p, O._u32p, ctypes.c_uint64]
    x = np.ascontiguousarray(x, dtype=np.uint32)
    y = np.empty((x.size, 4), np.uint32)
    L.crvec_oracle_direct_f32_batch(O.FN[fn], O._p32(x), O._p32(y), x.size)
    return y


def _threshold_inputs():
    thr = [2 ** -26, 2 ** -28, 2 ** -13, 2 ** -12, 88.8, 88.72, -104.0, -103.97, 38.6, 38.53,
           -45.2, -45.15, -18.0, 89.5, 89.4, 10.0, 9.0, 1.0, 128.0, -150.0, 0.0, 1e-45]
    thr += [float(10 ** k) for k in range(1, 11)] + [float(k) for k in range(1, 11)]
    thr += [4.0 ** k for k in range(-60, 60)] + [2.0 ** -148, 2.0 ** -146]
    out = []
    for t in thr:
        for s in (1, -1):
            b = f2u(s * t)
            out.extend(((b + d) & 0xFFFFFFFF) for d in range(-24, 25))
    return np.array(out, dtype=np.uint32)


@pytest.mark.parametrize("fn", ["exp", "exp10", "expm1", "log10", "log1p", "sin", "cos", "tan",
                                "asin", "acos", "atan", "sinh", "cosh", "tanh", "rsqrt",
                                "exp2", "log", "log2"])
def test_extension_vs_mpfr_direct(oracle, fn):
    rng = np.random.default_rng(606)
    x = np.concatenate([rng.integers(0, 2**32, 6000, dtype=np.uint64).astype(np.uint32),
                        rng.uniform(-100, 100, 3000).astype(np.float32).view(np.uint32),
                        _threshold_inputs()])
    a = oracle.f32(fn, x, None)
    b = _direct(oracle, fn, x)
    bad = np.nonzero((a != b).any(1))[0]
    assert len(bad) == 0, [hex(int(x[i])) for i in bad[:5]]


def test_extended_rung_never_changes_results(oracle):
    rng = np.random.default_rng(777)
    x = np.concatenate([rng.integers(0, 2**32, 20000, dtype=np.uint64).astype(np.uint32),
                        rng.uniform(-50, 50, 20000).astype(np.float32).view(np.uint32)])
    for fn in oracle.FN:
        a = oracle.f32(fn, x, None, use_ld=True)
        b = oracle.f32(fn, x, None, use_ld=False)
        assert (a == b).all(), fn


def test_golden_sweep_files_are_consistent(oracle):
    """Every committed sweep golden re-derives on a sampled chunk."""
    d = os.path.join(ROOT, "tests", "golden", "sweep")
    names = sorted(f[:-4] for f in os.listdir(d) if f.endswith(".npy") and not f.startswith("."))
    assert names, "no golden sweep data"
    for fn in names:
        g = np.load(os.path.join(d, fn + ".npy"))
        assert g.shape == (4096, 4) and g.dtype == np.uint64
        c = {"exp": 2047, "log": 1016}.get(fn, 1000)
        h = oracle.sweep_hashes(fn, c, c + 1)
        assert (h[0] == g[c]).all(), fn


def test_sweep_hash_definition(oracle):
    """Host restatement of the chunk hash on a slice (numpy mix64)."""
    p = np.arange(1000 << 20, (1000 << 20) + (1 << 20), dtype=np.uint64).astype(np.uint32)
    y = oracle.f32("exp", p, None)
    for m in range(4):
        h = oracle.mix64((y[:, m].astype(np.uint64) << np.uint64(32)) | p.astype(np.uint64))
        want = oracle.sweep_hashes("exp", 1000, 1001)[0, m]
        assert np.uint64(h.sum(dtype=np.uint64)) == want


def _bd(lib, fname, f, x):
    d, ex, dom = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
    getattr(lib, fname)(f, x, ctypes.byref(d), ctypes.byref(ex), ctypes.byref(dom))
    return d.value, ex.value, dom.value


def test_boundary_distance_and_hardest_case_search_match_reference(ref_oracle):
    """ref: proj/src/oracle.cpp:430-580; ref test proj/tests/test_oracle.cpp:221-246."""
    O = ref_oracle
    L, R = O.lib(), O.ref()
    for lib in (L, R):
        pfx = "crvec_oracle_" if lib is L else "crvec_ref_"
        getattr(lib, pfx + "boundary_distance_f32").argtypes = [ctypes.c_int, ctypes.c_uint32] + [ctypes.c_void_p] * 3
        getattr(lib, pfx + "boundary_distance_f64").argtypes = [ctypes.c_int, ctypes.c_uint64] + [ctypes.c_void_p] * 3
        getattr(lib, pfx + "hardest_case_search").restype = ctypes.c_uint64
        getattr(lib, pfx + "hardest_case_search").argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64]
    rng = np.random.default_rng(42)
    xs = rng.integers(0, 2 ** 32, 3000, dtype=np.uint64).astype(np.uint32)
    for fn in O.REF_FNS:
        f = O.FN[fn]
        for x in xs:
            assert _bd(L, "crvec_oracle_boundary_distance_f32", f, int(x)) == \
                _bd(R, "crvec_ref_boundary_distance_f32", f, int(x)), (fn, hex(int(x)))
    x64 = rng.integers(0, 2 ** 64, 1500, dtype=np.uint64)
    for fn in ("exp2", "log"):
        f = O.FN[fn]
        for x in x64:
            assert _bd(L, "crvec_oracle_boundary_distance_f64", f, int(x)) == \
                _bd(R, "crvec_ref_boundary_distance_f64", f, int(x)), (fn, hex(int(x)))
    lo, hi = f2u(1.0), f2u(1.0 + 2.0 ** -10)
    res = []
    for lib, pfx in ((L, "crvec_oracle_"), (R, "crvec_ref_")):
        n = getattr(lib, pfx + "hardest_case_search")(O.FN["exp2"], lo, hi, None, None, 0)
        bits, dist = np.zeros(n, np.uint32), np.zeros(n, np.float64)
        getattr(lib, pfx + "hardest_case_search")(O.FN["exp2"], lo, hi, bits.ctypes.data, dist.ctypes.data, 0)
        res.append((bits, dist))
    assert (res[0][0] == res[1][0]).all() and (res[0][1] == res[1][1]).all()
    assert (np.diff(res[0][1]) >= 0).all()
    assert _bd(L, "crvec_oracle_boundary_distance_f32", O.FN["log2"], f2u(4.0))[1] == 1  # exact


def test_hardcase_corpus_expected_outputs(oracle):
    """Expected outputs stored in the hard-case corpus equal the oracle's."""
    d = os.path.join(ROOT, "tests", "golden", "hardcases")
    if not os.path.isdir(d):
        pytest.skip("no hard-case corpus yet")
    import paper_2605_15547_b200 as crvec
    for f in sorted(os.listdir(d)):
        name = f[:-4]
        rows = [l.split() for l in open(os.path.join(d, f)) if l.strip() and not l.startswith("#")]
        x = np.array([int(r[0], 16) for r in rows], np.uint32)
        want = np.array([[int(v, 16) for v in r[3:7]] for r in rows], np.uint32)
        assert (oracle.f32(crvec.ORACLE_NAME[name], x, None, use_ld=False) == want).all(), name


# ---- the reference's own kernels (oracle/_ref/libcrvec_refk*.so) ----------
@pytest.fixture(scope="module")
def refk(ref_oracle):
    O = ref_oracle
    if not O.refk_available():
        pytest.skip("reference kernels not built")
    return O


def test_reference_table_artifact_roundtrip(refk):
    """tests/golden/ref_tables.txt is the reference's own text artifact
    (serialize_tables, FNV-1a header): its parse_tables accepts it and it equals
    the tables compiled into the reference kernels (ref: proj/src/tables.cpp:75-226)."""
    K = refk.refk()
    assert K.crvec_refk_tables_from_file(refk.REF_ARTIFACT.encode()) == 0
    assert K.crvec_refk_file_equals_builtin() == 1
    assert K.crvec_refk_tables_loaded() == 1


def test_reference_kernels_with_generated_tables_match_oracle(refk):
    """SPEC acceptance spot check (ref: SPEC.md:637): the reference's cr_exp2f /
    cr_log2f (both backends) and cr_exp2 / cr_log, run with the generated
    tables, agree with the oracle in all four modes."""
    O = refk
    rng = np.random.default_rng(777)
    x32 = np.concatenate([rng.integers(0, 2 ** 32, 3000, dtype=np.uint64).astype(np.uint32),
                          rng.uniform(-150, 130, 3000).astype(np.float32).view(np.uint32)])
    for fn in ("exp2", "log2"):
        want = O.f32(fn, x32, None)
        for m in range(4):
            for vec in (True, False):
                assert (O.refk_f32(fn, x32, m, vector=vec) == want[:, m]).all(), (fn, m, vec)
    x64 = {"exp2": np.concatenate([rng.uniform(-20, 20, 2000), rng.uniform(-1075, 1024, 1000)]),
           "log": np.concatenate([rng.uniform(0.125, 8, 2000),
                                  rng.integers(1, 0x7FF0000000000000, 1000, dtype=np.uint64).view(np.float64)])}
    for fn, xv in x64.items():
        want = O.f64(fn, xv.view(np.uint64), None)
        for m in range(4):
            got, _ = O.refk_f64(fn, xv.view(np.uint64), m)
            assert (got == want[:, m]).all(), (fn, m)


def test_gpu_round_test_fixture_matches_live_reference(refk):
    """tests/golden/ref_round_test.npz (the GPU round test's golden data) equals
    the live reference round_test_lane on a sample."""
    K = refk.refk()
    g = np.load(os.path.join(ROOT, "tests", "golden", "ref_round_test.npz"))
    v = ctypes.c_double()
    for i in range(0, g["hi"].size, 37):
        for m in range(4):
            dec = K.crvec_refk_round_test_lane(float(g["hi"][i]), float(g["lo"][i]), int(g["scale"][i]),
                                               float(g["eps_rel"][i]), float(g["eps_abs"][i]), m, ctypes.byref(v))
            assert dec == g["decided"][i, m]
            assert np.float64(v.value).view(np.uint64) == g["value"][i, m].view(np.uint64)


def test_golden_sweep_mpfr_only_dense_chunks(oracle):
    """Re-derive seeded numerically dense chunks (|x| in [2^-10, 2^7): exponent
    fields 117..134, chunk = pattern >> 20) of every committed exhaustive golden
    with the MPFR-only Ziv ladder (the x87 long-double rung OFF), so the golden
    hashes do not rest on glibc's *l() error bounds."""
    d = os.path.join(ROOT, "tests", "golden", "sweep")
    names = sorted(f[:-4] for f in os.listdir(d) if f.endswith(".npy") and not f.startswith("."))
    rng = np.random.default_rng(20240817)
    for fn in names:
        g = np.load(os.path.join(d, fn + ".npy"))
        for c in (int(rng.integers(117 * 8, 135 * 8)), 2048 + int(rng.integers(117 * 8, 135 * 8))):
            p = np.arange(c << 20, (c + 1) << 20, dtype=np.uint64).astype(np.uint32)
            y = oracle.f32(fn, p, None, use_ld=False)  # all host threads over elements
            for m in range(4):
                h = oracle.mix64((y[:, m].astype(np.uint64) << np.uint64(32)) | p.astype(np.uint64))
                assert np.uint64(h.sum(dtype=np.uint64)) == g[c, m], (fn, c, m)
