"""ctypes bindings for the CPU oracle — TEST INFRASTRUCTURE ONLY.

Importable only from tests/, ``__graft_entry__.smoke()`` and bench.py's CPU
baseline / reference arm (the checker, never the thing measured or shipped).

Two libraries:
  * ``oracle/libcrvec_oracle.so`` — the C restatement of the reference oracle
    (ref: proj/src/oracle.cpp) extended to the 18 MPFR functions;
  * ``oracle/_ref/libcrvec_ref.so`` — the reference's OWN oracle compiled from
    /root/reference/proj/src/{fpbits,oracle}.cpp (``make -C oracle ref``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcrvec_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libcrvec_ref.so")
# the reference's own kernels (AVX-512 build and an x86-64-v2 build)
REFK_PATHS = (os.path.join(HERE, "_ref", "libcrvec_refk.so"), os.path.join(HERE, "_ref", "libcrvec_refk_v2.so"))

# Oracle function ids (first three = reference FuncId order,
# ref: proj/include/crvec/oracle.hpp:21).
FN = {
    "exp2": 0, "log": 1, "log2": 2, "exp": 3, "exp10": 4, "expm1": 5,
    "log10": 6, "log1p": 7, "sin": 8, "cos": 9, "tan": 10, "asin": 11,
    "acos": 12, "atan": 13, "sinh": 14, "cosh": 15, "tanh": 16, "rsqrt": 17,
}
REF_FNS = ("exp2", "log", "log2")
MODES = ("rne", "rz", "ru", "rd")

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_lib = None
_ref = None
_refk = None


REF_ARTIFACT = os.path.join(os.path.dirname(HERE), "tests", "golden", "ref_tables.txt")
REF_GEN_INC = os.path.join(HERE, "_ref", "gen", "tables_data.inc")


def inc_from_artifact(path: str = REF_ARTIFACT, out: str = REF_GEN_INC) -> None:
    """The statements the reference's builtin_tables() includes
    (ref: proj/src/tables.cpp:233-240), from its text artifact
    (ref: proj/src/tables.cpp:75-120; tests/golden/ref_tables.txt, written by
    tools/gen_ref_tables.py through the reference's own serialize_tables)."""
    def f(h):
        return float(np.array([int(h, 16)], dtype=np.uint64).view(np.float64)[0]).hex()
    lines = ["// from " + os.path.relpath(path, os.path.dirname(HERE)) + " (oracle.inc_from_artifact)"]
    meta = {"fit.exp2f": "fit_exp2f", "fit.log2f": "fit_log2f", "fit.exp2d": "fit_exp2d", "fit.logd": "fit_logd",
            "eps.exp2d": "eps_exp2d", "eps.logd": "eps_logd", "quant.logd": "quant_logd"}
    for ln in open(path):
        if not ln.strip() or ln.startswith("#"):
            continue
        key, *v = ln.split()
        k = key.split(".")
        if key.startswith(("exp2f.T.", "exp2f.c.", "logd.rcp.")):
            lines.append(f"v.{k[0]}.{k[1]}[{k[2]}] = {f(v[0])};")
        elif key.startswith("log2f.c."):
            lines.append(f"v.log2f.c[{k[2]}][{k[3]}] = {f(v[0])};")
        elif k[0] == "exp2d" and k[1] in ("T1", "T2", "T3"):
            lines.append(f"v.exp2d.{k[1]}_hi[{k[2]}] = {f(v[0])}; v.exp2d.{k[1]}_lo[{k[2]}] = {f(v[1])};")
        elif key in ("exp2d.ln2", "logd.ln2"):
            lines.append(f"v.{k[0]}.ln2 = DD{{{f(v[0])}, {f(v[1])}}};")
        elif key.startswith("exp2d.c."):
            lines.append(f"v.exp2d.c[{int(k[2]) - 2}] = {f(v[0])};")
        elif key.startswith("logd.c."):
            lines.append(f"v.logd.c[{int(k[2]) - 3}] = {f(v[0])};")
        elif key.startswith("logd.L."):
            u = int(v[0], 16)
            lines.append(f"v.logd.L[{k[2]}] = static_cast<std::int64_t>({u - (1 << 64) if u >> 63 else u}LL);")
        elif key == "logd.degree":
            lines.append(f"v.logd.tail_degree = {int(v[0])};")
        elif key.startswith("meta."):
            lines.append(f"v.eps.{meta[key[5:]]} = {f(v[0])};")
        else:
            raise ValueError("unknown table record " + key)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def build(ref: bool = True) -> None:
    """Compile the oracle (and, when /root/reference exists, the reference's
    oracle and kernels; the kernels' table data comes from the committed
    artifact tests/golden/ref_tables.txt)."""
    subprocess.run(["make", "-s", "-C", HERE, "libcrvec_oracle.so"], check=True)
    if ref and os.path.isdir("/root/reference/proj"):
        if not os.path.exists(REF_GEN_INC) and os.path.exists(REF_ARTIFACT):
            inc_from_artifact()
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build(ref=False)
        L = ctypes.CDLL(LIB_PATH)
        L.crvec_oracle_f32.restype = ctypes.c_uint32
        L.crvec_oracle_f32.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.crvec_oracle_f64.restype = ctypes.c_uint64
        L.crvec_oracle_f64.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int)]
        L.crvec_oracle_f32_all_modes.argtypes = [ctypes.c_int, ctypes.c_uint32, _u32p, ctypes.c_int]
        L.crvec_oracle_f64_all_modes.argtypes = [ctypes.c_int, ctypes.c_uint64, _u64p]
        L.crvec_oracle_f32_batch.argtypes = [ctypes.c_int, _u32p, _u32p, ctypes.c_uint64,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.crvec_oracle_f64_batch.argtypes = [ctypes.c_int, _u64p, _u64p, ctypes.c_uint64,
                                             ctypes.c_int, ctypes.c_int]
        L.crvec_oracle_sweep_hashes.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                                _u64p, ctypes.c_int, ctypes.c_int]
        L.crvec_oracle_convert_f64_to_f32.restype = ctypes.c_uint32
        L.crvec_oracle_convert_f64_to_f32.argtypes = [ctypes.c_uint64, ctypes.c_int]
        for name in ("cap_failures", "cap_input", "mpfr_calls", "ld_decided"):
            getattr(L, "crvec_oracle_" + name).restype = ctypes.c_uint64
        L.crvec_oracle_mix64.restype = ctypes.c_uint64
        L.crvec_oracle_mix64.argtypes = [ctypes.c_uint64]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        R = ctypes.CDLL(REF_PATH)
        R.crvec_ref_ziv_f32.restype = ctypes.c_uint32
        R.crvec_ref_ziv_f32.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int)]
        R.crvec_ref_ziv_f64.restype = ctypes.c_uint64
        R.crvec_ref_ziv_f64.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int)]
        R.crvec_ref_all_modes_f32.argtypes = [ctypes.c_int, ctypes.c_uint32, _u32p]
        R.crvec_ref_all_modes_f64.argtypes = [ctypes.c_int, ctypes.c_uint64, _u64p]
        R.crvec_ref_convert_f64_to_f32.restype = ctypes.c_uint32
        R.crvec_ref_convert_f64_to_f32.argtypes = [ctypes.c_uint64, ctypes.c_int]
        R.crvec_ref_batch_f32.argtypes = [ctypes.c_int, _u32p, _u32p, ctypes.c_uint64, ctypes.c_int,
                                          ctypes.c_int]
        R.crvec_ref_batch_f64.argtypes = [ctypes.c_int, _u64p, _u64p, ctypes.c_uint64, ctypes.c_int,
                                          ctypes.c_int]
        _ref = R
    return _ref


def _host_has_avx512() -> bool:
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return all(f in flags for f in ("avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"))


def refk_path() -> str | None:
    """The reference-kernel library for this host (AVX-512 build if the host has it)."""
    p4, p2 = REFK_PATHS
    if _host_has_avx512() and os.path.exists(p4):
        return p4
    return p2 if os.path.exists(p2) else None


def refk_available() -> bool:
    return refk_path() is not None


def refk():
    """The REFERENCE's kernels (cr_exp2f/cr_log2f/cr_exp2/cr_log, round_test_lane)."""
    global _refk
    if _refk is None:
        p = refk_path()
        if p is None:
            raise RuntimeError("reference kernels not built: make -C oracle ref")
        K = ctypes.CDLL(p)
        K.crvec_refk_round_test_lane.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int64,
                                                 ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                                 ctypes.POINTER(ctypes.c_double)]
        K.crvec_refk_f32.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int]
        K.crvec_refk_f64.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                     ctypes.c_int, ctypes.c_int, _u64p]
        K.crvec_refk_bounds.argtypes = [ctypes.POINTER(ctypes.c_double)]
        _refk = K
    return _refk


def refk_f32(fn: str, xbits: np.ndarray, mode: int, threads: int = 0, vector: bool = True) -> np.ndarray:
    """The reference's cr_exp2f<16> / cr_log2f<16> (Backend::vector, or the
    per-lane Backend::reference) over an array, std::thread over chunks."""
    x = np.ascontiguousarray(xbits, dtype=np.uint32)
    y = np.empty_like(x)
    rc = refk().crvec_refk_f32(FN[fn], x.ctypes.data, y.ctypes.data, x.size, int(mode), int(vector), threads)
    if rc != 0:
        raise RuntimeError(f"reference kernel: no binary32 {fn}")
    return y


def refk_f64(fn: str, xbits: np.ndarray, mode: int, threads: int = 0):
    """The reference's cr_exp2<16> / cr_log<16> (counted); returns (y, callouts)."""
    x = np.ascontiguousarray(xbits, dtype=np.uint64)
    y = np.empty_like(x)
    und = ctypes.c_uint64(0)
    rc = refk().crvec_refk_f64(FN[fn], x.ctypes.data, y.ctypes.data, x.size, int(mode), threads,
                               ctypes.byref(und))
    if rc != 0:
        raise RuntimeError(f"reference kernel: no binary64 {fn}")
    return y, int(und.value)


def _p32(a):
    return a.ctypes.data_as(_u32p)


def _p64(a):
    return a.ctypes.data_as(_u64p)


def f32(fn: str, xbits: np.ndarray, mode: int | None = None, threads: int = 0,
        use_ld: bool = True) -> np.ndarray:
    """Correctly rounded binary32 results (as uint32 bit patterns).

    mode None -> array of shape (n, 4) indexed by RoundingMode."""
    x = np.ascontiguousarray(xbits, dtype=np.uint32)
    n = x.size
    if mode is None:
        y = np.empty((n, 4), dtype=np.uint32)
        m = -1
    else:
        y = np.empty(n, dtype=np.uint32)
        m = int(mode)
    before = lib().crvec_oracle_cap_failures()
    rc = lib().crvec_oracle_f32_batch(FN[fn], _p32(x), _p32(y), n, m, threads, int(use_ld))
    if rc != 0 or lib().crvec_oracle_cap_failures() != before:
        raise RuntimeError(f"oracle: {fn} undecidable at precision cap "
                           f"(input 0x{lib().crvec_oracle_cap_input():08x})")
    return y


def f64(fn: str, xbits: np.ndarray, mode: int | None = None, threads: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(xbits, dtype=np.uint64)
    n = x.size
    if mode is None:
        y = np.empty((n, 4), dtype=np.uint64)
        m = -1
    else:
        y = np.empty(n, dtype=np.uint64)
        m = int(mode)
    rc = lib().crvec_oracle_f64_batch(FN[fn], _p64(x), _p64(y), n, m, threads)
    if rc != 0:
        raise RuntimeError(f"oracle: {fn} f64 undecidable at precision cap")
    return y


def sweep_hashes(fn: str, chunk_lo: int = 0, chunk_hi: int = 4096, threads: int = 0,
                 use_ld: bool = True) -> np.ndarray:
    """Per-2^20-chunk, per-mode commutative hashes of the CR outputs."""
    h = np.zeros((chunk_hi - chunk_lo, 4), dtype=np.uint64)
    rc = lib().crvec_oracle_sweep_hashes(FN[fn], chunk_lo, chunk_hi, _p64(h), threads, int(use_ld))
    if rc != 0:
        raise RuntimeError(f"oracle: sweep {fn} failed rc={rc}")
    return h


def ref_f32(fn: str, xbits: np.ndarray, mode: int, threads: int = 0) -> np.ndarray:
    """The REFERENCE's ziv_correctly_round_f32 over an array (exp2/log/log2 only)."""
    x = np.ascontiguousarray(xbits, dtype=np.uint32)
    y = np.empty_like(x)
    rc = ref().crvec_ref_batch_f32(FN[fn], _p32(x), _p32(y), x.size, int(mode), threads)
    if rc != 0:
        raise RuntimeError("reference oracle threw")
    return y


def ref_f64(fn: str, xbits: np.ndarray, mode: int, threads: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(xbits, dtype=np.uint64)
    y = np.empty_like(x)
    rc = ref().crvec_ref_batch_f64(FN[fn], _p64(x), _p64(y), x.size, int(mode), threads)
    if rc != 0:
        raise RuntimeError("reference oracle threw")
    return y


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer (vectorized), the sweep hash mixer."""
    z = np.asarray(z, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z
