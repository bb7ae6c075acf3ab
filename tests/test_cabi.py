"""CPU tests of the drop-in boundary (no GPU needed): the C-ABI library loads,
exports every symbol include/crvec.h declares, validates arguments, and fails
loudly (CRVEC_ENODEV) without a device — there is no CPU fallback."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "crvec.h")


@pytest.fixture(scope="module")
def lib():
    import paper_2605_15547_b200 as crvec
    if not os.path.exists(crvec.LIB_PATH):
        from paper_2605_15547_b200 import build
        build.build()
    return crvec.lib()


def declared_symbols():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(crvec_\w+)\s*\(", txt, flags=re.M)))


def test_header_symbols_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 50, syms
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2605_15547_b200", "libcrvec.so")],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (crvec_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        getattr(lib, s)  # resolvable through ctypes


def test_no_torch_types_in_abi():
    txt = open(HDR).read()
    assert "torch" not in txt.lower().replace("no torch", "")
    assert "#include <cuda" not in txt


def test_argument_validation(lib):
    x = np.ones(4, np.float32)
    y = np.empty_like(x)
    vp = ctypes.c_void_p
    lib.crvec_eval_f32.argtypes = [ctypes.c_int, vp, vp, vp, ctypes.c_size_t, ctypes.c_int]
    assert lib.crvec_eval_f32(99, x.ctypes.data, y.ctypes.data, None, 4, 0) == -1
    assert lib.crvec_eval_f32(3, x.ctypes.data, y.ctypes.data, None, 4, 7) == -1
    assert lib.crvec_eval_f32(3, None, y.ctypes.data, None, 4, 0) == -1
    assert lib.crvec_eval_f32(18, x.ctypes.data, y.ctypes.data, None, 4, 0) == -1  # sincos needs y2
    assert lib.crvec_eval_f32(3, None, None, None, 0, 0) == 0  # empty input is fine
    lib.crvec_sweep_f32.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, vp, vp, vp, ctypes.c_int, vp]
    assert lib.crvec_sweep_f32(3, 10, 5, x.ctypes.data, None, x.ctypes.data, 0, None) == -1


def test_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2605_15547_b200 as crvec
    with pytest.raises(crvec.CrvecError):
        crvec.cr_expf(np.ones(8, np.float32))
    with pytest.raises(crvec.CrvecError):
        crvec.cr_exp2(np.ones(8))


def test_names_and_version(lib):
    import paper_2605_15547_b200 as crvec
    assert lib.crvec_fn_count() == 19
    for name, fid in crvec.FN_IDS.items():
        assert lib.crvec_fn_name(fid).decode() == name
    assert b"sm_100a" in lib.crvec_version()


def test_kernels_compiled_for_sm100a():
    so = os.path.join(ROOT, "paper_2605_15547_b200", "libcrvec.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    def sass(fn):
        return subprocess.run(["cuobjdump", "-sass", "-fun", fn, so], capture_output=True, text=True).stdout
    # logf: shared-memory (c, L) table read with one LDS.128 per element
    s = sass("_ZN5crvec9k_map_vecINS_6FnLogBILi0EEELi0EEEvPKfPfjPy")
    for op in ("DFMA", "LDS.128", "LDG.E.NA", "STG.E.EF", "F2F.F32.F64"):
        assert op in s, op
    # asinf: (C, S, angle) from the column-split shared table (round 2: the
    # angle moved from a __shfl_sync register table to a third column)
    s = sass("_ZN5crvec9k_map_vecINS_10FnAsinAcosILb0EEELi0EEEvPKfPfjPy")
    for op in ("DFMA", "LDS.64", "LDG.E", "STG.E", "F2F.F32.F64"):
        assert op in s, op
    assert "SHFL.IDX" not in s


def test_cpp_compat_header_compiles(lib, tmp_path):
    exe = tmp_path / "test_compat"
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "test_compat.cpp"),
                        "-L", os.path.join(ROOT, "paper_2605_15547_b200"), "-lcrvec",
                        f"-Wl,-rpath,{os.path.join(ROOT, 'paper_2605_15547_b200')}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rr = subprocess.run([str(exe)], capture_output=True, text=True)
    import torch
    assert rr.returncode == (0 if torch.cuda.is_available() else 77), rr.stdout


def test_tables_reproducible():
    """SPEC acceptance #8: the generator regenerates the checked-in tables."""
    r = subprocess.run(["python", os.path.join(ROOT, "tools", "gen_tables.py"), "--check"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_tables_at_most_16_entries_for_binary32():
    txt = open(os.path.join(ROOT, "paper_2605_15547_b200", "csrc", "crvec_tables.inc")).read()
    f32_part = txt.split("binary64 exp2")[0]
    for name, n in re.findall(r"CR_CONST \w+ (\w+)\[(\d+)\]", f32_part):
        if name.startswith(("INVFACT", "LOG1P_T", "SINT", "COST", "ATANT", "INV_PI_WORDS", "PH_T", "POW10")):
            continue  # accurate-path series coefficients / Payne-Hanek bits of 1/pi (PH_T: the same bits cut per exponent), not lookup tables
        if name.endswith("Q"):
            continue  # polynomial coefficients
        assert int(n) <= 16, (name, n)


def test_python_wrapper_rejects_host_tensors_before_the_abi(lib):
    """Tensors must be CUDA tensors of the path's dtype: a
    host tensor's pointer would fault the kernel, a float32 tensor in the
    binary64 path would be written out of bounds."""
    import torch
    import paper_2605_15547_b200 as crvec
    with pytest.raises(crvec.CrvecError):
        crvec.eval_f32("logf", torch.ones(8))
    with pytest.raises(crvec.CrvecError):
        crvec.cr_exp2(torch.ones(8, dtype=torch.float64))
    with pytest.raises(crvec.CrvecError):
        crvec.cr_log(torch.ones(8, dtype=torch.float32))
    # numpy outputs are validated too
    with pytest.raises(crvec.CrvecError):
        crvec.eval_f32("logf", np.ones(8, dtype=np.float32), out=np.empty(7, dtype=np.float32))
