"""crvec-b200: B200-native correctly rounded vector math (host-side mirror).

Python mirror of the reference's public kernel interface
(ref: proj/include/crvec/kernels_f32.hpp:25-49, kernels_f64.hpp:58-81) over the
C ABI of ``libcrvec.so`` (include/crvec.h):

    RoundingMode            <- crvec::RoundingMode (fpbits.hpp:13-18), same numbering
    cr_exp2f(x, mode)       <- cr_exp2f<W>(Batch<float,W>, RoundingMode, Backend)
    cr_exp2f_scalar(x, mode)<- cr_exp2f_scalar(float, RoundingMode)
    cr_log2f / cr_log2f_scalar, and the other 17 binary32 functions of PAPER.md:49
    cr_exp2 / cr_log (+ _counted with FastPathStats) for binary64

Arrays may be numpy arrays (host path: the library stages them through HBM
with pipelined copies) or CUDA torch tensors (device path, stream-ordered on
torch's current stream). The library has no CPU fallback: every call raises
``CrvecError`` when the CUDA library or an sm_100 device is missing.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CRVEC_LIB: developer override to load an A/B variant build (tools only).
LIB_PATH = os.environ.get("CRVEC_LIB") or os.path.join(_HERE, "libcrvec.so")


class CrvecError(RuntimeError):
    pass


class RoundingMode(enum.IntEnum):
    NearestEven = 0
    TowardZero = 1
    TowardPositive = 2
    TowardNegative = 3


class Backend(enum.IntEnum):
    """Accepted for source compatibility with the reference; ignored (the GPU
    kernel is the only backend)."""
    reference = 0
    vector = 1


# C-ABI function ids (include/crvec.h crvec_fn_t).
FN_IDS = {
    "exp2f": 0, "logf": 1, "log2f": 2, "expf": 3, "exp10f": 4, "expm1f": 5, "log10f": 6,
    "log1pf": 7, "sinf": 8, "cosf": 9, "tanf": 10, "asinf": 11, "acosf": 12, "atanf": 13,
    "sinhf": 14, "coshf": 15, "tanhf": 16, "rsqrtf": 17, "sincosf": 18,
}
F32_FUNCS = [k for k in FN_IDS if k != "sincosf"]
# oracle / MPFR function backing each binary32 function
ORACLE_NAME = {k: k[:-1] for k in F32_FUNCS}

CRVEC_OK, CRVEC_EINVAL, CRVEC_ECUDA, CRVEC_ENOMEM, CRVEC_ENODEV = 0, -1, -2, -3, -4

_lib = None


class Stats(ctypes.Structure):
    _fields_ = [("lanes", ctypes.c_uint64), ("fast_undecided", ctypes.c_uint64),
                ("accurate_undecided", ctypes.c_uint64), ("host_callouts", ctypes.c_uint64)]


@dataclass
class FastPathStats:
    """Mirror of crvec::FastPathStats (ref: proj/include/crvec/kernels_f64.hpp:72-81)."""
    lanes: int = 0
    undecided: int = 0
    accurate_undecided: int = 0
    host_callouts: int = 0


def lib() -> ctypes.CDLL:
    """The loaded C library; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CrvecError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
        L.crvec_eval_f32.argtypes = [i, vp, vp, vp, sz, i]
        L.crvec_eval_f32_dev.argtypes = [i, vp, vp, vp, sz, i, vp]
        L.crvec_sweep_f32.argtypes = [i, ctypes.c_uint32, ctypes.c_uint32, vp, vp, vp, i, vp]
        L.crvec_stats_get.argtypes = [ctypes.POINTER(Stats)]
        L.crvec_strerror.restype = ctypes.c_char_p
        L.crvec_last_cuda_error.restype = ctypes.c_char_p
        L.crvec_version.restype = ctypes.c_char_p
        L.crvec_fn_name.restype = ctypes.c_char_p
        if hasattr(L, "crvec_exp2"):
            for nm in ("crvec_exp2", "crvec_log"):
                getattr(L, nm).argtypes = [vp, vp, sz, i, ctypes.POINTER(Stats)]
            for nm in ("crvec_exp2_dev", "crvec_log_dev"):
                getattr(L, nm).argtypes = [vp, vp, sz, i, vp]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != CRVEC_OK:
        L = lib()
        raise CrvecError(f"crvec: {L.crvec_strerror(rc).decode()} ({rc}); "
                         f"{L.crvec_last_cuda_error().decode()}")


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _stream_ptr(t):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _check_out(t, ref, what):
    """A caller-supplied output tensor must match the input: same CUDA device,
    dtype and element count, and contiguous (the kernels write numel() elements
    through the raw pointer)."""
    if (not _is_torch(t) or t.device != ref.device or t.dtype != ref.dtype
            or t.numel() != ref.numel() or not t.is_contiguous()):
        raise CrvecError(f"{what} must be a contiguous {ref.dtype} tensor on {ref.device} "
                         f"with {ref.numel()} elements")


def _check_out_np(a, ref, what):
    if (not isinstance(a, np.ndarray) or a.dtype != ref.dtype or a.size != ref.size
            or not a.flags.c_contiguous or not a.flags.writeable):
        raise CrvecError(f"{what} must be a writeable contiguous {ref.dtype} array of {ref.size} elements")


def eval_f32(name: str, x, mode: int = RoundingMode.NearestEven, out=None, out2=None):
    """Evaluate binary32 function `name` elementwise; returns out (and out2 for sincosf)."""
    fn = FN_IDS[name]
    L = lib()
    if _is_torch(x):
        import torch
        if not x.is_cuda or x.dtype != torch.float32:
            raise CrvecError("torch input must be a CUDA float32 tensor")
        x = x.contiguous()
        out = torch.empty_like(x) if out is None else out
        _check_out(out, x, "out")
        if fn == FN_IDS["sincosf"]:
            out2 = torch.empty_like(x) if out2 is None else out2
            _check_out(out2, x, "out2")
        # the C ABI launches on the current device: make it the tensor's
        with torch.cuda.device(x.device):
            _check(L.crvec_eval_f32_dev(fn, x.data_ptr(), out.data_ptr(),
                                        out2.data_ptr() if out2 is not None else None,
                                        x.numel(), int(mode), _stream_ptr(x)))
    else:
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty_like(x) if out is None else out
        _check_out_np(out, x, "out")
        if fn == FN_IDS["sincosf"]:
            out2 = np.empty_like(x) if out2 is None else out2
            _check_out_np(out2, x, "out2")
        _check(L.crvec_eval_f32(fn, x.ctypes.data, out.ctypes.data,
                                out2.ctypes.data if out2 is not None else None, x.size, int(mode)))
    return (out, out2) if fn == FN_IDS["sincosf"] else out


def _make(name):
    def f(x, mode=RoundingMode.NearestEven, backend=Backend.vector, out=None):
        return eval_f32(name, x, mode, out)

    def f_scalar(x: float, mode=RoundingMode.NearestEven) -> float:
        return float(eval_f32(name, np.array([x], dtype=np.float32), mode)[0])

    f.__name__ = "cr_" + name
    f_scalar.__name__ = "cr_" + name + "_scalar"
    f.__doc__ = f"Correctly rounded {name} over an array (C ABI crvec_{name} / crvec_{name}_dev)."
    return f, f_scalar


for _n in F32_FUNCS:
    globals()["cr_" + _n], globals()["cr_" + _n + "_scalar"] = _make(_n)


def cr_sincosf(x, mode=RoundingMode.NearestEven):
    return eval_f32("sincosf", x, mode)


def _f64(name, x, mode, stats: FastPathStats | None):
    L = lib()
    if not hasattr(L, "crvec_" + name):
        raise CrvecError("binary64 kernels not built")
    if _is_torch(x):
        import torch
        if not x.is_cuda or x.dtype != torch.float64:
            raise CrvecError("torch input must be a CUDA float64 tensor")
        x = x.contiguous()
        out = torch.empty_like(x)
        if stats is None:
            with torch.cuda.device(x.device):
                _check(getattr(L, f"crvec_{name}_dev")(x.data_ptr(), out.data_ptr(), x.numel(),
                                                       int(mode), _stream_ptr(x)))
            return out
        # counted form: the device counters around a stream-ordered call
        with torch.cuda.device(x.device):
            torch.cuda.current_stream(x.device).synchronize()
            before = _read_stats()
            _check(getattr(L, f"crvec_{name}_dev")(x.data_ptr(), out.data_ptr(), x.numel(),
                                                   int(mode), _stream_ptr(x)))
            torch.cuda.current_stream(x.device).synchronize()
            after = _read_stats()
        stats.lanes += x.numel()
        stats.undecided += after.fast_undecided - before.fast_undecided
        stats.accurate_undecided += after.accurate_undecided - before.accurate_undecided
        stats.host_callouts += after.host_callouts - before.host_callouts
        return out
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    st = Stats()
    _check(getattr(L, "crvec_" + name)(x.ctypes.data, out.ctypes.data, x.size, int(mode),
                                        ctypes.byref(st)))
    if stats is not None:
        stats.lanes += st.lanes
        stats.undecided += st.fast_undecided
        stats.accurate_undecided += st.accurate_undecided
        stats.host_callouts += st.host_callouts
    return out


def cr_exp2(x, mode=RoundingMode.NearestEven, backend=Backend.vector):
    return _f64("exp2", x, mode, None)


def cr_log(x, mode=RoundingMode.NearestEven, backend=Backend.vector):
    return _f64("log", x, mode, None)


def cr_exp2_counted(x, mode, stats: FastPathStats):
    return _f64("exp2", x, mode, stats)


def cr_log_counted(x, mode, stats: FastPathStats):
    return _f64("log", x, mode, stats)


def cr_exp2_scalar(x: float, mode=RoundingMode.NearestEven) -> float:
    return float(cr_exp2(np.array([x]), mode)[0])


def cr_log_scalar(x: float, mode=RoundingMode.NearestEven) -> float:
    return float(cr_log(np.array([x]), mode)[0])


SWEEP_KERNELS, SWEEP_ACCURATE, SWEEP_MAP_KERNELS, SWEEP_ELEMENT_KERNELS = 0, 1, 3, 4  # crvec_sweep_f32 modes


def sweep_f32(name: str, chunk_lo: int = 0, chunk_hi: int = 4096, force_accurate: int = SWEEP_KERNELS,
              device=None):
    """Exhaustive sweep (C ABI crvec_sweep_f32) on the current CUDA device.
    force_accurate: SWEEP_KERNELS (0), SWEEP_ACCURATE (1 / True: every
    main-range lane through the accurate path), SWEEP_MAP_KERNELS (3: the
    product map kernels, crvec_<fn>f_dev, over every pattern, 4 modes) or
    SWEEP_ELEMENT_KERNELS (4: the same through the element kernel that serves
    relatively misaligned arrays).

    Returns (hashes[chunks, 4] uint64, hashes_cos or None, accurate_lanes)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    n = chunk_hi - chunk_lo
    h = torch.zeros((n, 4), dtype=torch.int64, device=dev)
    h2 = torch.zeros((n, 4), dtype=torch.int64, device=dev) if name == "sincosf" else None
    ctr = torch.zeros(4, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        _check(lib().crvec_sweep_f32(FN_IDS[name], chunk_lo, chunk_hi, h.data_ptr(),
                                     h2.data_ptr() if h2 is not None else None, ctr.data_ptr(),
                                     int(force_accurate), _stream_ptr(h)))
    torch.cuda.current_stream(dev).synchronize()
    to_np = lambda t: t.cpu().numpy().view(np.uint64)  # noqa: E731
    return to_np(h), (to_np(h2) if h2 is not None else None), int(ctr[0].item())


def _read_stats() -> Stats:
    st = Stats()
    _check(lib().crvec_stats_get(ctypes.byref(st)))
    return st


def stats() -> Stats:
    """Cumulative counters of the current device (crvec_stats_get)."""
    return _read_stats()


def reset_stats() -> None:
    _check(lib().crvec_stats_reset())


def version() -> str:
    return lib().crvec_version().decode()
