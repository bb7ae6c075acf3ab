"""Seeded synthetic inputs shared by tests and bench (counter-free, numpy)."""
import numpy as np

SPECIAL_F32 = np.array([
    0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00000, 0x7F800001,
    0xFF912345, 0x7FA00000, 0x00000001, 0x80000001, 0x007FFFFF, 0x807FFFFF, 0x00800000,
    0x80800000, 0x7F7FFFFF, 0xFF7FFFFF, 0x3F800000, 0xBF800000, 0x3F800001, 0x3F7FFFFF,
    0x40000000, 0xC0000000, 0x3F000000, 0x41200000, 0x42C80000, 0x447A0000, 0x43000000,
    0xC3160000, 0xC3150000, 0x42B17218, 0x42B17217, 0xC2CFF1B5, 0x33800000, 0xB3800000,
    0x32800000, 0x39800000, 0x3FC90FDB, 0x40490FDB, 0x4B000000, 0x4B800000, 0x47800000,
    0x5A000000, 0x7E000000, 0x3E800000,
], dtype=np.uint32)

RANGES = {
    "expf": (-110, 95), "exp2f": (-155, 135), "exp10f": (-50, 45), "expm1f": (-20, 95),
    "sinhf": (-95, 95), "coshf": (-95, 95), "tanhf": (-12, 12), "logf": (0, 10),
    "log2f": (0, 10), "log10f": (0, 10), "log1pf": (-1, 5), "sinf": (-100, 100),
    "cosf": (-100, 100), "tanf": (-100, 100), "sincosf": (-100, 100), "asinf": (-1, 1),
    "acosf": (-1, 1), "atanf": (-50, 50), "rsqrtf": (0, 100),
}


def mixed_f32(name: str, n: int, seed: int = 1) -> np.ndarray:
    """n/2 uniform bit patterns (all classes) + n/2 uniform reals over the
    function's interesting range + the special list. Returns uint32 bits."""
    rng = np.random.default_rng(seed)
    lo, hi = RANGES[name]
    a = rng.integers(0, 2**32, n // 2, dtype=np.uint64).astype(np.uint32)
    b = rng.uniform(lo, hi, n - n // 2).astype(np.float32).view(np.uint32)
    return np.concatenate([a, b, SPECIAL_F32])


def log_family_input(name: str, n: int, seed: int = 3) -> np.ndarray:
    """Config C2 (BASELINE.json configs[1]): 15/16 uniform positive bit patterns,
    ~1% injected subnormals, 0.1% each of +-0, +-Inf, qNaN/sNaN with payloads,
    negatives; log1pf adds U(-1, 0)."""
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 0x7F800000, n, dtype=np.uint64).astype(np.uint32)
    k = rng.integers(0, 1000, n)
    x = np.where(k < 10, rng.integers(1, 0x00800000, n, dtype=np.uint64).astype(np.uint32), x)
    x = np.where(k == 10, np.uint32(0), x)
    x = np.where(k == 11, np.uint32(0x80000000), x)
    x = np.where(k == 12, np.uint32(0x7F800000), x)
    x = np.where(k == 13, np.uint32(0xFF800000), x)
    x = np.where(k == 14, np.uint32(0x7FC12345), x)
    x = np.where(k == 15, np.uint32(0xFFA54321), x)
    x = np.where(k == 16, (x | np.uint32(0x80000000)), x)
    if name == "log1pf":
        neg = rng.uniform(-1, 0, n).astype(np.float32).view(np.uint32)
        x = np.where((k >= 17) & (k < 80), neg, x)
    return x


def trig_input(n: int, seed: int = 4) -> np.ndarray:
    """Config C3: 7/8 uniform real U[-100, 100]; 1/8 large-argument tail
    |x| in [2^15, 2^128) (random exponent 142..254, random mantissa and sign),
    randomly interleaved."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-100, 100, n).astype(np.float32).view(np.uint32)
    e = rng.integers(142, 255, n, dtype=np.uint64).astype(np.uint32)
    m = rng.integers(0, 1 << 23, n, dtype=np.uint64).astype(np.uint32)
    s = rng.integers(0, 2, n, dtype=np.uint64).astype(np.uint32) << np.uint32(31)
    big = s | (e << np.uint32(23)) | m
    return np.where(rng.integers(0, 8, n) == 0, big, x)


def device_input(name: str, n: int, dist: str = "config", seed: int = 7, device: str = "cuda",
                 specials: bool = True):
    """The same distributions as above generated on the device with torch (for
    the perf tools: 2^28-element inputs in milliseconds; not bit-identical to
    the numpy generators). Returns a float32 tensor."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def ubits(m, hi=2**32):
        return torch.randint(0, hi, (m,), generator=g, device=device, dtype=torch.int64)

    lo, hi = RANGES[name]
    if dist == "uniform" or name not in ("logf", "log2f", "log10f", "log1pf", "sinf", "cosf",
                                         "tanf", "sincosf"):
        u = torch.rand(n, generator=g, device=device, dtype=torch.float64)
        return (lo + (hi - lo) * u).to(torch.float32)
    if name in ("sinf", "cosf", "tanf", "sincosf"):
        u = torch.rand(n, generator=g, device=device, dtype=torch.float64)
        x = (-100 + 200 * u).to(torch.float32).view(torch.int32).to(torch.int64)
        e = torch.randint(142, 255, (n,), generator=g, device=device)
        m = ubits(n, 1 << 23)
        s = ubits(n, 2) << 31
        big = s | (e << 23) | m
        x = torch.where(torch.randint(0, 8, (n,), generator=g, device=device) == 0, big, x)
    else:
        x = ubits(n, 0x7F800000)
        k = torch.randint(0, 1000, (n,), generator=g, device=device)
        x = torch.where(k < 10, ubits(n, 0x00800000 - 1) + 1, x)
        if specials:
            for kk, v in ((10, 0), (11, 0x80000000), (12, 0x7F800000), (13, 0xFF800000),
                          (14, 0x7FC12345), (15, 0xFFA54321)):
                x = torch.where(k == kk, torch.full_like(x, v), x)
            x = torch.where(k == 16, x | 0x80000000, x)
        if name == "log1pf":
            u = torch.rand(n, generator=g, device=device, dtype=torch.float64)
            neg = (-u).to(torch.float32).view(torch.int32).to(torch.int64) & 0xFFFFFFFF
            x = torch.where((k >= 17) & (k < 80), neg, x)
    x = x & 0xFFFFFFFF
    x = torch.where(x >= 2**31, x - 2**32, x)
    return x.to(torch.int32).view(torch.float32)
