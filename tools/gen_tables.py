"""Offline table / coefficient generator for the crvec B200 kernels.

Emits ``paper_2605_15547_b200/csrc/crvec_tables.inc`` (checked in). Every table
has <= 16 entries (the paper's constraint, ref: PAPER.md:51) and every
polynomial is a Chebyshev (near-minimax) fit computed with mpmath at 60 digits
then rounded to binary64; the script prints each fast polynomial's worst
relative error so the rounding-test tolerances in the kernels can be checked
against it. ``--check`` regenerates into memory and compares with the
checked-in file byte for byte (SPEC acceptance #8, ref: SPEC.md:666).

This plays the role of the reference's empty coefficient generator
(ref: proj/include/crvec/coeffgen.hpp:16-67, proj/src/coeffgen.cpp:1).
"""
import hashlib
import os
import sys

import mpmath as mp

mp.mp.dps = 60
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_2605_15547_b200", "csrc", "crvec_tables.inc")


def d(x):
    """Round an mpf to the nearest binary64."""
    return float(mp.mpf(x))


def hx(x):
    return float(x).hex()


def dd(x):
    """Double-double split of an mpf: (hi, lo) with hi = RN(x)."""
    x = mp.mpf(x)
    hi = d(x)
    lo = d(x - hi)
    return hi, lo


def trunc_bits(x, bits):
    """x rounded to `bits` significant bits (as a double)."""
    x = mp.mpf(x)
    if x == 0:
        return 0.0
    e = int(mp.floor(mp.log(abs(x), 2)))
    q = mp.mpf(2) ** (e - bits + 1)
    return d(mp.nint(x / q) * q)


def split3(x, b1, b2):
    """x = h + m + l with h (b1 bits), m (b2 bits) and l = RN(x - h - m)."""
    x = mp.mpf(x)
    h = trunc_bits(x, b1)
    m = trunc_bits(x - h, b2)
    l = d(x - h - m)
    return h, m, l


def chebfit(f, a, b, deg):
    """Near-minimax polynomial (coefficients low->high, as mpf) for f on [a, b]."""
    coeffs, err = mp.chebyfit(f, [a, b], deg + 1, error=True)
    return list(reversed(coeffs)), err


def rel_err_of(poly_eval, f, a, b, n=4000):
    worst = mp.mpf(0)
    for i in range(n + 1):
        x = a + (b - a) * mp.mpf(i) / n
        if x == 0:
            continue
        fx = f(x)
        if fx == 0:
            continue
        e = abs((poly_eval(x) - fx) / fx)
        if e > worst:
            worst = e
    return worst


def horner(cs, x):
    acc = mp.mpf(0)
    for c in reversed(cs):
        acc = acc * x + c
    return acc


lines = []
report = []


def emit(s=""):
    lines.append(s)


def arr(name, vals, ctype="double"):
    emit(f"static CR_CONST {ctype} {name}[{len(vals)}] = {{")
    for i in range(0, len(vals), 4):
        emit("    " + ", ".join(hx(v) if ctype == "double" else repr(v) for v in vals[i:i + 4]) + ",")
    emit("};")


def scalar(name, v):
    # constant-bank scalar: FP64 instructions read it as a c[] operand
    emit(f"static CR_CONST double {name} = {hx(v)};")


def poly_block(name, cs):
    arr(name, [d(c) for c in cs])


# ------------------------------------------------------------------ exp ----
LN2 = mp.log(2)
R_EXP = LN2 / 32 * mp.mpf("1.0005")          # |r| bound after k = RN(x*16/ln2)


def gen_exp():
    emit("// ---- exp family: 2^(j/16) table, e^r - 1 polynomial ----")
    T = [mp.mpf(2) ** (mp.mpf(j) / 16) for j in range(16)]
    arr("EXP2J_HI", [dd(t)[0] for t in T])
    arr("EXP2J_LO", [dd(t)[1] for t in T])
    # e^r - 1 = r + r^2 * Q(r), Q degree 4 (fast path)
    g = lambda r: (mp.expm1(r) - r) / r ** 2 if r != 0 else mp.mpf(1) / 2
    for deg, name in ((3, "EXPQ3"), (4, "EXPQ")):
        cs, _ = chebfit(g, -R_EXP, R_EXP, deg)
        csd = [mp.mpf(d(c)) for c in cs]
        err = rel_err_of(lambda r: r + r * r * horner(csd, r), mp.expm1, -R_EXP, R_EXP)
        report.append(f"expm1 poly r+r^2*Q deg(Q)={deg}: max rel err 2^{float(mp.log(err, 2)):.1f}")
        poly_block(name, csd)
    # tanhf works on h = r/2 (the x2 of expm1(2|x|) folded into the reduction):
    # (e^(2h) - 1)/2 = h + h^2 * 2 Q(2h), coefficients EXPQ[i] * 2^(i+1) (exact)
    poly_block("EXPQ_HALF", [c * mp.mpf(2) ** (i + 1) for i, c in enumerate(csd)])
    h, m, l = split3(LN2 / 16, 40, 40)
    scalar("LN2_16_H", h); scalar("LN2_16_M", m); scalar("LN2_16_L", l)
    scalar("LN2_32_H", h / 2); scalar("LN2_32_M", m / 2)  # exact halves
    scalar("INV_LN2_16", d(16 / LN2))
    scalar("INV_LN2_32", d(32 / LN2))
    scalar("LN2_D", d(LN2))
    scalar("LN2_DL", d(LN2 - d(LN2)))
    LOG2_10 = mp.log(10, 2)
    scalar("LOG2_10_16", d(16 * LOG2_10))
    h, m, l = split3(mp.log(10), 29, 29)
    scalar("LN10_H", h); scalar("LN10_M", m); scalar("LN10_L", l)
    # slow path: 1/n! as double-doubles, n = 0..16
    inv_fact = [mp.mpf(1) / mp.factorial(n) for n in range(17)]
    arr("INVFACT_HI", [dd(v)[0] for v in inv_fact])
    arr("INVFACT_LO", [dd(v)[1] for v in inv_fact])
    # exact powers of ten for exp10f(k), k = 0..10
    arr("POW10_D", [float(10 ** k) for k in range(16)])
    # sinh / cosh of r polynomials (fast path), |r| <= R_EXP: degree 1 in r^2
    # (2^-48.5 / 2^-45.7 relative; the kernels' tolerance E = 512 covers them)
    gs = lambda r: (mp.sinh(r) - r) / r ** 3 if r != 0 else mp.mpf(1) / 6
    cs, _ = chebfit(lambda s: gs(mp.sqrt(s)) if s > 0 else mp.mpf(1) / 6, mp.mpf(0), R_EXP ** 2, 1)
    csd = [mp.mpf(d(c)) for c in cs]
    err = rel_err_of(lambda r: r + r ** 3 * horner(csd, r * r), mp.sinh, -R_EXP, R_EXP)
    report.append(f"sinh poly deg(S)=1 in r^2: max rel err 2^{float(mp.log(err, 2)):.1f}")
    poly_block("SINHQ", csd)
    gc = lambda s: (mp.cosh(mp.sqrt(s)) - 1) / s if s > 0 else mp.mpf(1) / 2
    cs, _ = chebfit(gc, mp.mpf(0), R_EXP ** 2, 1)
    csd = [mp.mpf(d(c)) for c in cs]
    err = rel_err_of(lambda r: 1 + r * r * horner(csd, r * r), mp.cosh, -R_EXP, R_EXP)
    report.append(f"cosh poly deg(C)=1 in r^2: max rel err 2^{float(mp.log(err, 2)):.1f}")
    poly_block("COSHQ", csd)


# ------------------------------------------------------------------ log ----
def gen_log():
    emit("// ---- log family: normalization window [0.765625, 1.53125), 16 bins ----")
    # bin i spans hi-words [OFF + i*2^16, OFF + (i+1)*2^16), OFF = 0x3FE88000
    OFFV = mp.mpf("0.765625")
    lo_edges = []
    for i in range(16):
        if i < 7:
            a = OFFV + mp.mpf(i) / 32
            b = a + mp.mpf(1) / 32
        elif i == 7:
            a, b = 1 - mp.mpf(1) / 64, 1 + mp.mpf(1) / 32
        else:
            a = 1 + mp.mpf(1) / 32 + mp.mpf(i - 8) / 16
            b = a + mp.mpf(1) / 16
        lo_edges.append((a, b))
    cs_, L, L2, L10 = [], [], [], []
    rmin, rmax = mp.mpf(0), mp.mpf(0)
    for i, (a, b) in enumerate(lo_edges):
        if i == 7:
            c = mp.mpf(1)
        else:
            c = mp.mpf(trunc_bits(2 / (a + b), 20))
        cs_.append(float(c))
        rmin = min(rmin, a * c - 1)
        rmax = max(rmax, b * c - 1)
        L.append(-mp.log(c))
        L2.append(-mp.log(c, 2))
        L10.append(-mp.log(c, 10))
    arr("LOG_C", cs_)
    assert all((int.from_bytes(__import__("struct").pack("<d", c), "little") & 0xFFFFFFFF) == 0 for c in cs_)
    emit("static CR_CONST int LOG_C_HI[16] = {")
    emit("    " + ", ".join(str(int.from_bytes(__import__("struct").pack("<d", c), "little") >> 32) for c in cs_) + ",")
    emit("};")
    arr("LOG_L_HI", [dd(v)[0] for v in L]); arr("LOG_L_LO", [dd(v)[1] for v in L])
    arr("LOG2_L_HI", [dd(v)[0] for v in L2]); arr("LOG2_L_LO", [dd(v)[1] for v in L2])
    arr("LOG10_L_HI", [dd(v)[0] for v in L10]); arr("LOG10_L_LO", [dd(v)[1] for v in L10])
    report.append(f"log r range [{float(rmin):.5f}, {float(rmax):.5f}]")
    a, b = rmin * mp.mpf("1.001"), rmax * mp.mpf("1.001")
    g = lambda r: (mp.log1p(r) - r) / r ** 2 if r != 0 else -mp.mpf(1) / 2
    for deg in (5,):  # 2^-43.3: the log kernels' tolerance E = 1024 covers it
        cs, _ = chebfit(g, a, b, deg)
        csd = [mp.mpf(d(c)) for c in cs]
        err = rel_err_of(lambda r: r + r * r * horner(csd, r), mp.log1p, a, b)
        report.append(f"log1p poly r+r^2*Q deg(Q)={deg}: max rel err 2^{float(mp.log(err, 2)):.1f}")
        poly_block("LOGQ", csd)
    h, m, l = split3(LN2, 40, 40)
    scalar("LN2_H", h); scalar("LN2_M", m); scalar("LN2_L", l)
    scalar("INV_LN2", d(1 / LN2)); scalar("INV_LN2_L", d(1 / LN2 - d(1 / LN2)))
    scalar("INV_LN10", d(1 / mp.log(10))); scalar("INV_LN10_L", d(1 / mp.log(10) - d(1 / mp.log(10))))
    scalar("LOG10_2", d(mp.log(2, 10))); scalar("LOG10_2_L", d(mp.log(2, 10) - d(mp.log(2, 10))))
    # slow path: log1p(r) = sum (-1)^(n+1) r^n / n as DD, n = 1..24
    inv = [mp.mpf((-1) ** (n + 1)) / n for n in range(1, 25)]
    arr("LOG1P_T_HI", [dd(v)[0] for v in inv]); arr("LOG1P_T_LO", [dd(v)[1] for v in inv])


# ----------------------------------------------------------------- trig ----
def gen_ph_table():
    """Exponent-indexed Payne-Hanek table of the fast path (every binary32
    exponent, so one reduction serves small and large arguments alike).

    x = M * 2^E (M < 2^24 an integer, E = max(b, 1) - 150 for biased exponent
    b). x*16/pi mod 32 = x * T_E mod 32 with T_E = (16/pi) mod 2^(5-E): the
    bits of 16/pi of weight >= 2^(5-E) only add multiples of 32*M. T_E is cut
    into hi (lsb 2^-L, L = 48 + E for E > 2, min(50, 53 + E) otherwise: hi has
    <= 53 bits and x*hi - RN(x*hi) is exact in binary64) and lo = RN(T_E - hi),
    so |x * (hi + lo - T_E)| < 2^-77. Row b (16 bytes: hi, lo) for b = 0..255
    (row 255, Inf/NaN, is never used on the main path)."""
    emit("// Payne-Hanek fast-path table: (hi, lo) of (16/pi) mod 2^(5-E) per binary32 exponent")
    rows = []
    with mp.workprec(1200):
        C = 16 / mp.pi
        for b in range(256):
            if b == 255:
                rows.extend([0.0, 0.0])
                continue
            E = max(b, 1) - 150
            T = C - mp.mpf(2) ** (5 - E) * mp.floor(C / mp.mpf(2) ** (5 - E)) if E > 2 else C
            L = 48 + E if E > 2 else min(50, 53 + E)
            hi = mp.floor(T * mp.mpf(2) ** L) / mp.mpf(2) ** L
            assert mp.mpf(d(hi)) == hi, b  # <= 53 bits
            lo = d(T - hi)
            rows.extend([d(hi), lo])
            # |x (hi + lo - T)| for the largest x of this exponent
            err = abs(mp.mpf(2) ** (E + 24) * (hi + mp.mpf(lo) - T))
            assert err < mp.mpf(2) ** -76, (b, float(mp.log(err, 2)))
    arr("PH_T", rows)


def gen_trig():
    emit("// ---- trig: k = RN(x*16/pi), sin(j*pi/16) table, sin/cos of r ----")
    PI = mp.pi
    S = [mp.sin(j * PI / 16) for j in range(16)]
    arr("SIN16_HI", [dd(v)[0] for v in S]); arr("SIN16_LO", [dd(v)[1] for v in S])
    arr("COS16_HI", [dd(mp.cos(j * PI / 16))[0] for j in range(16)])
    R = PI / 32 * mp.mpf("1.0005")
    gs = lambda s: (mp.sin(mp.sqrt(s)) - mp.sqrt(s)) / (mp.sqrt(s) * s) if s > 0 else -mp.mpf(1) / 6
    cs, _ = chebfit(gs, mp.mpf(0), R ** 2, 2)
    csd = [mp.mpf(d(c)) for c in cs]
    err = rel_err_of(lambda r: r + r ** 3 * horner(csd, r * r), mp.sin, -R, R)
    report.append(f"sin poly deg 2 in r^2: max rel err 2^{float(mp.log(err, 2)):.1f}")
    poly_block("SINQ", csd)
    gc = lambda s: (mp.cos(mp.sqrt(s)) - 1) / s if s > 0 else -mp.mpf(1) / 2
    cs, _ = chebfit(gc, mp.mpf(0), R ** 2, 2)
    csd = [mp.mpf(d(c)) for c in cs]
    err = rel_err_of(lambda r: 1 + r * r * horner(csd, r * r), mp.cos, -R, R)
    report.append(f"cos poly deg 2 in r^2: max rel err 2^{float(mp.log(err, 2)):.1f}")
    poly_block("COSQ", csd)
    # tan r = r + r^3 T(r^2), T of degree 3 (tanf's fast path: (S_j + C_j t) / (C_j - S_j t))
    gt = lambda s: (mp.tan(mp.sqrt(s)) - mp.sqrt(s)) / (mp.sqrt(s) * s) if s > 0 else mp.mpf(1) / 3
    cs, _ = chebfit(gt, mp.mpf(0), R ** 2, 3)
    csd = [mp.mpf(d(c)) for c in cs]
    err = rel_err_of(lambda r: r + r ** 3 * horner(csd, r * r), mp.tan, -R, R)
    report.append(f"tan poly deg 3 in r^2: max rel err 2^{float(mp.log(err, 2)):.1f}")
    poly_block("TANQ", csd)
    scalar("INV_PI_16", d(16 / PI))
    h, m, l = split3(PI / 16, 33, 33)
    scalar("PI_16_H", h); scalar("PI_16_M", m); scalar("PI_16_L", l)
    # two-part split for |x| < 2^12 (k < 2^14.4: k * PI_16_A exact with 36 bits)
    a = trunc_bits(PI / 16, 36)
    scalar("PI_16_A", a); scalar("PI_16_B", d(PI / 16 - a))
    # four-part split for the DD slow path
    p1, p2, rest = split3(PI / 16, 33, 33)
    p3 = trunc_bits(PI / 16 - p1 - p2, 33)
    p4 = d(PI / 16 - p1 - p2 - p3)
    scalar("PI_16_Q1", p1); scalar("PI_16_Q2", p2); scalar("PI_16_Q3", p3); scalar("PI_16_Q4", p4)
    # Payne-Hanek: bits of 1/pi, 32-bit words, word w holds bits [32w+1, 32w+32]
    # (bit j has weight 2^-j); 2 zero words of padding in front.
    # (320 bits of 1/pi need more than the module's working precision)
    with mp.workprec(1200):
        v = 1 / mp.pi
        words = [0, 0]
        for w in range(10):
            v = v * (mp.mpf(2) ** 32)
            iw = int(mp.floor(v))
            words.append(iw)
            v -= iw
    emit("static CR_CONST unsigned INV_PI_WORDS[12] = {")
    emit("    " + ", ".join(f"0x{w:08x}u" for w in words) + ",")
    emit("};")
    hi, lo = dd(PI / 16 * mp.mpf(2) ** -64)
    scalar("PI_16_2M64_H", hi); scalar("PI_16_2M64_L", lo)
    scalar("PI_16_RN", d(PI / 16))
    gen_ph_table()
    # slow path: sin/cos Taylor terms (-1)^n / (2n+1)!, (-1)^n / (2n)!
    sn = [mp.mpf((-1) ** n) / mp.factorial(2 * n + 1) for n in range(12)]
    cn = [mp.mpf((-1) ** n) / mp.factorial(2 * n) for n in range(12)]
    arr("SINT_HI", [dd(v)[0] for v in sn]); arr("SINT_LO", [dd(v)[1] for v in sn])
    arr("COST_HI", [dd(v)[0] for v in cn]); arr("COST_LO", [dd(v)[1] for v in cn])


# ---------------------------------------------------------- inverse trig ----
def gen_atrig():
    emit("// ---- inverse trig: theta_j = j*pi/30, j = 0..15, atan(t) polynomial ----")
    PI = mp.pi
    S = [mp.sin(j * PI / 30) for j in range(16)]
    arr("SIN30_HI", [dd(v)[0] for v in S]); arr("SIN30_LO", [dd(v)[1] for v in S])
    T = mp.tan(PI / 60 + mp.mpf("0.0065"))
    report.append(f"atan t bound {float(T):.5f}")
    g = lambda s: (mp.atan(mp.sqrt(s)) - mp.sqrt(s)) / (mp.sqrt(s) * s) if s > 0 else -mp.mpf(1) / 3
    for deg in (3,):
        cs, _ = chebfit(g, mp.mpf(0), T ** 2, deg)
        csd = [mp.mpf(d(c)) for c in cs]
        err = rel_err_of(lambda t: t + t ** 3 * horner(csd, t * t), mp.atan, -T, T)
        report.append(f"atan poly deg {deg} in t^2: max rel err 2^{float(mp.log(err, 2)):.1f}")
        poly_block("ATANQ", csd)
    h, l = dd(PI / 30)
    scalar("PI_30_H", h); scalar("PI_30_L", l)
    h, l = dd(PI)
    scalar("PI_H", h); scalar("PI_L", l)
    an = [mp.mpf((-1) ** n) / (2 * n + 1) for n in range(20)]
    arr("ATANT_HI", [dd(v)[0] for v in an]); arr("ATANT_LO", [dd(v)[1] for v in an])
    gen_asin()
    gen_atan()


def gen_atan():
    """atan by angle subtraction: atan z = A_k + atan((z C_k - S_k)/(C_k + z S_k))
    for any angle A_k (C, S = cos, sin A_k). Entry k = j + 8*up, up = (z > 1),
    j = RN(7.49 * min(z, 1/z)) in 0..7: A_j = atan(j/7.49), A_{8+j} = pi/2 - A_j,
    rounded to 21 bits (one 32-bit word per entry)."""
    emit("// ---- atan: angle-subtraction table, k = j + 8*up ----")
    K = mp.mpf("7.49")
    ang = []
    for k in range(16):
        j, up = k % 8, k >= 8
        th = mp.atan(mp.mpf(j) / K)
        ang.append(mp.pi / 2 - th if up else th)
    hv = [hi_word(a) for a in ang]
    emit("static CR_CONST int ATAN_A_HI[16] = {")
    emit("    " + ", ".join(str(h if h < 2**31 else h - 2**32) for _, h in hv) + ",")
    emit("};")
    arr("ATAN_C", [d(mp.cos(v)) for v, _ in hv])
    arr("ATAN_S", [d(mp.sin(v)) for v, _ in hv])
    worst = mp.mpf(0)
    for i in range(20001):
        p = mp.mpf(i) / 20000
        j = int(mp.nint(p * K))
        worst = max(worst, abs(mp.atan(p) - hv[j][0]))
    T = mp.tan(worst) * mp.mpf("1.02")
    report.append(f"atan (angle subtraction) reduced |t| <= {float(T):.5f}")
    g = lambda s: (mp.atan(mp.sqrt(s)) - mp.sqrt(s)) / (mp.sqrt(s) * s) if s > 0 else -mp.mpf(1) / 3
    cs, _ = chebfit(g, mp.mpf(0), T ** 2, 3)
    csd = [mp.mpf(d(c)) for c in cs]
    err = rel_err_of(lambda t: t + t ** 3 * horner(csd, t * t), mp.atan, -T, T)
    report.append(f"atan2 poly deg 3 in t^2 (|t| <= {float(T):.4f}): max rel err 2^{float(mp.log(err, 2)):.1f}")
    poly_block("ATANQ2", csd)


def hi_word(x):
    """x rounded to 21 significant bits: a double whose low word is zero."""
    v = trunc_bits(x, 21)
    b = int.from_bytes(__import__("struct").pack("<d", v), "little")
    assert b & 0xFFFFFFFF == 0
    return v, b >> 32


def gen_asin():
    """asin / acos by angle subtraction without division:
    asin(|x|) = A_k + asin(|x| cos A_k - s sin A_k), s = sqrt(1 - x^2), and
    acos(|x|) = B_k + asin(s cos B_k - |x| sin B_k). Entry k = j + 8*up,
    up = (|x| > s), j = RN(10.5 * min(|x|, s)) in 0..7; the angles are rounded
    to 21 bits (one 32-bit word per entry) and their sin / cos rounded to
    binary64, so sin(theta - A_k) is a two-term dot product."""
    emit("// ---- asin / acos: angle-subtraction tables, k = j + 8*up ----")
    PI2 = mp.pi / 2
    A, B = [], []
    for k in range(16):
        j, up = k % 8, k >= 8
        th = mp.asin(mp.mpf(j) / mp.mpf("10.5"))
        A.append(PI2 - th if up else th)
        B.append(th if up else PI2 - th)
    for name, ang in (("ASIN", A), ("ACOS", B)):
        hv = [hi_word(a) for a in ang]
        emit(f"static CR_CONST int {name}_A_HI[16] = {{")
        emit("    " + ", ".join(str(h if h < 2**31 else h - 2**32) for _, h in hv) + ",")
        emit("};")
        arr(f"{name}_C", [d(mp.cos(v)) for v, _ in hv])
        arr(f"{name}_S", [d(mp.sin(v)) for v, _ in hv])
    # reduced argument bound: |theta - A_k| over the grid (+ rounding slack)
    worst = mp.mpf(0)
    for i in range(20001):
        p = mp.sqrt(mp.mpf(1) / 2) * i / 20000
        j = int(mp.nint(p * mp.mpf("10.5")))
        worst = max(worst, abs(mp.asin(p) - mp.asin(mp.mpf(j) / mp.mpf("10.5"))))
    D = mp.sin(worst) * mp.mpf("1.02")
    report.append(f"asin reduced |d| <= {float(D):.5f}")
    g = lambda s: (mp.asin(mp.sqrt(s)) - mp.sqrt(s)) / (mp.sqrt(s) * s) if s > 0 else mp.mpf(1) / 6
    cs, _ = chebfit(g, mp.mpf(0), D ** 2, 3)
    csd = [mp.mpf(d(c)) for c in cs]
    err = rel_err_of(lambda t: t + t ** 3 * horner(csd, t * t), mp.asin, -D, D)
    report.append(f"asin poly deg 3 in d^2: max rel err 2^{float(mp.log(err, 2)):.1f}")
    poly_block("ASINQ", csd)


# ---------------------------------------------------------------- binary64 --
def gen_f64():
    """Tables for the binary64 exp2 / log fast paths (ref: PAPER.md II.B;
    ref: proj/include/crvec/tables.hpp:33-51) and the multiword constants of
    their accurate path."""
    emit("// ---- binary64 exp2: x = N + (i1*256 + i2*16 + i3)/4096 + R, three DD tables ----")
    for lvl, den in ((1, 16), (2, 256), (3, 4096)):
        T = [mp.mpf(2) ** (mp.mpf(j) / den) for j in range(16)]
        arr(f"EXP2D_T{lvl}_HI", [dd(t)[0] for t in T])
        arr(f"EXP2D_T{lvl}_LO", [dd(t)[1] for t in T])
    # 2^R = 1 + R ln2 + R^2 q(R), q Taylor (|R ln2| <= 2^-13.5, truncation < 2^-106)
    q = [LN2 ** n / mp.factorial(n) for n in range(2, 8)]
    arr("EXP2D_Q", [d(c) for c in q])
    # fast path: x = N + (ia*64 + ib)/4096 + R, two 64-entry DD tables, and a
    # degree-5 Taylor tail (R^6 term < 2^-84 relative for |R| <= 2^-13)
    emit("// ---- binary64 exp2 fast path: 2^(ia/64) * 2^(ib/4096), 64-entry DD tables ----")
    for nm, den in (("A", 64), ("B", 4096)):
        T = [mp.mpf(2) ** (mp.mpf(j) / den) for j in range(64)]
        arr(f"EXP2D_{nm}_HI", [dd(t)[0] for t in T])
        arr(f"EXP2D_{nm}_LO", [dd(t)[1] for t in T])
    arr("EXP2D_Q4", [d(LN2 ** n / mp.factorial(n)) for n in range(2, 6)])
    h, l = dd(LN2)
    scalar("LN2D_H", h); scalar("LN2D_L", l)
    emit("// ---- binary64 log: m in [0.75, 1.5), 128 bins, c_i = 1/mid (7 bits) ----")
    cs, Ls = [], []
    for i in range(128):
        if i < 64:
            a = mp.mpf("0.75") + mp.mpf(i) / 256
            b = a + mp.mpf(1) / 256
        else:
            a = 1 + mp.mpf(i - 64) / 128
            b = a + mp.mpf(1) / 128
        c = mp.mpf(1) if i in (63, 64) else mp.mpf(trunc_bits(2 / (a + b), 7))
        cs.append(float(c))
        Ls.append(-mp.log(c))
    arr("LOGD_C", cs)
    arr("LOGD_L_HI", [dd(v)[0] for v in Ls])
    arr("LOGD_L_LO", [dd(v)[1] for v in Ls])
    # L_i trimmed to the 2^-40 grid so e*LN2_H + L_i is exact in one add
    Lt = [mp.nint(v * mp.mpf(2) ** 40) / mp.mpf(2) ** 40 for v in Ls]
    arr("LOGD_LT_HI", [d(v) for v in Lt])
    arr("LOGD_LT_LO", [d(v - t) for v, t in zip(Ls, Lt)])
    # fast path (B200): 512 bins, c_i = 1/mid to 10 bits (r = m c_i - 1 exact,
    # |r| < 2^-9.4, 53 bits), -log c_i split on the 2^-40 grid, degree-6 tail
    emit("// ---- binary64 log fast path: 512 bins, |r| < 2^-9.4 ----")
    cs5, L5 = [], []
    for i in range(512):
        if i < 256:
            a = mp.mpf("0.75") + mp.mpf(i) / 1024
            b = a + mp.mpf(1) / 1024
        else:
            a = 1 + mp.mpf(i - 256) / 512
            b = a + mp.mpf(1) / 512
        c = mp.mpf(1) if i in (255, 256) else mp.mpf(trunc_bits(2 / (a + b), 10))
        cs5.append(float(c))
        L5.append(-mp.log(c))
    arr("LOGD5_C", cs5)
    Lt5 = [mp.nint(v * mp.mpf(2) ** 40) / mp.mpf(2) ** 40 for v in L5]
    arr("LOGD5_LT_HI", [d(v) for v in Lt5])
    arr("LOGD5_LT_LO", [d(v - t) for v, t in zip(L5, Lt5)])
    # log1p(r) = r - r^2/2 + r^3 P(r), P(r) = 1/3 - r/4 + ... + r^6/9
    arr("LOGD5_P", [d(mp.mpf((-1) ** n) / (n + 3)) for n in range(7)])
    h, m, l = split3(LN2, 40, 40)
    scalar("LN2_HD", h)
    scalar("LN2_LD", d(LN2 - h))
    arr("LOGD_TAIL", [d(mp.mpf((-1) ** (n + 1)) / n) for n in range(4, 13)])
    h, l = dd(mp.mpf(1) / 3)
    scalar("THIRD_H", h); scalar("THIRD_L", l)
    # multiword: ln2 to 288 bits as 9 x u32, most significant first (value = 0.w0 w1 ...)
    v = LN2
    words = []
    for _ in range(9):
        v *= mp.mpf(2) ** 32
        w = int(mp.floor(v))
        words.append(w)
        v -= w
    emit("static CR_CONST unsigned LN2_WORDS[9] = {")
    emit("    " + ", ".join(f"0x{w:08x}u" for w in words) + ",")
    emit("};")


def generate():
    lines.clear()
    report.clear()
    emit("// GENERATED by tools/gen_tables.py -- do not edit. Tables <= 16 entries.")
    emit("#pragma once")
    gen_exp()
    gen_log()
    gen_trig()
    gen_atrig()
    gen_f64()
    return "\n".join(lines) + "\n"


def main():
    text = generate()
    if "--check" in sys.argv:
        cur = open(OUT).read()
        ok = cur == text
        print("tables:", "reproducible" if ok else "MISMATCH", hashlib.sha256(text.encode()).hexdigest()[:16])
        sys.exit(0 if ok else 1)
    with open(OUT, "w") as f:
        f.write(text)
    for r in report:
        print(r)
    print("wrote", OUT, hashlib.sha256(text.encode()).hexdigest()[:16])


if __name__ == "__main__":
    main()
