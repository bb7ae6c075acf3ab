"""CPU checks of round-2 fast-path constants: the tanhf halved reduction, the
tanf polynomial, and the trig fast path's exponent-indexed Payne-Hanek table
(PH_T in csrc/crvec_tables.inc, tools/gen_tables.py gen_ph_table) and of the
reduction it feeds (red_trig_ph in csrc/crvec_fns_f32.cuh), restated in exact
rational arithmetic:

  x = M 2^E, row b: hi + lo ~ T_E = (16/pi) mod 2^(5-E)
  t = RN(x hi + 1.5 2^52), kd = t - 1.5 2^52, f0 = x hi - kd (must be exact),
  u = RN(x lo + f0),  k = kd mod 32,  u ~ x 16/pi - k  (mod 32)

The exhaustive GPU sweep checks every binary32 input end to end; these tests
pin the two properties the design relies on, on random mantissas of every
exponent: f0 is representable (so the FMA computes it exactly) and u differs
from the true reduced argument by < 2^-70 absolute plus u's own rounding."""
import os
import re
from fractions import Fraction

import numpy as np
import pytest

mp = pytest.importorskip("mpmath")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "paper_2605_15547_b200", "csrc", "crvec_tables.inc")
SHIFTER = Fraction(3, 2) * 2 ** 52


def _ph_table():
    txt = open(INC).read()
    m = re.search(r"PH_T\[(\d+)\] = \{(.*?)\};", txt, flags=re.S)
    vals = [float.fromhex(v.strip()) if "0x" in v else float(v) for v in m.group(2).split(",") if v.strip()]
    assert len(vals) == int(m.group(1)) == 512
    return vals


def _rn(q: Fraction) -> Fraction:
    """Round a rational to the nearest binary64 (ties to even), exactly."""
    if q == 0:
        return q
    f = float(q)  # correctly rounded by Python for Fractions
    return Fraction(f)


def _representable(q: Fraction) -> bool:
    return q == 0 or Fraction(float(q)) == q


@pytest.fixture(scope="module")
def table():
    return _ph_table()


@pytest.fixture(scope="module")
def sixteen_over_pi():
    with mp.workprec(1400):
        v = mp.mpf(16) / mp.pi
        return Fraction(int(mp.floor(v * mp.mpf(2) ** 1300)), 2 ** 1300)


@pytest.mark.parametrize("b", [1, 60, 100, 115, 126, 127, 130, 138, 139, 140, 150, 170, 200, 230, 254])
def test_row_reduction_exact_and_accurate(table, sixteen_over_pi, b):
    hi, lo = Fraction(table[2 * b]), Fraction(table[2 * b + 1])
    E = max(b, 1) - 150
    C = sixteen_over_pi
    rng = np.random.default_rng(b)
    for M in list(rng.integers(1 << 23, 1 << 24, 40)) + [(1 << 23), (1 << 24) - 1]:
        x = Fraction(int(M)) * Fraction(2) ** E
        t = _rn(x * hi + SHIFTER)
        kd = t - SHIFTER
        f0 = x * hi - kd
        assert _representable(f0), (b, M)          # the FMA computes it exactly
        assert abs(f0) <= Fraction(1, 2)
        u = _rn(x * lo + f0)
        # true reduced argument: x 16/pi - k, k = kd (mod 32 it is what the kernel uses)
        true_u = x * C - kd
        true_u -= 32 * round(true_u / 32)  # multiples of 32 in x C are dropped by T_E
        err = abs(u - true_u)
        bound = Fraction(1, 2 ** 70) + abs(u) * Fraction(1, 2 ** 52)
        assert err <= bound, (b, int(M), float(err))


def test_rows_cover_every_exponent(table):
    # row 255 (Inf / NaN) is never used on the main path; every other row is set
    assert table[2 * 255] == 0.0 and table[2 * 255 + 1] == 0.0
    assert all(table[2 * b] != 0.0 or table[2 * b + 1] != 0.0 for b in range(255))


def _arr(name):
    txt = open(INC).read()
    m = re.search(name + r"\[(\d+)\] = \{(.*?)\};", txt, flags=re.S)
    return [float.fromhex(v.strip()) if "0x" in v else float(v) for v in m.group(2).split(",") if v.strip()]


def _scalar(name):
    m = re.search(r"CR_CONST double " + name + r" = ([^;]+);", open(INC).read())
    v = m.group(1).strip()
    return float.fromhex(v) if "0x" in v else float(v)


def test_tanh_halved_constants_are_exact_scalings():
    """tanhf works on h = r/2 (FnTanh::fast): its coefficients and Cody-Waite
    constants must be exact power-of-two scalings of the exp family's."""
    q, qh = _arr("EXPQ"), _arr("EXPQ_HALF")
    assert len(q) == len(qh) == 5
    for i, (a, b) in enumerate(zip(q, qh)):
        assert Fraction(b) == Fraction(a) * 2 ** (i + 1)
    assert Fraction(_scalar("LN2_32_H")) * 2 == Fraction(_scalar("LN2_16_H"))
    assert Fraction(_scalar("LN2_32_M")) * 2 == Fraction(_scalar("LN2_16_M"))
    assert _scalar("INV_LN2_32") == 2 * _scalar("INV_LN2_16")


def test_tan_polynomial_accuracy():
    """t = r + r^3 T(r^2) on |r| <= pi/32 (1 + 5e-4): relative error < 2^-47
    (tanf's budget is E = 1024 double ulps, 2^-43)."""
    T = [Fraction(v) for v in _arr("TANQ")]
    with mp.workprec(200):
        R = mp.pi / 32 * mp.mpf("1.0005")
        worst = mp.mpf(0)
        for i in range(1, 801):
            r = R * i / 800
            s = r * r
            p = sum(mp.mpf(c.numerator) / c.denominator * s ** k for k, c in enumerate(T))
            worst = max(worst, abs((r + r * s * p) / mp.tan(r) - 1))
        assert worst < mp.mpf(2) ** -47
