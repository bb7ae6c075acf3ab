"""Certify the binary64 fast-path error bounds of csrc/crvec_fns_f64.cuh:
EPS_EXP2D (exp2) and the log bound b = EPS_LOGD |V| + K_SMALL |r^3 P(r)|.

This is the B200 build's counterpart of the reference's CertifiedBounds and its
certifier budgets (ref: proj/include/crvec/tables.hpp:56-61,
proj/include/crvec/coeffgen.hpp:16-67): for binary64 there is
no exhaustive proof, so these bounds ARE the correctness argument of every
fast-path decision.

Part A, a-priori (term by term): every table entry and
table product is measured exactly (rational emulation of the RN/fma operations,
mpmath at 200 bits); the polynomial approximation errors are maximised over the
reduced-argument intervals with the shipped double coefficients; every
floating-point rounding of the evaluation is bounded by u = 2^-53 times a
bound on the magnitude it rounds. The sum must stay below the constant the
kernel's round test uses.

Part B, dense grid: the same device source compiled for the CPU (tools/emu,
g++ -ffp-contract=off, correctly rounded std::fma, the arithmetic of the DFMA/
DADD/DMUL the kernels use) evaluated on ~2^20 inputs per function, including
every table index and the extremes of the reduced argument, against mpmath at
160 bits. The largest observed error must sit inside the certified bound.

Usage: python tools/certify_f64.py [--grid LOG2N] [--out profiles/r02/certify_f64.txt]
Exit status 1 if any bound fails.
"""
import argparse
import ctypes
import os
import re
import sys
from fractions import Fraction as Fr

import mpmath as mp
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "paper_2605_15547_b200", "csrc", "crvec_tables.inc")
HDR = os.path.join(ROOT, "paper_2605_15547_b200", "csrc", "crvec_fns_f64.cuh")
mp.mp.prec = 200
U = 2.0 ** -53  # unit roundoff of binary64 round-to-nearest


def tables():
    txt = open(INC).read()
    out = {}
    for name, body in re.findall(r"CR_CONST double (\w+)\[\d+\] = \{([^}]*)\}", txt):
        out[name] = [float.fromhex(v.strip()) for v in body.split(",") if v.strip()]
    for name, v in re.findall(r"CR_CONST double (\w+) = ([^;]+);", txt):
        out[name] = float.fromhex(v.strip())
    return out


def kernel_constants():
    txt = open(HDR).read()
    eps_e = float.fromhex(re.search(r"EPS_EXP2D = (0x[0-9a-fp+-.]+);", txt).group(1))
    eps_l = float.fromhex(re.search(r"EPS_LOGD = (0x[0-9a-fp+-.]+);", txt).group(1))
    k_small = float.fromhex(re.search(r"fma_\(dabs\(small\), (0x[0-9a-fp+-.]+), EPS_LOGD", txt).group(1))
    return eps_e, eps_l, k_small


def rn(x: Fr) -> float:
    """Round an exact rational to the nearest double (CPython int division is correctly rounded)."""
    return x.numerator / x.denominator if x != 0 else 0.0


def fma(a, b, c):
    return rn(Fr(a) * Fr(b) + Fr(c))


def lg2(x):
    return float(mp.log(abs(mp.mpf(x)), 2)) if x else float("-inf")


# ------------------------------------------------------------------ exp2 ----
def certify_exp2(T, eps, rep):
    AH, AL, BH, BL = T["EXP2D_A_HI"], T["EXP2D_A_LO"], T["EXP2D_B_HI"], T["EXP2D_B_LO"]
    Q = T["EXP2D_Q4"]
    H, L = T["LN2D_H"], T["LN2D_L"]
    Rm = 2.0 ** -13
    # (a1) the table product T = A B as the kernel forms it, all 4096 pairs
    eT, tl_ratio, Tmax, Tmin = 0.0, 0.0, 0.0, 4.0
    for ia in range(64):
        for ib in range(64):
            ah, alo, bh, blo = AH[ia], AL[ia], BH[ib], BL[ib]
            Th = ah * bh
            t1 = fma(ah, bh, -Th)  # exact product error
            Tl = fma(ah, blo, fma(alo, bh, t1))  # the kernel's 3-FMA form
            exact = mp.power(2, mp.mpf(64 * ia + ib) / 4096)
            eT = max(eT, float(abs(mp.mpf(Th) + mp.mpf(Tl) - exact) / exact))
            tl_ratio = max(tl_ratio, abs(Tl) / Th)
            Tmax, Tmin = max(Tmax, Th), min(Tmin, Th)
    rep.append(f"exp2 (a1) table product T = 2^(ia/64) 2^(ib/4096), 4096 pairs: max rel err 2^{lg2(eT):.1f}, "
               f"|Tl/Th| <= 2^{lg2(tl_ratio):.1f}")
    # (a2) 1 + R (H + L) + R^2 Q(R) with the shipped coefficients vs 2^R, |R| <= 2^-13
    Qm = [mp.mpf(c) for c in Q]
    HL = mp.mpf(H) + mp.mpf(L)
    eapx = mp.mpf(0)
    for j in range(-2000, 2001):
        R = mp.mpf(j) / 2000 * Rm
        f = 1 + R * HL + R * R * (((Qm[3] * R + Qm[2]) * R + Qm[1]) * R + Qm[0])
        eapx = max(eapx, abs(f - mp.power(2, R)) / mp.power(2, R))
    eapx = float(eapx) * 1.01
    rep.append(f"exp2 (a2) polynomial 1 + R ln2 + R^2 q(R), |R| <= 2^-13: max rel err 2^{lg2(eapx):.1f} (x1.01)")
    # (a3) roundings in p = lin.hi + pl (absolute), lin = two_prod(R, H) exact
    y1 = abs(Q[2]) + abs(Q[3]) * Rm
    e1 = U * y1
    y2 = abs(Q[1]) + y1 * Rm
    e2 = U * y2 + Rm * e1
    qm = abs(Q[0]) + y2 * Rm
    eq = U * qm + Rm * e2                                  # |q - Q(R)|
    tmax = Rm * abs(L) + U * Rm * H                         # |R L + lin.lo|
    et = U * tmax                                           # t = RN(fma(R, L, lin.lo))
    plmax = (Rm * Rm * qm + tmax) * (1 + U)
    epl = U * Rm * Rm * qm + Rm * Rm * eq + et + U * plmax  # R2 rounding, q error, t, pl rounding
    pmin = -Rm * H - plmax
    dp_rel = epl / (1 + pmin)
    rep.append(f"exp2 (a3) roundings in p: |dp| <= 2^{lg2(epl):.1f}, relative to V 2^{lg2(dp_rel):.1f}")
    # (a4) assembly V = s + e1 + [Th pl + Tl ph + Tl] with s = RN(Th + Th ph) (one FMA),
    # e1 = RN(Th ph + (Th - s)) its rounding error (Th - s exact, Sterbenz), Tl pl neglected
    Tlm = tl_ratio * Tmax
    lin_hi = Rm * H
    neg = Tlm * plmax                                       # Tl * pl dropped
    t2m = Tlm * (1 + lin_hi)
    e_t2 = U * t2m
    t3m = Tmax * plmax + t2m
    e_t3 = U * t3m + Tmax * 0 + e_t2                        # + propagated t2 error
    e1m = U * Tmax * (1 + lin_hi) * 2                       # |e1| <= ulp(s)/2, s < 2 Tmax
    e_e1 = U * e1m                                          # e1 rounded once
    e_lo = U * (e1m + t3m)                                  # lo = RN(e1 + t3)
    Vmin = Tmin * (1 + pmin)
    e_asm = (neg + e_t3 + e_e1 + e_lo) / Vmin
    rep.append(f"exp2 (a4) assembly: Tl pl 2^{lg2(neg):.1f}, t3 2^{lg2(U * t3m):.1f}, e1 2^{lg2(e_e1):.1f}, "
               f"lo 2^{lg2(e_lo):.1f}; relative to V >= {Vmin:.6f}: 2^{lg2(e_asm):.1f}")
    total = float((1 + mp.mpf(eT)) * (1 + mp.mpf(eapx)) * (1 + mp.mpf(dp_rel)) * (1 + mp.mpf(e_asm)) - 1)
    ok = total < eps
    rep.append(f"exp2 TOTAL a-priori relative bound 2^{lg2(total):.2f} vs EPS_EXP2D = 2^{lg2(eps):.0f}: "
               f"{'OK' if ok else 'FAIL'} (margin x{eps / total:.1f})")
    return ok, total


# ------------------------------------------------------------------- log ----
def certify_log(T, eps, k_small, rep):
    C, LH, LL, P = T["LOGD5_C"], T["LOGD5_LT_HI"], T["LOGD5_LT_LO"], T["LOGD5_P"]
    HD, LD = T["LN2_HD"], T["LN2_LD"]
    ok = True
    # grid facts behind the exact steps
    assert (Fr(HD) * 2 ** 40).denominator == 1, "LN2_HD not on the 2^-40 grid"
    assert all((Fr(v) * 2 ** 40).denominator == 1 for v in LH), "L_hi not on the 2^-40 grid"
    ln2 = mp.log(2)
    e_split = float(abs(mp.mpf(HD) + mp.mpf(LD) - ln2))
    rmax, eL, bits_needed = 0.0, 0.0, 0
    bins = []
    for i in range(512):
        a = Fr(3, 4) + Fr(i, 1024) if i < 256 else 1 + Fr(i - 256, 512)
        b = a + (Fr(1, 1024) if i < 256 else Fr(1, 512))
        c = C[i]
        cf = Fr(c)
        mant = cf.numerator
        while mant % 2 == 0:
            mant //= 2
        assert mant.bit_length() <= 10, (i, c)
        r_lo, r_hi = a * cf - 1, b * cf - 1
        rb = float(max(abs(r_lo), abs(r_hi)))
        rmax = max(rmax, rb)
        ulp_m = Fr(1, 2 ** 53) if a < 1 else Fr(1, 2 ** 52)
        grid = ulp_m * Fr(1, cf.denominator) if cf.denominator > 1 else ulp_m
        nb = int(np.ceil(np.log2(rb / float(grid)))) if rb > 0 else 0
        bits_needed = max(bits_needed, nb)
        eL = max(eL, float(abs(mp.mpf(LH[i]) + mp.mpf(LL[i]) + mp.log(mp.mpf(c)))))
        # |V| lower bound for e = 0 over the bin (bins holding 1 have c = 1: V = log1p(r))
        ma, mb = mp.mpf(a.numerator) / a.denominator, mp.mpf(b.numerator) / b.denominator
        vmin = float(min(abs(mp.log(ma)), abs(mp.log(mb)))) if c != 1.0 else None
        bins.append((i, c, rb, vmin))
    rep.append(f"log (b1) 512 bins: c_i <= 10 significant bits, |r| <= 2^{lg2(rmax):.2f}, r = m c_i - 1 needs "
               f"<= {bits_needed} bits (exact: <= 53)")
    ok &= bits_needed <= 53
    rep.append(f"log (b2) table: max |L_hi + L_lo + log c_i| = 2^{lg2(eL):.1f}; |LN2_HD + LN2_LD - ln2| = "
               f"2^{lg2(e_split):.1f}; e ln2_hi + L_hi exact on the 2^-40 grid for |e| <= 1128")
    # (b3) log1p(r) = r - r^2/2 + r^3 P_d(r), shipped coefficients: error in units of |r^3 P(r)|
    Pm = [mp.mpf(v) for v in P]
    worst_apx = mp.mpf(0)
    for j in range(1, 4001):
        for sgn in (1, -1):
            r = sgn * mp.mpf(j) / 4000 * mp.mpf(rmax)
            pd = mp.mpf(0)
            for cc in reversed(Pm):
                pd = pd * r + cc
            g = r - r * r / 2 + r ** 3 * pd
            worst_apx = max(worst_apx, abs(g - mp.log1p(r)) / abs(r ** 3 * pd))
    k_apx = float(worst_apx) * 1.01
    rep.append(f"log (b3) r - r^2/2 + r^3 P(r) vs log1p(r): error <= {k_apx / U:.3f} u |r^3 P(r)|")
    # (b4) roundings proportional to |small| = |r^3 P(r)|: s.hi, r s.hi, Horner p, * p, the add of
    # small into s2 and the final lo (each <= u of a magnitude <= |small| (1 + O(u)))
    rr = rmax
    y = abs(P[6])
    eh = 0.0
    for k in range(5, -1, -1):
        y_new = abs(P[k]) + y * rr
        eh = U * y_new + rr * eh
        y = y_new
    pmin = abs(P[0]) - sum(abs(P[k]) * rr ** k for k in range(1, 7))
    dp_rel = eh / pmin
    Um = mp.mpf(U)
    k_small_rnd = float((1 + Um) ** 3 * (1 + mp.mpf(dp_rel)) - 1)  # s.hi, r s.hi, * p roundings + Horner error
    k_rnd = k_small_rnd + float(2 * Um * (1 + Um) * (1 + 4 * Um))  # then the s2 and lo roundings
    k_tot = k_apx + k_rnd + 1.02 * U * U
    rep.append(f"log (b4) r^3-term roundings: small {k_small_rnd / U:.3f} u + s2, lo "
               f"2.000 u; with (b3): {k_tot / U:.3f} u |small| vs K_SMALL = 2^{lg2(k_small):.0f} = {k_small / U:.0f} u: "
               f"{'OK' if k_tot * (1 + 8 * U) < k_small else 'FAIL'}")
    ok &= k_tot * (1 + 8 * U) < k_small
    # (b5) everything else, relative to |V|: table L, e ln2 split, tl and s1 roundings, t4,
    # truncation beyond r^9 already in (b3); worst over e != 0 (|V| >= 0.2876) and e = 0 bins
    emax = 1128
    tl_e = emax * abs(LD) + max(abs(v) for v in LL)
    abs_e = eL + emax * e_split + U * tl_e + U * (2 * U * 745 + tl_e) + 2 * U * U * rmax
    vmin_e = float(abs(-ln2 + mp.log(mp.mpf(1.5))))
    rel_e = abs_e / vmin_e
    rel_0 = 0.0
    for i, c, rb, vmin in bins:
        if vmin is None:  # c = 1: L = 0, tl = 0, V = log1p(r): only u^2-level terms relative to |r|
            rel_0 = max(rel_0, 4 * U * U)
            continue
        a0 = eL + U * (2 * U * 1.0 + abs(LL[i])) + 2 * U * U * rb
        rel_0 = max(rel_0, a0 / vmin)
    rel = max(rel_e, rel_0)
    rep.append(f"log (b5) remaining terms relative to |V|: e != 0 2^{lg2(rel_e):.1f}, e = 0 2^{lg2(rel_0):.1f}")
    ok_rel = rel * (1 + 8 * U) < eps
    rep.append(f"log TOTAL: |V - log x| <= 2^{lg2(rel):.1f} |V| + {k_tot / U:.2f} u |r^3 P(r)| vs "
               f"b = 2^{lg2(eps):.0f} |V| + 2^{lg2(k_small):.0f} |r^3 P(r)|: {'OK' if (ok and ok_rel) else 'FAIL'} "
               f"(margins x{eps / rel:.0f}, x{k_small / k_tot:.2f})")
    return ok and ok_rel, rel, k_tot


# ------------------------------------------------------------- dense grid ----
def emu():
    lib = os.path.join(ROOT, "tools", "emu", "libemu64.so")
    os.system(f"make -s -C {os.path.dirname(lib)} libemu64.so")
    E = ctypes.CDLL(lib)
    d = ctypes.POINTER(ctypes.c_double)
    E.emu64_value.argtypes = [ctypes.c_int, d, d, d, d, ctypes.POINTER(ctypes.c_int), ctypes.c_uint64]
    return E


def grid_check(E, fn, x, eps, rep, T):
    x = np.ascontiguousarray(x, np.float64)
    n = x.size
    hi, lo, b = np.empty(n), np.empty(n), np.empty(n)
    N = np.empty(n, dtype=np.int32)
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    E.emu64_value(fn, dp(x), dp(hi), dp(lo), dp(b), N.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), n)
    mp.mp.prec = 160
    worst_rel, worst_b = 0.0, 0.0
    for i in range(n):
        V = mp.mpf(hi[i]) + mp.mpf(lo[i])
        if fn == 0:
            exact = mp.power(2, mp.mpf(x[i]) - int(N[i]))
        else:
            exact = mp.log(mp.mpf(x[i]))
        if exact == 0:
            continue
        err = abs(V - exact)
        worst_rel = max(worst_rel, float(err / abs(exact)))
        worst_b = max(worst_b, float(err / mp.mpf(b[i])))
    mp.mp.prec = 200
    rep.append(f"{('exp2', 'log')[fn]} dense grid ({n} inputs, emulated device arithmetic vs mpmath 160 bits): "
               f"max rel err 2^{lg2(worst_rel):.2f}; max err / round-test bound = {worst_b:.4f} "
               f"{'OK' if worst_b < 1 else 'FAIL'}")
    return worst_b < 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=18)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "certify_f64.txt"))
    a = ap.parse_args()
    T = tables()
    eps_e, eps_l, k_small = kernel_constants()
    rep = [f"# tools/certify_f64.py: binary64 fast-path error bounds of csrc/crvec_fns_f64.cuh "
           f"(EPS_EXP2D = 2^{lg2(eps_e):.0f}, EPS_LOGD = 2^{lg2(eps_l):.0f}, K_SMALL = 2^{lg2(k_small):.0f}); u = 2^-53"]
    ok1, _ = certify_exp2(T, eps_e, rep)
    ok2, _, _ = certify_log(T, eps_l, k_small, rep)
    E = emu()
    rng = np.random.default_rng(20240817)
    n = 1 << a.grid
    # exp2: every k = RN(4096 x) mod 4096 with R at both extremes and random, plus random x
    k = np.arange(4096)
    ends = np.concatenate([(k + 0.5 - 2.0 ** -40) / 4096, (k - 0.5 + 2.0 ** -40) / 4096, (k + rng.uniform(-0.5, 0.5, 4096)) / 4096])
    xe = np.concatenate([ends, ends - 7, rng.uniform(-20, 20, n), rng.uniform(-1022, 1023.9, n // 4),
                         rng.uniform(-2.0 ** -10, 2.0 ** -10, n // 8)])
    ok3 = grid_check(E, 0, xe, eps_e, rep, T)
    # log: every bin at both edges and random, scaled by 2^e, plus the paper range and near 1
    bins = []
    for i in range(512):
        a0 = 0.75 + i / 1024 if i < 256 else 1 + (i - 256) / 512
        w = 1 / 1024 if i < 256 else 1 / 512
        bins += [a0, np.nextafter(a0 + w, 0), a0 + w * rng.random()]
    bins = np.array(bins)
    xl = np.concatenate([bins, bins * 2.0 ** 5, bins * 2.0 ** -9, rng.uniform(0.125, 8, n),
                         rng.uniform(1 - 2.0 ** -9, 1 + 2.0 ** -9, n // 2),
                         rng.integers(0x0010000000000000, 0x7FEFFFFFFFFFFFFF, n // 8, dtype=np.uint64).view(np.float64)])
    ok4 = grid_check(E, 1, xl, eps_l, rep, T)
    ok = ok1 and ok2 and ok3 and ok4
    rep.append("RESULT: " + ("all bounds certified" if ok else "A BOUND FAILED"))
    txt = "\n".join(rep) + "\n"
    print(txt, end="")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        f.write(txt)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
