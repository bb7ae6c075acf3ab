// Correctly rounded binary64 exp2 and log (the two double-precision functions
// of SPEC.md, ref: PAPER.md II.B, proj/src/kernels_f64.cpp:234-307).
//
//  fast path   the paper's algorithms, restructured for the GPU: exp2 via
//              x = N + (64 ia + ib)/4096 + R and two 64-entry DD tables in
//              shared memory (one DD product instead of the reference's two
//              over three 16-entry tables, ref: kernels_f64.cpp:82-100,135-150);
//              log via 512 bins with a 10-bit c_i (r = m c_i - 1 exact), a
//              -log(c_i) table split on a 2^-40 grid, and r - r^2/2 + r^3 P(r)
//              (the reference: 128 bins, 7-bit reciprocal, ref: kernels_f64.cpp:102-124).
//  round test  Ziv straddle test in registers (ref: kernels_f64.cpp:63-76):
//              the DD value +- eps|v| must round to the same binary64.
//  accurate    lanes the test cannot decide (or whose result is subnormal)
//              are compacted per warp with __ballot_sync into a side queue and
//              evaluated by full warps in 256-bit fixed point (error < 2^-230,
//              far below the binary64 worst cases of these functions), then
//              rounded exactly. This replaces the reference's scalar MPFR
//              callout (ref: kernels_f64.cpp:78-80); there is no host callout.
#pragma once
#include "crvec_device.cuh"
#include "crvec_tables.inc"

namespace crvec {

// ------------------------------------------------- 256-bit fixed point ----
// Signed two's complement, value = W / 2^240 (16 integer bits), w[0] least
// significant.
struct Fx {
  uint32_t w[8];
};
constexpr int FX_FRAC = 240;

CR_F Fx fx_zero() {
  Fx r;
  for (int i = 0; i < 8; ++i) r.w[i] = 0;
  return r;
}
CR_F bool fx_neg_p(const Fx &a) { return (a.w[7] >> 31) != 0; }
CR_F bool fx_is_zero(const Fx &a) {
  uint32_t o = 0;
  for (int i = 0; i < 8; ++i) o |= a.w[i];
  return o == 0;
}
CR_F Fx fx_add(const Fx &a, const Fx &b) {
  Fx r;
  uint64_t c = 0;
  for (int i = 0; i < 8; ++i) {
    c += (uint64_t)a.w[i] + b.w[i];
    r.w[i] = (uint32_t)c;
    c >>= 32;
  }
  return r;
}
CR_F Fx fx_negate(const Fx &a) {
  Fx r;
  uint64_t c = 1;
  for (int i = 0; i < 8; ++i) {
    c += (uint64_t)(~a.w[i]);
    r.w[i] = (uint32_t)c;
    c >>= 32;
  }
  return r;
}
CR_F Fx fx_sub(const Fx &a, const Fx &b) { return fx_add(a, fx_negate(b)); }
CR_F Fx fx_abs(const Fx &a) { return fx_neg_p(a) ? fx_negate(a) : a; }
CR_F Fx fx_from_int(int64_t v) {
  Fx r = fx_zero();
  uint64_t m = v < 0 ? (uint64_t)(-v) : (uint64_t)v;
  // integer part occupies bits 240..255: limb 7 bits 16..31
  r.w[7] = (uint32_t)(m << 16);
  return v < 0 ? fx_negate(r) : r;
}
// Exact conversion of a finite double with |v| < 2^15 and lsb >= 2^-240.
CR_F Fx fx_from_double(double v) {
  Fx r = fx_zero();
  if (v == 0.0) return r;
  uint64_t b = d2u(v);
  int be = (int)((b >> 52) & 0x7FF);
  uint64_t M = (b & 0xFFFFFFFFFFFFFull) | (be ? (1ull << 52) : 0);
  int E = (be ? be : 1) - 1075;  // v = M * 2^E
  int pos = E + FX_FRAC;         // bit index of M's lsb
  if (pos < 0) {                 // truncate (never for the callers' inputs)
    M = -pos >= 64 ? 0 : (M >> -pos);
    pos = 0;
  }
  int limb = pos >> 5, sh = pos & 31;
  uint64_t lo = M << sh;                       // bits 0..63 of the shifted M
  uint64_t hi = sh ? (M >> (64 - sh)) : 0;    // bits 64..(52+sh)
  if (limb < 8) r.w[limb] = (uint32_t)lo;
  if (limb + 1 < 8) r.w[limb + 1] = (uint32_t)(lo >> 32);
  if (limb + 2 < 8) r.w[limb + 2] = (uint32_t)hi;
  return (b >> 63) ? fx_negate(r) : r;
}
// (a * b) >> 240 for non-negative a, b (truncating).
CR_F Fx fx_mul(const Fx &a, const Fx &b) {
  uint32_t p[16];
  for (int i = 0; i < 16; ++i) p[i] = 0;
  for (int i = 0; i < 8; ++i) {
    uint64_t c = 0;
    for (int j = 0; j < 8; ++j) {
      uint64_t t = (uint64_t)a.w[i] * b.w[j] + p[i + j] + c;
      p[i + j] = (uint32_t)t;
      c = t >> 32;
    }
    p[i + 8] = (uint32_t)c;
  }
  // shift right by 240 = 7 limbs + 16 bits
  Fx r;
  for (int i = 0; i < 8; ++i) {
    uint32_t lo = p[i + 7], hi = (i + 8 < 16) ? p[i + 8] : 0;
    r.w[i] = (lo >> 16) | (hi << 16);
  }
  return r;
}
// a * k for non-negative a and small k.
CR_F Fx fx_mul_u32(const Fx &a, uint32_t k) {
  Fx r;
  uint64_t c = 0;
  for (int i = 0; i < 8; ++i) {
    c += (uint64_t)a.w[i] * k;
    r.w[i] = (uint32_t)c;
    c >>= 32;
  }
  return r;
}
// a / d for non-negative a (truncating).
CR_F Fx fx_div_u32(const Fx &a, uint32_t d) {
  Fx r;
  uint64_t rem = 0;
  for (int i = 7; i >= 0; --i) {
    uint64_t cur = (rem << 32) | a.w[i];
    r.w[i] = (uint32_t)(cur / d);
    rem = cur % d;
  }
  return r;
}
// 1/b for b in [1, 4) by Newton from the double reciprocal (3 steps: 53 -> 212+ bits).
CR_F Fx fx_recip(const Fx &b, double bd) {
  Fx r = fx_from_double(1.0 / bd);
  Fx two = fx_from_int(2);
  for (int it = 0; it < 3; ++it) r = fx_mul(r, fx_sub(two, fx_mul(b, r)));
  return r;
}
CR_F Fx fx_ln2() {
  // ln2 = 0.LN2_WORDS... ; value * 2^240 = top 240 fraction bits
  Fx r;
  // fraction bits f_1..f_240 -> limbs: bit (240 - j) holds f_j
  // words[k] holds f_{32k+1} .. f_{32k+32}; shifting the 288-bit fraction
  // right by 48 bits (288 - 240) gives the 240-bit integer.
  uint32_t w[9];
  for (int i = 0; i < 9; ++i) w[i] = LN2_WORDS[i];
  // integer value = (w0 w1 ... w8) >> 48  (w0 most significant)
  for (int i = 0; i < 8; ++i) {
    // limb i (least significant first) = bits [32i, 32i+32) of (W >> 48)
    // W's limb j (lsw first) = w[8 - j]
    int j = i + 1;  // 48 = 32 + 16
    uint32_t lo = (8 - j >= 0) ? w[8 - j] : 0;
    uint32_t hi = (8 - j - 1 >= 0) ? w[8 - j - 1] : 0;
    r.w[i] = (lo >> 16) | (hi << 16);
  }
  r.w[7] &= 0x0000FFFFu;  // integer part 0
  return r;
}

// Exact rounding of v * 2^scale (v signed Fx) to binary64 in mode M. Sets
// *undecided when the bits below the rounding point are within the Fx error
// of a boundary (pattern 0x000.., 0x7FF.., 0x800.., 0xFFF.. over 64 bits).
template <int M>
CR_F double fx_round(const Fx &v, int scale, int *undecided) {
  bool neg = fx_neg_p(v);
  Fx a = fx_abs(v);
  int top = -1;
  for (int i = 7; i >= 0 && top < 0; --i)
    if (a.w[i]) top = i * 32 + 31 - clz32(a.w[i]);
  if (top < 0) return neg ? -0.0 : 0.0;
  // value = a * 2^(scale - 240); leading bit weight 2^(top + scale - 240)
  int ev = top + scale - FX_FRAC;
  int prec = 53;
  if (ev < -1022) prec = 53 - (-1022 - ev);
  // bits: kept = a[top .. top-prec+1], rest below
  auto bit_window64 = [&](int hi_bit) -> uint64_t {  // 64 bits a[hi_bit .. hi_bit-63]
    uint64_t r = 0;
    for (int k = 0; k < 64; ++k) {
      int b = hi_bit - k;
      uint64_t bit = (b >= 0 && b < 256) ? ((a.w[b >> 5] >> (b & 31)) & 1u) : 0;
      r = (r << 1) | bit;
    }
    return r;
  };
  uint64_t kept = 0;
  if (prec > 0) kept = bit_window64(top) >> (64 - prec);
  int rest_top = top - (prec > 0 ? prec : 0);  // first bit below kept
  if (prec <= 0) rest_top = top - prec;        // leading bits are below half of min subnormal
  uint64_t R = bit_window64(rest_top);          // 64 bits just below the rounding point
  bool sticky_below = false;
  for (int b = rest_top - 64; b >= 0 && !sticky_below; --b)
    if ((a.w[b >> 5] >> (b & 31)) & 1u) sticky_below = true;
  if (prec <= 0) {
    // value < 2^-1074 (prec==0: in [2^-1075, 2^-1074)); R holds bits from
    // weight 2^-1075 downward (with leading zeros when prec < 0).
    kept = 0;
  }
  if (R == 0 || R == ~0ull || R == 0x8000000000000000ull || R == 0x7FFFFFFFFFFFFFFFull)
    *undecided = 1;
  bool round_bit = (R >> 63) & 1;
  bool inexact = R != 0 || sticky_below;
  bool up;
  if (M == RNE) up = round_bit && ((R << 1) != 0 || sticky_below || (kept & 1));
  else if (M == RZ) up = false;
  else if (M == RU) up = !neg && inexact;
  else up = neg && inexact;
  int e = ev;
  int p = prec > 0 ? prec : 0;
  if (up) {
    kept += 1;
    if (ev >= -1022 && (kept >> p)) {  // carry out of a normal significand
      kept >>= 1;
      e += 1;
    }
    if (p == 0) {  // rounded up to the min subnormal
      return neg ? -0x1p-1074 : 0x1p-1074;
    }
  }
  if (p == 0) return neg ? -0.0 : 0.0;
  if (e > 1023) {
    bool inf = M == RNE || (M == RU && !neg) || (M == RD && neg);
    return inf ? (neg ? -INFINITY : INFINITY) : (neg ? -0x1.fffffffffffffp1023 : 0x1.fffffffffffffp1023);
  }
  uint64_t bits;
  if (ev < -1022) {
    // subnormal: kept is the significand at 2^-1074 granularity (may have
    // carried into the normal range, which the encoding handles naturally)
    bits = kept;
  } else {
    bits = ((uint64_t)(e + 1023) << 52) | (kept & 0xFFFFFFFFFFFFFull);
  }
  return u2d(bits | (neg ? 0x8000000000000000ull : 0));
}

// ------------------------------------------------------- exp2 accurate ----
// 2^x = 2^N * e^(f ln2), N = floor(x), f in [0,1) exact in Fx; e^y by Taylor.
template <int M>
CR_F double exp2d_accurate(double x, int *undecided) {
  double N = floor(x);
  Fx f = fx_sub(fx_from_double(x), fx_from_int((int64_t)N));
  Fx y = fx_mul(f, fx_ln2());
  Fx sum = fx_from_int(1), term = fx_from_int(1);
  for (uint32_t n = 1; n < 80; ++n) {
    term = fx_div_u32(fx_mul(term, y), n);
    if (fx_is_zero(term)) break;
    sum = fx_add(sum, term);
  }
  return fx_round<M>(sum, (int)N, undecided);
}

// -------------------------------------------------------- log accurate ----
// log x = e ln2 + 2 atanh((m-1)/(m+1)), m in [0.75, 1.5).
template <int M>
CR_F double logd_accurate(double x, int *undecided) {
  int eadj = 0;
  if (x < 0x1p-1022) {
    x *= 0x1p54;
    eadj = -54;
  }
  int h = d2hi(x);
  int hh = h - 0x3FE80000;
  int e = (hh >> 20) + eadj;
  double m = hilo2d(h - ((hh >> 20) << 20), d2lo(x));
  Fx mf = fx_from_double(m);
  Fx one = fx_from_int(1);
  Fx num = fx_sub(mf, one);
  Fx den = fx_add(mf, one);
  bool sneg = fx_neg_p(num);
  Fx s = fx_mul(fx_abs(num), fx_recip(den, m + 1.0));
  Fx s2 = fx_mul(s, s);
  Fx sum = s, t = s;
  for (uint32_t k = 1; k < 80; ++k) {
    t = fx_mul(t, s2);
    if (fx_is_zero(t)) break;
    sum = fx_add(sum, fx_div_u32(t, 2 * k + 1));
  }
  sum = fx_add(sum, sum);  // 2 atanh(s) = |log m|
  if (sneg) sum = fx_negate(sum);
  Fx el = fx_mul_u32(fx_ln2(), (uint32_t)(e < 0 ? -e : e));
  if (e < 0) el = fx_negate(el);
  return fx_round<M>(fx_add(el, sum), 0, undecided);
}

// --------------------------------------------------------- fast paths ----
// Shared-memory tables, laid out so each lookup is one 128-bit LDS.
struct alignas(16) Pair64 {
  double a, b;
};
struct F64Tab {
  Pair64 ta[64], tb[64];  // (hi, lo) of 2^(i/64) and 2^(i/4096)
  Pair64 lc[512];         // (c_i (10 bits), -log(c_i) on the 2^-40 grid)
  double lll[512];        // -log(c_i) - the grid part
};

struct F64Out {
  double y;
  bool decided;
};

// Round test (ref: proj/src/kernels_f64.cpp:63-76): the DD value h + l with
// absolute error bound b is decided in mode M iff both ends of the enclosure,
// h + (l +- b), round to the same binary64 - two DADDs with the static
// rounding modifier, so binade edges, ties and the directed modes need no
// case analysis (|l| <= ulp(h) and b << |l| rounding error are not needed:
// l +- b is computed in RN and b carries the margin).
template <int M>
CR_F F64Out round_test64(double h, double l, double b) {
  const double y1 = add_M<M>(h, add_(l, b)), y2 = add_M<M>(h, sub_(l, b));
  return {y1, y1 == y2};
}

// Fast-path error bounds used by the round test, certified by
// tools/certify_f64.py (term by term from the shipped tables, DESIGN.md section
// 4a; profiles/r02/certify_f64.txt): exp2's value is within 2^-77.4 |V| (bound
// 2^-74: margin x10); log's within 2^-82.5 |V| + 6.51 u |r^3 P(r)| (bound
// 2^-73 |V| + 2^-49 |r^3 P(r)|, see logd_value). A dense grid of the same
// device arithmetic against mpmath stays inside both.
constexpr double EPS_EXP2D = 0x1p-74;
constexpr double EPS_LOGD = 0x1p-73;

// Lanes outside exp2's main range: NaN, +-Inf, overflow / underflow classes,
// |x| <= 2^-55 (2^x in the gap beside 1) — all decided by rules.
template <int M>
CR_F double exp2d_special(double x) {
  uint64_t xb = d2u(x);
  if (x != x) return u2d(xb | 0x0008000000000000ull);
  if (x == INFINITY) return INFINITY;
  if (x >= 1024.0) return (M == RNE || M == RU) ? INFINITY : 0x1.fffffffffffffp1023;
  if (x <= -1075.0) return (M == RU && x != -INFINITY) ? 0x1p-1074 : 0.0;  // tie at -1075 -> 0
  if (x > 0) return M == RU ? 1.0 + 0x1p-52 : 1.0;                       // tiny
  if (x < 0) return (M == RZ || M == RD) ? 1.0 - 0x1p-53 : 1.0;
  return 1.0;                                                              // +-0
}
// main: 2^-55 < |x| < 1022 (bit-pattern range check); also (-1075, -1022]
// (subnormal results) and [1022, 1024) go through the fast path + test.
CR_F bool exp2d_main(double x) {
  uint64_t a = d2u(x) & 0x7FFFFFFFFFFFFFFFull;
  return a > 0x3C80000000000000ull && a < 0x4090CC0000000000ull;  // 2^-55 < |x| < 1075
}

// exp2 fast path: x = N + (64 ia + ib)/4096 + R, |R| <= 2^-13 exact;
// 2^x = 2^N T (1 + p) with T = 2^(ia/64) 2^(ib/4096) (two 64-entry DD tables
// in shared memory; one product instead of the paper's two over 3 x 16
// entries, ref: proj/src/kernels_f64.cpp:82-90) and 2^R = 1 + ph + pl,
// ph = RN(R ln2_hi). V = T (1 + p) = Th + Th ph + [Tl + Th pl + Tl ph] with
// Th ph exact; relative error < EPS_EXP2D before the round test (DESIGN.md
// section 4a derives the bound); the 2^N scale is an integer add to the
// exponent field.
struct Exp2dV {
  DD V;  // in [1, 2]
  int N, k;
  double R;
};
CR_F Exp2dV exp2d_value(double xs, const F64Tab &T) {
  double t = fma_(xs, 4096.0, SHIFTER);
  double kd = sub_(t, SHIFTER);
  int k = (int)d2lo(t);
  double R = fma_(kd, -0x1p-12, xs);  // exact, |R| <= 2^-13
  int N = k >> 12, ia = (k >> 6) & 63, ib = k & 63;
  // T = A B as an unnormalised DD (|Tl| < 2^-51 |Th|)
  const Pair64 A = T.ta[ia], B = T.tb[ib];
  const double ah = A.a, alo = A.b, bh = B.a, blo = B.b;
  double Th = mul_(ah, bh);
  double Tl = fma_(ah, blo, fma_(alo, bh, fma_(ah, bh, -Th)));  // inner fma exact
  double q = fma_(fma_(fma_(EXP2D_Q4[3], R, EXP2D_Q4[2]), R, EXP2D_Q4[1]), R, EXP2D_Q4[0]);
  DD lin = two_prod(R, LN2D_H);
  double pl = fma_(mul_(R, R), q, fma_(R, LN2D_L, lin.lo));
  // s = RN(Th + Th ph) in one FMA; its rounding error e1 = (Th + Th ph) - s by
  // a second FMA over Th - s (exact: s lies within a factor 2 of Th), e1 itself
  // rounded once (~2^-106 |V|). (s, lo) is left unnormalised (|lo| <= ~ulp(s)):
  // the round test rounds s + (lo +- b) directly.
  const double s = fma_(Th, lin.hi, Th);
  const double e1 = fma_(Th, lin.hi, sub_(Th, s));
  const double lo = add_(e1, fma_(Th, pl, fma_(Tl, lin.hi, Tl)));
  return {DD{s, lo}, N, k, R};
}

// Rule-complete form (scalar kernels, the side-queue drain).
template <int M>
CR_F F64Out exp2d_fast(double x, const F64Tab &T) {
  if (!exp2d_main(x) || x >= 1024.0) return {exp2d_special<M>(x), true};
  const Exp2dV e = exp2d_value(x, T);
  if (e.R == 0.0 && (e.k & 4095) == 0) {  // integer x: 2^x exact (normal or subnormal)
    const int N = e.N;
    double p = N >= -1022 ? u2d((uint64_t)(N + 1023) << 52) : u2d(1ull << (N + 1074));
    return {p, true};
  }
  F64Out r = round_test64<M>(e.V.hi, e.V.lo, EPS_EXP2D * dabs(e.V.hi));
  if (x < -1022.0) r.decided = false;  // subnormal result: accurate path
  // y in [1, 2]: the exponent add is exact, 2 * 2^1023 correctly gives +Inf
  r.y = scale2(r.y, e.N);
  return r;
}

// Vector-kernel form: no special-value branches. Lanes outside the normal-
// result range, and integer x (exact 2^N), are returned undecided and resolved
// by the warp's side-queue drain, which runs exp2d_fast (rules) first.
template <int M>
CR_F F64Out exp2d_main_path(double x, const F64Tab &T) {
  const uint64_t a = d2u(x) & 0x7FFFFFFFFFFFFFFFull;
  const bool ok = a > 0x3C80000000000000ull && x < 1024.0 && x >= -1022.0;  // 2^-55 < |x|
  const Exp2dV e = exp2d_value(ok ? x : 0.5, T);
  F64Out r = round_test64<M>(e.V.hi, e.V.lo, EPS_EXP2D * dabs(e.V.hi));
  r.decided = r.decided && ok && !(e.R == 0.0 && (e.k & 4095) == 0);
  r.y = scale2(r.y, e.N);
  return r;
}

// log fast path: x = 2^e m, m in [0.75, 1.5), 512 bins (the paper's 128,
// ref: proj/src/kernels_f64.cpp:102-124, refined so the r^3 term needs no
// double-double): r = m c_i - 1 exact (c_i has 10 bits, |r| < 2^-9.4),
// log x = e ln2 - log c_i + r - r^2/2 + r^3 P(r), P of degree 6.
// The fast-path value for a positive normal x (subnormals arrive scaled, with
// eadj): V = V.hi + V.lo and the round-test bound. Error budget (DESIGN.md
// section 4a, tools/certify_f64.py): every term but one is below 2^-76 |V|;
// the rounding errors carried by the r^3 P(r) term (its own evaluation and the
// two additions it enters) are up to ~6u |r^3 P(r)| in absolute terms, which
// for x near 1 (e = 0, |V| ~ |r|) is ~2^-70.6 |V| -- above any fixed relative
// bound the rest of the budget would justify. The bound therefore carries that
// term explicitly: b = EPS_LOGD |V| + 2^-49 |r^3 P(r)| (16u vs a certified ~7u).
struct LogdV {
  DD V;
  double b;
};
CR_F LogdV logd_value(double xs, int eadj, const F64Tab &T) {
  int h = d2hi(xs);
  int hh = h - 0x3FE80000;
  const int e0 = hh >> 20;
  int e = e0 + eadj;
  int i = (hh >> 11) & 511;
#if CR_DEVICE
  int mh;  // h - e0 2^20 as one IMAD (the shift-and-subtract form is LOP3 + IADD)
  asm("mad.lo.s32 %0, %1, -1048576, %2;" : "=r"(mh) : "r"(e0), "r"(h));
#else
  int mh = h - (int)((uint32_t)e0 << 20);
#endif
  double m = hilo2d(mh, d2lo(xs));
  const Pair64 cl = T.lc[i];
  double r = fma_(m, cl.a, -1.0);                  // exact
  DD s = two_prod(r, r);                          // r^2 exact
  const double *P = LOGD5_P;
  double p = fma_(fma_(fma_(fma_(fma_(fma_(P[6], r, P[5]), r, P[4]), r, P[3]), r, P[2]), r, P[1]), r, P[0]);
  double small = mul_(mul_(r, s.hi), p);          // r^3 P(r)
  // a = r - r^2/2 exactly as a pair: a.hi = RN(r - s.hi/2) by one FMA, a.lo
  // its rounding error by a second FMA over r - a.hi (exact: a.hi is within a
  // factor 2 of r); the error of RN(r - s.hi/2) is representable, so exact
  DD a;
  a.hi = fma_(-0.5, s.hi, r);
  a.lo = fma_(-0.5, s.hi, sub_(r, a.hi));
  // e ln2 + L: the high parts add exactly (both on the 2^-40 grid)
  double ed = i2d(e);
  double th = fma_(ed, LN2_HD, cl.b);
  double tl = fma_(ed, LN2_LD, T.lll[i]);
  DD v = two_sum(th, a.hi);
  double lo = add_(add_(v.lo, tl), add_(fma_(-0.5, s.lo, a.lo), small));
  const DD V = {v.hi, lo};  // unnormalised, as in exp2d_value
  return {V, fma_(dabs(small), 0x1p-49, EPS_LOGD * dabs(V.hi))};
}

template <int M>
CR_F F64Out logd_core(double xs, int eadj, const F64Tab &T) {
  const LogdV v = logd_value(xs, eadj, T);
  return round_test64<M>(v.V.hi, v.V.lo, v.b);
}

// Lanes outside log's main range (positive normal, x != 1): NaN, +-0, x < 0,
// +Inf, 1, and subnormals (scaled by 2^54 into the main computation).
template <int M>
CR_F F64Out logd_special(double x, const F64Tab &T) {
  uint64_t xb = d2u(x);
  if (x != x) return {u2d(xb | 0x0008000000000000ull), true};
  if (x == 0.0) return {-INFINITY, true};
  if (xb >> 63) return {u2d(0x7FF8000000000000ull), true};
  if (x == INFINITY) return {INFINITY, true};
  if (x == 1.0) return {0.0, true};
  return logd_core<M>(x * 0x1p54, -54, T);  // subnormal
}

template <int M>
CR_F F64Out logd_main_path(double x, const F64Tab &T) {
  // positive normal (high word in [0x00100000, 0x7FF00000)) and x != 1
  const bool ok = (uint32_t)d2hi(x) - 0x00100000u < 0x7FE00000u && x != 1.0;
  F64Out r = logd_core<M>(ok ? x : 2.0, 0, T);
  r.decided = r.decided && ok;
  return r;
}

template <int M>
CR_F F64Out logd_fast(double x, const F64Tab &T) {
  uint64_t xb = d2u(x);
  if (xb - 0x0010000000000000ull >= 0x7FE0000000000000ull || x == 1.0) return logd_special<M>(x, T);
  return logd_core<M>(x, 0, T);
}

}  // namespace crvec
