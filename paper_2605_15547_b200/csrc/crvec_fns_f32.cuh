// The 19 correctly rounded binary32 functions of the paper (ref: PAPER.md:49):
// fast path (branch-free fp64 range reduction + <=16-entry table held in
// shared memory or in registers read with __shfl_sync, per function by
// measurement + fp64 polynomial + one static-mode conversion) and a rare
// double-double accurate path for lanes the rounding test cannot decide.
//
// The reference implements exp2f / log2f only (ref: proj/src/kernels_f32.cpp:
// 36-157, Figs. 1-2 of PAPER.md); its algorithms need ten 8-entry permutes
// per element for log2f, which on a GPU is 20 SHFL per element. These kernels
// instead follow the paper's own "one larger table and constant coefficients"
// variant (ref: PAPER.md:130) and replace the RZ+sticky final step with an
// explicit Ziv straddle test on the fp64 result (ref: proj/src/kernels_f64.cpp:
// 63-76) so every fast-path lane is provably decided; correctness of the
// whole (fast + accurate path) is established exhaustively against the CPU
// oracle over all 2^32 inputs in all four modes.
#pragma once
#include "crvec_device.cuh"
#include "crvec_tables.inc"

namespace crvec {

// A 16-byte pair: one LDS.128 reads both halves of a shared-table entry.
struct alignas(16) D2 {
  double x, y;
};



// Column-split shared 16-entry tables: NC columns of 16 doubles (128 bytes
// each, one column per value). A warp's LDS.64 moves 256 bytes in two
// 128-byte wavefronts and a column spans each bank exactly once, so any mix
// of rows is conflict-free; the interleaved 16-byte-pair form (LDS.128)
// conflicts whenever two lanes of a quarter-warp read rows r and r + 8
// (ncu: 6.7 wavefronts per LDS.128 instead of 4 in sinf, round 2). Column c
// of row j: base + 128 c + 8 (j & 15), one address per row and immediate
// column offsets. W gives a third column as hilo2d(W[i], 0).
template <int TAG, int NC>
CR_F const double *sh_split16(const double *A, const double *B, const int *W) {
#if CR_DEVICE
  __shared__ __align__(16) double tab[16 * NC];
#else
  static double tab[16 * NC];
#endif
#if CR_DEVICE
  if (threadIdx.x < 16) {
    const int i = threadIdx.x;
#else
  for (int i = 0; i < 16; ++i) {
#endif
    tab[i] = A[i];
    if (NC > 1) tab[16 + i] = B[i];
    if (NC > 2) tab[32 + i] = hilo2d(W[i], 0u);
    if (NC > 3) tab[48 + i] = PI_H - hilo2d(W[i], 0u);  // exact (see FnAsinAcos)
  }
#if CR_DEVICE
  __syncthreads();
#endif
  return tab;
}
struct SplitRow {
#if CR_DEVICE
  uint32_t a;  // shared address of column 0, row j
#else
  const double *p;
#endif
};
CR_F SplitRow split_row(const double *t, int j) {
#if CR_DEVICE
  return {(uint32_t)__cvta_generic_to_shared(t) + ((uint32_t)(j & 15) << 3)};
#else
  return {t + (j & 15)};
#endif
}
// Row j + 8 up of a sh_split16 table, j in [0, 7] left by the shifter trick
// in the low bits of kb = bits of (float)(j + 1.5 2^23): the shifter bias and
// the +8 rows ride in one select-constant of an IMAD (kb 8 + c), no masking.
CR_F SplitRow split_row_kb(const double *t, uint32_t kb, bool up) {
#if CR_DEVICE
  const uint32_t c = (up ? 64u : 0u) - (0x4B400000u << 3);
  return {(uint32_t)__cvta_generic_to_shared(t) + (kb * 8u + c)};
#else
  return {t + ((kb & 7u) + (up ? 8u : 0u))};
#endif
}
// Column at a run-time byte offset (a multiple of 128) of a split row.
CR_F double split_get_dyn(SplitRow r, uint32_t off) {
#if CR_DEVICE
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(r.a + off));
  return v;
#else
  return r.p[off / 8];
#endif
}
template <int COL>
CR_F double split_get(SplitRow r) {
#if CR_DEVICE
  double v;
  asm("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(r.a), "n"(COL * 128));
  return v;
#else
  return r.p[16 * COL];
#endif
}

// Polynomials (Horner, coefficients from tools/gen_tables.py).
CR_F double expq(double r) {
  return fma_(fma_(fma_(fma_(EXPQ[4], r, EXPQ[3]), r, EXPQ[2]), r, EXPQ[1]), r, EXPQ[0]);
}
CR_F double logq(double r) {
  double q = fma_(LOGQ[5], r, LOGQ[4]);
  q = fma_(q, r, LOGQ[3]);
  q = fma_(q, r, LOGQ[2]);
  q = fma_(q, r, LOGQ[1]);
  return fma_(q, r, LOGQ[0]);
}

// Copy the sign of binary32 bits xb onto a double (integer op on the high word).
CR_F double with_sign(double a, uint32_t xb) {
  return hilo2d(d2hi(a) ^ (int)(xb & 0x80000000u), d2lo(a));
}

// ============================================================ exp family ====
// The 2^(j/16) table: shared memory, one LDS.64 per lookup instead of two SHFL
// (+1..5% with the shapes re-tuned, profiles/r01/ab_shtab_exp.txt). The
// register form (exp_t(double, k)) stays for the emulation build and A/B.
template <int TAG>
CR_F const double *exp_tab() {
#if CR_DEVICE
  __shared__ double tab[16];
  if (threadIdx.x < 16) tab[threadIdx.x] = EXP2J_HI[threadIdx.x];
  __syncthreads();
  return tab;
#else
  return EXP2J_HI;
#endif
}
CR_F double exp_t(const double *tab, int k) { return tab[k & 15]; }
CR_F double exp_t(double reg, int k) { return CR_TAB(reg, EXP2J_HI, k); }  // lane k mod 32 -> entry k & 15
// exp_core: 2^(k/16) * e^r with |r| <= ln2/32 (fast path).
template <class Tab>
CR_F double exp_core(int k, double r, Tab tab) {
  double T = exp_t(tab, k);
  double p = fma_(mul_(r, r), expq(r), r);  // e^r - 1
  return scale2_imad(fma_(T, p, T), k >> 4);
}

// Cubic-Q variant (2^-40.1 relative on e^r - 1, i.e. < 2^-45.5 on the
// result): the rounding-test tolerance E = 512 covers it with margin.
CR_F double expq3(double r) { return fma_(fma_(fma_(EXPQ3[3], r, EXPQ3[2]), r, EXPQ3[1]), r, EXPQ3[0]); }
template <class Tab>
CR_F double exp_core3(int k, double r, Tab tab) {
  double T = exp_t(tab, k);
  double p = fma_(mul_(r, r), expq3(r), r);  // e^r - 1
  return scale2_imad(fma_(T, p, T), k >> 4);
}
// Non-main lanes of exp / exp2 / exp10: NaN, +-0 -> 1, +Inf -> +Inf,
// -Inf -> +0, tiny |x|: b^x lies in the gap beside 1 (above for x > 0).
template <int M>
CR_F uint32_t exp_like_special(uint32_t xb) {
  uint32_t az = xb << 1;
  if (nan_bits(xb)) return quiet_bits(xb);
  if (az == 0) return 0x3F800000u;
  if (az == 0xFF000000u) return (int)xb < 0 ? 0u : 0x7F800000u;
  return f2u(cvt_f32<M>((int)xb > 0 ? 1.0 + 0x1p-30 : 1.0 - 0x1p-31));
}

// Double-double e^r, |r| <= ln2/32: Taylor to r^13 (error < 2^-104).
CR_F DD exp_r_dd(DD r) {
  DD p = {INVFACT_HI[13], INVFACT_LO[13]};
  for (int n = 12; n >= 0; --n) p = dd_add(dd_mul(p, r), DD{INVFACT_HI[n], INVFACT_LO[n]});
  return p;
}
// 2^(k/16) * e^r as DD, exponent applied (results stay normal in binary64).
CR_F DD exp_dd(int k, DD r) {
  int j = k & 15, e = k >> 4;
  DD v = dd_mul(DD{EXP2J_HI[j], EXP2J_LO[j]}, exp_r_dd(r));
  double s = scale2(1.0, e);
  return DD{v.hi * s, v.lo * s};
}

// Argument reduction x = k*ln2/16 + r for the natural-base functions.
struct RedExp {
  int k;
  double kd, r;
};
CR_F RedExp red_exp(double xc) {
  double t = fma_(xc, INV_LN2_16, SHIFTER);
  double kd = sub_(t, SHIFTER);
  double r = fma_(kd, -LN2_16_H, xc);  // exact (Cody-Waite)
  r = fma_(kd, -LN2_16_M, r);
  return {(int)d2lo(t), kd, r};
}
CR_F DD red_exp_dd(double xc, int &k) {
  double t = fma_(xc, INV_LN2_16, SHIFTER);
  double kd = sub_(t, SHIFTER);
  k = (int)d2lo(t);
  double r1 = fma_(kd, -LN2_16_H, xc);       // exact
  DD r = two_sum(r1, -mul_(kd, LN2_16_M));   // kd*M exact
  return dd_add_d(r, -mul_(kd, LN2_16_L));
}

struct FnExp {
  static constexpr uint32_t E = 512;
  struct Regs { const double *t; };
  CR_F static void load(Regs &R) { R.t = exp_tab<121>(); }
  CR_F static Fast fast(float x, const Regs &R) {
    RedExp q = red_exp(f2d(fminf(fmaxf(x, -104.5f), 89.5f)));
    // main: 2^-26 < |x| < inf (saturation is handled by the clamp)
    return Fast{exp_core3(q.k, q.r, R.t), in_main(f2u(x))};
  }
  CR_F static bool in_main(uint32_t xb) { return in_range(xb << 1, 0x65000002u, 0xFF000000u); }
  // map kernels: main <=> 2^-26 < |x| <= FLT_MAX (float compares, same set as in_main)
  static constexpr bool kMainAbs = true;
  static constexpr float kMainLo = 0x1p-26f, kMainHi = 0x1.fffffep127f;
  template <int M>
  CR_F static uint32_t special(float x) { return exp_like_special<M>(f2u(x)); }
  CR_F static DD slow(float x) {
    double xc = fmin(fmax(f2d(x), -104.5), 89.5);
    int k;
    DD r = red_exp_dd(xc, k);
    return exp_dd(k, r);
  }
};

struct FnExp2 {
  static constexpr uint32_t E = 512;
  struct Regs { const double *t; };
  CR_F static void load(Regs &R) { R.t = exp_tab<130>(); }
  CR_F static Fast fast(float x, const Regs &R) {
    double xc = f2d(fminf(fmaxf(x, -151.5f), 129.5f));
    double t = fma_(xc, 16.0, SHIFTER);
    double kd = sub_(t, SHIFTER);
    double u = fma_(kd, -0.0625, xc);  // exact
    // integer x gives 2^x exactly: the rounding test sends it to the accurate
    // path, whose exact-value snap returns it in every mode.
    return Fast{exp_core3((int)d2lo(t), mul_(u, LN2_D), R.t), in_main(f2u(x))};
  }
  CR_F static bool in_main(uint32_t xb) { return in_range(xb << 1, 0x65000002u, 0xFF000000u); }
  // map kernels: main <=> 2^-26 < |x| <= FLT_MAX (float compares, same set as in_main)
  static constexpr bool kMainAbs = true;
  static constexpr float kMainLo = 0x1p-26f, kMainHi = 0x1.fffffep127f;
  template <int M>
  CR_F static uint32_t special(float x) { return exp_like_special<M>(f2u(x)); }
  CR_F static DD slow(float x) {
    double xc = fmin(fmax(f2d(x), -151.5), 129.5);
    double t = fma_(xc, 16.0, SHIFTER);
    double kd = sub_(t, SHIFTER);
    double u = fma_(kd, -0.0625, xc);
    DD r = two_prod(u, LN2_D);
    r = dd_add_d(r, mul_(u, LN2_DL));
    return exp_dd((int)d2lo(t), r);
  }
};

struct FnExp10 {
  static constexpr uint32_t E = 512;
  struct Regs { const double *t; };
  CR_F static void load(Regs &R) { R.t = exp_tab<123>(); }
  CR_F static Fast fast(float x, const Regs &R) {
    double xc = f2d(fminf(fmaxf(x, -45.5f), 39.5f));
    double t = fma_(xc, LOG2_10_16, SHIFTER);
    double kd = sub_(t, SHIFTER);
    double r = fma_(xc, LN10_H, -mul_(kd, LN2_16_H));
    r = fma_(xc, LN10_M, r);
    r = fma_(kd, -LN2_16_M, r);
    r = fma_(xc, LN10_L, r);
    return Fast{exp_core3((int)d2lo(t), r, R.t), in_main(f2u(x))};
  }
  CR_F static bool in_main(uint32_t xb) { return in_range(xb << 1, 0x63000002u, 0xFF000000u); }
  // map kernels: main <=> 2^-28 < |x| <= FLT_MAX (float compares, same set as in_main)
  static constexpr bool kMainAbs = true;
  static constexpr float kMainLo = 0x1p-28f, kMainHi = 0x1.fffffep127f;
  template <int M>
  CR_F static uint32_t special(float x) { return exp_like_special<M>(f2u(x)); }
  CR_F static DD slow(float x) {
    double xc = fmin(fmax(f2d(x), -45.5), 39.5);
    double t = fma_(xc, LOG2_10_16, SHIFTER);
    double kd = sub_(t, SHIFTER);
    // x*ln10 - k*ln2/16 in DD: all partial products exact except the last.
    DD r = two_sum(mul_(xc, LN10_H), -mul_(kd, LN2_16_H));
    r = dd_add_d(r, mul_(xc, LN10_M));
    r = dd_add_d(r, -mul_(kd, LN2_16_M));
    r = dd_add(r, two_prod(xc, LN10_L));
    r = dd_add_d(r, -mul_(kd, LN2_16_L));
    return exp_dd((int)d2lo(t), r);
  }
};

struct FnExpm1 {
  static constexpr uint32_t E = 128;
  struct Regs { const double *t; };
  CR_F static void load(Regs &R) { R.t = exp_tab<131>(); }
  CR_F static Fast fast(float x, const Regs &R) {
    uint32_t xb = f2u(x);
    RedExp q = red_exp(f2d(fminf(fmaxf(x, -18.5f), 89.5f)));
    int e = q.k >> 4;
    double T = scale2_imad(exp_t(R.t, q.k), e);
    double p = fma_(mul_(q.r, q.r), expq(q.r), q.r);
    // main: 2^-26 < |x| < inf and x >= -18
    return Fast{fma_(T, p, sub_(T, 1.0)), in_main(xb)};
  }
  // main: 2^-26 < |x| < inf. x < -18.5 takes the clamp: expm1(-18.5) lies in
  // (-1, -1 + 2^-26), which holds no binary32 rounding boundary, so it rounds
  // like the true value in every mode.
  CR_F static bool in_main(uint32_t xb) { return in_range(xb << 1, 0x65000002u, 0xFF000000u); }
  template <int M>
  CR_F static uint32_t special(float x) {
    uint32_t xb = f2u(x), az = xb << 1;
    if (nan_bits(xb)) return quiet_bits(xb);
    if (az == 0) return xb;
    if (az == 0xFF000000u) return (int)xb < 0 ? 0xBF800000u : 0x7F800000u;
    double xd = f2d(x);
    if (x < -18.0f) return f2u(cvt_f32<M>(-1.0 + 0x1p-40));  // (-1, -1 + 2^-25)
    return f2u(cvt_f32<M>(fma_(dabs(xd), 0x1p-36, xd)));     // x + x^2/2 beside x
  }
  CR_F static DD slow(float x) {
    double xc = fmin(fmax(f2d(x), -18.5), 89.5);
    int k;
    DD r = red_exp_dd(xc, k);
    if (k == 0) {  // e^r - 1 = sum_{n>=1} r^n/n!, no cancellation
      DD p = {INVFACT_HI[14], INVFACT_LO[14]};
      for (int n = 13; n >= 1; --n) p = dd_add(dd_mul(p, r), DD{INVFACT_HI[n], INVFACT_LO[n]});
      return dd_mul(p, r);
    }
    return dd_add_d(exp_dd(k, r), -1.0);
  }
};

// Hyperbolics share the exp reduction: x = a + r, a = k ln2/16,
// sinh x = sinh a cosh r + cosh a sinh r, cosh x = cosh a cosh r + sinh a sinh r.
struct HypParts {
  double Sa, Ca, sr, cr;
};
// Fast path uses the rounded table (2^-54 relative per entry): for k = +-1 the
// difference E+ - E- loses ~5 bits, which the sinh/tanh tolerances cover.
// Shared table of (2^(j/16), 2^(-j/16 mod 1)): e^(+a) and e^(-a) come from
// row k mod 16 (entry k holds T[k mod 16] and T[-k mod 16]), column-split
// (two conflict-free LDS.64, see sh_split16; the interleaved LDS.128 form
// measured 7.4 wavefronts per load in sinhf) - one table read per element
// was 4-5% faster than four SHFL (profiles/r01/ab_shtab_hyp.txt).
template <int TAG>
CR_F const double *exp_pm_pairs() {
#if CR_DEVICE
  __shared__ __align__(16) double tab[32];
  if (threadIdx.x < 16) {
    tab[threadIdx.x] = 0.5 * EXP2J_HI[threadIdx.x];  // halved: e^(+-a)/2 (exact)
    tab[16 + threadIdx.x] = 0.5 * EXP2J_HI[(16 - threadIdx.x) & 15];
  }
  __syncthreads();
  return tab;
#else
  static double tab[32];
  for (int i = 0; i < 16; ++i) {
    tab[i] = 0.5 * EXP2J_HI[i];
    tab[16 + i] = 0.5 * EXP2J_HI[(16 - i) & 15];
  }
  return tab;
#endif
}
using HypTab = const double *;
CR_F HypParts hyp_parts(double ax, HypTab tab) {
  RedExp q = red_exp(ax);
  const int kp = q.k;
  // e^(+-a)/2 from the halved table: 2^(k>>4) and 2^((-k)>>4) = 2^-((k+15)>>4)
  // as one IMAD each on the exponent field
  const SplitRow pm = split_row(tab, kp);
  double Ep = scale2_imad(split_get<0>(pm), kp >> 4);
  double Em = scale2_imad_neg(split_get<1>(pm), (kp + 15) >> 4);
  double s = mul_(q.r, q.r);
  double sr = fma_(mul_(q.r, s), fma_(SINHQ[1], s, SINHQ[0]), q.r);
  double cr = fma_(s, fma_(COSHQ[1], s, COSHQ[0]), 1.0);
  return {sub_(Ep, Em), add_(Ep, Em), sr, cr};
}
struct HypDD {
  DD Sa, Ca, sr, cr;
};
CR_F HypDD hyp_parts_dd(double ax) {
  int k;
  DD r = red_exp_dd(ax, k);
  DD s = dd_mul(r, r);
  // sinh r = r * sum s^n/(2n+1)!, cosh r = sum s^n/(2n)!  (n <= 6)
  DD ps = {INVFACT_HI[13], INVFACT_LO[13]}, pc = {INVFACT_HI[12], INVFACT_LO[12]};
  for (int n = 5; n >= 0; --n) {
    ps = dd_add(dd_mul(ps, s), DD{INVFACT_HI[2 * n + 1], INVFACT_LO[2 * n + 1]});
    pc = dd_add(dd_mul(pc, s), DD{INVFACT_HI[2 * n], INVFACT_LO[2 * n]});
  }
  DD sr = dd_mul(ps, r);
  int kp = k, km = -k;
  double s1 = scale2(1.0, kp >> 4), s2 = scale2(1.0, km >> 4);
  DD Ep = {EXP2J_HI[kp & 15] * s1, EXP2J_LO[kp & 15] * s1};
  DD Em = {EXP2J_HI[km & 15] * s2, EXP2J_LO[km & 15] * s2};
  DD Sa = dd_add(Ep, dd_neg(Em)), Ca = dd_add(Ep, Em);
  Sa = DD{Sa.hi * 0.5, Sa.lo * 0.5};
  Ca = DD{Ca.hi * 0.5, Ca.lo * 0.5};
  return {Sa, Ca, sr, pc};
}

struct FnSinh {
  static constexpr uint32_t E = 512;
  struct Regs { HypTab t; };
  CR_F static void load(Regs &R) { R.t = exp_pm_pairs<110>(); }
  CR_F static Fast fast(float x, const Regs &R) {
    uint32_t xb = f2u(x);
    HypParts h = hyp_parts(f2d(fminf(fabs_(x), 90.0f)), R.t);
    return Fast{with_sign(fma_(h.Sa, h.cr, mul_(h.Ca, h.sr)), xb), in_main(xb)};
  }
  CR_F static bool in_main(uint32_t xb) { return in_range(xb << 1, 0x73000002u, 0xFF000000u); }  // 2^-12 < |x| < inf
  // map kernels: main <=> 2^-12 < |x| <= FLT_MAX (float compares, same set as in_main)
  static constexpr bool kMainAbs = true;
  static constexpr float kMainLo = 0x1p-12f, kMainHi = 0x1.fffffep127f;
  template <int M>
  CR_F static uint32_t special(float x) {
    uint32_t xb = f2u(x), az = xb << 1;
    if (nan_bits(xb)) return quiet_bits(xb);
    if (az == 0 || az == 0xFF000000u) return xb;
    double xd = f2d(x);
    return f2u(cvt_f32<M>(fma_(xd, 0x1p-36, xd)));  // x + x^3/6 just above |x|
  }
  CR_F static DD slow(float x) {
    double xd = f2d(x);
    HypDD h = hyp_parts_dd(fmin(dabs(xd), 90.0));
    DD v = dd_add(dd_mul(h.Sa, h.cr), dd_mul(h.Ca, h.sr));
    return xd < 0 ? dd_neg(v) : v;
  }
};

struct FnCosh {
  static constexpr uint32_t E = 512;
  struct Regs { HypTab t; };
  CR_F static void load(Regs &R) { R.t = exp_pm_pairs<111>(); }
  CR_F static Fast fast(float x, const Regs &R) {
    HypParts h = hyp_parts(f2d(fminf(fabs_(x), 90.0f)), R.t);
    return Fast{fma_(h.Ca, h.cr, mul_(h.Sa, h.sr)), in_main(f2u(x))};
  }
  CR_F static bool in_main(uint32_t xb) { return in_range(xb << 1, 0x72000002u, 0xFF000000u); }  // 2^-13 < |x| < inf
  // map kernels: main <=> 2^-13 < |x| <= FLT_MAX (float compares, same set as in_main)
  static constexpr bool kMainAbs = true;
  static constexpr float kMainLo = 0x1p-13f, kMainHi = 0x1.fffffep127f;
  template <int M>
  CR_F static uint32_t special(float x) {
    uint32_t xb = f2u(x), az = xb << 1;
    if (nan_bits(xb)) return quiet_bits(xb);
    if (az == 0) return 0x3F800000u;
    if (az == 0xFF000000u) return 0x7F800000u;
    return f2u(cvt_f32<M>(1.0 + 0x1p-30));  // 1 + x^2/2 in (1, 1 + 2^-24)
  }
  CR_F static DD slow(float x) {
    HypDD h = hyp_parts_dd(fmin(dabs(f2d(x)), 90.0));
    return dd_add(dd_mul(h.Ca, h.cr), dd_mul(h.Sa, h.sr));
  }
};

struct FnTanh {
  // tanh|x| = E / (E + 2), E = expm1(2|x|) = T (1 + p) - 1 (T rounded: for
  // k = +-1 the cancellation costs ~2^-49.5, covered by E).
  static constexpr uint32_t E = 512;
  struct Regs { const double *t; };
  CR_F static void load(Regs &R) { R.t = exp_tab<125>(); }
  CR_F static Fast fast(float x, const Regs &R) {
    uint32_t xb = f2u(x);
    // reduction of 2|x| with the x2 folded in: k = RN(2|x| 16/ln2), h = r/2 =
    // |x| - k ln2/32 (Cody-Waite on the halved constants, exact first step),
    // (e^r - 1)/2 = h + h^2 2Q(2h); E = T e^r - 1 = 2T (e^r - 1)/2 + (T - 1)
    const double xd = f2d_posnorm(f2u(fminf(fabs_(x), 10.0f)));  // exact on the main range (normal |x|)
    const double t = fma_(xd, INV_LN2_32, SHIFTER);
    const double kd = sub_(t, SHIFTER);
    double h = fma_(kd, -LN2_32_H, xd);  // exact
    h = fma_(kd, -LN2_32_M, h);
    const int k = (int)d2lo(t), e = k >> 4;
    const double Tj = exp_t(R.t, k);
    const double T = scale2_imad(Tj, e), T2 = scale2_imad(Tj, e + 1);
    const double q = fma_(fma_(fma_(fma_(EXPQ_HALF[4], h, EXPQ_HALF[3]), h, EXPQ_HALF[2]), h, EXPQ_HALF[1]), h,
                          EXPQ_HALF[0]);
    const double ph = fma_(mul_(h, h), q, h);
    double em1 = fma_(T2, ph, sub_(T, 1.0));
    return Fast{with_sign(div_fast(em1, add_(em1, 2.0)), xb), in_main(xb)};
  }
  // main: 2^-12 < |x| < inf. |x| > 10 takes the clamp: tanh(10) lies in
  // (1 - 2^-27, 1), which holds no binary32 rounding boundary, so it rounds
  // like the true value in every mode.
  CR_F static bool in_main(uint32_t xb) { return in_range(xb << 1, 0x73000002u, 0xFF000000u); }
  // map kernels: main <=> 2^-12 < |x| <= FLT_MAX (float compares, same set as in_main)
  static constexpr bool kMainAbs = true;
  static constexpr float kMainLo = 0x1p-12f, kMainHi = 0x1.fffffep127f;
  template <int M>
  CR_F static uint32_t special(float x) {
    uint32_t xb = f2u(x), az = xb << 1;
    if (nan_bits(xb)) return quiet_bits(xb);
    if (az == 0) return xb;
    if (az == 0xFF000000u) return (int)xb < 0 ? 0xBF800000u : 0x3F800000u;
    double xd = f2d(x);
    if (az >= 0x82400000u) return f2u(cvt_f32<M>(with_sign(1.0 - 0x1p-40, xb)));  // |x| >= 10
    return f2u(cvt_f32<M>(fma_(-xd, 0x1p-36, xd)));  // x - x^3/3 just below |x|
  }
  CR_F static DD slow(float x) {
    double xd = f2d(x);
    HypDD h = hyp_parts_dd(fmin(dabs(xd), 10.0));
    DD sh = dd_add(dd_mul(h.Sa, h.cr), dd_mul(h.Ca, h.sr));
    DD ch = dd_add(dd_mul(h.Ca, h.cr), dd_mul(h.Sa, h.sr));
    DD v = dd_div(sh, ch);
    return xd < 0 ? dd_neg(v) : v;
  }
};

// ============================================================ log family ====
// Log family: the 16-entry table of (c_i, L_i) pairs lives in shared memory,
// one LDS.128 per lookup instead of three SHFL (+ a register move to pair the
// words): 6-16% faster than the register-table form with the shapes re-tuned
// (profiles/r01/ab_shtab_log.txt). Filled by the block's first 16 threads at
// kernel entry (every kernel calls F::load() unconditionally in its prologue).
template <int TAG>
CR_F const D2 *log_pairs(const double *L) {
#if CR_DEVICE
  __shared__ __align__(256) D2 tab[16];  // 256-aligned: see log_pair()
  // The OR-ed row offset needs the shared *address* 256-aligned. User shared
  // memory starts 1 KiB into the CTA's window (sm_100 reserves the first
  // 1 KiB), so declared alignments up to 1 KiB hold for absolute addresses
  // (a 4 KiB alignment did not: an OR-addressed Payne-Hanek table read wrong
  // rows in a round-2 build). The check costs one test per thread.
  if (((uint32_t)__cvta_generic_to_shared(tab) & 255u) != 0u) __trap();
  if (threadIdx.x < 16) tab[threadIdx.x] = D2{hilo2d(LOG_C_HI[threadIdx.x], 0u), L[threadIdx.x]};
  __syncthreads();
  return tab;
#else
  static D2 tab[16];
  for (int i = 0; i < 16; ++i) tab[i] = D2{hilo2d(LOG_C_HI[i], 0u), L[i]};
  return tab;
#endif
}

// Entry (i & 15) of a log_pairs table for the raw bin index i = hh >> 16:
// byte offset (hh >> 12) & 0xF0 OR-ed into the 256-aligned shared address
// (SHF + one 3-input LOP3, then LDS.128 [R]; the indexed C++ form adds the
// table base with an extra IADD per element).
CR_F D2 log_pair(const D2 *t, int hh) {
#if CR_DEVICE
  const uint32_t a = (((uint32_t)hh >> 12) & 0xF0u) | (uint32_t)__cvta_generic_to_shared(t);
  D2 r;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(a));
  return r;
#else
  return t[(hh >> 16) & 15];
#endif
}

// Interleaved shared 16-entry pair table {A[i], B[i]} (one LDS.128 per
// lookup; used where the column-split form measured slower: tanf).
template <int TAG>
CR_F const D2 *sh_pair16(const double *A, const double *B) {
#if CR_DEVICE
  __shared__ __align__(16) D2 tab[16];
  if (threadIdx.x < 16) tab[threadIdx.x] = D2{A[threadIdx.x], B[threadIdx.x]};
  __syncthreads();
#else
  static D2 tab[16];
  for (int i = 0; i < 16; ++i) tab[i] = D2{A[i], B[i]};
#endif
  return tab;
}



// x = 2^e * m, m in [0.765625, 1.53125); bin i = 4 bits after the window
// offset (16 bins, 1.0 at the centre of bin 7 with c_7 = 1 so log near 1 is
// relative-accurate); r = m*c_i - 1 (exact when m has <= 24 bits).
struct RedLog {
  int e, i, hh;
  double m;
};
// `i` is the raw bin index (bits above the 16-bin field included): table
// reads use i & 15.
CR_F RedLog red_log(double xd) {
  int h = d2hi(xd);
  int hh = h - 0x3FE88000;
  int e = hh >> 20;
#if CR_DEVICE
  // m's high word h - e 2^20 as one IMAD (the shift-and-subtract form compiles
  // to LOP3 + IADD on the ALU pipe)
  int mh;
  asm("mad.lo.s32 %0, %1, -1048576, %2;" : "=r"(mh) : "r"(e), "r"(h));
#else
  int mh = h - (int)((uint32_t)e << 20);
#endif
  return {e, hh >> 16, hh, hilo2d(mh, d2lo(xd))};
}

template <int BASE>  // 0: ln, 2: log2, 10: log10
struct FnLogB {
  static constexpr uint32_t E = 1024;
  struct Regs { const D2 *t; };
  CR_F static void load(Regs &R) {
    R.t = log_pairs<BASE>(BASE == 0 ? LOG_L_HI : BASE == 2 ? LOG2_L_HI : LOG10_L_HI);
  }
  CR_F static Fast fast(float x, const Regs &R) {
    uint32_t xb = f2u(x);
    RedLog q = red_log(f2d(x));
    const D2 cl = log_pair(R.t, q.hh);
    const double c = cl.x, L = cl.y;
    double r = fma_(q.m, c, -1.0);  // exact
    double p = fma_(mul_(r, r), logq(r), r);
    double ed = i2d(q.e), a;
    if (BASE == 0) a = add_(fma_(ed, LN2_D, L), p);
    else if (BASE == 2) a = fma_(p, INV_LN2, add_(ed, L));
    else a = fma_(p, INV_LN10, fma_(ed, LOG10_2, L));
    // main: 0 < x < +Inf. Exact results (x = 1, 2^k, 10^k) fail the rounding
    // test and are returned exactly by the accurate path's snap.
    return Fast{a, in_main(xb)};
  }
  CR_F static bool in_main(uint32_t xb) { return xb - 1u < 0x7F7FFFFFu; }  // 0 < x < +Inf
  // map kernels: main <=> 0 < x <= FLT_MAX (float compares, same set as in_main)
  static constexpr bool kMainAbs = false;
  static constexpr float kMainLo = 0.0f, kMainHi = 0x1.fffffep127f;
  // branch-free: +-0 -> -Inf, +Inf -> +Inf, NaN -> quiet(x), x < 0 -> qNaN
  template <int M>
  CR_F static uint32_t special(float x) {
    const uint32_t xb = f2u(x);
    uint32_t r = (xb << 1) == 0 ? 0xFF800000u : 0x7FC00000u;
    r = xb == 0x7F800000u ? 0x7F800000u : r;
    return nan_bits(xb) ? quiet_bits(xb) : r;
  }
  CR_F static DD log_dd_core(int e, int i, DD r) {
    // log1p(r) = sum_{n=1}^{24} (-1)^(n+1) r^n / n
    DD p = dd_mul(dd_horner(LOG1P_T_HI, LOG1P_T_LO, 24, r), r);
    double ed = i2d(e);
    DD el = two_sum(mul_(ed, LN2_H), mul_(ed, LN2_M));
    el = dd_add_d(el, mul_(ed, LN2_L));
    DD v = dd_add(dd_add(el, DD{LOG_L_HI[i], LOG_L_LO[i]}), p);
    if (BASE == 2) v = dd_mul(v, DD{INV_LN2, INV_LN2_L});
    if (BASE == 10) v = dd_mul(v, DD{INV_LN10, INV_LN10_L});
    return v;
  }
  CR_F static DD slow(float x) {
    RedLog q = red_log(f2d(x));
    double r = fma_(q.m, (double)LOG_C[q.i & 15], -1.0);  // exact
    return log_dd_core(q.e, q.i & 15, DD{r, 0.0});
  }
};
using FnLog = FnLogB<0>;
using FnLog2 = FnLogB<2>;
using FnLog10 = FnLogB<10>;

struct FnLog1p {
  static constexpr uint32_t E = 1024;
  struct Regs { const D2 *t; };
  CR_F static void load(Regs &R) { R.t = log_pairs<1>(LOG_L_HI); }
  CR_F static Fast fast(float x, const Regs &R) {
    uint32_t xb = f2u(x);
    double y = add_(1.0, f2d(x));
    RedLog q = red_log(y);
    const D2 cl = log_pair(R.t, q.hh);
    const double c = cl.x, L = cl.y;
    double r = fma_(q.m, c, -1.0);
    double p = fma_(mul_(r, r), logq(r), r);
    double a = add_(fma_(i2d(q.e), LN2_D, L), p);
    // fast-path main: -1 < x < +Inf (two float compares; NaN fails both).
    // +-0 is "main" here only because the tiny rule (which the kernels apply
    // to every tiny lane, zeros included) returns it exactly; in_main() below
    // keeps the zeros on the rule path for the rare / accurate routing.
    (void)xb;
    const bool main = (x > -1.0f) & (x <= 0x1.fffffep127f);
    return Fast{a, main};
  }
  // |x| <= 2^-26 is ~40% of all bit patterns (79% of the config-2 mix): its
  // rule stays on the main path, applied to the result bits after the
  // conversion. log1p(x) = x - x^2/2 + ... lies strictly below x and within
  // x^2/2 < 2^-27 |x| of it, so in mode M it rounds to x (RNE, RU), to the
  // float below x (RD), or toward zero from there (RZ): an integer +-1.
  // log1p(+-0) = +-0 exactly in every mode: the zeros are tiny and keep xb.
  static constexpr float kTiny = 0x1p-26f;  // the map kernels' tiny test: |x| <= kTiny
  static constexpr bool kMainAbs = false;   // map kernels: -1 < x <= FLT_MAX
  static constexpr float kMainLo = -1.0f, kMainHi = 0x1.fffffep127f;
  CR_F static bool is_tiny(uint32_t xb) { return (xb << 1) <= 0x65000000u; }  // = |x| <= 2^-26
  template <int M>
  CR_F static uint32_t tiny_bits(uint32_t xb) {
    if (M == RNE || M == RU) return xb;
    if (M == RZ) return (int)xb > 0 ? xb - 1u : xb;  // positive: the float below x
    // RD: next float toward -Inf (x > 0: down; x < 0: magnitude up; zeros kept)
    return (int)xb > 0 ? xb - 1u : (xb > 0x80000000u ? xb + 1u : xb);
  }
  CR_F static bool in_main(uint32_t xb) { return in_range(xb << 1, 2u, 0xFF000000u) && xb < 0xBF800000u; }
  template <int M>
  CR_F static uint32_t special(float x) {
    // branch-free (the rare loop runs it divergently): the tiny rule, then
    // +Inf, x <= -1 and NaN by selects
    const uint32_t xb = f2u(x);
    uint32_t r = tiny_bits<M>(xb);                                  // +-0 and |x| <= 2^-26
    r = xb == 0x7F800000u ? xb : r;                                 // +Inf
    r = xb >= 0xBF800000u ? (xb == 0xBF800000u ? 0xFF800000u : 0x7FC00000u) : r;  // x <= -1
    return nan_bits(xb) ? quiet_bits(xb) : r;
  }
  CR_F static DD slow(float x) {
    double xd = f2d(x);
    // tiny |x|: the main path's rule (x - x^2/2 strictly inside the gap below
    // x) — a plain DD here would be snapped to x by round_dd.
    if ((f2u(x) << 1) <= 0x65000000u) return DD{xd, -dabs(xd) * 0x1p-36};
    DD y = two_sum(1.0, xd);  // 1 + x = y.hi + y.lo exactly
    RedLog q = red_log(y.hi);
    DD pm = two_prod(q.m, (double)LOG_C[q.i & 15]);
    DD r = fast_two_sum(sub_(pm.hi, 1.0), pm.lo);
    DD v = FnLogB<0>::log_dd_core(q.e, q.i & 15, r);
    // log(1 + x) = log(y.hi) + log1p(u), u = y.lo / y.hi (|u| <= 2^-53, or
    // u = x itself when x is tiny and y.hi == 1): u - u^2/2 + u^3/3 - u^4/4.
    double u = y.lo / y.hi;
    double tail = mul_(u, fma_(u, fma_(u, fma_(u, -0.25, 1.0 / 3.0), -0.5), 0.0));
    return dd_add(v, fast_two_sum(u, tail));
  }
};

// ================================================================== trig ====
// x = k*pi/16 + r, |r| <= pi/32; sin(x) = S_k cos r + C_k sin r with
// S_k = sin(k pi/16) = +-SIN16[k & 15] (sign from k & 16), C_k = S_{k+8}.
struct RedTrig {
  int k;
  double r;
};
CR_F RedTrig red_trig_small(double xd) {
  double t = fma_(xd, INV_PI_16, SHIFTER);
  double kd = sub_(t, SHIFTER);
  // two-part Cody-Waite, valid for |x| < 2^12 (larger |x| take Payne-Hanek):
  // k * PI_16_A is exact (36-bit constant), the tail error is < 2^-76
  double r = fma_(kd, -PI_16_A, xd);
  r = fma_(kd, -PI_16_B, r);
  return {(int)d2lo(t), r};
}

// Payne-Hanek for |x| >= 2^12 (binary32 x = M * 2^(ex-23)):
// x*16/pi mod 32 from a 32*NW-bit window of 1/pi times the 24-bit M.
// Returns k mod 32 (of |x|) and the 64-bit signed fraction (units 2^-64),
// plus the next 64 (NW >= 5) or 59 (NW = 4) fraction bits.
struct PH {
  int k;
  int64_t f;      // fraction * 2^64, in [-2^63, 2^63)
  uint64_t f2;    // following 64 bits (accurate path only)
};
template <int NW>
CR_F PH payne_hanek(uint32_t xb, const unsigned *words) {
  int ex = (int)((xb >> 23) & 0xFF) - 127;
  uint32_t M = (xb & 0x7FFFFFu) | 0x800000u;
  int g0 = ex + 40;  // bit index of j0 = ex - 23 in the padded word array
  int w0 = g0 >> 5, sh = g0 & 31;
  uint32_t W[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    uint32_t a = words[w0 + i], b = words[w0 + i + 1];
    W[i] = sh ? (a << sh) | (b >> (32 - sh)) : a;
  }
  // P = M * W (little-endian limbs L[0..NW]); W[0] is the most significant.
  uint32_t L[NW + 1];
  uint64_t carry = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    uint64_t p = (uint64_t)M * W[NW - 1 - i] + carry;
    L[i] = (uint32_t)p;
    carry = p >> 32;
  }
  L[NW] = (uint32_t)carry;
  // value = P * 2^-(32*NW - 5): integer part mod 32 = top 5 bits of limb NW-1.
  uint32_t top = L[NW - 1];
  uint32_t kk = top >> 27;
  uint64_t f = ((uint64_t)(top & 0x07FFFFFFu) << 37) | ((uint64_t)L[NW - 2] << 5) | (L[NW - 3] >> 27);
  static_assert(NW >= 4, "window too short");
  uint64_t f2 = ((uint64_t)(L[NW - 3] & 0x07FFFFFFu) << 37) | ((uint64_t)L[NW - 4] << 5);
  if constexpr (NW >= 5) f2 |= L[NW - 5] >> 27;
  kk += (uint32_t)(f >> 63);
  return {(int)kk, (int64_t)f, f2};
}

CR_F double sin_r(double r, double s) {
  return fma_(mul_(r, s), fma_(fma_(SINQ[2], s, SINQ[1]), s, SINQ[0]), r);
}
CR_F double cos_r(double s) { return fma_(s, fma_(fma_(COSQ[2], s, COSQ[1]), s, COSQ[0]), 1.0); }
// tan r = r + r^3 T(r^2), |r| <= pi/32 (relative error 2^-47.3, tools/gen_tables.py)
CR_F double tan_r(double r, double s) {
  return fma_(mul_(r, s), fma_(fma_(fma_(TANQ[3], s, TANQ[2]), s, TANQ[1]), s, TANQ[0]), r);
}
// DD sin/cos of r (|r| <= pi/32), Taylor to r^23.
CR_F void sincos_r_dd(DD r, DD &sr, DD &cr) {
  DD s = dd_mul(r, r);
  DD ps = {SINT_HI[11], SINT_LO[11]}, pc = {COST_HI[11], COST_LO[11]};
  for (int n = 10; n >= 0; --n) {
    ps = dd_add(dd_mul(ps, s), DD{SINT_HI[n], SINT_LO[n]});
    pc = dd_add(dd_mul(pc, s), DD{COST_HI[n], COST_LO[n]});
  }
  sr = dd_mul(ps, r);
  cr = pc;
}
CR_F DD sin16_dd(int k) {
  DD v = {SIN16_HI[k & 15], SIN16_LO[k & 15]};
  return (k & 16) ? dd_neg(v) : v;
}
// Accurate reduction: k and r (DD) for any finite binary32 x.
CR_F DD red_trig_dd(float x, int &k) {
  double xd = f2d(x);
  uint32_t xb = f2u(x);
  if (dabs(xd) < 0x1p17) {
    double t = fma_(xd, INV_PI_16, SHIFTER);
    double kd = sub_(t, SHIFTER);
    k = (int)d2lo(t);
    double r1 = fma_(kd, -PI_16_Q1, xd);            // exact
    DD r = two_sum(r1, -mul_(kd, PI_16_Q2));         // exact product
    r = dd_add_d(r, -mul_(kd, PI_16_Q3));            // exact product
    return dd_add_d(r, -mul_(kd, PI_16_Q4));
  }
  PH p = payne_hanek<6>(xb & 0x7FFFFFFFu, INV_PI_WORDS);
  // fraction = f*2^-64 + f2*2^-128 (f signed), times pi/16
  double fh = (double)(p.f >> 11) * 0x1p11;          // exact (53 bits)
  double fl = (double)(p.f & 2047) + (double)(p.f2 >> 11) * 0x1p-53;
  DD fr = fast_two_sum(fh, fl);
  DD r = dd_mul(fr, DD{PI_16_2M64_H, PI_16_2M64_L});
  k = p.k;
  if (xb >> 31) { k = -k; r = dd_neg(r); }
  return r;
}

// Exponent-indexed Payne-Hanek reduction (the fast path of every lane of a
// warp step that holds a large argument; tools/gen_tables.py gen_ph_table):
// x = M 2^E, row b = biased exponent holds hi + lo = (16/pi) mod 2^(5-E) with
// |x (hi + lo - T_E)| < 2^-77 and hi short enough that f0 = x hi - RN(x hi)
// is exact; then u = f0 + x lo in one FMA (relative 2^-53) and r = u pi/16.
// k = RN(x hi) (mod 32 from the shifter's low word). x*16/pi has at most ~30
// leading zero fraction bits for a binary32 x, so r keeps > 2^-46 relative
// accuracy (the fast path's budget is 2^-44); |u| <= 1/2 + 2^-24.
// Row address: the table's shared address + (b << 4).
// The table is column-split (hi[256] then lo[256], two LDS.64: exponents of
// neighbouring lanes map to distinct banks, see sh_split16).
CR_F D2 ph_row(const double *tab, uint32_t xb) {
#if CR_DEVICE
  const uint32_t a = ((xb >> 20) & 0x7F8u) + (uint32_t)__cvta_generic_to_shared(tab);
  D2 r;
  asm("ld.shared.f64 %0, [%1];" : "=d"(r.x) : "r"(a));
  asm("ld.shared.f64 %0, [%1+2048];" : "=d"(r.y) : "r"(a));
  return r;
#else
  return D2{tab[(xb >> 23) & 0xFFu], tab[256 + ((xb >> 23) & 0xFFu)]};
#endif
}
CR_F RedTrig red_trig_ph(float x, const double *tab) {
  const D2 h = ph_row(tab, f2u(x));
  const double xd = f2d(x);
  const double t = fma_(xd, h.x, SHIFTER);
  const double kd = sub_(t, SHIFTER);
  const double f0 = fma_(xd, h.x, -kd);  // exact, |f0| <= 1/2
  const double u = fma_(xd, h.y, f0);
  return {(int)d2lo(t), mul_(u, PI_16_RN)};
}

// One 16-entry shared table of (sin(j pi/16), cos(j pi/16)) pairs, j = k mod
// 16, read with one LDS.128 (5-8% faster than two register tables read with
// four SHFL: profiles/r01/ab_shtab_trig.txt). With m = bit 4 of k,
// sin(x) = (-1)^m (S_j cos r + C_j sin r) and cos(x) = (-1)^m (C_j cos r -
// S_j sin r): one sign flip of the result (none for tan).
CR_F double flip_k16(double v, int k) { return hilo2d(d2hi(v) ^ ((k << 27) & (int)0x80000000), d2lo(v)); }
template <int WHICH>  // 0: sin, 1: cos, 2: tan
struct FnTrig {
  static constexpr uint32_t E = WHICH == 2 ? 1024 : 512;
  // (S_j, C_j): column-split (conflict-free LDS.64) for all three. tanf had
  // interleaved pairs (round 2 r2q: split -2.6%); after its shorter division
  // the pair LDS.128 conflicts were its top stall and split measured +8.9% on
  // the config mix, -0.9% uniform (profiles/r02/ab_tan_split_r3a.txt)
  static constexpr bool kSplit = true;
  struct Regs {
    const double *t;
    const D2 *p;
  };
  CR_F static void load(Regs &R) {
    if (kSplit) R.t = sh_split16<100, 2>(SIN16_HI, COS16_HI, nullptr);
    else R.p = sh_pair16<104>(SIN16_HI, COS16_HI);
  }
  CR_F static void sc_get(const Regs &R, int k, double &Sj, double &Cj) {
    if (kSplit) {
      const SplitRow sc = split_row(R.t, k);
      Sj = split_get<0>(sc);
      Cj = split_get<1>(sc);
    } else {
      const D2 sc = R.p[k & 15];
      Sj = sc.x;
      Cj = sc.y;
    }
  }
  CR_F static Fast from_red(float x, RedTrig q, const Regs &R) {
    double s = mul_(q.r, q.r);
    double Sj, Cj;
    sc_get(R, q.k, Sj, Cj);
    double a;
    if (WHICH == 2) {
      // tan(a + r) = (S_j + C_j t) / (C_j - S_j t), t = tan r (divided by
      // cos r > 0; period pi, so no sign flip): 13 FP64 operations + one
      // MUFU where sin/cos of r and the two products took 17
      const double t = tan_r(q.r, s);
      a = div_fast(fma_(Cj, t, Sj), fma_(-Sj, t, Cj));
    } else {
      const double sr = sin_r(q.r, s), cr = cos_r(s);
      if (WHICH == 0) a = flip_k16(fma_(Sj, cr, mul_(Cj, sr)), q.k);
      else a = flip_k16(fma_(Cj, cr, -mul_(Sj, sr)), q.k);
    }
    // main: tiny threshold < |x| < inf (sin 2^-12, cos/tan 2^-13)
    return Fast{a, in_main(f2u(x))};
  }
  CR_F static bool in_main(uint32_t xb) {
    return in_range(xb << 1, WHICH == 0 ? 0x73000002u : 0x72000002u, 0xFF000000u);
  }
  // map kernels: main <=> 2^-12 (sin) / 2^-13 < |x| <= FLT_MAX (float compares, same set as in_main)
  static constexpr bool kMainAbs = true;
  static constexpr float kMainLo = WHICH == 0 ? 0x1p-12f : 0x1p-13f, kMainHi = 0x1.fffffep127f;
  // sin and cos from one reduction and one table read.
  CR_F static void sincos_from_red(float x, RedTrig q, const Regs &R, Fast &fs, Fast &fc) {
    double s = mul_(q.r, q.r);
    double sr = sin_r(q.r, s), cr = cos_r(s);
    double Sj, Cj;
    sc_get(R, q.k, Sj, Cj);
    const uint32_t xb = f2u(x);
    fs = Fast{flip_k16(fma_(Sj, cr, mul_(Cj, sr)), q.k), FnTrig<0>::in_main(xb)};
    fc = Fast{flip_k16(fma_(Cj, cr, -mul_(Sj, sr)), q.k), FnTrig<1>::in_main(xb)};
  }
  template <int M>
  CR_F static uint32_t special(float x) {
    uint32_t xb = f2u(x), az = xb << 1;
    if (nan_bits(xb)) return quiet_bits(xb);
    if (az == 0xFF000000u) return 0x7FC00000u;  // sin/cos/tan(+-Inf) invalid
    if (az == 0) return WHICH == 1 ? 0x3F800000u : xb;
    double xd = f2d(x);
    if (WHICH == 0) return f2u(cvt_f32<M>(fma_(-xd, 0x1p-36, xd)));  // x - x^3/6
    if (WHICH == 2) return f2u(cvt_f32<M>(fma_(xd, 0x1p-36, xd)));   // x + x^3/3
    return f2u(cvt_f32<M>(1.0 - 0x1p-31));                          // 1 - x^2/2
  }
  CR_F static Fast fast(float x, const Regs &R) { return from_red(x, red_trig_small(f2d(x)), R); }
  CR_F static DD slow(float x) {
    int k;
    DD r = red_trig_dd(x, k);
    DD sr, cr;
    sincos_r_dd(r, sr, cr);
    DD Sk = sin16_dd(k), Ck = sin16_dd(k + 8);
    DD sn = dd_add(dd_mul(Sk, cr), dd_mul(Ck, sr));
    DD cs = dd_add(dd_mul(Ck, cr), dd_neg(dd_mul(Sk, sr)));
    if (WHICH == 0) return sn;
    if (WHICH == 1) return cs;
    return dd_div(sn, cs);
  }
};
using FnSin = FnTrig<0>;
using FnCos = FnTrig<1>;
using FnTan = FnTrig<2>;

// ========================================================== inverse trig ====
// atan2-style core for Y, X >= 0: theta_j = j*pi/30 (j = 0..15), t =
// tan(angle - theta_j) = (Y cos - X sin)/(X cos + Y sin), result theta_j +
// atan(t); sin/cos of theta_j from one 16-entry table (cos theta_j = sin
// theta_{15-j}).
// theta_j index from a cheap fp32 angle estimate (|error| < 0.004 rad, far
// inside the half-spacing pi/60); inputs are binary32 copies of Y, X >= 0.
CR_F int atan_index_f(float yf, float xf) {
  float mn = fminf(yf, xf), mx = fmaxf(yf, xf);
#if CR_DEVICE
  float q = __fdividef(mn, mx);
#else
  float q = mn / mx;
#endif
  q = mx > 0.0f ? q : 0.0f;
  float at = q * fmaf(0.273f, 1.0f - q, 0.78539816f);
  float ang = yf > xf ? 1.57079633f - at : at;
  int j = (int)rintf(ang * 9.5492966f);  // 30/pi
  return j < 0 ? 0 : (j > 15 ? 15 : j);
}
CR_F int atan_index(double Y, double X) { return atan_index_f((float)Y, (float)X); }
CR_F DD atan2_core_dd(DD Y, DD X) {
  int j = atan_index(Y.hi, X.hi);
  DD S = {SIN30_HI[j], SIN30_LO[j]}, C = {SIN30_HI[15 - j], SIN30_LO[15 - j]};
  DD num = dd_add(dd_mul(Y, C), dd_neg(dd_mul(X, S)));
  DD den = dd_add(dd_mul(X, C), dd_mul(Y, S));
  DD t = dd_div(num, den);
  DD s = dd_mul(t, t);
  DD p = dd_mul(dd_horner(ATANT_HI, ATANT_LO, 14, s), t);
  double jd = i2d(j);
  DD th = two_prod(jd, PI_30_H);
  th = dd_add_d(th, mul_(jd, PI_30_L));
  return dd_add(th, p);
}

// atan by angle subtraction (tools/gen_tables.py gen_atan): with z = |x| and
// a table angle A_k near atan z, atan z = A_k + atan((z C_k - S_k)/(C_k + z S_k)),
// |t| <= 0.069. Entry k = j + 8*up, up = (z > 1), j = RN(7.49 * min(z, 1/z)):
// the index needs one fp32 reciprocal, no angle estimate.
CR_F double atan_t2(double t) {
  double s = mul_(t, t);
  double q = fma_(fma_(fma_(ATANQ2[3], s, ATANQ2[2]), s, ATANQ2[1]), s, ATANQ2[0]);
  return fma_(mul_(t, s), q, t);
}

struct FnAtan {
  static constexpr uint32_t E = 512;
  struct Regs { const double *t; };
  CR_F static void load(Regs &R) { R.t = sh_split16<101, 3>(ATAN_C, ATAN_S, ATAN_A_HI); }
  CR_F static Fast fast(float x, const Regs &R) {
    uint32_t xb = f2u(x);
    float axf = fminf(fabs_(x), 0x1p127f);
    double z = f2d_posnorm(f2u(axf));  // exact on the main range (normal |x|)
    bool up = axf > 1.0f;
    const uint32_t kb = f2u(fmaf(up ? rcp_approx_f(axf) : axf, 7.49f, 0x1.8p23f));  // j <= 7
    const SplitRow cs = split_row_kb(R.t, kb, up);
    const double C = split_get<0>(cs), S = split_get<1>(cs), A = split_get<2>(cs);
    double t = div_fast(fma_(z, C, -S), fma_(z, S, C));
    return Fast{with_sign(add_(A, atan_t2(t)), xb), in_main(xb)};
  }
  CR_F static bool in_main(uint32_t xb) { return in_range(xb << 1, 0x73000002u, 0xFF000002u); }  // 2^-12 < |x| <= inf
  // map kernels: main <=> 2^-12 < |x| <= +Inf (float compares, same set as in_main)
  static constexpr bool kMainAbs = true;
  static constexpr float kMainLo = 0x1p-12f, kMainHi = __builtin_huge_valf();
  template <int M>
  CR_F static uint32_t special(float x) {
    uint32_t xb = f2u(x);
    if (nan_bits(xb)) return quiet_bits(xb);
    if ((xb << 1) == 0) return xb;
    double xd = f2d(x);
    return f2u(cvt_f32<M>(fma_(-xd, 0x1p-36, xd)));  // x - x^3/3 just below |x|
  }
  CR_F static DD slow(float x) {
    double xd = f2d(x);
    DD v = atan2_core_dd(DD{fmin(dabs(xd), 0x1p127), 0.0}, DD{1.0, 0.0});
    return xd < 0 ? dd_neg(v) : v;
  }
};

// asin / acos without a division: with theta = asin|x| (or acos|x|), s =
// sqrt(1 - x^2) and a table angle A_k near theta,
//   sin(theta - A_k) = |x| cos A_k - s sin A_k        (asin)
//   sin(phi - B_k)   = s cos B_k - |x| sin B_k        (acos, phi = acos|x|)
// so the result is A_k + asin(d) with |d| <= 0.064 and a degree-3 odd
// polynomial in d^2. Entry k = j + 8*up: up = (|x| > s) selects the upper
// half-angle range and j = RN(10.5 * min(|x|, s)) (tools/gen_tables.py
// gen_asin). The angles have 21 significant bits: one shuffled word each.
CR_F double asinq(double d) {
  double z = mul_(d, d);
  double q = fma_(fma_(fma_(ASINQ[3], z, ASINQ[2]), z, ASINQ[1]), z, ASINQ[0]);
  return fma_(mul_(d, z), q, d);
}

template <bool ACOS>
struct FnAsinAcos {
  static constexpr uint32_t E = 64;
  struct Regs { const double *t; };
  CR_F static void load(Regs &R) {
    // (cos, sin, angle) columns: the angle is a third conflict-free LDS.64 off
    // the same row address (one SHFL + a zero-word move before)
    // acos: a fourth column pi_H - angle for x < 0 (acos(-|x|) = pi - acos|x|)
    R.t = ACOS ? sh_split16<102, 4>(ACOS_C, ACOS_S, ACOS_A_HI) : sh_split16<103, 3>(ASIN_C, ASIN_S, ASIN_A_HI);
  }
  CR_F static Fast fast(float x, const Regs &R) {
    uint32_t xb = f2u(x);
    float axf = fminf(fabs_(x), 1.0f);
    // |x| as a double and sqrt(1 - x^2) as a float by exponent-field
    // arithmetic (integer pipes, not two conversions): exact for the normal
    // |x| of asin's main range; acos's zero / subnormal lanes get a value
    // below 2^-126, and acos of that rounds like acos(x) (pi/2 is nowhere near
    // a binary32 rounding boundary)
    double ax = f2d_posnorm(f2u(axf));
    double s = sqrt_fast(fma_(-ax, ax, 1.0));  // 1 - x^2 exact
    float sf = d2f_trunc(s);
    bool up = axf > sf;
    // j = RN(10.5 * min) in the low bits of the 1.5*2^23-shifted sum; (cos,
    // sin, angle) from three columns of one shared row (round 2; round 1 had
    // the angle in a register table, profiles/r01/ab_shtab_trig.txt)
    const uint32_t kb = f2u(fmaf(up ? sf : axf, 10.5f, 0x1.8p23f));  // j <= 7
    const SplitRow cs = split_row_kb(R.t, kb, up);
    const double C = split_get<0>(cs), S = split_get<1>(cs);
    double a;
    if (!ACOS) {
      const double d = fma_(ax, C, -mul_(s, S));
      a = with_sign(add_(split_get<2>(cs), asinq(d)), xb);
    } else {
      // x < 0: (pi_H - A) + asin(-d) from the fourth column and a sign flip
      // of d (one LOP3), instead of pi_H - (A + asin d) (one DADD + selects)
      const double d = with_sign(fma_(s, C, -mul_(ax, S)), xb);
      a = add_(split_get_dyn(cs, (int)xb < 0 ? 384u : 256u), asinq(d));
    }
    return Fast{a, in_main(xb)};
  }
  // asin main: 2^-12 < |x| < 1; acos main: |x| < 1 (s > 0 on the main path)
  CR_F static bool in_main(uint32_t xb) {
    return ACOS ? (xb << 1) < 0x7F000000u : in_range(xb << 1, 0x73000002u, 0x7F000000u);
  }
  // map kernels: main <=> (acos: any, asin: 2^-12 <) |x| < 1 (float compares, same set as in_main)
  static constexpr bool kMainAbs = true;
  static constexpr float kMainLo = ACOS ? -1.0f : 0x1p-12f, kMainHi = 0x1.fffffep-1f;
  template <int M>
  CR_F static uint32_t special(float x) {
    uint32_t xb = f2u(x);
    if (nan_bits(xb)) return quiet_bits(xb);
    if ((xb << 1) > 0x7F000000u) return 0x7FC00000u;  // |x| > 1
    if ((xb << 1) == 0x7F000000u) {                   // |x| = 1: +-pi/2, 0, pi
      if (!ACOS) return f2u(cvt_f32<M>(with_sign(0.5 * PI_H, xb)));
      return (int)xb < 0 ? f2u(cvt_f32<M>(PI_H)) : 0u;
    }
    if ((xb << 1) == 0) return xb;                    // asin(+-0)
    double xd = f2d(x);
    return f2u(cvt_f32<M>(fma_(xd, 0x1p-36, xd)));   // asin: x + x^3/6 just above |x|
  }
  CR_F static DD slow(float x) {
    double xd = f2d(x), ax = fmin(dabs(xd), 1.0);
    DD s = dd_sqrt(DD{fma_(-ax, ax, 1.0), 0.0});
    if (!ACOS) {
      DD v = atan2_core_dd(DD{ax, 0.0}, s);
      return xd < 0 ? dd_neg(v) : v;
    }
    DD v = atan2_core_dd(s, DD{ax, 0.0});
    return xd < 0 ? dd_add(DD{PI_H, PI_L}, dd_neg(v)) : v;
  }
};
using FnAsin = FnAsinAcos<false>;
using FnAcos = FnAsinAcos<true>;

// ================================================================= rsqrt ====
struct FnRsqrt {
  static constexpr uint32_t E = 8;
  struct Regs {};
  CR_F static void load(Regs &) {}
  CR_F static double newton(double xd) {
    double y = rsqrt_approx(xd);
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      double e = fma_(-mul_(xd, y), y, 1.0);
      y = fma_(mul_(y, 0.5), e, y);
    }
    return y;
  }
  CR_F static Fast fast(float x, const Regs &) {
    return Fast{newton(f2d(x)), in_main(f2u(x))};
  }
  CR_F static bool in_main(uint32_t xb) { return xb - 1u < 0x7F7FFFFFu; }  // 0 < x < inf
  // map kernels: main <=> 0 < x <= FLT_MAX (float compares, same set as in_main)
  static constexpr bool kMainAbs = false;
  static constexpr float kMainLo = 0.0f, kMainHi = 0x1.fffffep127f;
  template <int M>
  CR_F static uint32_t special(float x) {
    uint32_t xb = f2u(x);
    if (nan_bits(xb)) return quiet_bits(xb);
    if (xb == 0u) return 0x7F800000u;
    if (xb == 0x80000000u) return 0xFF800000u;
    if (xb == 0x7F800000u) return 0u;
    return 0x7FC00000u;  // x < 0
  }
  CR_F static DD slow(float x) {
    double xd = f2d(x);
    double y = newton(xd);
    // e = 1 - x y^2 exactly in DD; y' = y (1 + e/2 + 3e^2/8)
    DD y2 = two_prod(y, y);
    DD xy2 = dd_mul_d(y2, xd);
    DD e = dd_add_d(dd_neg(xy2), 1.0);
    double corr = mul_(y, fma_(0.375, e.hi * e.hi, 0.5 * e.hi));
    return fast_two_sum(y, corr);
  }
};

}  // namespace crvec
