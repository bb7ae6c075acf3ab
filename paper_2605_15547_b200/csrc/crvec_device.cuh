// crvec device primitives for sm_100a.
//
// The B200 has what the paper's GPUs lacked (ref: PAPER.md:208): per-
// instruction static rounding. Every helper here maps to 1-3 SASS
// instructions: the reference's AVX-512 helper-op contracts
// (ref: proj/include/crvec/lanes.hpp:53-224) and its software rounding engine
// (ref: proj/src/fpbits.cpp:33-187) collapse to DFMA/DADD plus one
// cvt.{rn,rz,rp,rm}.f32.f64.
//
// The same header also compiles under g++ (CRVEC_EMU) for the developer-only
// algorithm harness in tools/emu/ — that build is never part of libcrvec.so
// and is not a fallback; on the device every helper is a hardware op.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__) && !defined(CRVEC_EMU)
#define CR_F __device__ __forceinline__
#define CR_NOINLINE __device__ __noinline__
#define CR_CONST __device__ __constant__
#define CR_DEVICE 1
#else
#include <cmath>
#include <cstring>
#define CR_F inline
#define CR_NOINLINE
#define CR_CONST const
#define CR_DEVICE 0
#endif

namespace crvec {

// 1.5 * 2^52: adding it rounds to an integer kept in the low mantissa bits.
#define SHIFTER 0x1.8p52

// RoundingMode numbering of ref: proj/include/crvec/fpbits.hpp:13-18.
enum : int { RNE = 0, RZ = 1, RU = 2, RD = 3 };

// ------------------------------------------------------------- bit views ----
#if CR_DEVICE
CR_F uint32_t f2u(float f) { return __float_as_uint(f); }
CR_F float u2f(uint32_t u) { return __uint_as_float(u); }
CR_F uint64_t d2u(double d) { return (uint64_t)__double_as_longlong(d); }
CR_F double u2d(uint64_t u) { return __longlong_as_double((long long)u); }
CR_F int d2hi(double d) { return __double2hiint(d); }
CR_F uint32_t d2lo(double d) { return (uint32_t)__double2loint(d); }
CR_F double hilo2d(int hi, uint32_t lo) { return __hiloint2double(hi, (int)lo); }
CR_F double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
CR_F double add_(double a, double b) { return __dadd_rn(a, b); }
CR_F double sub_(double a, double b) { return __dsub_rn(a, b); }
CR_F double mul_(double a, double b) { return __dmul_rn(a, b); }
CR_F double i2d(int i) { return __int2double_rn(i); }
// a + b rounded in mode M (one DADD with a static rounding modifier)
template <int M>
CR_F double add_M(double a, double b) {
  if (M == RNE) return __dadd_rn(a, b);
  if (M == RZ) return __dadd_rz(a, b);
  if (M == RU) return __dadd_ru(a, b);
  return __dadd_rd(a, b);
}
CR_F double f2d(float f) { return (double)f; }
CR_F double dabs(double a) { return fabs(a); }
CR_F float fabs_(float a) { return fabsf(a); }
// MUFU.RCP64H / MUFU.RSQ64H seeds (~2^-22 relative), refined by Newton steps.
CR_F double rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
CR_F double rsqrt_approx(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));  // one MUFU.RSQ64H (the non-ftz form adds a range fix-up call)
  return r;
}
CR_F float rcp_approx_f(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));  // one MUFU.RCP
  return r;
}
CR_F double sqrt_rn(double x) { return __dsqrt_rn(x); }
CR_F int clz32(uint32_t v) { return __clz((int)v); }
template <int M>
CR_F float cvt_f32(double a) {
  if (M == RNE) return __double2float_rn(a);
  if (M == RZ) return __double2float_rz(a);
  if (M == RU) return __double2float_ru(a);
  return __double2float_rd(a);
}
#else
CR_F uint32_t f2u(float f) { uint32_t u; std::memcpy(&u, &f, 4); return u; }
CR_F float u2f(uint32_t u) { float f; std::memcpy(&f, &u, 4); return f; }
CR_F uint64_t d2u(double d) { uint64_t u; std::memcpy(&u, &d, 8); return u; }
CR_F double u2d(uint64_t u) { double d; std::memcpy(&d, &u, 8); return d; }
CR_F int d2hi(double d) { return (int)(d2u(d) >> 32); }
CR_F uint32_t d2lo(double d) { return (uint32_t)d2u(d); }
CR_F double hilo2d(int hi, uint32_t lo) { return u2d(((uint64_t)(uint32_t)hi << 32) | lo); }
CR_F double fma_(double a, double b, double c) { return std::fma(a, b, c); }
CR_F double add_(double a, double b) { volatile double r = a + b; return r; }
CR_F double sub_(double a, double b) { volatile double r = a - b; return r; }
CR_F double mul_(double a, double b) { volatile double r = a * b; return r; }
CR_F double i2d(int i) { return (double)i; }
template <int M>
CR_F double add_M(double a, double b) {
  double s = add_(a, b), bb = sub_(s, a);
  double e = add_(sub_(a, sub_(s, bb)), sub_(b, bb));  // a + b = s + e exactly
  if (M == RNE || e == 0.0) return s;
  if (M == RZ && (e > 0) != (s > 0)) return std::nextafter(s, 0.0);
  if (M == RU && e > 0) return std::nextafter(s, INFINITY);
  if (M == RD && e < 0) return std::nextafter(s, -INFINITY);
  return s;
}
CR_F double f2d(float f) { return (double)f; }
CR_F double dabs(double a) { return std::fabs(a); }
CR_F float fabs_(float a) { return std::fabs(a); }
// MUFU.RCP64H / RSQ64H seeds modelled pessimistically: the exact value cut
// to 19 fraction bits (relative error < 2^-19; measured on B200: 2^-19.9 /
// 2^-19.0 for |1 - x r| / |1 - x y^2|, tools/mufu_probe.cu)
CR_F double seed19(double v) { uint64_t u; std::memcpy(&u, &v, 8); u &= ~((1ull << 33) - 1); std::memcpy(&v, &u, 8); return v; }
CR_F double rcp_approx(double x) { return seed19(1.0 / x); }
CR_F double rsqrt_approx(double x) { return seed19(1.0 / std::sqrt(x)); }
CR_F float rcp_approx_f(float x) { return 1.0f / x; }
CR_F double sqrt_rn(double x) { return std::sqrt(x); }
CR_F int clz32(uint32_t v) { return v ? __builtin_clz(v) : 32; }
template <int M>
CR_F float cvt_f32(double a) {
  float f = (float)a;  // RNE with gradual underflow / overflow to inf
  if (a != a) return f;
  if (M == RZ && std::fabs((double)f) > std::fabs(a)) f = std::nextafterf(f, 0.0f);
  if (M == RU && (double)f < a) f = std::nextafterf(f, INFINITY);
  if (M == RD && (double)f > a) f = std::nextafterf(f, -INFINITY);
  if (M == RU && (double)f > a && std::isinf(f) && a < 0) f = -3.40282347e38f;
  if (M == RD && (double)f < a && std::isinf(f) && a > 0) f = 3.40282347e38f;
  return f;
}
#endif

// ------------------------------------------------------ 16-entry tables ----
// A table of <= 16 entries lives in registers: lane l holds entry (l & 15);
// a lookup is __shfl_sync (2 SHFL per double), standing in for the AVX-512
// permute of ref: proj/include/crvec/lanes.hpp:320-328. Requires the whole
// warp to be converged (the main paths are branch-free).
#if CR_DEVICE
#define CR_TAB_LOAD(arr) (arr[threadIdx.x & 15])
#define CR_TAB(reg, arr, idx) __shfl_sync(0xffffffffu, (reg), (idx))
#else
#define CR_TAB_LOAD(arr) (arr[0])
#define CR_TAB(reg, arr, idx) (arr[(idx) & 15])
#endif

// ---------------------------------------------------- double-double EFTs ----
// ref: proj/include/crvec/dd.hpp:11-68 (Dekker / Knuth / Joldes-Muller-Popescu).
struct DD {
  double hi, lo;
};
CR_F DD two_sum(double a, double b) {
  double s = add_(a, b);
  double bb = sub_(s, a);
  double e = add_(sub_(a, sub_(s, bb)), sub_(b, bb));
  return {s, e};
}
CR_F DD fast_two_sum(double a, double b) {
  double s = add_(a, b);
  double e = sub_(b, sub_(s, a));
  return {s, e};
}
CR_F DD two_prod(double a, double b) {
  double p = mul_(a, b);
  return {p, fma_(a, b, -p)};
}
CR_F DD dd_add(DD x, DD y) {
  DD s = two_sum(x.hi, y.hi);
  DD t = two_sum(x.lo, y.lo);
  DD v = fast_two_sum(s.hi, add_(s.lo, t.hi));
  return fast_two_sum(v.hi, add_(t.lo, v.lo));
}
CR_F DD dd_add_d(DD x, double y) {
  DD s = two_sum(x.hi, y);
  return fast_two_sum(s.hi, add_(x.lo, s.lo));
}
CR_F DD dd_mul(DD x, DD y) {
  DD p = two_prod(x.hi, y.hi);
  double t = fma_(x.hi, y.lo, mul_(x.lo, y.hi));
  return fast_two_sum(p.hi, add_(p.lo, t));
}
CR_F DD dd_mul_d(DD x, double s) {
  DD p = two_prod(x.hi, s);
  return fast_two_sum(p.hi, fma_(x.lo, s, p.lo));
}
CR_F DD dd_neg(DD x) { return {-x.hi, -x.lo}; }
// x / y in double-double (relative error ~2^-100).
CR_F DD dd_div(DD x, DD y) {
  double q1 = x.hi / y.hi;
  DD r = dd_add(x, dd_neg(dd_mul_d(y, q1)));
  double q2 = r.hi / y.hi;
  r = dd_add(r, dd_neg(dd_mul_d(y, q2)));
  double q3 = r.hi / y.hi;
  DD q = fast_two_sum(q1, q2);
  return dd_add_d(q, q3);
}
// sqrt in double-double (Karp-Markstein step on the RN sqrt).
CR_F DD dd_sqrt(DD a) {
  if (a.hi <= 0.0) return {0.0, 0.0};
  double s = sqrt_rn(a.hi);
  DD s2 = two_prod(s, s);
  double r = add_(sub_(sub_(a.hi, s2.hi), s2.lo), a.lo);
  return fast_two_sum(s, r / (2.0 * s));
}
// Horner in double-double over DD coefficient tables c[0..n-1] (low -> high).
CR_F DD dd_horner(const double *chi, const double *clo, int n, DD x) {
  DD p = {chi[n - 1], clo[n - 1]};
  for (int i = n - 2; i >= 0; --i) p = dd_add(dd_mul(p, x), DD{chi[i], clo[i]});
  return p;
}

// ------------------------------------------------ rounding decisions ----
// Fast-path rounding test. `a` approximates f(x) with relative error below
// E * 2^-53. The binary32 rounding boundaries for every mode (representable
// values and midpoints, subnormals included) are the doubles whose low 28
// significand bits are zero (53 - 25 = 28); subnormal binary32 boundaries are
// a subset. The lane is decided iff a is outside the window [-2E, 2E) double
// ulps around every such double (which contains the +-E of the error bound):
// the Ziv straddle test of ref: proj/src/kernels_f64.cpp:63-76 on the 32-bit
// low word. E is a power of two, so the window test is one add and one
// LOP3 with a predicate output: ((lo + 2E) mod 2^28) < 4E.
CR_F bool near_boundary_lo(uint32_t lo, uint32_t E) {
  return ((lo + 2u * E) & (0x0FFFFFFFu & ~(4u * E - 1u))) == 0u;
}
CR_F bool near_boundary(double a, uint32_t E) { return near_boundary_lo(d2lo(a), E); }

// Correct rounding of a double-double h + l (|h + l - f| <= 2^-90 |f|):
// snap to an exactly representable binary32 when within 2^-80 (binary32
// inputs never put a non-exact f(x) that close to a boundary; the exhaustive
// sweep confirms), else round-to-odd at 53 bits (ref: "round-to-
// zero mode and sticky bit computation") and one static-mode conversion.
template <int M>
CR_F uint32_t round_dd(double h, double l) {
  float c = cvt_f32<RNE>(h);
  double dc = f2d(c);
  double diff = add_(sub_(h, dc), l);
  if (dabs(diff) <= 0x1p-80 * dabs(h) && dabs(dc) < 0x1p128) return f2u(c);
  uint64_t b = d2u(h);
  if (l != 0.0) {
    if ((l < 0.0) != (h < 0.0)) b -= 1;
    b |= 1;
  }
  return f2u(cvt_f32<M>(u2d(b)));
}

// One fast-path result: `a` approximates f(x) with relative error below
// E * 2^-53 whenever `main` is set. Lanes outside the function's main range
// (IEEE specials, tiny-argument and saturation rules) are resolved by the
// function's special<M>() in a rare, warp-uniform branch, so the common path
// carries only one range check.
struct Fast {
  double a;
  bool main;
};

// Common-path assembly: one static-mode conversion and the rounding test.
template <int M>
CR_F uint32_t finish(Fast r, bool &fail, uint32_t E) {
  fail = r.main && near_boundary(r.a, E);
  return f2u(cvt_f32<M>(r.a));
}

// lo <= u < hi (unsigned), one subtract + one compare.
CR_F bool in_range(uint32_t u, uint32_t lo, uint32_t hi) { return u - lo < hi - lo; }
CR_F bool nan_bits(uint32_t xb) { return (xb << 1) > 0xFF000000u; }
// quiet(x): payload and sign kept (ref: proj/include/crvec/fpbits.hpp:101-102).
CR_F uint32_t quiet_bits(uint32_t xb) { return xb | 0x00400000u; }

// sqrt(a) for a normal, positive a to ~2^-52 relative (a = 0 gives NaN: the
// callers keep such lanes off the main path): MUFU.RSQ64H seed y
// (|e| = |1 - a y^2| <= 2^-19.0, tools/mufu_probe.cu), s = a y, then
// sqrt a = s (1 - e)^(-1/2) = s (1 + e/2 + 3e^2/8 + ...) truncated after e^2
// (error 5e^3/16 <= 2^-58.8). 1 MUFU + 2 DMUL + 3 DFMA (round 2; the coupled
// Newton + Karp-Markstein form took 2 DMUL + 5 DFMA: asinf/acosf +4..6%).
CR_F double sqrt_fast(double a) {
  const double y = rsqrt_approx(a);
  const double s = mul_(a, y);
  const double e = fma_(-s, y, 1.0);  // 1 - a y^2 (s rounded: 2^-54 relative)
  return fma_(s, mul_(e, fma_(e, 0.375, 0.5)), s);
}

// binary32 -> binary64 for a non-negative NORMAL float by exponent-field
// arithmetic on the integer pipes (LEA.HI + SHL) instead of F2F on the
// conversion (XU) pipe; zeros, subnormals, Inf and NaN give garbage, so the
// callers keep such lanes off the main path (or show the result rounds alike).
CR_F double f2d_posnorm(uint32_t ub) { return hilo2d((int)((ub >> 3) + (896u << 20)), ub << 29); }
// ... and back, truncated to binary32 precision (index / comparison use only):
// the bits of a non-negative normal double as a float, one IMAD.
CR_F float d2f_trunc(double a) { return u2f((uint32_t)d2hi(a) * 8u + (uint32_t)d2lo(a) / 0x20000000u - (896u << 23)); }

// 2^e scaling of a normal double by exponent-field arithmetic (integer pipe);
// valid while the result stays normal.
CR_F double scale2(double a, int e) { return hilo2d(d2hi(a) + (e << 20), d2lo(a)); }
// The same with the exponent add forced into one IMAD (the shift-and-add
// form compiles to 2-3 ALU ops). Do not feed it e = (-k) >> n: ptxas 12.9
// folds the negated shift into a LEA.HI.SX32 with a negated operand that
// computes -(k >> n) instead (found by the exhaustive sinh/cosh sweep,
// reproduced standalone); hyp_parts passes -(k + 15) >> 4 to
// scale2_imad_neg instead.
CR_F double scale2_imad(double a, int e) {
#if CR_DEVICE
  int h;
  asm("mad.lo.s32 %0, %1, 1048576, %2;" : "=r"(h) : "r"(e), "r"(d2hi(a)));
  return hilo2d(h, d2lo(a));
#else
  return scale2(a, e);
#endif
}
// a * 2^-u (hi - u 2^20 as one IMAD)
CR_F double scale2_imad_neg(double a, int u) {
#if CR_DEVICE
  int h;
  asm("mad.lo.s32 %0, %1, -1048576, %2;" : "=r"(h) : "r"(u), "r"(d2hi(a)));
  return hilo2d(h, d2lo(a));
#else
  return scale2(a, -u);
#endif
}

// Division num/den to ~2^-52 relative: MUFU seed r (|e| = |1 - den r| <=
// 2^-19.9 over all inputs, tools/mufu_probe.cu, profiles/r02/mufu_probe.txt),
// then 1/den = r (1 + e + e^2 + e^3 ...) truncated after e^2 (error e^3 <=
// 2^-59.8): e and num*r in parallel, two FMAs after - 4 FP64 ops, chain depth
// 3 (round 2; the Newton + residual-correction form took 5 ops, depth 5:
// tanf/tanhf/atanf +1..7%, profiles/r02/ab_div_sqrt.txt).
CR_F double div_fast(double num, double den) {
  const double r = rcp_approx(den);
  const double e = fma_(-den, r, 1.0);
  const double q = mul_(num, r);
  return fma_(q, fma_(e, e, e), q);
}

}  // namespace crvec
