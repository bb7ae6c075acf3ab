/* crvec CPU oracle — TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity checker for the B200 kernels. It may be called only
 * from tests/, from __graft_entry__.smoke() and from bench.py's CPU-baseline /
 * reference arm. The product library (libcrvec.so) never links it, and the
 * product path has no CPU fallback.
 *
 * It is a plain-C restatement of the reference's correctly rounding oracle,
 * /root/reference/proj/src/oracle.cpp (Ziv ladder over MPFR), together with
 * the software rounding engine of /root/reference/proj/src/fpbits.cpp that
 * the oracle feeds, extended from the reference's three functions
 * (FuncId {exp2, log, log2}, ref: proj/include/crvec/oracle.hpp:21) to the 18
 * distinct MPFR functions behind the paper's 19 binary32 CR functions
 * (ref: PAPER.md:49; sincosf = sin + cos).
 *
 * Third-party dependency: MPFR 4.2.1 + GMP 6.3.0 (ref: proj/CMakeLists.txt:26-27),
 * the image's runtime libraries, declared through oracle/mpfr_shim.h.
 *
 * Parity pinning (see tests/test_oracle_*.py):
 *   - every known-answer case of ref: proj/tests/test_oracle.cpp:52-110 and
 *     ref: proj/tests/test_fpbits.cpp:69-93;
 *   - bit equality with the reference oracle itself, compiled from
 *     /root/reference by `make -C oracle ref` into oracle/_ref/ (exp2/log/log2,
 *     f32 and f64 targets) on random and boundary inputs;
 *   - for the 15 extension functions, bit equality with direct MPFR rounding
 *     under an emulated binary32 exponent range (the idiom of
 *     ref: proj/tests/test_oracle.cpp:193-217) on random + boundary samples.
 *
 * One addition to the reference's structure: an optional first Ziv rung at
 * 64 bits evaluated with the host's x87 extended-precision libm (the paper's
 * "quad precision functions" validation idea, ref: PAPER.md:122). Its error is
 * bounded by LD_REL_EPS (2^-51, >= 2^11 times glibc's documented long-double
 * error); it decides a lane only when the whole interval rounds identically,
 * and otherwise falls through to the MPFR ladder unchanged. It is switched
 * off for the reference-equality tests and checked against the MPFR-only
 * ladder on random samples.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "mpfr_shim.h"

#define EXPORT __attribute__((visibility("default")))

/* ---------------------------------------------------------------- ids ---- */
/* The first three ids keep the reference's FuncId order
 * (ref: proj/include/crvec/oracle.hpp:21). */
enum {
  FN_EXP2 = 0, FN_LOG, FN_LOG2, FN_EXP, FN_EXP10, FN_EXPM1, FN_LOG10, FN_LOG1P,
  FN_SIN, FN_COS, FN_TAN, FN_ASIN, FN_ACOS, FN_ATAN, FN_SINH, FN_COSH, FN_TANH,
  FN_RSQRT, FN_COUNT
};

static const char *const fn_names[FN_COUNT] = {
    "exp2", "log", "log2", "exp", "exp10", "expm1", "log10", "log1p", "sin",
    "cos", "tan", "asin", "acos", "atan", "sinh", "cosh", "tanh", "rsqrt"};

EXPORT const char *crvec_oracle_fn_name(int f) {
  return (f >= 0 && f < FN_COUNT) ? fn_names[f] : "?";
}
EXPORT int crvec_oracle_fn_count(void) { return FN_COUNT; }

/* ---------------------------------------------------------- fpbits ------ */
/* RoundingMode numbering of ref: proj/include/crvec/fpbits.hpp:13-18. */
enum { RNE = 0, RZ = 1, RU = 2, RD = 3 };

typedef struct {
  int sign;
  int64_t exponent; /* floor(log2|value|) */
  uint64_t mant;    /* bit 63 set unless zero */
  int sticky;
} SigParts;

typedef struct {
  int sign;
  int64_t exponent;
  uint64_t mantissa;
  int inexact, overflow, is_zero;
} RoundedRaw;

/* ref: proj/src/fpbits.cpp:33-118 (round_sig). */
static RoundedRaw round_sig(const SigParts *p, int mode, int prec, int64_t emin,
                            int64_t emax) {
  RoundedRaw out = {p->sign, 0, 0, 0, 0, 0};
  if (p->mant == 0) {
    out.is_zero = 1;
    out.inexact = p->sticky;
    if (p->sticky) {
      int up = (mode == RU && !p->sign) || (mode == RD && p->sign);
      if (up) {
        out.is_zero = 0;
        out.exponent = emin - (prec - 1);
        out.mantissa = 1;
      }
    }
    return out;
  }
  int64_t e = p->exponent;
  int64_t drop64 = 64 - prec;
  if (e < emin) drop64 += emin - e;
  int drop = drop64 > 65 ? 65 : (int)drop64;
  uint64_t kept, rem_high, rem_rest;
  if (drop >= 65) {
    kept = 0; rem_high = 0; rem_rest = 1;
  } else if (drop == 64) {
    kept = 0; rem_high = p->mant >> 63; rem_rest = (p->mant << 1) != 0;
  } else {
    kept = p->mant >> drop;
    uint64_t rem = drop ? (p->mant << (64 - drop)) : 0;
    rem_high = drop ? (rem >> 63) : 0;
    rem_rest = drop ? ((rem << 1) != 0) : 0;
  }
  int inexact = rem_high || rem_rest || p->sticky;
  int up = 0;
  switch (mode) {
    case RNE: up = rem_high && (rem_rest || p->sticky || (kept & 1)); break;
    case RZ: up = 0; break;
    case RU: up = !p->sign && inexact; break;
    case RD: up = p->sign && inexact; break;
  }
  if (up) {
    kept += 1;
    if (kept >> prec) { kept >>= 1; e += 1; }
  }
  if (e < emin && (kept >> (prec - 1))) e = emin;
  if (kept == 0) { out.is_zero = 1; out.inexact = inexact; return out; }
  if (e > emax) { out.overflow = 1; out.inexact = 1; return out; }
  out.exponent = e;
  out.mantissa = kept;
  out.inexact = inexact;
  return out;
}

/* ref: proj/src/fpbits.cpp:122-141 (round_sig_to_binary32). */
static uint32_t round_sig_to_binary32(const SigParts *p, int mode, int *inexact) {
  RoundedRaw r = round_sig(p, mode, 24, -126, 127);
  uint32_t s = r.sign ? 0x80000000u : 0u;
  if (inexact) *inexact = r.inexact;
  if (r.is_zero) return s;
  if (r.overflow) {
    int to_inf = mode == RNE || (mode == RU && !r.sign) || (mode == RD && r.sign);
    return s | (to_inf ? 0x7F800000u : 0x7F7FFFFFu);
  }
  uint32_t mant = (uint32_t)r.mantissa, be;
  if (mant >> 23) { be = (uint32_t)(r.exponent + 127); mant &= 0x7FFFFFu; }
  else be = 0;
  return s | (be << 23) | mant;
}

/* ref: proj/src/fpbits.cpp:143-162 (round_sig_to_binary64). */
static uint64_t round_sig_to_binary64(const SigParts *p, int mode, int *inexact) {
  RoundedRaw r = round_sig(p, mode, 53, -1022, 1023);
  uint64_t s = r.sign ? 0x8000000000000000ull : 0ull;
  if (inexact) *inexact = r.inexact;
  if (r.is_zero) return s;
  if (r.overflow) {
    int to_inf = mode == RNE || (mode == RU && !r.sign) || (mode == RD && r.sign);
    return s | (to_inf ? 0x7FF0000000000000ull : 0x7FEFFFFFFFFFFFFFull);
  }
  uint64_t mant = r.mantissa, be;
  if (mant >> 52) { be = (uint64_t)(r.exponent + 1023); mant &= 0xFFFFFFFFFFFFFull; }
  else be = 0;
  return s | (be << 52) | mant;
}

static inline uint64_t dbits(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static inline double bitsd(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static inline uint32_t fbits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float bitsf(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* Exact SigParts of a finite binary64 value. */
static SigParts sig_of_double(double d) {
  SigParts p = {0, 0, 0, 0};
  uint64_t b = dbits(d);
  p.sign = (int)(b >> 63);
  uint64_t mant = b & 0xFFFFFFFFFFFFFull;
  int64_t be = (int64_t)((b >> 52) & 0x7FF);
  if (be == 0 && mant == 0) return p;
  if (be == 0) {
    int msb = 63 - __builtin_clzll(mant);
    p.exponent = -1074 + msb;
    p.mant = mant << (63 - msb);
  } else {
    p.exponent = be - 1023;
    p.mant = (mant | 0x10000000000000ull) << 11;
  }
  return p;
}

/* ref: proj/src/fpbits.cpp:164-187 (convert_f64_to_f32). */
static uint32_t convert_f64_to_f32(uint64_t v, int mode) {
  uint32_t s32 = (uint32_t)(v >> 63) << 31;
  uint64_t be = (v >> 52) & 0x7FF, mf = v & 0xFFFFFFFFFFFFFull;
  if (be == 0x7FF && mf) return s32 | 0x7FC00000u | ((uint32_t)(mf >> 29) & 0x3FFFFFu);
  if (be == 0x7FF) return s32 | 0x7F800000u;
  if ((v << 1) == 0) return s32;
  SigParts p = sig_of_double(bitsd(v));
  return round_sig_to_binary32(&p, mode, NULL);
}

EXPORT uint32_t crvec_oracle_convert_f64_to_f32(uint64_t v, int mode) {
  return convert_f64_to_f32(v, mode);
}

/* ------------------------------------------------- SigParts helpers ----- */
/* ref: proj/src/oracle.cpp:147-189. */
static SigParts integer_sig(int64_t n) {
  SigParts p = {0, 0, 0, 0};
  if (n == 0) return p;
  p.sign = n < 0;
  uint64_t mag = p.sign ? 0 - (uint64_t)n : (uint64_t)n;
  int msb = 63 - __builtin_clzll(mag);
  p.exponent = msb;
  p.mant = mag << (63 - msb);
  return p;
}
static SigParts pow2_sig(int64_t n) {
  SigParts p = {0, n, 1ull << 63, 0};
  return p;
}
static SigParts open_interval_above_pow2(int64_t n) {
  SigParts p = pow2_sig(n);
  p.sticky = 1;
  return p;
}
static SigParts open_interval_below_one(void) {
  SigParts p = {0, -1, ~0ull, 1};
  return p;
}
/* Extension helpers: "strictly inside (|d|, |d|(1+2^-63))" (dir=+1) or
 * "strictly inside (|d|(1-2^-63), |d|)" (dir=-1), sign of d. Used for tiny
 * arguments where f(x) provably sits in the rounding gap beside x. */
static SigParts beside(double d, int dir) {
  SigParts p = sig_of_double(d);
  if (dir > 0) {
    p.sticky = 1;
  } else if (p.mant == (1ull << 63)) {
    p.exponent -= 1;
    p.mant = ~0ull;
    p.sticky = 1;
  } else {
    p.mant -= 1;
    p.sticky = 1;
  }
  return p;
}

/* ------------------------------------------------------ shortcuts ------- */
/* ref: proj/src/oracle.cpp:191-277 (Shortcut / shortcut_eval). */
enum { SC_NONE = 0, SC_DIRECT, SC_PARTS };
typedef struct {
  int kind;
  uint64_t direct; /* binary64 bits */
  SigParts parts;
  int value_exact;
} Shortcut;

static const uint64_t F64_PINF = 0x7FF0000000000000ull;
static const uint64_t F64_NINF = 0xFFF0000000000000ull;
static const uint64_t F64_QNAN = 0x7FF8000000000000ull;

static Shortcut sc_direct(uint64_t v) { Shortcut s = {SC_DIRECT, v, {0, 0, 0, 0}, 0}; return s; }
static Shortcut sc_parts(SigParts p, int exact) { Shortcut s = {SC_PARTS, 0, p, exact}; return s; }
static Shortcut sc_none(void) { Shortcut s = {SC_NONE, 0, {0, 0, 0, 0}, 0}; return s; }

static Shortcut sc_below_one(int sign) {
  SigParts p = open_interval_below_one();
  p.sign = sign;
  return sc_parts(p, 0);
}
static Shortcut sc_above(int64_t n, int sign) {
  SigParts p = open_interval_above_pow2(n);
  p.sign = sign;
  return sc_parts(p, 0);
}

/* The reference's exp2 / log / log2 shortcuts, restated verbatim. */
static Shortcut shortcut_ref(int f, double xd, uint64_t xb, int target_f32) {
  if (f == FN_EXP2) {
    if (xd == 0.0) return sc_parts(integer_sig(1), 1);
    if (xb == F64_PINF) return sc_direct(F64_PINF);
    if (xb == F64_NINF) return sc_direct(0);
    if (xd == floor(xd) && fabs(xd) <= 0x1p40) return sc_parts(pow2_sig((int64_t)xd), 1);
    double sat_hi = target_f32 ? 128.0 : 1024.0;
    double sat_lo = target_f32 ? -150.0 : -1075.0;
    if (xd > sat_hi) return sc_parts(open_interval_above_pow2((int64_t)sat_hi), 0);
    if (xd < sat_lo) return sc_parts(open_interval_above_pow2((int64_t)sat_lo - 1), 0);
    double tiny = target_f32 ? 0x1p-26 : 0x1p-55;
    if (fabs(xd) <= tiny)
      return sc_parts(xd > 0.0 ? open_interval_above_pow2(0) : open_interval_below_one(), 0);
    return sc_none();
  }
  /* log / log2 */
  if (xd == 0.0) return sc_direct(F64_NINF);
  if (xb >> 63) return sc_direct(F64_QNAN);
  if (xb == F64_PINF) return sc_direct(F64_PINF);
  if (xd == 1.0) { SigParts z = {0, 0, 0, 0}; return sc_parts(z, 1); }
  if (f == FN_LOG2) {
    int e2;
    if (frexp(xd, &e2) == 0.5) return sc_parts(integer_sig(e2 - 1), 1);
  }
  return sc_none();
}

/* Extension: the same rule classes (IEEE specials, algebraically exact
 * results, saturation, tiny-argument gaps) for the other 15 functions, binary32
 * target only. Conventions follow the reference: NaN in -> quiet(x) (handled by
 * the callers), invalid -> +qNaN 0x7FC00000, IEEE signed zeros. Thresholds are
 * chosen so the claimed interval lies strictly inside one binary32 rounding
 * gap; each is validated against direct MPFR rounding in tests. */
static Shortcut shortcut_ext(int f, double x, uint64_t xb) {
  int sgn = (int)(xb >> 63);
  int isinf = (xb << 1) == (F64_PINF << 1);
  double ax = fabs(x);
  switch (f) {
    case FN_EXP:
    case FN_EXP10: {
      if (x == 0.0) return sc_parts(integer_sig(1), 1);
      if (xb == F64_PINF) return sc_direct(F64_PINF);
      if (xb == F64_NINF) return sc_direct(0);
      double hi = f == FN_EXP ? 88.8 : 38.6, lo = f == FN_EXP ? -104.0 : -45.2;
      if (x > hi) return sc_parts(open_interval_above_pow2(128), 0);
      if (x < lo) return sc_parts(open_interval_above_pow2(-151), 0);
      if (f == FN_EXP10 && x == floor(x) && x >= 1.0 && x <= 10.0) {
        int64_t v = 1;
        for (int i = 0; i < (int)x; ++i) v *= 10;
        return sc_parts(integer_sig(v), 1);
      }
      double tiny = f == FN_EXP ? 0x1p-26 : 0x1p-28;
      if (ax <= tiny)
        return sc_parts(x > 0.0 ? open_interval_above_pow2(0) : open_interval_below_one(), 0);
      return sc_none();
    }
    case FN_EXPM1:
      if (x == 0.0) return sc_direct(xb);
      if (xb == F64_PINF) return sc_direct(F64_PINF);
      if (xb == F64_NINF) return sc_direct(dbits(-1.0));
      if (x > 88.8) return sc_parts(open_interval_above_pow2(128), 0);
      if (x < -18.0) return sc_below_one(1);
      if (ax <= 0x1p-26) return sc_parts(beside(x, x > 0 ? +1 : -1), 0);
      return sc_none();
    case FN_LOG10:
      if (x == 0.0) return sc_direct(F64_NINF);
      if (sgn) return sc_direct(F64_QNAN);
      if (xb == F64_PINF) return sc_direct(F64_PINF);
      {
        double p = 1.0;
        for (int k = 0; k <= 10; ++k, p *= 10.0)
          if (x == p) return sc_parts(integer_sig(k), 1);
      }
      return sc_none();
    case FN_LOG1P:
      if (x == 0.0) return sc_direct(xb);
      if (x == -1.0) return sc_direct(F64_NINF);
      if (x < -1.0) return sc_direct(F64_QNAN);
      if (xb == F64_PINF) return sc_direct(F64_PINF);
      if (ax <= 0x1p-26) return sc_parts(beside(x, x > 0 ? -1 : +1), 0);
      return sc_none();
    case FN_SIN:
    case FN_TAN:
      if (isinf) return sc_direct(F64_QNAN);
      if (x == 0.0) return sc_direct(xb);
      if (ax <= 0x1p-26) return sc_parts(beside(x, f == FN_SIN ? -1 : +1), 0);
      return sc_none();
    case FN_COS:
      if (isinf) return sc_direct(F64_QNAN);
      if (x == 0.0) return sc_parts(integer_sig(1), 1);
      if (ax <= 0x1p-13) return sc_below_one(0);
      return sc_none();
    case FN_ASIN:
      if (ax > 1.0) return sc_direct(F64_QNAN);
      if (x == 0.0) return sc_direct(xb);
      if (ax <= 0x1p-26) return sc_parts(beside(x, +1), 0);
      return sc_none();
    case FN_ACOS:
      if (ax > 1.0) return sc_direct(F64_QNAN);
      if (x == 1.0) { SigParts z = {0, 0, 0, 0}; return sc_parts(z, 1); }
      return sc_none();
    case FN_ATAN:
      if (x == 0.0) return sc_direct(xb);
      if (ax <= 0x1p-26) return sc_parts(beside(x, -1), 0);
      return sc_none();
    case FN_SINH:
      if (x == 0.0) return sc_direct(xb);
      if (isinf) return sc_direct(xb);
      if (ax > 89.5) return sc_above(128, sgn);
      if (ax <= 0x1p-26) return sc_parts(beside(x, +1), 0);
      return sc_none();
    case FN_COSH:
      if (x == 0.0) return sc_parts(integer_sig(1), 1);
      if (isinf) return sc_direct(F64_PINF);
      if (ax > 89.5) return sc_above(128, 0);
      if (ax <= 0x1p-13) return sc_parts(open_interval_above_pow2(0), 0);
      return sc_none();
    case FN_TANH:
      if (x == 0.0) return sc_direct(xb);
      if (isinf) return sc_direct(dbits(sgn ? -1.0 : 1.0));
      if (ax >= 10.0) return sc_below_one(sgn);
      if (ax <= 0x1p-26) return sc_parts(beside(x, -1), 0);
      return sc_none();
    case FN_RSQRT:
      if (xb == 0) return sc_direct(F64_PINF);
      if (xb == 0x8000000000000000ull) return sc_direct(F64_NINF);
      if (sgn) return sc_direct(F64_QNAN);
      if (xb == F64_PINF) return sc_direct(0);
      {
        int e2;
        if (frexp(x, &e2) == 0.5 && ((e2 - 1) & 1) == 0)
          return sc_parts(pow2_sig(-(int64_t)(e2 - 1) / 2), 1);
      }
      return sc_none();
  }
  return sc_none();
}

static Shortcut shortcut_eval(int f, double xd, int target_f32) {
  uint64_t xb = dbits(xd);
  if (f == FN_EXP2 || f == FN_LOG || f == FN_LOG2) return shortcut_ref(f, xd, xb, target_f32);
  return shortcut_ext(f, xd, xb);
}

/* ---------------------------------------------------- MPFR ladder ------- */
/* ref: proj/include/crvec/oracle.hpp:27 */
static const int ziv_ladder[] = {96, 160, 256, 512, 1024, 2048, 4096};
#define ZIV_RUNGS 7

/* Per-thread MPFR scratch (ref: proj/src/oracle.cpp:93-124). */
typedef struct {
  mpfr_t x, v, err, lo, hi, t;
  mpz_t z;
  int init;
} Scratch;

static __thread Scratch tls;

static Scratch *scratch(void) {
  Scratch *s = &tls;
  if (!s->init) {
    mpfr_init2(s->x, 64);
    mpfr_init2(s->v, 160);
    mpfr_init2(s->err, 64);
    mpfr_init2(s->lo, 168);
    mpfr_init2(s->hi, 168);
    mpfr_init2(s->t, 224);
    mpz_init(s->z);
    s->init = 1;
  }
  return s;
}

static void scratch_release(void) {
  Scratch *s = &tls;
  if (s->init) {
    mpfr_clear(s->x); mpfr_clear(s->v); mpfr_clear(s->err);
    mpfr_clear(s->lo); mpfr_clear(s->hi); mpfr_clear(s->t); mpz_clear(s->z);
    mpfr_free_cache();
    s->init = 0;
  }
}

/* ref: proj/src/oracle.cpp:128-145 (sig_parts_from). */
static SigParts sig_parts_from(mpfr_srcptr m, mpz_ptr z) {
  SigParts p = {0, 0, 0, 0};
  p.sign = mpfr_sgn(m) < 0;
  if (mpfr_zero_p(m)) return p;
  mpfr_exp_t e = mpfr_get_z_2exp(z, m);
  mpz_abs(z, z);
  int64_t msb = (int64_t)mpz_sizeinbase(z, 2) - 1;
  p.exponent = (int64_t)e + msb;
  if (msb >= 64) {
    unsigned long shift = (unsigned long)(msb - 63);
    p.sticky = mpz_scan1(z, 0) < shift;
    mpz_fdiv_q_2exp(z, z, shift);
  }
  uint64_t mant = mpz_get_ui(z);
  if (msb < 63) mant <<= (63 - msb);
  p.mant = mant;
  return p;
}

/* ref: proj/src/oracle.cpp:279-285 (eval_into), extended. */
static void eval_into(mpfr_ptr out, int f, mpfr_srcptr x) {
  switch (f) {
    case FN_EXP2: mpfr_exp2(out, x, MPFR_RNDN); break;
    case FN_LOG: mpfr_log(out, x, MPFR_RNDN); break;
    case FN_LOG2: mpfr_log2(out, x, MPFR_RNDN); break;
    case FN_EXP: mpfr_exp(out, x, MPFR_RNDN); break;
    case FN_EXP10: mpfr_exp10(out, x, MPFR_RNDN); break;
    case FN_EXPM1: mpfr_expm1(out, x, MPFR_RNDN); break;
    case FN_LOG10: mpfr_log10(out, x, MPFR_RNDN); break;
    case FN_LOG1P: mpfr_log1p(out, x, MPFR_RNDN); break;
    case FN_SIN: mpfr_sin(out, x, MPFR_RNDN); break;
    case FN_COS: mpfr_cos(out, x, MPFR_RNDN); break;
    case FN_TAN: mpfr_tan(out, x, MPFR_RNDN); break;
    case FN_ASIN: mpfr_asin(out, x, MPFR_RNDN); break;
    case FN_ACOS: mpfr_acos(out, x, MPFR_RNDN); break;
    case FN_ATAN: mpfr_atan(out, x, MPFR_RNDN); break;
    case FN_SINH: mpfr_sinh(out, x, MPFR_RNDN); break;
    case FN_COSH: mpfr_cosh(out, x, MPFR_RNDN); break;
    case FN_TANH: mpfr_tanh(out, x, MPFR_RNDN); break;
    case FN_RSQRT: mpfr_rec_sqrt(out, x, MPFR_RNDN); break;
  }
}

/* ref: proj/src/oracle.cpp:289-298 (enclose). */
static void enclose(Scratch *s, int f, int prec) {
  mpfr_set_prec(s->v, prec);
  eval_into(s->v, f, s->x);
  mpfr_set_prec(s->lo, prec + 8);
  mpfr_set_prec(s->hi, prec + 8);
  mpfr_abs(s->err, s->v, MPFR_RNDU);
  mpfr_mul_2si(s->err, s->err, 1 - prec, MPFR_RNDU);
  mpfr_sub(s->lo, s->v, s->err, MPFR_RNDD);
  mpfr_add(s->hi, s->v, s->err, MPFR_RNDU);
}

/* Error reporting: the reference throws std::runtime_error at the precision
 * cap (ref: proj/src/oracle.cpp:323,387); a C oracle counts the event and
 * remembers the input instead, and every caller surfaces it as a failure. */
static volatile uint64_t g_cap_failures = 0;
static volatile uint64_t g_cap_input = 0;
static volatile uint64_t g_mpfr_calls = 0;
static volatile uint64_t g_ld_decided = 0;

EXPORT uint64_t crvec_oracle_cap_failures(void) { return g_cap_failures; }
EXPORT uint64_t crvec_oracle_cap_input(void) { return g_cap_input; }
EXPORT uint64_t crvec_oracle_mpfr_calls(void) { return g_mpfr_calls; }
EXPORT uint64_t crvec_oracle_ld_decided(void) { return g_ld_decided; }
EXPORT void crvec_oracle_reset_counters(void) {
  g_cap_failures = 0; g_cap_input = 0; g_mpfr_calls = 0; g_ld_decided = 0;
}

static void cap_fail(uint64_t xbits) {
  __atomic_fetch_add(&g_cap_failures, 1, __ATOMIC_RELAXED);
  __atomic_store_n(&g_cap_input, xbits, __ATOMIC_RELAXED);
}

/* ----------------------------------------- 64-bit extended rung (ext) --- */
#define LD_REL_UNITS 4096ull /* 2^12 units of a 64-bit significand = 2^-51 rel */

static long double ld_eval(int f, long double x) {
  switch (f) {
    case FN_EXP2: return exp2l(x);
    case FN_LOG: return logl(x);
    case FN_LOG2: return log2l(x);
    case FN_EXP: return expl(x);
    case FN_EXP10: return exp10l(x);
    case FN_EXPM1: return expm1l(x);
    case FN_LOG10: return log10l(x);
    case FN_LOG1P: return log1pl(x);
    case FN_SIN: return sinl(x);
    case FN_COS: return cosl(x);
    case FN_TAN: return tanl(x);
    case FN_ASIN: return asinl(x);
    case FN_ACOS: return acosl(x);
    case FN_ATAN: return atanl(x);
    case FN_SINH: return sinhl(x);
    case FN_COSH: return coshl(x);
    case FN_TANH: return tanhl(x);
    case FN_RSQRT: return 1.0L / sqrtl(x);
  }
  return 0.0L;
}

/* Try to decide all four binary32 modes from the extended-precision value.
 * Returns a bitmask of decided modes. */
static int ld_rung_f32(int f, double xd, uint32_t out[4]) {
  long double v = ld_eval(f, (long double)xd);
  if (!isfinite(v) || v == 0.0L) return 0;
  int e;
  long double m = frexpl(fabsl(v), &e); /* [0.5, 1) */
  if (m < 0.5L) return 0;               /* denormal long double */
  uint64_t mant = (uint64_t)ldexpl(m, 64);
  if (mant < (1ull << 63) + 2 * LD_REL_UNITS || mant > ~0ull - 2 * LD_REL_UNITS) return 0;
  SigParts lo = {v < 0, e - 1, mant - LD_REL_UNITS, 0};
  SigParts hi = {v < 0, e - 1, mant + LD_REL_UNITS, 0};
  int decided = 0;
  for (int mo = 0; mo < 4; ++mo) {
    uint32_t a = round_sig_to_binary32(&lo, mo, NULL);
    uint32_t b = round_sig_to_binary32(&hi, mo, NULL);
    if (a == b) { out[mo] = a; decided |= 1 << mo; }
  }
  return decided;
}

/* --------------------------------------------------- binary32 API ------- */
/* ref: proj/src/oracle.cpp:302-324 (ziv_correctly_round_f32). Returns the
 * result bits; *prec_out = deciding precision (0 = shortcut). */
EXPORT uint32_t crvec_oracle_f32(int f, uint32_t xbits, int mode, int start_prec,
                                 int *prec_out, int *exact_out) {
  if (prec_out) *prec_out = 0;
  if (exact_out) *exact_out = 0;
  if ((xbits & 0x7F800000u) == 0x7F800000u && (xbits & 0x7FFFFFu)) return xbits | 0x00400000u;
  double wide = (double)bitsf(xbits);
  Shortcut s = shortcut_eval(f, wide, 1);
  if (s.kind == SC_DIRECT) return convert_f64_to_f32(s.direct, mode);
  if (s.kind == SC_PARTS) {
    int inexact;
    uint32_t r = round_sig_to_binary32(&s.parts, mode, &inexact);
    if (exact_out) *exact_out = s.value_exact && !inexact;
    return r;
  }
  Scratch *sc = scratch();
  mpfr_set_d(sc->x, wide, MPFR_RNDN);
  __atomic_fetch_add(&g_mpfr_calls, 1, __ATOMIC_RELAXED);
  for (int i = 0; i < ZIV_RUNGS; ++i) {
    int prec = ziv_ladder[i];
    if (prec < start_prec) continue;
    enclose(sc, f, prec);
    SigParts plo = sig_parts_from(sc->lo, sc->z);
    SigParts phi = sig_parts_from(sc->hi, sc->z);
    uint32_t a = round_sig_to_binary32(&plo, mode, NULL);
    uint32_t b = round_sig_to_binary32(&phi, mode, NULL);
    if (a == b) { if (prec_out) *prec_out = prec; return a; }
  }
  cap_fail(xbits);
  return 0x7FC00000u;
}

/* ref: proj/src/oracle.cpp:347-388 (oracle_all_modes_f32), plus the optional
 * extended rung. out[m] indexed by RoundingMode. Returns 0 on success. */
static int all_modes_f32(int f, uint32_t xbits, uint32_t out[4], int use_ld) {
  if ((xbits & 0x7F800000u) == 0x7F800000u && (xbits & 0x7FFFFFu)) {
    for (int m = 0; m < 4; ++m) out[m] = xbits | 0x00400000u;
    return 0;
  }
  double wide = (double)bitsf(xbits);
  Shortcut s = shortcut_eval(f, wide, 1);
  if (s.kind == SC_DIRECT) {
    for (int m = 0; m < 4; ++m) out[m] = convert_f64_to_f32(s.direct, m);
    return 0;
  }
  if (s.kind == SC_PARTS) {
    for (int m = 0; m < 4; ++m) out[m] = round_sig_to_binary32(&s.parts, m, NULL);
    return 0;
  }
  int undecided = 0xF;
  if (use_ld) {
    undecided &= ~ld_rung_f32(f, wide, out);
    if (!undecided) {
      __atomic_fetch_add(&g_ld_decided, 1, __ATOMIC_RELAXED);
      return 0;
    }
  }
  Scratch *sc = scratch();
  mpfr_set_d(sc->x, wide, MPFR_RNDN);
  __atomic_fetch_add(&g_mpfr_calls, 1, __ATOMIC_RELAXED);
  for (int i = 0; i < ZIV_RUNGS; ++i) {
    enclose(sc, f, ziv_ladder[i]);
    SigParts plo = sig_parts_from(sc->lo, sc->z);
    SigParts phi = sig_parts_from(sc->hi, sc->z);
    for (int m = 0; m < 4; ++m) {
      if (!(undecided & (1 << m))) continue;
      uint32_t a = round_sig_to_binary32(&plo, m, NULL);
      uint32_t b = round_sig_to_binary32(&phi, m, NULL);
      if (a == b) { out[m] = a; undecided &= ~(1 << m); }
    }
    if (!undecided) return 0;
  }
  cap_fail(xbits);
  for (int m = 0; m < 4; ++m) if (undecided & (1 << m)) out[m] = 0x7FC00000u;
  return -1;
}

EXPORT int crvec_oracle_f32_all_modes(int f, uint32_t xbits, uint32_t out[4], int use_ld) {
  if (f < 0 || f >= FN_COUNT) return -2;
  return all_modes_f32(f, xbits, out, use_ld);
}

/* --------------------------------------------------- binary64 API ------- */
/* ref: proj/src/oracle.cpp:326-345 (ziv_correctly_round_f64); reference
 * functions only (exp2, log, log2), as in the reference. */
EXPORT uint64_t crvec_oracle_f64(int f, uint64_t xbits, int mode, int start_prec,
                                 int *prec_out) {
  if (prec_out) *prec_out = 0;
  if (f != FN_EXP2 && f != FN_LOG && f != FN_LOG2) return F64_QNAN;
  double xd = bitsd(xbits);
  if (isnan(xd)) return xbits | 0x0008000000000000ull;
  Shortcut s = shortcut_eval(f, xd, 0);
  if (s.kind == SC_DIRECT) return s.direct;
  if (s.kind == SC_PARTS) return round_sig_to_binary64(&s.parts, mode, NULL);
  Scratch *sc = scratch();
  mpfr_set_d(sc->x, xd, MPFR_RNDN);
  __atomic_fetch_add(&g_mpfr_calls, 1, __ATOMIC_RELAXED);
  for (int i = 0; i < ZIV_RUNGS; ++i) {
    int prec = ziv_ladder[i];
    if (prec < start_prec) continue;
    enclose(sc, f, prec);
    SigParts plo = sig_parts_from(sc->lo, sc->z);
    SigParts phi = sig_parts_from(sc->hi, sc->z);
    uint64_t a = round_sig_to_binary64(&plo, mode, NULL);
    uint64_t b = round_sig_to_binary64(&phi, mode, NULL);
    if (a == b) { if (prec_out) *prec_out = prec; return a; }
  }
  cap_fail(xbits);
  return F64_QNAN;
}

/* ref: proj/src/oracle.cpp:390-429 (oracle_all_modes_f64). */
static int all_modes_f64(int f, uint64_t xbits, uint64_t out[4]) {
  double xd = bitsd(xbits);
  if (isnan(xd)) {
    for (int m = 0; m < 4; ++m) out[m] = xbits | 0x0008000000000000ull;
    return 0;
  }
  Shortcut s = shortcut_eval(f, xd, 0);
  if (s.kind == SC_DIRECT) { for (int m = 0; m < 4; ++m) out[m] = s.direct; return 0; }
  if (s.kind == SC_PARTS) {
    for (int m = 0; m < 4; ++m) out[m] = round_sig_to_binary64(&s.parts, m, NULL);
    return 0;
  }
  Scratch *sc = scratch();
  mpfr_set_d(sc->x, xd, MPFR_RNDN);
  __atomic_fetch_add(&g_mpfr_calls, 1, __ATOMIC_RELAXED);
  int undecided = 0xF;
  for (int i = 0; i < ZIV_RUNGS; ++i) {
    enclose(sc, f, ziv_ladder[i]);
    SigParts plo = sig_parts_from(sc->lo, sc->z);
    SigParts phi = sig_parts_from(sc->hi, sc->z);
    for (int m = 0; m < 4; ++m) {
      if (!(undecided & (1 << m))) continue;
      uint64_t a = round_sig_to_binary64(&plo, m, NULL);
      uint64_t b = round_sig_to_binary64(&phi, m, NULL);
      if (a == b) { out[m] = a; undecided &= ~(1 << m); }
    }
    if (!undecided) return 0;
  }
  cap_fail(xbits);
  return -1;
}

EXPORT int crvec_oracle_f64_all_modes(int f, uint64_t xbits, uint64_t out[4]) {
  if (f != FN_EXP2 && f != FN_LOG && f != FN_LOG2) return -2;
  return all_modes_f64(f, xbits, out);
}



/* ------------------------------------------ boundary distance / search --- */
/* ref: proj/src/oracle.cpp:430-580 (consider_candidate, boundary_distance_f32/
 * f64, hardest_case_search): distance of f(x) (160-bit evaluation) to the
 * nearest rounding boundary (the RN result and the two flanking midpoints), in
 * units of 2^-160; exact results are flagged, specials / saturated inputs are
 * outside the domain. */
static void consider_candidate(Scratch *s, double *best) {
  mpfr_sub(s->t, s->v, s->t, MPFR_RNDN);
  mpfr_abs(s->t, s->t, MPFR_RNDN);
  mpfr_mul_2si(s->t, s->t, 160, MPFR_RNDN);
  double d = mpfr_get_d(s->t, MPFR_RNDU);
  if (d < *best) *best = d;
}

static int64_t ordered32(uint32_t b) {
  int64_t mag = b & 0x7FFFFFFFu;
  return (b >> 31) ? -mag - 1 : mag;
}
static uint32_t from_ordered32(int64_t o) {
  if (o >= 0) return (uint32_t)o;
  return 0x80000000u | (uint32_t)(-(o + 1));
}

EXPORT int crvec_oracle_boundary_distance_f32(int f, uint32_t xb, double *dist, int *exact,
                                              int *domain) {
  *dist = 0.0; *exact = 0; *domain = 1;
  if ((xb & 0x7F800000u) == 0x7F800000u) { *domain = 0; return 0; }
  double xd = (double)bitsf(xb);
  if ((f == FN_LOG || f == FN_LOG2) && xd <= 0.0) { *domain = 0; return 0; }
  Shortcut sc = shortcut_eval(f, xd, 1);
  if (sc.kind == SC_PARTS && sc.value_exact) { *exact = 1; return 0; }
  if (sc.kind != SC_NONE) { *domain = 0; return 0; }
  Scratch *s = scratch();
  mpfr_set_d(s->x, xd, MPFR_RNDN);
  mpfr_set_prec(s->v, 160);
  eval_into(s->v, f, s->x);
  SigParts p = sig_parts_from(s->v, s->z);
  int inexact;
  uint32_t rn = round_sig_to_binary32(&p, RNE, &inexact);
  if (!inexact) { *exact = 1; return 0; }
  double best = INFINITY;
  mpfr_set_prec(s->t, 224);
  mpfr_set_d(s->t, (double)bitsf(rn), MPFR_RNDN);
  consider_candidate(s, &best);
  int64_t o = ordered32(rn);
  for (int dir = -1; dir <= 1; dir += 2) {
    uint32_t nb = from_ordered32(o + dir);
    double nbv = ((nb & 0x7F800000u) == 0x7F800000u) ? (dir > 0 ? 0x1p128 : -0x1p128)
                                                      : (double)bitsf(nb);
    mpfr_set_prec(s->t, 224);
    mpfr_set_d(s->t, (double)bitsf(rn), MPFR_RNDN);
    mpfr_add_d(s->t, s->t, nbv, MPFR_RNDN);
    mpfr_div_2si(s->t, s->t, 1, MPFR_RNDN);
    consider_candidate(s, &best);
  }
  *dist = best;
  return 0;
}

EXPORT int crvec_oracle_boundary_distance_f64(int f, uint64_t xbits, double *dist, int *exact,
                                              int *domain) {
  *dist = 0.0; *exact = 0; *domain = 1;
  if (f != FN_EXP2 && f != FN_LOG && f != FN_LOG2) return -2;
  double xd = bitsd(xbits);
  if (!isfinite(xd)) { *domain = 0; return 0; }
  if (f != FN_EXP2 && xd <= 0.0) { *domain = 0; return 0; }
  Shortcut sc = shortcut_eval(f, xd, 0);
  if (sc.kind == SC_PARTS && sc.value_exact) { *exact = 1; return 0; }
  if (sc.kind != SC_NONE) { *domain = 0; return 0; }
  Scratch *s = scratch();
  mpfr_set_d(s->x, xd, MPFR_RNDN);
  mpfr_set_prec(s->v, 160);
  eval_into(s->v, f, s->x);
  SigParts p = sig_parts_from(s->v, s->z);
  int inexact;
  uint64_t rn = round_sig_to_binary64(&p, RNE, &inexact);
  if (!inexact) { *exact = 1; return 0; }
  double best = INFINITY, rd = bitsd(rn);
  mpfr_set_prec(s->t, 288);
  mpfr_set_d(s->t, rd, MPFR_RNDN);
  consider_candidate(s, &best);
  for (int dir = -1; dir <= 1; dir += 2) {
    uint64_t nb;
    if ((rn << 1) == 0) {
      nb = ((dir > 0) == ((rn >> 63) == 0)) ? 0x1ull : 0x8000000000000001ull;
    } else {
      int away = (dir > 0) == ((rn >> 63) == 0);
      nb = rn + (away ? 1 : (uint64_t)-1);
    }
    mpfr_set_prec(s->t, 288);
    mpfr_set_d(s->t, rd, MPFR_RNDN);
    double nbd = bitsd(nb);
    if (!isfinite(nbd)) {
      mpfr_t big;
      mpfr_init2(big, 64);
      mpfr_set_ui_2exp(big, 1, 1024, MPFR_RNDN);
      if (dir < 0) mpfr_neg(big, big, MPFR_RNDN);
      mpfr_add(s->t, s->t, big, MPFR_RNDN);
      mpfr_clear(big);
    } else {
      mpfr_add_d(s->t, s->t, nbd, MPFR_RNDN);
    }
    mpfr_div_2si(s->t, s->t, 1, MPFR_RNDN);
    consider_candidate(s, &best);
  }
  *dist = best;
  return 0;
}

typedef struct { uint32_t bits; double d; } HardCase;
static int hc_cmp(const void *a, const void *b) {
  const HardCase *x = (const HardCase *)a, *y = (const HardCase *)b;
  if (x->d < y->d) return -1;
  if (x->d > y->d) return 1;
  return x->bits < y->bits ? -1 : (x->bits > y->bits);  /* stable: input order */
}

/* Every non-exact in-domain input in [lo, hi] ranked ascending by boundary
 * distance; writes up to cap entries (cap 0 = all; buffers sized by caller
 * via a first call with out == NULL). Returns the number of candidates. */
EXPORT uint64_t crvec_oracle_hardest_case_search(int f, uint32_t lo, uint32_t hi, uint32_t *out_bits,
                                                 double *out_dist, uint64_t cap) {
  uint64_t n = (uint64_t)hi - lo + 1, k = 0;
  HardCase *v = (HardCase *)malloc(sizeof(HardCase) * n);
  for (uint64_t b = lo; b <= hi; ++b) {
    double d;
    int ex, dom;
    crvec_oracle_boundary_distance_f32(f, (uint32_t)b, &d, &ex, &dom);
    if (!dom || ex) continue;
    v[k].bits = (uint32_t)b;
    v[k].d = d;
    ++k;
  }
  qsort(v, k, sizeof(HardCase), hc_cmp);
  uint64_t m = (cap && cap < k) ? cap : k;
  if (out_bits)
    for (uint64_t i = 0; i < m; ++i) { out_bits[i] = v[i].bits; out_dist[i] = v[i].d; }
  free(v);
  return k;
}

/* ------------------------------------- independent MPFR-direct check ---- */
/* Cross-check for the shortcut extension: f(x) correctly rounded by MPFR
 * straight to 24 bits under an emulated binary32 exponent range, the idiom of
 * ref: proj/tests/test_oracle.cpp:193-217 and test_fpbits.cpp:17-41. IEEE
 * conventions (NaN -> quiet(x), invalid -> +qNaN, rsqrt(-0) = -Inf) applied
 * first, as in Appendix A of SURVEY.md. */
static int direct_f32(int f, uint32_t xbits, uint32_t out[4]) {
  float xf = bitsf(xbits);
  if (isnan(xf)) { for (int m = 0; m < 4; ++m) out[m] = xbits | 0x00400000u; return 0; }
  if (f == FN_RSQRT && xbits == 0x80000000u) { for (int m = 0; m < 4; ++m) out[m] = 0xFF800000u; return 0; }
  if (f == FN_EXPM1 && xbits == 0x80000000u) { for (int m = 0; m < 4; ++m) out[m] = xbits; return 0; }
  if (f == FN_LOG1P && xbits == 0x80000000u) { for (int m = 0; m < 4; ++m) out[m] = xbits; return 0; }
  mpfr_t xm, w;
  mpfr_init2(xm, 64);
  mpfr_init2(w, 24);
  mpfr_set_flt(xm, xf, MPFR_RNDN);
  mpfr_exp_t oemin = mpfr_get_emin(), oemax = mpfr_get_emax();
  static const mpfr_rnd_t rm[4] = {MPFR_RNDN, MPFR_RNDZ, MPFR_RNDU, MPFR_RNDD};
  for (int m = 0; m < 4; ++m) {
    mpfr_set_emin(-148);
    mpfr_set_emax(128);
    int t = 0;
    switch (f) {
      case FN_EXP2: t = mpfr_exp2(w, xm, rm[m]); break;
      case FN_LOG: t = mpfr_log(w, xm, rm[m]); break;
      case FN_LOG2: t = mpfr_log2(w, xm, rm[m]); break;
      case FN_EXP: t = mpfr_exp(w, xm, rm[m]); break;
      case FN_EXP10: t = mpfr_exp10(w, xm, rm[m]); break;
      case FN_EXPM1: t = mpfr_expm1(w, xm, rm[m]); break;
      case FN_LOG10: t = mpfr_log10(w, xm, rm[m]); break;
      case FN_LOG1P: t = mpfr_log1p(w, xm, rm[m]); break;
      case FN_SIN: t = mpfr_sin(w, xm, rm[m]); break;
      case FN_COS: t = mpfr_cos(w, xm, rm[m]); break;
      case FN_TAN: t = mpfr_tan(w, xm, rm[m]); break;
      case FN_ASIN: t = mpfr_asin(w, xm, rm[m]); break;
      case FN_ACOS: t = mpfr_acos(w, xm, rm[m]); break;
      case FN_ATAN: t = mpfr_atan(w, xm, rm[m]); break;
      case FN_SINH: t = mpfr_sinh(w, xm, rm[m]); break;
      case FN_COSH: t = mpfr_cosh(w, xm, rm[m]); break;
      case FN_TANH: t = mpfr_tanh(w, xm, rm[m]); break;
      case FN_RSQRT: t = mpfr_rec_sqrt(w, xm, rm[m]); break;
    }
    t = mpfr_check_range(w, t, rm[m]);
    mpfr_subnormalize(w, t, rm[m]);
    float r = mpfr_get_flt(w, rm[m]);
    mpfr_set_emin(oemin);
    mpfr_set_emax(oemax);
    out[m] = mpfr_nan_p(w) ? 0x7FC00000u : fbits(r);
  }
  mpfr_clear(xm);
  mpfr_clear(w);
  return 0;
}

EXPORT int crvec_oracle_direct_f32_batch(int f, const uint32_t *x, uint32_t *y, uint64_t n) {
  if (f < 0 || f >= FN_COUNT) return -2;
  for (uint64_t i = 0; i < n; ++i) direct_f32(f, x[i], y + 4 * i);
  return 0;
}

/* ----------------------------------------- threaded batch drivers ------- */
typedef struct {
  int kind; /* 0 = f32 batch, 1 = f64 batch, 2 = sweep hashes */
  int f, mode, use_ld;
  const void *x;
  void *y;
  uint64_t n;       /* elements (batch) or chunks (sweep) */
  uint64_t base;    /* first chunk index (sweep) */
  uint64_t grain;
  uint64_t next;    /* atomic work counter */
  int rc;
} Job;

static inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27; z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

#define SWEEP_CHUNK_BITS 20

static void run_range(Job *j, uint64_t b, uint64_t e) {
  if (j->kind == 0) {
    const uint32_t *x = (const uint32_t *)j->x;
    uint32_t *y = (uint32_t *)j->y;
    for (uint64_t i = b; i < e; ++i) {
      uint32_t o[4];
      if (all_modes_f32(j->f, x[i], o, j->use_ld)) j->rc = -1;
      if (j->mode < 0) memcpy(y + 4 * i, o, 16);
      else y[i] = o[j->mode];
    }
  } else if (j->kind == 1) {
    const uint64_t *x = (const uint64_t *)j->x;
    uint64_t *y = (uint64_t *)j->y;
    for (uint64_t i = b; i < e; ++i) {
      uint64_t o[4];
      if (all_modes_f64(j->f, x[i], o)) j->rc = -1;
      if (j->mode < 0) memcpy(y + 4 * i, o, 32);
      else y[i] = o[j->mode];
    }
  } else {
    uint64_t *h = (uint64_t *)j->y; /* [chunk][mode] */
    for (uint64_t c = b; c < e; ++c) {
      uint64_t chunk = j->base + c;
      uint64_t acc[4] = {0, 0, 0, 0};
      uint64_t p0 = chunk << SWEEP_CHUNK_BITS;
      for (uint64_t p = p0; p < p0 + (1ull << SWEEP_CHUNK_BITS); ++p) {
        uint32_t o[4];
        if (all_modes_f32(j->f, (uint32_t)p, o, j->use_ld)) j->rc = -1;
        for (int m = 0; m < 4; ++m) acc[m] += mix64(((uint64_t)o[m] << 32) | p);
      }
      memcpy(h + 4 * c, acc, 32);
    }
  }
}

static void *worker(void *arg) {
  Job *j = (Job *)arg;
  for (;;) {
    uint64_t b = __atomic_fetch_add(&j->next, j->grain, __ATOMIC_RELAXED);
    if (b >= j->n) break;
    uint64_t e = b + j->grain < j->n ? b + j->grain : j->n;
    run_range(j, b, e);
  }
  scratch_release();
  return NULL;
}

static int run_job(Job *j, int threads) {
  if (threads <= 0) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    threads = c > 0 ? (int)c : 1;
  }
  if ((uint64_t)threads > j->n) threads = j->n ? (int)j->n : 1;
  j->next = 0;
  j->rc = 0;
  if (threads == 1) {
    worker(j);
    return j->rc;
  }
  pthread_t *t = (pthread_t *)malloc(sizeof(pthread_t) * threads);
  for (int i = 0; i < threads; ++i) pthread_create(&t[i], NULL, worker, j);
  for (int i = 0; i < threads; ++i) pthread_join(t[i], NULL);
  free(t);
  return j->rc;
}

/* y gets n results for mode in 0..3, or 4n results ([i][mode]) for mode < 0. */
EXPORT int crvec_oracle_f32_batch(int f, const uint32_t *x, uint32_t *y, uint64_t n,
                                  int mode, int threads, int use_ld) {
  if (f < 0 || f >= FN_COUNT || mode > 3) return -2;
  Job j = {0, f, mode, use_ld, x, y, n, 0, 256, 0, 0};
  return run_job(&j, threads);
}

EXPORT int crvec_oracle_f64_batch(int f, const uint64_t *x, uint64_t *y, uint64_t n,
                                  int mode, int threads) {
  if ((f != FN_EXP2 && f != FN_LOG && f != FN_LOG2) || mode > 3) return -2;
  Job j = {1, f, mode, 0, x, y, n, 0, 64, 0, 0};
  return run_job(&j, threads);
}

/* Exhaustive-sweep golden: for chunks [chunk_lo, chunk_hi) of 2^20 binary32
 * patterns, h[(c - chunk_lo)*4 + mode] = sum over p in chunk of
 * mix64((out_bits << 32) | p) mod 2^64 (commutative, order-free; the chunking
 * rule of ref: SPEC.md:289-290). */
EXPORT int crvec_oracle_sweep_hashes(int f, uint32_t chunk_lo, uint32_t chunk_hi,
                                     uint64_t *h, int threads, int use_ld) {
  if (f < 0 || f >= FN_COUNT || chunk_hi > 4096 || chunk_lo >= chunk_hi) return -2;
  Job j = {2, f, -1, use_ld, NULL, h, chunk_hi - chunk_lo, chunk_lo, 1, 0, 0};
  return run_job(&j, threads);
}

EXPORT uint64_t crvec_oracle_mix64(uint64_t z) { return mix64(z); }
