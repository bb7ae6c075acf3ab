// DEVELOPER TOOL ONLY (never shipped, never a fallback): compiles the device
// math of paper_2605_15547_b200/csrc/crvec_fns_f32.cuh with g++ so algorithm
// bugs can be caught on a GPU-less box against the CPU oracle. The GPU
// kernels are the only product path.
#define CRVEC_EMU 1
#include <cstdint>
#include <cstdio>
#include <type_traits>
#include "../../paper_2605_15547_b200/csrc/crvec_fns_f32.cuh"
using namespace crvec;

// the kernels' exponent-indexed Payne-Hanek table (PHBlock: hi at [b], lo at
// [256 + b]); big arguments (|x| >= 2^12) take red_trig_ph as in a warp that
// holds one
static const double *ph_tab() {
  static double t[512];
  for (int i = 0; i < 256; ++i) {
    t[i] = PH_T[2 * i];
    t[256 + i] = PH_T[2 * i + 1];
  }
  return t;
}
static bool trig_big(float x) { return std::fabs(x) >= 0x1p12f; }

template <class F> struct is_trig : std::false_type {};
template <int W> struct is_trig<FnTrig<W>> : std::true_type {};

template <class F, int M>
static uint32_t eval1(float x, int force, uint64_t *slow) {
  typename F::Regs R;
  F::load(R);
  Fast f;
  if constexpr (is_trig<F>::value) {
    RedTrig q = trig_big(x) ? red_trig_ph(x, ph_tab()) : red_trig_small(f2d(x));
    f = F::from_red(x, q, R);
  } else {
    f = F::fast(x, R);
  }
  if (!f.main) return F::template special<M>(x);
  if constexpr (std::is_same<F, FnLog1p>::value) {
    if (!force && F::is_tiny(f2u(x))) return F::template tiny_bits<M>(f2u(x));  // kernels' rule
  }
  bool fail;
  uint32_t y = finish<M>(f, fail, F::E);
  if (fail || force) {
    ++*slow;
    DD v = F::slow(x);
    y = round_dd<M>(v.hi, v.lo);
  }
  return y;
}

template <class F>
static void run(const uint32_t *x, uint32_t *y, uint64_t n, int force, uint64_t *slow) {
  for (uint64_t i = 0; i < n; ++i) {
    float xf = u2f(x[i]);
    y[4 * i + 0] = eval1<F, RNE>(xf, force, slow);
    y[4 * i + 1] = eval1<F, RZ>(xf, force, slow);
    y[4 * i + 2] = eval1<F, RU>(xf, force, slow);
    y[4 * i + 3] = eval1<F, RD>(xf, force, slow);
  }
}

extern "C" int emu_eval(int fn, const uint32_t *x, uint32_t *y, uint64_t n, int force, uint64_t *slow) {
  switch (fn) {
    case 0: run<FnExp2>(x, y, n, force, slow); break;
    case 1: run<FnLog>(x, y, n, force, slow); break;
    case 2: run<FnLog2>(x, y, n, force, slow); break;
    case 3: run<FnExp>(x, y, n, force, slow); break;
    case 4: run<FnExp10>(x, y, n, force, slow); break;
    case 5: run<FnExpm1>(x, y, n, force, slow); break;
    case 6: run<FnLog10>(x, y, n, force, slow); break;
    case 7: run<FnLog1p>(x, y, n, force, slow); break;
    case 8: run<FnSin>(x, y, n, force, slow); break;
    case 9: run<FnCos>(x, y, n, force, slow); break;
    case 10: run<FnTan>(x, y, n, force, slow); break;
    case 11: run<FnAsin>(x, y, n, force, slow); break;
    case 12: run<FnAcos>(x, y, n, force, slow); break;
    case 13: run<FnAtan>(x, y, n, force, slow); break;
    case 14: run<FnSinh>(x, y, n, force, slow); break;
    case 15: run<FnCosh>(x, y, n, force, slow); break;
    case 16: run<FnTanh>(x, y, n, force, slow); break;
    case 17: run<FnRsqrt>(x, y, n, force, slow); break;
    default: return -1;
  }
  return 0;
}

// Max |a - f(x)| of the fast path in units of ulp(a) (f from the accurate DD
// path), over main lanes: the observed margin against the tolerance F::E.
template <class F>
static double probe(const uint32_t *x, uint64_t n, uint32_t *E) {
  double worst = 0;
  *E = F::E;
  for (uint64_t i = 0; i < n; ++i) {
    float xf = u2f(x[i]);
    typename F::Regs R;
    F::load(R);
    Fast f;
    if constexpr (is_trig<F>::value) {
      RedTrig q = trig_big(xf) ? red_trig_ph(xf, ph_tab()) : red_trig_small(f2d(xf));
      f = F::from_red(xf, q, R);
    } else {
      f = F::fast(xf, R);
    }
    if (!f.main || !std::isfinite(f.a) || f.a == 0) continue;
    if constexpr (std::is_same<F, FnLog1p>::value) {
      if (F::is_tiny(x[i])) continue;  // the kernels apply the result-bits rule there
    }
    DD v = F::slow(xf);
    double ulp = std::ldexp(1.0, std::ilogb(f.a) - 52);
    double err = std::fabs((f.a - v.hi) - v.lo) / ulp;
    if (err > worst) worst = err;
  }
  return worst;
}

extern "C" double emu_probe(int fn, const uint32_t *x, uint64_t n, uint32_t *E) {
  switch (fn) {
    case 0: return probe<FnExp2>(x, n, E);
    case 1: return probe<FnLog>(x, n, E);
    case 2: return probe<FnLog2>(x, n, E);
    case 3: return probe<FnExp>(x, n, E);
    case 4: return probe<FnExp10>(x, n, E);
    case 5: return probe<FnExpm1>(x, n, E);
    case 6: return probe<FnLog10>(x, n, E);
    case 7: return probe<FnLog1p>(x, n, E);
    case 8: return probe<FnSin>(x, n, E);
    case 9: return probe<FnCos>(x, n, E);
    case 10: return probe<FnTan>(x, n, E);
    case 11: return probe<FnAsin>(x, n, E);
    case 12: return probe<FnAcos>(x, n, E);
    case 13: return probe<FnAtan>(x, n, E);
    case 14: return probe<FnSinh>(x, n, E);
    case 15: return probe<FnCosh>(x, n, E);
    case 16: return probe<FnTanh>(x, n, E);
    case 17: return probe<FnRsqrt>(x, n, E);
  }
  return -1;
}
