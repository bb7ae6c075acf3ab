// crvec/crvec.hpp — C++ source-compatibility layer over the C ABI (crvec.h).
//
// Re-exposes the reference's public kernel surface so reference-style caller
// code compiles unchanged against the B200 library (C++17 or later):
//
//   RoundingMode, all_rounding_modes, rounding_mode_name
//                                        ref: proj/include/crvec/fpbits.hpp:13-24
//   Binary32 / Binary64, f32_* / f64_* constants, quiet()
//                                        ref: proj/include/crvec/fpbits.hpp:28-102
//   Batch<T, W> (lane, width, W in {1,4,8,16}), LaneMask<W>
//                                        ref: proj/include/crvec/lanes.hpp:21-47
//   DD                                   ref: proj/include/crvec/dd.hpp:11-14
//   Backend                              ref: proj/include/crvec/kernels_f32.hpp:25 (accepted and
//                                        ignored: the sm_100a kernel is the only backend)
//   cr_exp2f<W>, cr_log2f<W>, *_scalar   ref: proj/include/crvec/kernels_f32.hpp:27-35
//   cr_<fn>f<W> for the 17 other binary32 functions (same contract)
//   exp2f_poly, log2f_poly, Exp2fTables, Log2fTables (certifier hooks)
//                                        ref: proj/include/crvec/kernels_f32.hpp:37-40,
//                                        proj/include/crvec/tables.hpp:19-29
//   FuncId                               ref: proj/include/crvec/oracle.hpp:21
//   DDBatch<W>, RoundTestOutcome<W>, RoundTestLane, round_test_lane, round_test<W>
//                                        ref: proj/include/crvec/kernels_f64.hpp:22-56
//   callout(FuncId, double, RoundingMode) ref: proj/include/crvec/kernels_f64.hpp:58-59
//   cr_exp2<W>, cr_log<W>, *_scalar, *_counted, FastPathStats
//                                        ref: proj/include/crvec/kernels_f64.hpp:61-81
//
// plus array overloads (the form a vector application actually wants). Every
// kernel, the round test and the callout run on the GPU through the C ABI;
// errors surface as crvec::Error (the reference kernels have no error path,
// the GPU library can: no device, CUDA failure). The two certifier hooks are
// pure polynomial evaluations over caller-supplied reference-format tables,
// inline exactly as the reference defines them (ref: proj/src/kernels_f32.cpp:
// 25-34,161-168); the reference's certifier runs them offline, and the B200
// kernels do not use the reference's table layout.
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../crvec.h"

namespace crvec {

// ------------------------------------------------------------ fpbits ----
enum class RoundingMode : unsigned {
  NearestEven = 0,
  TowardZero = 1,
  TowardPositive = 2,
  TowardNegative = 3,
};
inline constexpr RoundingMode all_rounding_modes[4] = {
    RoundingMode::NearestEven, RoundingMode::TowardZero, RoundingMode::TowardPositive,
    RoundingMode::TowardNegative};

inline const char *rounding_mode_name(RoundingMode m) noexcept {
  switch (m) {
    case RoundingMode::NearestEven: return "rne";
    case RoundingMode::TowardZero: return "rz";
    case RoundingMode::TowardPositive: return "ru";
    case RoundingMode::TowardNegative: return "rd";
  }
  return "?";
}

namespace detail {
template <class To, class From>
inline To bitcast(From f) noexcept {
  static_assert(sizeof(To) == sizeof(From), "size");
  To t;
  std::memcpy(&t, &f, sizeof(To));
  return t;
}
}  // namespace detail

struct Binary32 {
  std::uint32_t bits = 0;
  Binary32() = default;
  constexpr explicit Binary32(std::uint32_t b) : bits(b) {}
  static Binary32 from_float(float f) noexcept { return Binary32(detail::bitcast<std::uint32_t>(f)); }
  float to_float() const noexcept { return detail::bitcast<float>(bits); }
  constexpr std::uint32_t sign() const noexcept { return bits >> 31; }
  constexpr std::uint32_t biased_exponent() const noexcept { return (bits >> 23) & 0xFFu; }
  constexpr std::uint32_t mantissa_field() const noexcept { return bits & 0x7FFFFFu; }
  constexpr bool is_nan() const noexcept { return biased_exponent() == 0xFF && mantissa_field() != 0; }
  constexpr bool is_inf() const noexcept { return biased_exponent() == 0xFF && mantissa_field() == 0; }
  constexpr bool is_zero() const noexcept { return (bits & 0x7FFFFFFFu) == 0; }
  constexpr bool is_finite() const noexcept { return biased_exponent() != 0xFF; }
  constexpr bool is_subnormal() const noexcept { return biased_exponent() == 0 && mantissa_field() != 0; }
  friend constexpr bool operator==(Binary32 a, Binary32 b) noexcept { return a.bits == b.bits; }
  friend constexpr bool operator!=(Binary32 a, Binary32 b) noexcept { return a.bits != b.bits; }
};

struct Binary64 {
  std::uint64_t bits = 0;
  Binary64() = default;
  constexpr explicit Binary64(std::uint64_t b) : bits(b) {}
  static Binary64 from_double(double d) noexcept { return Binary64(detail::bitcast<std::uint64_t>(d)); }
  double to_double() const noexcept { return detail::bitcast<double>(bits); }
  constexpr std::uint64_t sign() const noexcept { return bits >> 63; }
  constexpr std::uint64_t biased_exponent() const noexcept { return (bits >> 52) & 0x7FFu; }
  constexpr std::uint64_t mantissa_field() const noexcept { return bits & 0xFFFFFFFFFFFFFull; }
  constexpr bool is_nan() const noexcept { return biased_exponent() == 0x7FF && mantissa_field() != 0; }
  constexpr bool is_inf() const noexcept { return biased_exponent() == 0x7FF && mantissa_field() == 0; }
  constexpr bool is_zero() const noexcept { return (bits & 0x7FFFFFFFFFFFFFFFull) == 0; }
  constexpr bool is_finite() const noexcept { return biased_exponent() != 0x7FF; }
  constexpr bool is_subnormal() const noexcept { return biased_exponent() == 0 && mantissa_field() != 0; }
  friend constexpr bool operator==(Binary64 a, Binary64 b) noexcept { return a.bits == b.bits; }
  friend constexpr bool operator!=(Binary64 a, Binary64 b) noexcept { return a.bits != b.bits; }
};

inline constexpr Binary32 f32_pos_inf{0x7F800000u};
inline constexpr Binary32 f32_neg_inf{0xFF800000u};
inline constexpr Binary32 f32_pos_zero{0x00000000u};
inline constexpr Binary32 f32_neg_zero{0x80000000u};
inline constexpr Binary32 f32_qnan{0x7FC00000u};
inline constexpr Binary32 f32_max_finite{0x7F7FFFFFu};
inline constexpr Binary64 f64_pos_inf{0x7FF0000000000000ull};
inline constexpr Binary64 f64_neg_inf{0xFFF0000000000000ull};
inline constexpr Binary64 f64_qnan{0x7FF8000000000000ull};
inline constexpr Binary64 f64_max_finite{0x7FEFFFFFFFFFFFFFull};

constexpr Binary32 quiet(Binary32 x) noexcept { return Binary32(x.bits | 0x00400000u); }
constexpr Binary64 quiet(Binary64 x) noexcept { return Binary64(x.bits | 0x0008000000000000ull); }

// ------------------------------------------------------------- lanes ----
template <typename T, int W>
struct Batch {
  static_assert(W == 1 || W == 4 || W == 8 || W == 16, "Batch width must be 1, 4, 8 or 16");
  std::array<T, W> lane{};

  static constexpr int width = W;
  T &operator[](int i) { return lane[static_cast<std::size_t>(i)]; }
  const T &operator[](int i) const { return lane[static_cast<std::size_t>(i)]; }

  static Batch broadcast(T v) {
    Batch b;
    b.lane.fill(v);
    return b;
  }
};

template <int W>
struct LaneMask {
  std::array<bool, W> bit{};
  bool &operator[](int i) { return bit[static_cast<std::size_t>(i)]; }
  bool operator[](int i) const { return bit[static_cast<std::size_t>(i)]; }
  bool any() const {
    for (bool b : bit)
      if (b) return true;
    return false;
  }
};

// hi + lo with hi == RN(hi + lo), |lo| <= ulp(hi)/2.
struct DD {
  double hi = 0.0;
  double lo = 0.0;
};

enum class Backend { reference, vector };
enum class FuncId { exp2, log, log2 };

// Fast-path accounting (ref: kernels_f64.hpp:72-76), extended with the
// accurate-path tiers of this implementation.
struct FastPathStats {
  std::uint64_t lanes = 0;
  std::uint64_t undecided = 0;
  std::uint64_t accurate_undecided = 0;
  std::uint64_t host_callouts = 0;
};

class Error : public std::runtime_error {
 public:
  explicit Error(int code)
      : std::runtime_error(std::string("crvec: ") + crvec_strerror(code) + " " +
                           crvec_last_cuda_error()),
        code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

namespace detail {
inline void check(int rc) {
  if (rc != CRVEC_OK) throw Error(rc);
}
inline crvec_mode_t mode(RoundingMode m) { return static_cast<crvec_mode_t>(m); }
inline void add(FastPathStats &s, const crvec_stats_t &st) {
  s.lanes += st.lanes;
  s.undecided += st.fast_undecided;
  s.accurate_undecided += st.accurate_undecided;
  s.host_callouts += st.host_callouts;
}
}  // namespace detail

// -------------------------------------------------------- binary32 ----
inline void eval(crvec_fn_t fn, const float *x, float *y, std::size_t n,
                 RoundingMode m = RoundingMode::NearestEven) {
  detail::check(crvec_eval_f32(fn, x, y, nullptr, n, detail::mode(m)));
}

#define CRVEC_CXX_F32(name, id)                                                              \
  template <int W>                                                                         \
  Batch<float, W> cr_##name(const Batch<float, W> &x, RoundingMode m,                      \
                            Backend = Backend::vector) {                                   \
    Batch<float, W> y;                                                                     \
    eval(id, x.lane.data(), y.lane.data(), W, m);                                          \
    return y;                                                                              \
  }                                                                                        \
  inline float cr_##name##_scalar(float x, RoundingMode m) {                               \
    float y;                                                                               \
    eval(id, &x, &y, 1, m);                                                                \
    return y;                                                                              \
  }                                                                                        \
  inline void cr_##name(const float *x, float *y, std::size_t n,                           \
                        RoundingMode m = RoundingMode::NearestEven) {                      \
    eval(id, x, y, n, m);                                                                  \
  }

CRVEC_CXX_F32(exp2f, CRVEC_FN_EXP2F)
CRVEC_CXX_F32(log2f, CRVEC_FN_LOG2F)
CRVEC_CXX_F32(expf, CRVEC_FN_EXPF)
CRVEC_CXX_F32(exp10f, CRVEC_FN_EXP10F)
CRVEC_CXX_F32(expm1f, CRVEC_FN_EXPM1F)
CRVEC_CXX_F32(logf, CRVEC_FN_LOGF)
CRVEC_CXX_F32(log10f, CRVEC_FN_LOG10F)
CRVEC_CXX_F32(log1pf, CRVEC_FN_LOG1PF)
CRVEC_CXX_F32(sinf, CRVEC_FN_SINF)
CRVEC_CXX_F32(cosf, CRVEC_FN_COSF)
CRVEC_CXX_F32(tanf, CRVEC_FN_TANF)
CRVEC_CXX_F32(asinf, CRVEC_FN_ASINF)
CRVEC_CXX_F32(acosf, CRVEC_FN_ACOSF)
CRVEC_CXX_F32(atanf, CRVEC_FN_ATANF)
CRVEC_CXX_F32(sinhf, CRVEC_FN_SINHF)
CRVEC_CXX_F32(coshf, CRVEC_FN_COSHF)
CRVEC_CXX_F32(tanhf, CRVEC_FN_TANHF)
CRVEC_CXX_F32(rsqrtf, CRVEC_FN_RSQRTF)
#undef CRVEC_CXX_F32

inline void cr_sincosf(const float *x, float *s, float *c, std::size_t n,
                       RoundingMode m = RoundingMode::NearestEven) {
  detail::check(crvec_sincosf(x, s, c, n, detail::mode(m)));
}

// Certifier hooks over the reference's table formats (tables.hpp:19-29).
struct Exp2fTables {
  std::array<double, 8> T{};
  std::array<double, 7> c{};
};
struct Log2fTables {
  std::array<std::array<double, 8>, 10> c{};
};
// (2^R - 1)/R: Horner c6 .. c0, each step one fma rounded to nearest.
inline double exp2f_poly(const Exp2fTables &t, double R) {
  double p = t.c[6];
  for (int d = 5; d >= 0; --d) p = std::fma(p, R, t.c[static_cast<std::size_t>(d)]);
  return p;
}
// Sub-interval `interval & 7` of log2f: Horner c9 .. c0 with fma.
inline double log2f_poly(const Log2fTables &t, int interval, double R) {
  const std::size_t j = static_cast<std::size_t>(interval & 7);
  double p = t.c[9][j];
  for (int d = 8; d >= 0; --d) p = std::fma(p, R, t.c[static_cast<std::size_t>(d)][j]);
  return p;
}

// -------------------------------------------------------- binary64 ----
template <int W>
struct DDBatch {
  Batch<double, W> hi, lo;
};

template <int W>
struct RoundTestOutcome {
  Batch<double, W> fast_result;
  LaneMask<W> decided;
  double error_bound = 0.0;
};

struct RoundTestLane {
  Binary64 value;
  bool decided;
};

// One lane of the Ziv straddle test (evaluated on the GPU, crvec_round_test_f64).
inline RoundTestLane round_test_lane(DD v, std::int64_t scale_pow2, double eps_rel, double eps_abs,
                                     RoundingMode mode) {
  double val = 0.0;
  unsigned char dec = 0;
  const std::int64_t sc = scale_pow2;
  detail::check(crvec_round_test_f64(&v.hi, &v.lo, &sc, &eps_rel, &eps_abs, detail::mode(mode), &val,
                                     &dec, 1));
  return {Binary64::from_double(val), dec != 0};
}

// Unscaled batch form (one GPU call for the W lanes).
template <int W>
RoundTestOutcome<W> round_test(const DDBatch<W> &v, double eps, RoundingMode mode) {
  RoundTestOutcome<W> out;
  out.error_bound = eps;
  std::array<unsigned char, W> dec{};
  std::array<double, W> e;
  e.fill(eps);
  detail::check(crvec_round_test_f64(v.hi.lane.data(), v.lo.lane.data(), nullptr, e.data(), nullptr,
                                     detail::mode(mode), out.fast_result.lane.data(), dec.data(), W));
  for (int i = 0; i < W; ++i) out.decided[i] = dec[static_cast<std::size_t>(i)] != 0;
  return out;
}

// Guaranteed-correct fallback for one lane: the GPU accurate path (binary64
// exp2 and log; FuncId::log2 has no binary64 function in the reference's
// SPEC scope and raises CRVEC_EINVAL).
inline double callout(FuncId f, double x, RoundingMode mode) {
  if (f == FuncId::log2) throw Error(CRVEC_EINVAL);
  double y = 0.0;
  detail::check(crvec_callout_f64(f == FuncId::exp2 ? 0 : 1, &x, &y, 1, detail::mode(mode)));
  return y;
}

#define CRVEC_CXX_F64(name)                                                                  \
  template <int W>                                                                         \
  Batch<double, W> cr_##name(const Batch<double, W> &x, RoundingMode m,                    \
                             Backend = Backend::vector) {                                  \
    Batch<double, W> y;                                                                    \
    detail::check(crvec_##name(x.lane.data(), y.lane.data(), W, detail::mode(m), nullptr)); \
    return y;                                                                              \
  }                                                                                        \
  template <int W>                                                                         \
  Batch<double, W> cr_##name##_counted(const Batch<double, W> &x, RoundingMode m,          \
                                       FastPathStats &stats) {                             \
    Batch<double, W> y;                                                                    \
    crvec_stats_t st{};                                                                    \
    detail::check(crvec_##name(x.lane.data(), y.lane.data(), W, detail::mode(m), &st));    \
    detail::add(stats, st);                                                                \
    return y;                                                                              \
  }                                                                                        \
  inline double cr_##name##_scalar(double x, RoundingMode m) {                             \
    double y;                                                                              \
    detail::check(crvec_##name(&x, &y, 1, detail::mode(m), nullptr));                      \
    return y;                                                                              \
  }                                                                                        \
  inline void cr_##name(const double *x, double *y, std::size_t n,                         \
                        RoundingMode m = RoundingMode::NearestEven,                        \
                        FastPathStats *stats = nullptr) {                                  \
    crvec_stats_t st{};                                                                    \
    detail::check(crvec_##name(x, y, n, detail::mode(m), stats ? &st : nullptr));          \
    if (stats) detail::add(*stats, st);                                                    \
  }

CRVEC_CXX_F64(exp2)
CRVEC_CXX_F64(log)
#undef CRVEC_CXX_F64

}  // namespace crvec
