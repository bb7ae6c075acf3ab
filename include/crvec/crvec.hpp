// crvec/crvec.hpp — C++ source-compatibility layer over the C ABI (crvec.h).
//
// Re-exposes the reference's public kernel signatures so reference-style
// caller code compiles unchanged against the B200 library:
//
//   RoundingMode, all_rounding_modes     ref: proj/include/crvec/fpbits.hpp:13-22
//   Batch<T, W>                          ref: proj/include/crvec/lanes.hpp:21-35
//   Backend                              ref: proj/include/crvec/kernels_f32.hpp:25 (ignored:
//                                        the sm_100a kernel is the only backend)
//   cr_exp2f<W>, cr_log2f<W>, *_scalar   ref: proj/include/crvec/kernels_f32.hpp:27-35
//   cr_<fn>f<W> for the 17 other binary32 functions (same contract)
//   cr_exp2<W>, cr_log<W>, *_scalar, *_counted, FastPathStats
//                                        ref: proj/include/crvec/kernels_f64.hpp:58-81
//
// plus array overloads (the form a vector application actually wants). Every
// call goes through the GPU; errors surface as crvec::Error (the reference
// kernels have no error path, the GPU library can: no device, CUDA failure).
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../crvec.h"

namespace crvec {

enum class RoundingMode : unsigned {
  NearestEven = 0,
  TowardZero = 1,
  TowardPositive = 2,
  TowardNegative = 3,
};
inline constexpr RoundingMode all_rounding_modes[4] = {
    RoundingMode::NearestEven, RoundingMode::TowardZero, RoundingMode::TowardPositive,
    RoundingMode::TowardNegative};

enum class Backend { reference, vector };

template <class T, int W>
struct Batch {
  std::array<T, W> v{};
  T &operator[](int i) { return v[static_cast<std::size_t>(i)]; }
  const T &operator[](int i) const { return v[static_cast<std::size_t>(i)]; }
  static Batch broadcast(T x) {
    Batch b;
    b.v.fill(x);
    return b;
  }
};

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
}  // namespace detail

// ---- arrays (host pointers) ----
inline void eval(crvec_fn_t fn, const float *x, float *y, std::size_t n,
                 RoundingMode m = RoundingMode::NearestEven) {
  detail::check(crvec_eval_f32(fn, x, y, nullptr, n, detail::mode(m)));
}

#define CRVEC_CXX_F32(name, id)                                                              \
  template <int W>                                                                         \
  Batch<float, W> cr_##name(const Batch<float, W> &x, RoundingMode m,                      \
                            Backend = Backend::vector) {                                   \
    Batch<float, W> y;                                                                     \
    eval(id, x.v.data(), y.v.data(), W, m);                                                \
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

// ---- binary64 ----
#define CRVEC_CXX_F64(name)                                                                  \
  template <int W>                                                                         \
  Batch<double, W> cr_##name(const Batch<double, W> &x, RoundingMode m,                    \
                             Backend = Backend::vector) {                                  \
    Batch<double, W> y;                                                                    \
    detail::check(crvec_##name(x.v.data(), y.v.data(), W, detail::mode(m), nullptr));      \
    return y;                                                                              \
  }                                                                                        \
  template <int W>                                                                         \
  Batch<double, W> cr_##name##_counted(const Batch<double, W> &x, RoundingMode m,          \
                                       FastPathStats &stats) {                             \
    Batch<double, W> y;                                                                    \
    crvec_stats_t st{};                                                                    \
    detail::check(crvec_##name(x.v.data(), y.v.data(), W, detail::mode(m), &st));          \
    stats.lanes += st.lanes;                                                               \
    stats.undecided += st.fast_undecided;                                                  \
    stats.accurate_undecided += st.accurate_undecided;                                     \
    stats.host_callouts += st.host_callouts;                                               \
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
    if (stats) {                                                                           \
      stats->lanes += st.lanes;                                                            \
      stats->undecided += st.fast_undecided;                                               \
      stats->accurate_undecided += st.accurate_undecided;                                  \
    }                                                                                      \
  }

CRVEC_CXX_F64(exp2)
CRVEC_CXX_F64(log)
#undef CRVEC_CXX_F64

}  // namespace crvec
