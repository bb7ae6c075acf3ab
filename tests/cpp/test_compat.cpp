// Reference-style C++ caller of the B200 library through include/crvec/crvec.hpp.
// Mirrors SPEC examples for cr_exp2f / cr_log2f / cr_exp2 / cr_log
// (ref: SPEC.md kernels_f32 / kernels_f64 examples). Exit code 0 = pass,
// 77 = no usable device (the library reported CRVEC_ENODEV: no CPU fallback).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>

#include "crvec/crvec.hpp"

using namespace crvec;

static int fails = 0;
#define CHECK(c) do { if (!(c)) { std::printf("FAILED %s:%d %s\n", __FILE__, __LINE__, #c); ++fails; } } while (0)

static uint32_t bits(float f) { uint32_t u; std::memcpy(&u, &f, 4); return u; }

int main() {
  try {
    for (auto m : all_rounding_modes) {
      CHECK(cr_exp2f_scalar(0.0f, m) == 1.0f);
      CHECK(cr_exp2f_scalar(127.0f, m) == 0x1p127f);
      CHECK(cr_log2f_scalar(1.0f, m) == 0.0f);
      CHECK(cr_log2f_scalar(8.0f, m) == 3.0f);
      CHECK(cr_exp2_scalar(10.0, m) == 1024.0);
      CHECK(cr_log_scalar(1.0, m) == 0.0 && !std::signbit(cr_log_scalar(1.0, m)));
    }
    CHECK(cr_exp2f_scalar(128.0f, RoundingMode::TowardZero) == std::numeric_limits<float>::max());
    CHECK(std::isinf(cr_exp2f_scalar(128.0f, RoundingMode::NearestEven)));
    CHECK(bits(cr_log2f_scalar(-1.0f, RoundingMode::NearestEven)) == 0x7FC00000u);
    Batch<float, 16> x = Batch<float, 16>::broadcast(0.5f);
    for (int i = 0; i < 16; ++i) x[i] = static_cast<float>(i) - 4.0f;
    auto y = cr_exp2f<16>(x, RoundingMode::NearestEven);
    for (int i = 0; i < 16; ++i) CHECK(y[i] == std::ldexp(1.0f, i - 4));
    Batch<double, 8> xd = Batch<double, 8>::broadcast(2.0);
    FastPathStats st;
    auto yd = cr_log_counted<8>(xd, RoundingMode::NearestEven, st);
    CHECK(yd[3] == 0x1.62e42fefa39efp-1);  // RN(ln 2)
    CHECK(st.lanes == 8);
  } catch (const Error &e) {
    if (e.code() == CRVEC_ENODEV) {
      std::printf("no device: %s\n", e.what());
      return 77;
    }
    std::printf("error: %s\n", e.what());
    return 1;
  }
  std::printf("%s (%d failures)\n", fails ? "FAIL" : "PASS", fails);
  return fails ? 1 : 0;
}
