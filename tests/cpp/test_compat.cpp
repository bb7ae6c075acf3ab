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

    // reference-style lane access (ref: proj/tests/test_lanes.cpp:231-248)
    static_assert(Batch<float, 4>::width == 4, "width");
    static_assert(Batch<double, 16>::width == 16, "width");
    Batch<float, 4> b;
    b.lane = {0.5f, 1.0f, 2.0f, -3.0f};
    auto lb = cr_log2f<4>(b, RoundingMode::TowardZero, Backend::reference);
    CHECK(lb.lane[0] == -1.0f && lb.lane[1] == 0.0f && lb.lane[2] == 1.0f);
    CHECK(Binary32::from_float(lb.lane[3]) == f32_qnan);
    CHECK(quiet(Binary32(0xFF812345u)).bits == 0xFFC12345u);
    LaneMask<4> mk;
    CHECK(!mk.any());
    mk[2] = true;
    CHECK(mk.any() && mk[2] && !mk[0]);
    Batch<double, 4> b64;
    b64.lane = {1.0, -1075.0, 1024.0, 0.5};
    auto e64 = cr_exp2<4>(b64, RoundingMode::TowardPositive);
    CHECK(e64.lane[0] == 2.0 && e64.lane[1] == 0x1p-1074 && std::isinf(e64.lane[2]));
    CHECK(e64.lane[3] == 0x1.6a09e667f3bcdp+0);  // RU(sqrt 2)

    // round test (the reference's semantics): the low end of the enclosure is
    // the reported value; an exactly representable value with a positive
    // bound is decided in RNE only (the directed modes see it straddled)
    {
      RoundTestLane r = round_test_lane(DD{1.5, 0.0}, 3, 0x1p-70, 0.0, RoundingMode::NearestEven);
      CHECK(r.value.to_double() == 12.0 && r.decided);
      r = round_test_lane(DD{1.5, 0.0}, 3, 0x1p-70, 0.0, RoundingMode::TowardZero);
      CHECK(r.value.to_double() == std::nextafter(12.0, 0.0) && !r.decided);
      r = round_test_lane(DD{1.5, 0x1p-60}, 3, 0x1p-70, 0.0, RoundingMode::TowardPositive);
      CHECK(r.value.to_double() == std::nextafter(12.0, 13.0) && r.decided);
    }
    RoundTestLane tie = round_test_lane(DD{1.0, 0x1p-53}, 0, 0x1p-70, 0.0, RoundingMode::NearestEven);
    CHECK(!tie.decided);
    RoundTestLane sub = round_test_lane(DD{1.0, 0x1p-60}, -1074, 0.0, 0.0, RoundingMode::TowardPositive);
    CHECK(sub.value.to_double() == 0x1p-1073 && sub.decided);  // 2^-1074 (1 + 2^-60) rounds up
    DDBatch<4> v;
    v.hi.lane = {1.0, 2.0, 3.0, 1.0};
    v.lo.lane = {0.0, 0x1p-60, -0x1p-60, 0x1p-53};
    auto rt = round_test<4>(v, 0x1p-80, RoundingMode::TowardZero);
    // lane 3: 1 + 2^-53 +- 2^-80 rounds to 1.0 toward zero at both ends (decided;
    // the reference's round_test_lane agrees, oracle/_ref crvec_refk_round_test_lane)
    CHECK(!rt.decided[0] && rt.decided[1] && rt.decided[2] && rt.decided[3]);
    CHECK(rt.fast_result[1] == 2.0 && rt.fast_result[2] == std::nextafter(3.0, 0.0));
    CHECK(rt.fast_result[3] == 1.0);
    CHECK(rt.error_bound == 0x1p-80);

    // callout: the GPU accurate path
    CHECK(callout(FuncId::exp2, 0.5, RoundingMode::NearestEven) == 0x1.6a09e667f3bcdp+0);
    CHECK(callout(FuncId::log, 2.0, RoundingMode::NearestEven) == 0x1.62e42fefa39efp-1);
    bool threw = false;
    try { callout(FuncId::log2, 2.0, RoundingMode::NearestEven); } catch (const Error &e) { threw = e.code() == CRVEC_EINVAL; }
    CHECK(threw);

    // certifier hooks over reference-format tables
    Exp2fTables et;
    et.c = {1.0, 0.5, 0.25, 0.0, 0.0, 0.0, 0.0};
    CHECK(exp2f_poly(et, 2.0) == 1.0 + 2.0 * (0.5 + 2.0 * 0.25));
    Log2fTables lt;
    lt.c[0][5] = 3.0;
    lt.c[1][5] = 1.0;
    CHECK(log2f_poly(lt, 13, 0.5) == 3.5);  // interval & 7 == 5

    // array overloads (host pointers), stats carry all fields
    float xa[37], ya[37];
    for (int i = 0; i < 37; ++i) xa[i] = static_cast<float>(i);
    cr_exp2f(xa, ya, 37, RoundingMode::NearestEven);
    for (int i = 0; i < 37; ++i) CHECK(ya[i] == std::ldexp(1.0f, i));
    double xl[5] = {1.0, 2.0, 4.0, 0.5, 8.0}, yl[5];
    FastPathStats s2;
    cr_log(xl, yl, 5, RoundingMode::NearestEven, &s2);
    CHECK(s2.lanes == 5 && yl[0] == 0.0 && yl[1] == 0x1.62e42fefa39efp-1);
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
