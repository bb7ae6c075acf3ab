/* TEST INFRASTRUCTURE ONLY: a minimal stand-in for doctest (absent from the
 * reference tree, ref: proj/CMakeLists.txt:5) covering exactly the macros the
 * reference's unit tests use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS, CAPTURE. */
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <vector>
namespace mini_doctest {
struct Abort {};
struct Reg { const char* name; void (*fn)(); };
inline std::vector<Reg>& regs() { static std::vector<Reg> r; return r; }
inline long& checks() { static long c = 0; return c; }
inline long& fails() { static long f = 0; return f; }
struct Adder { Adder(const char* n, void (*f)()) { regs().push_back({n, f}); } };
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++checks();
  if (!ok) {
    ++fails();
    if (fails() < 50) std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
    if (fatal) throw Abort{};
  }
}
}  // namespace mini_doctest
#define MDT_CAT2(a, b) a##b
#define MDT_CAT(a, b) MDT_CAT2(a, b)
#define TEST_CASE(name)                                                     \
  static void MDT_CAT(mdt_fn_, __LINE__)();                                 \
  static mini_doctest::Adder MDT_CAT(mdt_add_, __LINE__)(name, &MDT_CAT(mdt_fn_, __LINE__)); \
  static void MDT_CAT(mdt_fn_, __LINE__)()
#define CHECK(e) mini_doctest::report(static_cast<bool>(e), #e, __FILE__, __LINE__, false)
#define REQUIRE(e) mini_doctest::report(static_cast<bool>(e), #e, __FILE__, __LINE__, true)
#define CHECK_THROWS(e)                                                     \
  do { bool t_ = false; try { (void)(e); } catch (...) { t_ = true; }        \
       mini_doctest::report(t_, "THROWS " #e, __FILE__, __LINE__, false); } while (0)
#define CAPTURE(x) (void)(x)
#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  for (auto& r : mini_doctest::regs()) {
    try { r.fn(); } catch (mini_doctest::Abort&) {
    } catch (std::exception& e) { ++mini_doctest::fails(); std::fprintf(stderr, "%s: exception %s\n", r.name, e.what()); }
  }
  std::printf("test cases: %zu | checks: %ld | failed: %ld\n", mini_doctest::regs().size(),
              mini_doctest::checks(), mini_doctest::fails());
  return mini_doctest::fails() ? 1 : 0;
}
#endif
