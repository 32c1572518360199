// doctest.h -- minimal stand-in for the doctest subset the reference's unit
// tests use (TEST_CASE, SUBCASE, CHECK, REQUIRE, CHECK_THROWS_AS, FAIL,
// doctest::Approx), so those test sources compile unchanged against the
// drop-in header (bitkv_b200.hpp).  The reference tree ships no doctest
// (vendor/ is absent).  SUBCASEs run in sequence inside one pass.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {
struct TestCase {
  const char* name;
  void (*fn)();
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Register {
  Register(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double x, const Approx& a) {
    const double scale = std::max(std::fabs(x), std::fabs(a.v_));
    return std::fabs(x - a.v_) <= a.eps_ * (scale + 1.0);  // doctest's relative epsilon
  }
  friend bool operator==(const Approx& a, double x) { return x == a; }
  friend bool operator!=(double x, const Approx& a) { return !(x == a); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-05;  // doctest default: FLT_EPSILON * 100
};

inline void report(const char* file, int line, const char* what) {
  ++failures();
  std::printf("%s:%d: FAILED: %s\n", file, line, what);
}
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                        \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                            \
  static doctest::Register DOCTEST_CAT(doctest_reg_, __LINE__)(                \
      name, &DOCTEST_CAT(doctest_fn_, __LINE__));                              \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define SUBCASE(name) if (true)
#define CHECK(...)                                                             \
  do {                                                                         \
    if (!(__VA_ARGS__)) doctest::report(__FILE__, __LINE__, #__VA_ARGS__);     \
  } while (0)
#define REQUIRE(...)                                                           \
  do {                                                                         \
    if (!(__VA_ARGS__)) {                                                      \
      doctest::report(__FILE__, __LINE__, #__VA_ARGS__);                       \
      throw doctest::RequireFailed{};                                          \
    }                                                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                            \
  do {                                                                         \
    bool caught_ = false;                                                      \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const type&) {                                                    \
      caught_ = true;                                                          \
    } catch (...) {                                                            \
    }                                                                          \
    if (!caught_) doctest::report(__FILE__, __LINE__, "throws " #type ": " #expr); \
  } while (0)
#define FAIL(msg)                                                              \
  do {                                                                         \
    doctest::report(__FILE__, __LINE__, msg);                                  \
    throw doctest::RequireFailed{};                                            \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int cases_failed = 0;
  for (const auto& tc : doctest::registry()) {
    const int before = doctest::failures();
    try {
      tc.fn();
    } catch (const doctest::RequireFailed&) {
    } catch (const std::exception& e) {
      doctest::report("<exception>", 0, e.what());
    }
    const bool ok = doctest::failures() == before;
    cases_failed += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
  }
  std::printf("test cases: %zu | passed: %zu | failed: %d | failed checks: %d\n",
              doctest::registry().size(), doctest::registry().size() - cases_failed, cases_failed,
              doctest::failures());
  return cases_failed ? 1 : 0;
}
#endif
