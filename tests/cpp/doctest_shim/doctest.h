// doctest.h -- a minimal stand-in for the doctest framework (absent from the image), covering
// what the reference's unit suites use: TEST_SUITE, TEST_CASE, SUBCASE (one level), CHECK, REQUIRE,
// CHECK_THROWS_AS, doctest::Approx. Test infrastructure: lets tests/cpp/Makefile build the
// reference's own unit suites (/root/reference/proj/tests/test_*.cpp, unmodified) against the
// B200 C++ drop-in. A case runs once per SUBCASE leaf (plus once when it has none), like doctest.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) { eps = e; return *this; }
  Approx& scale(double s) { scl = s; return *this; }
  double value, eps = 1.19209290e-07 * 100, scl = 1.0;
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.value) < b.eps * (b.scl + std::max(std::fabs(a), std::fabs(b.value)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.value || a == b; }
  friend bool operator>=(double a, const Approx& b) { return a > b.value || a == b; }
  friend bool operator<(double a, const Approx& b) { return a < b.value && !(a == b); }
  friend bool operator>(double a, const Approx& b) { return a > b.value && !(a == b); }
};

namespace detail {
struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct RequireFailed {};
struct State {
  int failures = 0, checks = 0;
  int sub_target = -1;  // leaf SUBCASE to enter this run (-1: discovery run)
  int sub_seen = 0, sub_entered = 0;
  bool case_failed = false;
};
inline State& st() {
  static State s;
  return s;
}
inline void fail(const char* file, int line, const std::string& what) {
  st().failures += 1;
  st().case_failed = true;
  std::cout << "  " << file << ":" << line << ": FAILED: " << what << "\n";
}
struct Subcase {
  bool on;
  explicit Subcase(const char*) {
    State& s = st();
    const int idx = s.sub_seen++;
    on = s.sub_target < 0 ? (s.sub_entered == 0) : (idx == s.sub_target);
    if (on) s.sub_entered += 1;
  }
  explicit operator bool() const { return on; }
};
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                         \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                          \
  static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,     \
                                                                  &DOCTEST_CAT(doctest_case_, __LINE__)); \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define TEST_SUITE(name) namespace
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name})
#define DOCTEST_CHECK_IMPL(expr, fatal)                                                          \
  do {                                                                                            \
    doctest::detail::st().checks += 1;                                                           \
    bool doctest_ok_ = false;                                                                    \
    try {                                                                                         \
      doctest_ok_ = static_cast<bool>(expr);                                                     \
    } catch (const std::exception& e) {                                                         \
      doctest::detail::fail(__FILE__, __LINE__, std::string(#expr) + " threw " + e.what());     \
      if (fatal) throw doctest::detail::RequireFailed{};                                        \
      break;                                                                                      \
    }                                                                                             \
    if (!doctest_ok_) {                                                                          \
      doctest::detail::fail(__FILE__, __LINE__, #expr);                                         \
      if (fatal) throw doctest::detail::RequireFailed{};                                        \
    }                                                                                             \
  } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), false)
#define CHECK_THROWS_AS(expr, type)                                                              \
  do {                                                                                            \
    doctest::detail::st().checks += 1;                                                           \
    bool doctest_thrown_ = false;                                                                \
    try {                                                                                         \
      (void)(expr);                                                                              \
    } catch (const type&) {                                                                      \
      doctest_thrown_ = true;                                                                    \
    } catch (const std::exception& e) {                                                         \
      doctest::detail::fail(__FILE__, __LINE__, std::string(#expr) + " threw another type: " + e.what()); \
      doctest_thrown_ = true;                                                                    \
    }                                                                                             \
    if (!doctest_thrown_) doctest::detail::fail(__FILE__, __LINE__, std::string(#expr) + " did not throw " #type); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::detail;
  const std::string filter = argc > 1 ? argv[1] : "";
  int cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    if (!filter.empty() && std::string(c.name).find(filter) == std::string::npos) continue;
    cases += 1;
    State& s = st();
    s.case_failed = false;
    // discovery run enters the first SUBCASE (if any); then one run per further leaf
    s.sub_target = -1;
    s.sub_seen = s.sub_entered = 0;
    auto run = [&]() {
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
      }
    };
    run();
    const int leaves = s.sub_seen;
    for (int k = 1; k < leaves; ++k) {
      s.sub_target = k;
      s.sub_seen = s.sub_entered = 0;
      run();
    }
    std::cout << (s.case_failed ? "[FAIL] " : "[PASS] ") << c.name << "  (" << c.file << ":" << c.line << ")\n";
    if (s.case_failed) failed_cases += 1;
  }
  std::cout << "cases: " << cases << " failed: " << failed_cases << " checks: " << st().checks
            << " failed checks: " << st().failures << "\n";
  return failed_cases == 0 ? 0 : 1;
}
#endif
