// TEST INFRASTRUCTURE ONLY (oracle/): a tiny stand-in for the doctest API the
// reference unit tests use (/root/reference/proj/tests/test_*.cpp):
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS and
// doctest::Approx(...).epsilon(). doctest is not vendored in the reference
// (proj/.gitignore:2) and not installed here. Used only to
// prove that the in-place build of the reference under oracle/_ref is
// faithful; never part of the product.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  // doctest semantics: |lhs - v| < eps * (scale + max(|lhs|, |v|)).
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) <
           a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Stats {
  long long checks = 0;
  long long failed_checks = 0;
  bool current_failed = false;
};

inline Stats& stats() {
  static Stats s;
  return s;
}

struct RequireAbort {};

inline int reg(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}

inline void record(bool ok, const char* expr, const char* file, int line,
                   bool is_require) {
  auto& s = stats();
  ++s.checks;
  if (!ok) {
    ++s.failed_checks;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line,
                 is_require ? "REQUIRE" : "CHECK", expr);
    if (is_require) throw RequireAbort{};
  }
}

inline int run_all(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "--tc=", 5) == 0) filter = argv[i] + 5;
  }
  int failed_cases = 0, ran = 0;
  for (const auto& tc : registry()) {
    if (filter && std::strstr(tc.name, filter) == nullptr) continue;
    ++ran;
    stats().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", tc.file, tc.line,
                   tc.name, e.what());
      stats().current_failed = true;
      ++stats().failed_checks;
    }
    if (stats().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[doctest-shim] FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", ran,
              ran - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %lld | %lld passed | %lld failed\n",
              stats().checks, stats().checks - stats().failed_checks,
              stats().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                 \
  static void fn();                                                               \
  [[maybe_unused]] static const int DOCTEST_CAT(fn, _reg) =                       \
      ::doctest::detail::reg(name, __FILE__, __LINE__, &fn);                      \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...) \
  ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  ::doctest::detail::record(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
  ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                          \
  do {                                                                       \
    bool doctest_ok_ = false;                                                \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const type&) {                                                  \
      doctest_ok_ = true;                                                    \
    } catch (...) {                                                          \
    }                                                                        \
    ::doctest::detail::record(doctest_ok_, #expr " throws " #type, __FILE__, \
                              __LINE__, false);                              \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
