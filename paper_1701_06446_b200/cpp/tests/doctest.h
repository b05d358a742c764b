// Minimal doctest-compatible test harness (our own implementation; the real
// single-header doctest is not vendored in this environment).  It supports
// the subset the reference's unit tests use -- TEST_CASE, SUBCASE, CHECK,
// REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx -- so those
// test files compile unchanged against the cumstream_b200 drop-in API
// (tools/build_refsuite.sh).  SUBCASEs run once each, in order, inside a
// single execution of their test case.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
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
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
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

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct State {
  int checks = 0;
  int failures = 0;
  bool current_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++state().checks;
  if (ok) return;
  ++state().failures;
  state().current_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

}  // namespace detail

inline int run_all() {
  int failed_cases = 0, n = 0;
  for (const auto& tc : detail::registry()) {
    ++n;
    detail::state().current_failed = false;
    try {
      tc.fn();
    } catch (const detail::RequireAbort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: TEST_CASE(%s) threw: %s\n", tc.file, tc.line, tc.name, e.what());
      detail::state().current_failed = true;
      ++detail::state().failures;
    }
    if (detail::state().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[FAIL] %s\n", tc.name);
    } else {
      std::fprintf(stdout, "[ ok ] %s\n", tc.name);
    }
  }
  std::fprintf(stdout, "test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", n,
               n - failed_cases, failed_cases, detail::state().checks, detail::state().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                        \
  static void fn();                                                                  \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (true)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                         \
  do {                                                                                      \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                \
    doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);      \
    if (!doctest_ok_) throw doctest::detail::RequireAbort{};                                \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                           \
  do {                                                                                      \
    bool doctest_ok_ = false;                                                               \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__&) {                                                          \
      doctest_ok_ = true;                                                                   \
    } catch (...) {                                                                         \
    }                                                                                       \
    doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);     \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                  \
  do {                                                                                      \
    bool doctest_ok_ = true;                                                                \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (...) {                                                                         \
      doctest_ok_ = false;                                                                  \
    }                                                                                       \
    doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);       \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
