// TEST INFRASTRUCTURE ONLY (oracle).  A small, self-written stand-in for the
// doctest single header (absent from this image), providing exactly the
// macros the reference's unit tests use: TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx(..).epsilon
// and doctest::Contains.  Approx follows doctest's published comparison rule
// |a-b| < eps * (scale + max(|a|, |b|)) with scale = 1.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    scl = s;
    return *this;
  }
  double value;
  double eps = 1.1920928955078125e-07 * 100.0;  // FLT_EPSILON * 100, doctest's default
  double scl = 1.0;
  bool matches(double lhs) const {
    return std::fabs(lhs - value) < eps * (scl + std::max(std::fabs(lhs), std::fabs(value)));
  }
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

struct Contains {
  explicit Contains(std::string s) : needle(std::move(s)) {}
  std::string needle;
  bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
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
struct RequireAbort {};
struct Stats {
  long checks = 0;
  long failed_checks = 0;
  bool current_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}
inline void report(bool ok, const char* file, int line, const char* macro, const char* expr) {
  ++stats().checks;
  if (ok) return;
  ++stats().failed_checks;
  stats().current_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) failed\n", file, line, macro, expr);
}
inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    stats().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      stats().current_failed = true;
      std::fprintf(stderr, "%s:%d: ERROR: test case threw: %s\n", tc.file, tc.line, e.what());
    } catch (...) {
      stats().current_failed = true;
      std::fprintf(stderr, "%s:%d: ERROR: test case threw a non-std exception\n", tc.file,
                   tc.line);
    }
    if (stats().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - static_cast<std::size_t>(failed_cases), failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", stats().checks,
              stats().checks - stats().failed_checks, stats().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                   \
  static void fn();                                                                 \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                              &fn);                 \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define DOCTEST_EVAL_(macro, expr, is_require, want)                                \
  do {                                                                              \
    bool ok_ = false;                                                               \
    try {                                                                           \
      ok_ = static_cast<bool>(expr) == (want);                                      \
    } catch (...) {                                                                 \
      ok_ = false;                                                                  \
    }                                                                               \
    ::doctest::detail::report(ok_, __FILE__, __LINE__, macro, #expr);               \
    if (!ok_ && (is_require)) throw ::doctest::detail::RequireAbort{};             \
  } while (0)

#define CHECK(...) DOCTEST_EVAL_("CHECK", (__VA_ARGS__), false, true)
#define CHECK_FALSE(...) DOCTEST_EVAL_("CHECK_FALSE", (__VA_ARGS__), false, false)
#define REQUIRE(...) DOCTEST_EVAL_("REQUIRE", (__VA_ARGS__), true, true)
#define REQUIRE_FALSE(...) DOCTEST_EVAL_("REQUIRE_FALSE", (__VA_ARGS__), true, false)

#define CHECK_THROWS_AS(expr, ...)                                                  \
  do {                                                                              \
    bool ok_ = false;                                                               \
    try {                                                                           \
      static_cast<void>(expr);                                                      \
    } catch (const __VA_ARGS__&) {                                                  \
      ok_ = true;                                                                   \
    } catch (...) {                                                                 \
    }                                                                               \
    ::doctest::detail::report(ok_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr);   \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                    \
  do {                                                                              \
    bool ok_ = false;                                                               \
    try {                                                                           \
      static_cast<void>(expr);                                                      \
    } catch (const __VA_ARGS__& e_) {                                               \
      ok_ = (matcher).matches(e_.what());                                           \
    } catch (...) {                                                                 \
    }                                                                               \
    ::doctest::detail::report(ok_, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS", #expr); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
