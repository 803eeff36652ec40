// Test infrastructure only: a minimal restatement of the doctest macros the
// reference's unit tests use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// doctest::Approx with .epsilon / .scale), so those test files compile here
// unmodified (doctest itself is not vendored in /root/reference). Semantics
// follow doctest's published behaviour: a failed CHECK records and continues,
// a failed REQUIRE ends the test case, Approx compares
// |a - b| < eps * (scale + max(|a|, |b|)) with eps = 100 * FLT_EPSILON and
// scale = 1 by default. With DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN the including
// file gets a main() that runs every case and returns the failure count.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
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
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) <
           a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

namespace detail {

struct Case {
  const char* name;
  const char* file;
  int line;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures_in_case() {
  static int f = 0;
  return f;
}
struct RequireFailed {};
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
inline void report(const char* kind, const char* expr, const char* file, int line,
                   const char* extra = "") {
  ++failures_in_case();
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED %s\n", file, line, kind, expr, extra);
}
inline int run_all() {
  int failed_cases = 0, checks_failed = 0;
  for (const auto& c : registry()) {
    failures_in_case() = 0;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      report("TEST_CASE", "unexpected exception", c.file, c.line, e.what());
    } catch (...) {
      report("TEST_CASE", "unexpected exception", c.file, c.line);
    }
    const int f = failures_in_case();
    checks_failed += f;
    std::printf("[%s] %s\n", f ? "FAIL" : "ok", c.name);
    if (f) ++failed_cases;
  }
  std::printf("test cases: %zu | %zu passed | %d failed | checks failed: %d\n",
              registry().size(), registry().size() - failed_cases, failed_cases, checks_failed);
  return failed_cases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                               \
  static void fn();                                                                    \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                            &fn);                      \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...)                                                                    \
  do {                                                                                \
    try {                                                                             \
      if (!(__VA_ARGS__)) ::doctest::detail::report("CHECK", #__VA_ARGS__, __FILE__, \
                                                    __LINE__);                        \
    } catch (const std::exception& e) {                                               \
      ::doctest::detail::report("CHECK", #__VA_ARGS__, __FILE__, __LINE__, e.what()); \
    }                                                                                 \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                    \
  do {                                                                                  \
    if (!(__VA_ARGS__)) {                                                               \
      ::doctest::detail::report("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);           \
      throw ::doctest::detail::RequireFailed{};                                         \
    }                                                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                     \
  do {                                                                                 \
    bool doctest_ok_ = false;                                                          \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (const __VA_ARGS__&) {                                                     \
      doctest_ok_ = true;                                                              \
    } catch (...) {                                                                    \
    }                                                                                  \
    if (!doctest_ok_)                                                                  \
      ::doctest::detail::report("CHECK_THROWS_AS", #expr, __FILE__, __LINE__, #__VA_ARGS__); \
  } while (0)
#define CHECK_THROWS(expr)                                                             \
  do {                                                                                 \
    bool doctest_ok_ = false;                                                          \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (...) {                                                                    \
      doctest_ok_ = true;                                                              \
    }                                                                                  \
    if (!doctest_ok_) ::doctest::detail::report("CHECK_THROWS", #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                            \
  do {                                                                                 \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (...) {                                                                    \
      ::doctest::detail::report("CHECK_NOTHROW", #expr, __FILE__, __LINE__);           \
    }                                                                                  \
  } while (0)
#define INFO(...) (void)0
#define CAPTURE(...) (void)0
#define MESSAGE(...) (void)0

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
