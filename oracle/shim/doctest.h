// ORACLE TEST INFRASTRUCTURE — not product code.
//
// A from-scratch, minimal test-macro header implementing the subset of the
// doctest API that the reference's hot-path test files use
// (proj/tests/test_{kernel,nn_index,fast_predict}.cpp): TEST_CASE, SUBCASE
// (one nesting level, each leaf run in its own pass as doctest does), CHECK,
// CHECK_THROWS_AS, FAIL and doctest::Approx with .epsilon(). doctest itself is
// un-vendored in the reference (proj/.gitignore:2) and absent from the image.
// The same header is used by this repo's C++ facade tests (tests/cpp/).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
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
  // doctest's rule: |lhs - rhs| < eps * (scale + max(|lhs|, |rhs|)).
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) <
           r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator<=(double lhs, const Approx& r) { return lhs < r.value_ || lhs == r; }
  friend bool operator>=(double lhs, const Approx& r) { return lhs > r.value_ || lhs == r; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {

struct Registry {
  struct Case {
    const char* name;
    void (*fn)();
  };
  std::vector<Case> cases;
  int checks = 0;
  int failures = 0;
  bool current_failed = false;
  // SUBCASE bookkeeping for the current pass.
  int subcase_target = 0;
  int subcase_seen = 0;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

struct Registrar {
  Registrar(const char* name, void (*fn)()) { Registry::get().cases.push_back({name, fn}); }
};

inline void report(bool ok, const char* expr, const char* file, int line) {
  auto& r = Registry::get();
  ++r.checks;
  if (!ok) {
    ++r.failures;
    r.current_failed = true;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
  }
}

struct SubcaseGuard {
  bool enter;
  explicit SubcaseGuard(const char*) {
    auto& r = Registry::get();
    enter = (r.subcase_seen == r.subcase_target);
    ++r.subcase_seen;
  }
  explicit operator bool() const { return enter; }
};

inline int run_all() {
  auto& r = Registry::get();
  int failed_cases = 0;
  for (auto& c : r.cases) {
    r.current_failed = false;
    r.subcase_target = 0;
    for (;;) {
      r.subcase_seen = 0;
      try {
        c.fn();
      } catch (const std::exception& e) {
        std::fprintf(stderr, "TEST CASE '%s' threw: %s\n", c.name, e.what());
        r.current_failed = true;
        ++r.failures;
      } catch (...) {
        std::fprintf(stderr, "TEST CASE '%s' threw an unknown exception\n", c.name);
        r.current_failed = true;
        ++r.failures;
      }
      if (r.subcase_seen > r.subcase_target + 1) {
        ++r.subcase_target;
        continue;
      }
      break;
    }
    std::printf("[%s] %s\n", r.current_failed ? "FAIL" : "PASS", c.name);
    if (r.current_failed) ++failed_cases;
  }
  std::printf("test cases: %zu | failed: %d | checks: %d | failed checks: %d\n",
              r.cases.size(), failed_cases, r.checks, r.failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                       \
  static void fn();                                                            \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);        \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (::doctest::detail::SubcaseGuard DOCTEST_CAT(doctest_sub_, __LINE__){name})
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                           \
  do {                                                                         \
    bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                         \
    ::doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);  \
    if (!doctest_ok_) throw std::runtime_error("REQUIRE failed");              \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, type)                                            \
  do {                                                                         \
    bool doctest_thrown_ = false;                                              \
    try {                                                                      \
      static_cast<void>(expr);                                                 \
    } catch (const type&) {                                                    \
      doctest_thrown_ = true;                                                  \
    } catch (...) {                                                            \
    }                                                                          \
    ::doctest::detail::report(doctest_thrown_, "CHECK_THROWS_AS(" #expr ", " #type ")", __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                    \
  do {                                                                         \
    bool doctest_ok_ = true;                                                   \
    try {                                                                      \
      static_cast<void>(expr);                                                 \
    } catch (...) {                                                            \
      doctest_ok_ = false;                                                     \
    }                                                                          \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW(" #expr ")", __FILE__, __LINE__); \
  } while (0)
#define FAIL(msg) ::doctest::detail::report(false, msg, __FILE__, __LINE__)
#define MESSAGE(msg) std::printf("%s\n", std::string(msg).c_str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
