// TEST INFRASTRUCTURE ONLY. A minimal stand-in for the doctest header the reference's unit
// tests include (proj/tests/test_*.cpp; doctest itself is fetched by the reference's CMake and
// is not in this image). It implements exactly what those files use: TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS (+ doctest::Contains) and doctest::Approx with doctest's comparison rule
// (|a - b| < eps * (scale + max(|a|, |b|)), eps default 100 * FLT_EPSILON, scale 1), and a main
// that runs every case and prints one "[PASS]/[FAIL] case" line each plus a summary.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
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
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) <
           r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};

class Contains {
 public:
  explicit Contains(const char* s) : s_(s) {}
  bool matches(const std::string& what) const { return what.find(s_) != std::string::npos; }

 private:
  std::string s_;
};

namespace detail {

inline bool message_matches(const Contains& c, const std::string& what) { return c.matches(what); }
inline bool message_matches(const char* exact, const std::string& what) { return what == exact; }

struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline long long& assertions() {
  static long long a = 0;
  return a;
}
inline void report(bool ok, const char* what, const char* expr, const char* file, int line) {
  ++assertions();
  if (ok) return;
  ++failures();
  std::printf("  %s:%d: %s( %s ) failed\n", file, line, what, expr);
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, reg, name)                         \
  static void fn();                                          \
  static const ::doctest::detail::Reg reg(name, &fn);        \
  static void fn()
#define TEST_CASE(name) \
  DOCTEST_CASE_(DOCTEST_CAT(doctest_case_fn_, __LINE__), DOCTEST_CAT(doctest_case_reg_, __LINE__), name)

#define CHECK(...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                             \
  do {                                                                                           \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                     \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);         \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                                  \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                           \
  do {                                                                                       \
    bool doctest_ok_ = false;                                                                \
    try {                                                                                    \
      static_cast<void>(expr);                                                               \
    } catch (const __VA_ARGS__&) {                                                           \
      doctest_ok_ = true;                                                                    \
    } catch (...) {                                                                          \
    }                                                                                        \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);    \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                \
  do {                                                                                       \
    bool doctest_ok_ = false;                                                                \
    try {                                                                                    \
      static_cast<void>(expr);                                                               \
    } catch (const __VA_ARGS__& e) {                                                         \
      doctest_ok_ = ::doctest::detail::message_matches(with, e.what());                     \
    } catch (...) {                                                                          \
    }                                                                                        \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  const auto& cases = ::doctest::detail::registry();
  for (const auto& c : cases) {
    const int before = ::doctest::detail::failures();
    bool threw = false;
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
      threw = true;
    } catch (const std::exception& e) {
      std::printf("  unexpected exception: %s\n", e.what());
      threw = true;
    } catch (...) {
      std::printf("  unexpected exception\n");
      threw = true;
    }
    const bool ok = !threw && ::doctest::detail::failures() == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("test cases: %zu | %zu passed | %d failed | assertions: %lld | %d failed\n",
              cases.size(), cases.size() - static_cast<size_t>(failed_cases), failed_cases,
              ::doctest::detail::assertions(), ::doctest::detail::failures());
  return failed_cases ? 1 : 0;
}
#endif
