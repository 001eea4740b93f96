// TEST INFRASTRUCTURE ONLY (oracle/). A minimal, self-written stand-in for
// the doctest macros the reference unit suites use (proj/tests/*.cpp);
// doctest itself is expected in proj/vendor/, which is absent
// (proj/CMakeLists.txt:8, proj/.gitignore:2). Supports TEST_CASE, CHECK,
// REQUIRE, CHECK_FALSE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CHECK_NOTHROW,
// CHECK_MESSAGE, doctest::Approx and doctest::Contains.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <stdexcept>
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
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }
  friend bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.value_ && lhs != rhs; }
  friend bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.value_ && lhs != rhs; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(std::string s) : needle(std::move(s)) {}
  std::string needle;
};

namespace detail {

struct RequireFailure {};

struct Registry {
  struct Case {
    const char* name;
    void (*fn)();
  };
  std::vector<Case> cases;
  int failed_checks = 0;
  int passed_checks = 0;
  const char* current = "";
  static Registry& get() {
    static Registry r;
    return r;
  }
};

inline int add_case(const char* name, void (*fn)()) {
  Registry::get().cases.push_back({name, fn});
  return 0;
}

inline void report(bool ok, const char* file, int line, const char* expr) {
  auto& r = Registry::get();
  if (ok) {
    ++r.passed_checks;
    return;
  }
  ++r.failed_checks;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, r.current, expr);
}

inline bool matches(const std::string& what, const Contains& c) {
  return what.find(c.needle) != std::string::npos;
}
inline bool matches(const std::string& what, const char* s) { return what == s; }
inline bool matches(const std::string& what, const std::string& s) { return what == s; }

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                      \
  static void fn();                                                           \
  [[maybe_unused]] static const int DOCTEST_CAT(fn, _reg) =                   \
      doctest::detail::add_case(name, &fn);                                   \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define CHECK_MESSAGE(cond, ...) doctest::detail::report(static_cast<bool>(cond), __FILE__, __LINE__, #cond)
#define REQUIRE(...)                                                          \
  do {                                                                        \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                  \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, #__VA_ARGS__);   \
    if (!doctest_ok_) throw doctest::detail::RequireFailure{};                \
  } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, type)                                           \
  do {                                                                        \
    bool doctest_ok_ = false;                                                 \
    try {                                                                     \
      (void)(expr);                                                           \
    } catch (const type&) {                                                   \
      doctest_ok_ = true;                                                     \
    } catch (...) {                                                           \
    }                                                                         \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "throws " #type ": " #expr); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, type)                                \
  do {                                                                        \
    bool doctest_ok_ = false;                                                 \
    try {                                                                     \
      (void)(expr);                                                           \
    } catch (const type& e) {                                                 \
      doctest_ok_ = doctest::detail::matches(e.what(), with);                 \
    } catch (...) {                                                           \
    }                                                                         \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "throws-with " #type ": " #expr); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                   \
  do {                                                                        \
    bool doctest_ok_ = true;                                                  \
    try {                                                                     \
      (void)(expr);                                                           \
    } catch (...) {                                                           \
      doctest_ok_ = false;                                                    \
    }                                                                         \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "nothrow: " #expr); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  auto& r = doctest::detail::Registry::get();
  int failed_cases = 0;
  for (const auto& c : r.cases) {
    r.current = c.name;
    const int before = r.failed_checks;
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "test case \"%s\" threw: %s\n", c.name, e.what());
      ++r.failed_checks;
    }
    if (r.failed_checks != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d passed, %d failed\n",
              r.cases.size(), r.cases.size() - static_cast<std::size_t>(failed_cases), failed_cases,
              r.passed_checks, r.failed_checks);
  return failed_cases == 0 ? 0 : 1;
}
#endif
