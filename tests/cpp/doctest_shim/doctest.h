// Minimal doctest-compatible test runner (own code; the real doctest is not
// in this image).  Enough of doctest's interface to build the reference's
// unit tests (proj/tests/test_*.cpp) unchanged against include/lpmc:
// TEST_CASE, CHECK / CHECK_FALSE / REQUIRE, CHECK_THROWS / CHECK_THROWS_AS /
// CHECK_NOTHROW and doctest::Approx(...).epsilon(...), plus a main() under
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Output: one line per failed check and
// a summary; exit status 1 if any check failed.
//
//   unit_tests [substring]   run the test cases whose name contains substring
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
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
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
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

struct Stats {
  long checks = 0;
  long failed = 0;
  const char* current = "";
};

inline Stats& stats() {
  static Stats s;
  return s;
}

struct RequireFailed {};

inline int add(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}

inline bool check(bool ok, const char* what, const char* file, int line, bool require) {
  Stats& s = stats();
  ++s.checks;
  if (!ok) {
    ++s.failed;
    std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, s.current, what);
  }
  if (!ok && require) throw RequireFailed{};
  return ok;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(fn, name)                                                   \
  static void fn();                                                                    \
  static const int DOCTEST_CAT(fn, _reg) = doctest::detail::add(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::check(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                 \
  do {                                                                             \
    bool doctest_ok_ = false;                                                      \
    try {                                                                          \
      static_cast<void>(expr);                                                     \
    } catch (const __VA_ARGS__&) {                                                 \
      doctest_ok_ = true;                                                          \
    } catch (...) {                                                                \
    }                                                                              \
    doctest::detail::check(doctest_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS(expr)                                                         \
  do {                                                                             \
    bool doctest_ok_ = false;                                                      \
    try {                                                                          \
      static_cast<void>(expr);                                                     \
    } catch (...) {                                                                \
      doctest_ok_ = true;                                                          \
    }                                                                              \
    doctest::detail::check(doctest_ok_, #expr " throws", __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                        \
  do {                                                                             \
    bool doctest_ok_ = true;                                                       \
    try {                                                                          \
      static_cast<void>(expr);                                                     \
    } catch (...) {                                                                \
      doctest_ok_ = false;                                                         \
    }                                                                              \
    doctest::detail::check(doctest_ok_, #expr " does not throw", __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::detail;
  const char* filter = argc > 1 ? argv[1] : nullptr;
  long cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    if (filter != nullptr && std::strstr(c.name, filter) == nullptr) continue;
    ++cases;
    Stats& s = stats();
    s.current = c.name;
    const long before = s.failed;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++s.failed;
      std::printf("%s:%d: \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
    } catch (...) {
      ++s.failed;
      std::printf("%s:%d: \"%s\" threw a non-std exception\n", c.file, c.line, c.name);
    }
    const bool ok = s.failed == before;
    failed_cases += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("test cases: %ld | %ld passed | %ld failed; assertions: %ld | %ld failed\n", cases,
              cases - failed_cases, failed_cases, stats().checks, stats().failed);
  return stats().failed == 0 ? 0 : 1;
}
#endif
