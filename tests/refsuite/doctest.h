// Minimal doctest-compatible shim: TEST INFRASTRUCTURE ONLY.
//
// doctest.h is not in this image, so the reference's own unit
// tests (/root/reference/proj/tests/test_*.cpp) are compiled against this
// subset: TEST_CASE, SUBCASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, INFO (ignored), doctest::Approx (epsilon/scale, doctest's rule
// |a - b| < eps * (scale + max(|a|, |b|)), default eps = FLT_EPSILON * 100)
// and doctest::Contains.  Every SUBCASE of a test case runs in one pass (the
// reference's subcases are independent blocks, so re-entry is not needed).
//
// The binary takes optional substring filters on the test-case name (a
// leading '!' excludes) and
// prints one summary line that tests/test_refsuite_gpu.py parses:
//   [refsuite] cases N passed P failed F checks C failed_checks X
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <type_traits>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double a) const {
    return std::fabs(a - v_) < eps_ * (scale_ + std::max(std::fabs(a), std::fabs(v_)));
  }
  double value() const { return v_; }

 private:
  double v_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

template <class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator==(T a, const Approx& b) { return b.matches(static_cast<double>(a)); }
template <class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator==(const Approx& b, T a) { return b.matches(static_cast<double>(a)); }
template <class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator!=(T a, const Approx& b) { return !b.matches(static_cast<double>(a)); }
template <class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator!=(const Approx& b, T a) { return !b.matches(static_cast<double>(a)); }

struct Contains {
  explicit Contains(const char* s) : text(s) {}
  std::string text;
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
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
};

inline Stats& stats() {
  static Stats s;
  return s;
}

struct Register {
  Register(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

inline void report(bool ok, const char* file, int line, const char* what, bool fatal) {
  ++stats().checks;
  if (ok) return;
  ++stats().failed_checks;
  stats().case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
  if (fatal) throw RequireFailed{};
}

inline bool matches(const char* want, const std::string& what) { return what == want; }
inline bool matches(const std::string& want, const std::string& what) { return what == want; }
inline bool matches(const Contains& want, const std::string& what) {
  return what.find(want.text) != std::string::npos;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                                  \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                      \
  static doctest::detail::Register DOCTEST_CAT(doctest_reg_, __LINE__)(                  \
      name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_fn_, __LINE__));                    \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define SUBCASE(name) if (true)
#define DOCTEST_INFO(...) static_cast<void>(0)
#define INFO(...) static_cast<void>(0)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) doctest::detail::report(!(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)

#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__&) {                                                         \
      doctest_ok_ = true;                                                                  \
    } catch (...) {                                                                        \
    }                                                                                      \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "throws " #__VA_ARGS__ ": " #expr, \
                            false);                                                        \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                           \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__& e) {                                                       \
      doctest_ok_ = doctest::detail::matches(matcher, std::string(e.what()));              \
      if (!doctest_ok_) std::fprintf(stderr, "  message was: %s\n", e.what());             \
    } catch (...) {                                                                        \
    }                                                                                      \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__,                               \
                            "throws " #__VA_ARGS__ " with " #matcher ": " #expr, false);   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::detail;
  long cases = 0, failed = 0;
  for (const Case& c : registry()) {
    bool any_pos = false, selected = false, excluded = false;
    for (int i = 1; i < argc; ++i) {
      if (argv[i][0] == '!') {
        excluded |= std::strstr(c.name, argv[i] + 1) != nullptr;
      } else {
        any_pos = true;
        selected |= std::strstr(c.name, argv[i]) != nullptr;
      }
    }
    if ((any_pos && !selected) || excluded) continue;
    ++cases;
    stats().case_failed = false;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: test case threw: %s\n", c.file, c.line, e.what());
      stats().case_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: test case threw a non-std exception\n", c.file, c.line);
      stats().case_failed = true;
    }
    if (stats().case_failed) {
      ++failed;
      std::fprintf(stderr, "[refsuite] FAILED case: %s\n", c.name);
    }
  }
  std::printf("[refsuite] cases %ld passed %ld failed %ld checks %ld failed_checks %ld\n", cases,
              cases - failed, failed, stats().checks, stats().failed_checks);
  return failed ? 1 : 0;
}
#endif
