// doctest_lite — TEST INFRASTRUCTURE. A from-scratch stand-in for the part of doctest the
// reference's test suites use (proj/tests/*.cpp; doctest itself is vendored upstream and absent
// here, proj/.gitignore:2): TEST_CASE, CHECK / CHECK_FALSE / REQUIRE, CHECK_NOTHROW,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS (with doctest::Contains), INFO, doctest::Approx and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN. Each assertion prints file:line on failure; the runner
// executes every registered case, reports counts and exits non-zero on any failure. An optional
// argument filters cases by substring of their name.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
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
  // doctest: |lhs - value| < eps * (scale + max(|lhs|, |value|))
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};
template <class T>
bool operator==(const T& lhs, const Approx& a) {
  return a.matches(double(lhs));
}
template <class T>
bool operator==(const Approx& a, const T& rhs) {
  return a.matches(double(rhs));
}
template <class T>
bool operator!=(const T& lhs, const Approx& a) {
  return !a.matches(double(lhs));
}
template <class T>
bool operator<=(const T& lhs, const Approx& a) {
  return double(lhs) < a.value() || a.matches(double(lhs));
}
template <class T>
bool operator>=(const T& lhs, const Approx& a) {
  return double(lhs) > a.value() || a.matches(double(lhs));
}

struct Contains {
  explicit Contains(const char* s) : str(s) {}
  std::string str;
};
namespace detail {
inline const std::string& contains_text(const Contains& c) { return c.str; }
inline std::string contains_text(const char* s) { return s; }
}  // namespace detail

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
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  std::vector<std::string> info;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireFailure {};
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool require) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  for (const auto& m : s.info) std::fprintf(stderr, "  with: %s\n", m.c_str());
  if (require) throw RequireFailure{};
}
struct InfoScope {
  explicit InfoScope(std::string m) { state().info.push_back(std::move(m)); }
  ~InfoScope() { state().info.pop_back(); }
};
inline int run(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  long cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    state().case_failed = false;
    try {
      c.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
      state().case_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw an unknown exception\n", c.file, c.line, c.name);
      state().case_failed = true;
    }
    if (state().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST CASE \"%s\"\n", c.name);
    }
  }
  std::printf("[doctest_lite] test cases: %ld | %ld passed | %ld failed; assertions: %ld | %ld passed | %ld failed\n",
              cases, cases - failed_cases, failed_cases, state().checks, state().checks - state().failed_checks,
              state().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_LITE_CAT2(a, b) a##b
#define DOCTEST_LITE_CAT(a, b) DOCTEST_LITE_CAT2(a, b)
#define DOCTEST_LITE_CASE(fn, name)                                                                         \
  static void fn();                                                                                         \
  static ::doctest::detail::Registrar DOCTEST_LITE_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);             \
  static void fn()
#define TEST_CASE(name) DOCTEST_LITE_CASE(DOCTEST_LITE_CAT(doctest_lite_case_, __COUNTER__), name)

#define DOCTEST_LITE_CHECK(kind, cond, require, expr_text)                                                  \
  do {                                                                                                      \
    bool doctest_lite_ok = false;                                                                           \
    try {                                                                                                   \
      doctest_lite_ok = static_cast<bool>(cond);                                                            \
    } catch (const std::exception& e) {                                                                     \
      std::fprintf(stderr, "%s:%d: %s threw: %s\n", __FILE__, __LINE__, kind, e.what());                   \
    }                                                                                                       \
    ::doctest::detail::report(doctest_lite_ok, kind, expr_text, __FILE__, __LINE__, require);               \
  } while (0)
#define CHECK(...) DOCTEST_LITE_CHECK("CHECK", (__VA_ARGS__), false, #__VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_LITE_CHECK("CHECK_FALSE", !(__VA_ARGS__), false, #__VA_ARGS__)
#define REQUIRE(...) DOCTEST_LITE_CHECK("REQUIRE", (__VA_ARGS__), true, #__VA_ARGS__)
#define REQUIRE_FALSE(...) DOCTEST_LITE_CHECK("REQUIRE_FALSE", !(__VA_ARGS__), true, #__VA_ARGS__)

#define CHECK_NOTHROW(...)                                                                                  \
  do {                                                                                                      \
    bool doctest_lite_ok = true;                                                                            \
    try {                                                                                                   \
      __VA_ARGS__;                                                                                          \
    } catch (...) {                                                                                         \
      doctest_lite_ok = false;                                                                              \
    }                                                                                                       \
    ::doctest::detail::report(doctest_lite_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, false);   \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                          \
  do {                                                                                                      \
    bool doctest_lite_ok = false;                                                                           \
    try {                                                                                                   \
      expr;                                                                                                 \
    } catch (const __VA_ARGS__&) {                                                                          \
      doctest_lite_ok = true;                                                                               \
    } catch (...) {                                                                                         \
    }                                                                                                       \
    ::doctest::detail::report(doctest_lite_ok, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__, false);        \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                               \
  do {                                                                                                      \
    bool doctest_lite_ok = false;                                                                           \
    try {                                                                                                   \
      expr;                                                                                                 \
    } catch (const __VA_ARGS__& e) {                                                                        \
      doctest_lite_ok = std::string(e.what()).find(::doctest::detail::contains_text(with)) != std::string::npos; \
     \
    } catch (...) {                                                                                         \
    }                                                                                                       \
    ::doctest::detail::report(doctest_lite_ok, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, false);   \
  } while (0)
#define INFO(...)                                                                                           \
  ::doctest::detail::InfoScope DOCTEST_LITE_CAT(doctest_lite_info_, __LINE__)(                              \
      (std::ostringstream() << __VA_ARGS__).str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
