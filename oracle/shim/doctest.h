// doctest.h (shim) — TEST INFRASTRUCTURE ONLY.  A minimal stand-in for the
// subset of the doctest 2.x API the reference's test sources use
// (/root/reference/proj/tests: TEST_CASE, CHECK, REQUIRE, CHECK_FALSE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx, doctest::Contains),
// so those sources compile unchanged against (a) the reference itself built
// here (oracle/_ref) and (b) the drop-in GPU implementation of its hot path.
// Written for this repository; not doctest's code.  Approx follows doctest's
// documented rule |a - b| < eps * (scale + max(|a|, |b|)), eps default
// 100 * FLT_EPSILON, scale 1.
#pragma once
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <utility>
#include <vector>

namespace doctest {

class Approx {
 public:
  Approx(double v) : v_(v) {}  // NOLINT(google-explicit-constructor)
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool eq(double x) const { return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_))); }
  friend bool operator==(double x, const Approx& a) { return a.eq(x); }
  friend bool operator==(const Approx& a, double x) { return a.eq(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.eq(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.eq(x); }
  friend bool operator<=(double x, const Approx& a) { return x < a.v_ || a.eq(x); }
  friend bool operator>=(double x, const Approx& a) { return x > a.v_ || a.eq(x); }

 private:
  double v_, eps_ = 100.0 * FLT_EPSILON, scale_ = 1.0;
};

struct Contains {
  std::string needle;
  Contains(const char* s) : needle(s) {}  // NOLINT(google-explicit-constructor)
  bool matches(const std::string& m) const { return m.find(needle) != std::string::npos; }
};

namespace detail {
struct Case {
  const char* name;
  const char* file;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct State {
  int checks = 0, failed_checks = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}
struct Reg {
  Reg(const char* name, const char* file, void (*fn)()) { registry().push_back({name, file, fn}); }
};
struct RequireAbort {};
inline void result(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++state().checks;
  if (ok) return;
  ++state().failed_checks;
  state().case_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
}
inline bool msg_matches(const std::string& m, const Contains& c) { return c.matches(m); }
inline bool msg_matches(const std::string& m, const char* s) { return m == s; }
inline bool msg_matches(const std::string& m, const std::string& s) { return m == s; }

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    state().case_failed = false;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s: ERROR: test case \"%s\" threw: %s\n", c.file, c.name, e.what());
      state().case_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s: ERROR: test case \"%s\" threw a non-std exception\n", c.file, c.name);
      state().case_failed = true;
    }
    if (state().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", c.name);
    }
  }
  std::printf("[doctest] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - static_cast<size_t>(failed_cases), failed_cases);
  std::printf("[doctest] assertions: %d | %d passed | %d failed\n", state().checks,
              state().checks - state().failed_checks, state().failed_checks);
  std::printf("[doctest] Status: %s!\n", failed_cases ? "FAILURE" : "SUCCESS");
  return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                   \
  static void fn();                                                                             \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, &fn);                    \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::result(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::result(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                          \
  do {                                                                                        \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                  \
    ::doctest::detail::result(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);     \
    if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                        \
    bool doctest_ok_ = false;                                                                 \
    try {                                                                                     \
      static_cast<void>(expr);                                                                \
    } catch (const __VA_ARGS__&) {                                                            \
      doctest_ok_ = true;                                                                     \
    } catch (...) {                                                                           \
    }                                                                                         \
    ::doctest::detail::result(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                 \
  do {                                                                                        \
    bool doctest_ok_ = false;                                                                 \
    try {                                                                                     \
      static_cast<void>(expr);                                                                \
    } catch (const __VA_ARGS__& e) {                                                          \
      doctest_ok_ = ::doctest::detail::msg_matches(std::string(e.what()), with);             \
    } catch (...) {                                                                           \
    }                                                                                         \
    ::doctest::detail::result(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr ", " #with, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
