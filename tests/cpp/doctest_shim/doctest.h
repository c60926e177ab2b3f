// doctest.h -- TEST-ONLY minimal stand-in for the doctest framework (the
// reference's unit tests include "doctest.h", which is not vendored in the
// reference tree: proj/vendor/ is absent).  Implements just
// the subset those tests use -- TEST_CASE, flat SUBCASE, CHECK / REQUIRE /
// CHECK_FALSE, CHECK_THROWS_AS / CHECK_THROWS_WITH_AS / CHECK_NOTHROW, FAIL,
// doctest::Approx(.epsilon) and doctest::Contains -- so the reference's own
// unit tests can be compiled unmodified against the drop-in
// (tests/test_gpu_ref_unit.py).  Not part of the product.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double value;
  double eps = 1.1920928955078125e-07 * 100;  // doctest's default: float epsilon x 100
  double scale = 1.0;
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value) <
           rhs.eps * (rhs.scale + std::max(std::fabs(lhs), std::fabs(rhs.value)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
};

struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  bool matches(const std::string& what) const { return what.find(s) != std::string::npos; }
};

namespace shim {

struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct State {
  int failed_checks = 0, passed_checks = 0;
  bool case_failed = false;
  int subcase_target = 0, subcase_seen = 0;
};

inline State& state() {
  static State s;
  return s;
}

struct Abort {};  // REQUIRE / FAIL end the test case

inline void report(bool ok, const char* file, int line, const char* what, bool fatal) {
  State& s = state();
  if (ok) {
    ++s.passed_checks;
    return;
  }
  ++s.failed_checks;
  s.case_failed = true;
  std::printf("%s:%d: FAILED: %s\n", file, line, what);
  if (fatal) throw Abort{};
}

inline bool matches(const Contains& m, const std::string& what) { return m.matches(what); }
inline bool matches(const char* m, const std::string& what) { return what == m; }

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

// Flat subcases: run k of a test case enters only the k-th SUBCASE it meets.
inline bool enter_subcase() { return state().subcase_seen++ == state().subcase_target; }

// DOCTEST_SKIP: comma-separated substrings of test case names not to run.
inline bool skipped(const char* name) {
  const char* env = std::getenv("DOCTEST_SKIP");
  if (!env) return false;
  std::string list(env);
  for (size_t a = 0; a <= list.size();) {
    size_t b = list.find(',', a);
    if (b == std::string::npos) b = list.size();
    const std::string part = list.substr(a, b - a);
    if (!part.empty() && std::strstr(name, part.c_str())) return true;
    a = b + 1;
  }
  return false;
}

inline int run_all() {
  int cases = 0, failed = 0, skipped_n = 0;
  for (const Case& c : registry()) {
    if (skipped(c.name)) {
      ++skipped_n;
      continue;
    }
    State& s = state();
    s.case_failed = false;
    for (int target = 0;; ++target) {
      s.subcase_target = target;
      s.subcase_seen = 0;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        report(false, c.file, c.line, (std::string("unexpected exception: ") + e.what()).c_str(),
               false);
      }
      if (s.subcase_seen <= target + 1) break;  // no further subcase to enter
    }
    ++cases;
    if (s.case_failed) {
      ++failed;
      std::printf("test case FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", cases,
              cases - failed, failed, skipped_n);
  std::printf("[doctest] assertions: %d | %d passed | %d failed\n",
              state().passed_checks + state().failed_checks, state().passed_checks,
              state().failed_checks);
  return failed == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                          \
  static void fn();                                                                      \
  static const ::doctest::shim::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__,    \
                                                                 __LINE__);             \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::shim::enter_subcase())

#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", true)
#define FAIL(msg) ::doctest::shim::report(false, __FILE__, __LINE__, "FAIL", true)

#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                      \
    bool ok_ = false;                                                                       \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__&) {                                                          \
      ok_ = true;                                                                           \
    } catch (...) {                                                                         \
    }                                                                                       \
    ::doctest::shim::report(ok_, __FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ")", false); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                              \
  do {                                                                                     \
    bool ok_ = false;                                                                      \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__& e_) {                                                      \
      ok_ = ::doctest::shim::matches(with, e_.what());                                     \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::shim::report(ok_, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ")",   \
                            false);                                                        \
  } while (0)

#define CHECK_NOTHROW(expr)                                                                \
  do {                                                                                     \
    bool ok_ = true;                                                                       \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (...) {                                                                        \
      ok_ = false;                                                                         \
    }                                                                                      \
    ::doctest::shim::report(ok_, __FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")", false);  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
