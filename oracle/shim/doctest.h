// Minimal doctest-compatible test harness.
//
// TEST INFRASTRUCTURE ONLY. The reference vendors doctest under
// proj/vendor/ (absent: proj/.gitignore:2); this header implements just the
// macros its hot-path suites use (TEST_CASE, SUBCASE with re-run-per-leaf
// semantics for one nesting level, CHECK*, REQUIRE*, CHECK_THROWS_*,
// CAPTURE, doctest::Approx, doctest::Contains) so that
// tests/test_{index_oodgraph,attention,engine,index_flat,util}.cpp compile
// unchanged against oracle/_ref and validate the shimmed oracle build.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.v_) <
           rhs.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(rhs.v_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

 private:
  double v_;
  double eps_ = double(std::numeric_limits<float>::epsilon()) * 100;
};

struct Contains {
  explicit Contains(const char* s) : s_(s) {}
  bool matches(const std::string& what) const {
    return what.find(s_) != std::string::npos;
  }
  std::string s_;
};

namespace detail {

inline bool msg_matches(const std::string& what, const char* want) {
  return what == want;
}
inline bool msg_matches(const std::string& what, const Contains& want) {
  return want.matches(what);
}

struct RequireFailed {};

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
struct State {
  int failed_checks = 0;
  int total_checks = 0;
  bool case_failed = false;
  int subcase_target = 0;
  int subcase_seen = 0;
  const char* current = "";
};
inline State& state() {
  static State s;
  return s;
}

inline void report(bool ok, const char* file, int line, const char* expr) {
  auto& s = state();
  ++s.total_checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, s.current, expr);
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

// SUBCASE: each run of a test case enters exactly one top-level subcase
// (the `subcase_target`-th encountered); runs repeat until all are covered.
inline bool enter_subcase() {
  auto& s = state();
  return s.subcase_seen++ == s.subcase_target;
}

inline int run_all() {
  auto& s = state();
  int failed_cases = 0;
  const bool verbose = std::getenv("DOCTEST_SHIM_VERBOSE") != nullptr;
  for (const auto& tc : registry()) {
    s.current = tc.name;
    if (verbose) std::fprintf(stderr, "[doctest-shim] running \"%s\"\n", tc.name), std::fflush(stderr);
    s.case_failed = false;
    s.subcase_target = 0;
    for (;;) {
      s.subcase_seen = 0;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: \"%s\" threw: %s\n", tc.file, tc.line, tc.name,
                     e.what());
        s.case_failed = true;
        ++s.failed_checks;
      }
      if (++s.subcase_target >= s.subcase_seen) break;
    }
    if (s.case_failed) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n",
              registry().size(), registry().size() - size_t(failed_cases), failed_cases);
  std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", s.total_checks,
              s.total_checks - s.failed_checks, s.failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                         \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                             \
  static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(      \
      name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_fn_, __LINE__));           \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define SUBCASE(name) if (::doctest::detail::enter_subcase())

#define CHECK(...) \
  ::doctest::detail::report(bool(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!bool(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...)                                                            \
  do {                                                                          \
    bool ok_ = bool(__VA_ARGS__);                                               \
    ::doctest::detail::report(ok_, __FILE__, __LINE__, #__VA_ARGS__);           \
    if (!ok_) throw ::doctest::detail::RequireFailed{};                         \
  } while (0)
#define REQUIRE_MESSAGE(cond, msg) REQUIRE(cond)
#define CAPTURE(x) ((void)0)

#define CHECK_THROWS_AS(expr, type)                                             \
  do {                                                                          \
    bool ok_ = false;                                                           \
    try {                                                                       \
      (void)(expr);                                                             \
    } catch (const type&) {                                                     \
      ok_ = true;                                                               \
    } catch (...) {                                                             \
    }                                                                           \
    ::doctest::detail::report(ok_, __FILE__, __LINE__, "throws " #type ": " #expr); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, msg, type)                                   \
  do {                                                                          \
    bool ok_ = false;                                                           \
    try {                                                                       \
      (void)(expr);                                                             \
    } catch (const type& e_) {                                                  \
      ok_ = ::doctest::detail::msg_matches(e_.what(), msg);                     \
    } catch (...) {                                                             \
    }                                                                           \
    ::doctest::detail::report(ok_, __FILE__, __LINE__,                          \
                              "throws " #type " with " #msg ": " #expr);        \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
