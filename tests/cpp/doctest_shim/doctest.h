// Minimal doctest-compatible test harness (the vendored doctest.h of the
// reference is absent in this image).  Implements exactly what the
// reference's unit tests use -- TEST_CASE, SUBCASE (re-run until every leaf
// has executed once), CHECK / CHECK_FALSE / REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS with doctest::Contains, doctest::Approx -- so
// /root/reference/proj/tests/test_*.cpp compile unchanged against the B200
// lcnn library (tests/cpp/build_ref_tests.sh).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    scl = s;
    return *this;
  }
  double value;
  double eps = 1.1920928955078125e-05;  // FLT_EPSILON * 100
  double scl = 1.0;
};
inline bool operator==(double lhs, const Approx& a) {
  return std::fabs(lhs - a.value) <
         a.eps * (a.scl + std::max(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }
inline bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
  bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

namespace detail {

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

struct RequireAbort {};

struct State {
  int failures = 0;
  int checks = 0;
  bool case_failed = false;
  // subcase exploration
  std::set<std::vector<std::string>> done;
  std::vector<std::string> path;
  std::vector<bool> entered_at_depth = std::vector<bool>(64, false);
  int pending = 0;
};

inline State& st() {
  static State s;
  return s;
}

inline void report_failure(const char* file, int line, const char* what) {
  State& s = st();
  ++s.failures;
  s.case_failed = true;
  std::printf("%s:%d: CHECK FAILED: %s\n", file, line, what);
}

inline void check(bool ok, const char* file, int line, const char* what) {
  ++st().checks;
  if (!ok) report_failure(file, line, what);
}

inline void require(bool ok, const char* file, int line, const char* what) {
  ++st().checks;
  if (!ok) {
    report_failure(file, line, what);
    throw RequireAbort{};
  }
}

inline bool match(const std::string& what, const char* exact) { return what == exact; }
inline bool match(const std::string& what, const Contains& c) { return c.matches(what); }

struct Subcase {
  explicit Subcase(const char* name) {
    State& s = st();
    const std::size_t depth = s.path.size();
    std::vector<std::string> cand = s.path;
    cand.emplace_back(name);
    if (s.done.count(cand)) return;
    if (s.entered_at_depth[depth]) {
      ++s.pending;  // another sibling is still to run
      return;
    }
    entered = true;
    owner = true;
    s.entered_at_depth[depth] = true;
    s.entered_at_depth[depth + 1] = false;
    s.path = cand;
    pending_before = s.pending;
  }
  ~Subcase() {
    if (!owner) return;
    State& s = st();
    if (s.pending == pending_before) s.done.insert(s.path);
    s.path.pop_back();
  }
  bool entered = false;
  bool owner = false;
  int pending_before = 0;
  // the for-loop flips `entered` after one pass; `owner` keeps the cleanup
  explicit operator bool() const { return entered; }
};

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

inline int run_all() {
  State& s = st();
  int cases_failed = 0;
  for (const TestCase& tc : registry()) {
    s.done.clear();
    s.case_failed = false;
    for (int pass = 0; pass < 10000; ++pass) {
      s.path.clear();
      std::fill(s.entered_at_depth.begin(), s.entered_at_depth.end(), false);
      s.pending = 0;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        report_failure(tc.file, tc.line, (std::string("unexpected exception: ") + e.what()).c_str());
      } catch (...) {
        report_failure(tc.file, tc.line, "unexpected non-std exception");
      }
      if (s.pending == 0) break;
    }
    if (s.case_failed) {
      ++cases_failed;
      std::printf("[FAIL] %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d | failed checks: %d\n",
              registry().size(), registry().size() - cases_failed, cases_failed, s.checks,
              s.failures);
  return cases_failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                  \
  static void fn();                                                                       \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define SUBCASE(name) \
  for (doctest::detail::Subcase DOCTEST_CAT(sc_, __LINE__)(name); DOCTEST_CAT(sc_, __LINE__).entered; \
       DOCTEST_CAT(sc_, __LINE__).entered = false)

#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) \
  doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...) doctest::detail::require(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)

#define CHECK_THROWS_AS(expr, ...)                                                     \
  do {                                                                                 \
    bool doctest_ok_ = false;                                                          \
    try {                                                                              \
      expr;                                                                            \
    } catch (const __VA_ARGS__&) {                                                     \
      doctest_ok_ = true;                                                              \
    } catch (...) {                                                                    \
    }                                                                                  \
    doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "throws " #__VA_ARGS__ ": " #expr); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                       \
  do {                                                                                 \
    bool doctest_ok_ = false;                                                          \
    try {                                                                              \
      expr;                                                                            \
    } catch (const __VA_ARGS__& e) {                                                   \
      doctest_ok_ = doctest::detail::match(e.what(), matcher);                         \
    } catch (...) {                                                                    \
    }                                                                                  \
    doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "throws-with " #__VA_ARGS__ ": " #expr); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
