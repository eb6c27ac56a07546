// doctest-lite — ORACLE / TEST INFRASTRUCTURE ONLY.
//
// The reference's unit tests (proj/tests/unit/*.cpp) use doctest (proj/tests/unit/main.cpp:1-2),
// which is vendored in the reference's absent vendor/ directory.  This header implements the
// subset those hot-path tests use so they compile unmodified against (a) the reference's own
// moe.cpp/placement.cpp (oracle validation) and (b) this repo's GPU shim (drop-in proof):
// TEST_CASE, SUBCASE (flat; each leaf subcase re-runs the test body from the top, as doctest
// does), CHECK/CHECK_FALSE/REQUIRE, CHECK_THROWS/_AS/_WITH_AS, CHECK_NOTHROW, doctest::Approx,
// doctest::Contains.  DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN supplies main().
#pragma once

#include <cmath>
#include <cstdio>
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
  double value;
  double eps = 1.1920928955078125e-07 * 100;  // doctest default: FLT_EPSILON * 100
};
inline bool operator==(double lhs, const Approx& rhs) {
  const double scale = std::max(std::fabs(lhs), std::fabs(rhs.value));
  return std::fabs(lhs - rhs.value) < rhs.eps * (1.0 + scale);
}
inline bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
inline bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& what) const { return what.find(needle) != std::string::npos; }
  std::string needle;
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

struct State {
  long checks = 0;
  long failures = 0;
  bool current_failed = false;
  // flat subcase bookkeeping for the test case being run
  std::set<int> done;
  bool entered = false;
  bool pending = false;
};
inline State& state() {
  static State s;
  return s;
}

struct Register {
  Register(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

inline void record(bool ok, const char* kind, const char* expr, const char* file, int line) {
  auto& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
  }
}

struct Subcase {
  Subcase(const char* name, int line) : name_(name) {
    auto& s = state();
    if (!s.entered && !s.done.count(line)) {
      s.entered = true;
      s.done.insert(line);
      enter_ = true;
    } else if (!s.done.count(line)) {
      s.pending = true;
    }
  }
  explicit operator bool() const { return enter_; }
  const char* name_;
  bool enter_ = false;
};

inline int run_all() {
  auto& s = state();
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    s.done.clear();
    s.current_failed = false;
    do {
      s.entered = false;
      s.pending = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
        s.current_failed = true;
        ++s.failures;
      }
    } while (s.pending);
    if (s.current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[FAIL] %s\n", tc.name);
    }
  }
  std::printf("[doctest-lite] test cases: %zu | %zu passed | %d failed | checks: %ld | failures: %ld\n",
              registry().size(), registry().size() - static_cast<std::size_t>(failed_cases),
              failed_cases, s.checks, s.failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                        \
  static void fn();                                                                     \
  static ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __LINE__})

#define CHECK(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::record(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                          \
  do {                                                                                        \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                  \
    ::doctest::detail::record(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);      \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                               \
  } while (0)
#define CHECK_THROWS(...)                                                                     \
  do {                                                                                        \
    bool doctest_threw_ = false;                                                              \
    try {                                                                                     \
      (void)(__VA_ARGS__);                                                                    \
    } catch (...) {                                                                           \
      doctest_threw_ = true;                                                                  \
    }                                                                                         \
    ::doctest::detail::record(doctest_threw_, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                        \
    bool doctest_threw_ = false;                                                              \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const __VA_ARGS__&) {                                                            \
      doctest_threw_ = true;                                                                  \
    } catch (...) {                                                                           \
    }                                                                                         \
    ::doctest::detail::record(doctest_threw_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);  \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                              \
  do {                                                                                        \
    bool doctest_ok_ = false;                                                                 \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const __VA_ARGS__& e) {                                                          \
      doctest_ok_ = (matcher).matches(e.what());                                              \
    } catch (...) {                                                                           \
    }                                                                                         \
    ::doctest::detail::record(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                                    \
  do {                                                                                        \
    bool doctest_ok_ = true;                                                                  \
    try {                                                                                     \
      (void)(__VA_ARGS__);                                                                    \
    } catch (...) {                                                                           \
      doctest_ok_ = false;                                                                    \
    }                                                                                         \
    ::doctest::detail::record(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
