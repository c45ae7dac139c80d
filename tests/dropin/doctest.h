// doctest.h -- minimal doctest-compatible test harness (the subset the
// reference's unit tests use: TEST_CASE, SUBCASE, CHECK, CHECK_FALSE,
// CHECK_THROWS, CHECK_THROWS_WITH_AS + doctest::Contains, doctest::Approx
// with .epsilon / .scale, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN).  doctest
// itself is not vendored in the reference; this lets its test files
// (/root/reference/proj/tests/test_*.cpp) compile unmodified against the
// B200 drop-in (include/dtq).  Test infrastructure only.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double lhs) const {
    // doctest semantics: |lhs - v| < eps * (scale + max(|lhs|, |v|))
    return std::fabs(lhs - value_) <
           eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.matches(lhs); }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.matches(lhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

// CHECK_THROWS_WITH_AS(expr, doctest::Contains("..."), Ex): what() contains
struct Contains {
  explicit Contains(const char* s) : sub(s) {}
  std::string sub;
};

namespace detail {

inline bool message_matches(const std::string& what, const Contains& c) {
  return what.find(c.sub) != std::string::npos;
}

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

struct State {
  long checks = 0;
  long failed_checks = 0;
  bool case_failed = false;
  int sub_target = 0;  // SUBCASE: the one entered on this run of the case
  int sub_seen = 0;    // SUBCASEs met on this run
};

inline State& state() {
  static State s;
  return s;
}

inline int reg(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}

inline void report(bool ok, const char* expr, const char* file, int line) {
  ++state().checks;
  if (!ok) {
    ++state().failed_checks;
    state().case_failed = true;
    std::fprintf(stderr, "%s:%d: CHECK( %s ) failed\n", file, line, expr);
  }
}

// doctest re-runs a test case once per SUBCASE, entering exactly one of
// them each time (flat subcases only, as the reference tests use them)
inline bool enter_subcase() { return state().sub_seen++ == state().sub_target; }

inline bool message_matches(const std::string& what, const char* exact) { return what == exact; }
inline bool message_matches(const std::string& what, const std::string& exact) {
  return what == exact;
}

template <typename E, typename F, typename M>
void check_throws_with_as(F&& f, const M& matcher, const char* expr, const char* file, int line) {
  bool ok = false;
  try {
    f();
  } catch (const E& e) {
    ok = message_matches(std::string(e.what()), matcher);
  } catch (...) {
  }
  ++state().checks;
  if (!ok) {
    ++state().failed_checks;
    state().case_failed = true;
    std::fprintf(stderr, "%s:%d: CHECK_THROWS_WITH_AS( %s ) failed\n", file, line, expr);
  }
}

template <typename F>
void check_throws(F&& f, const char* expr, const char* file, int line) {
  bool threw = false;
  try {
    f();
  } catch (...) {
    threw = true;
  }
  ++state().checks;
  if (!threw) {
    ++state().failed_checks;
    state().case_failed = true;
    std::fprintf(stderr, "%s:%d: CHECK_THROWS( %s ) did not throw\n", file, line, expr);
  }
}

inline int run_all(int argc, char** argv) {
  std::string filter = argc > 1 ? argv[1] : "";
  int failed = 0, ran = 0;
  for (const Case& c : registry()) {
    if (!filter.empty() && std::string(c.name).find(filter) == std::string::npos) continue;
    ++ran;
    state().case_failed = false;
    state().sub_target = 0;
    try {
      do {  // once, or once per SUBCASE
        state().sub_seen = 0;
        c.fn();
      } while (++state().sub_target < state().sub_seen);
    } catch (const std::exception& e) {
      state().case_failed = true;
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
    } catch (...) {
      state().case_failed = true;
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw an unknown exception\n", c.file,
                   c.line, c.name);
    }
    if (state().case_failed) {
      ++failed;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", ran, ran - failed, failed);
  std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", state().checks,
              state().checks - state().failed_checks, state().failed_checks);
  return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                   \
  static void fn();                                                                        \
  static const int DOCTEST_CAT(fn, _reg) = doctest::detail::reg(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...) CHECK(__VA_ARGS__)
#define CHECK_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE_FALSE(...) CHECK_FALSE(__VA_ARGS__)
#define SUBCASE(name) if (doctest::detail::enter_subcase())
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                        \
  doctest::detail::check_throws_with_as<__VA_ARGS__>([&] { (void)(expr); }, matcher, #expr, \
                                                     __FILE__, __LINE__)
#define CHECK_THROWS(...) \
  doctest::detail::check_throws([&] { (void)(__VA_ARGS__); }, #__VA_ARGS__, __FILE__, __LINE__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
