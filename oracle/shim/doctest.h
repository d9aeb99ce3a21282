// Minimal doctest-compatible test runner. TEST INFRASTRUCTURE ONLY: lets the
// reference's own tests (/root/reference/proj/tests/test_{engine,layouts,vmm,
// kv}.cpp) compile unmodified into oracle/_ref. Implements the macro subset
// they use: TEST_CASE, SUBCASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CAPTURE, doctest::Approx(x).epsilon(e). SUBCASE follows doctest's
// re-execution model for sibling subcases (each run of a TEST_CASE enters the
// next not-yet-run subcase).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <type_traits>
#include <set>
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
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {

struct RequireAbort {};

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
  // subcase bookkeeping for the currently running test case
  std::set<std::string> done;
  bool entered = false;
  bool pending = false;
  std::vector<std::string> captures;
};

inline State& st() {
  static State s;
  return s;
}

inline int reg(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++st().checks;
  if (ok) return;
  ++st().failures;
  std::printf("%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
  for (const auto& c : st().captures) std::printf("    with %s\n", c.c_str());
}

struct Subcase {
  bool active = false;
  std::string key;
  Subcase(const char* name, const char* file, int line) {
    key = std::string(file) + ":" + std::to_string(line) + ":" + name;
    if (st().done.count(key)) return;
    if (st().entered) {
      st().pending = true;  // another sibling still to run
      return;
    }
    st().entered = true;
    active = true;
  }
  ~Subcase() {
    if (active) st().done.insert(key);
  }
  explicit operator bool() const { return active; }
};

struct Capture {
  Capture(const std::string& s) { st().captures.push_back(s); }
  ~Capture() { st().captures.pop_back(); }
};

template <class T>
std::string to_str(const T& v) {
  if constexpr (std::is_arithmetic_v<T>)
    return std::to_string(v);
  else if constexpr (std::is_convertible_v<T, std::string>)
    return std::string(v);
  else
    return "?";
}

inline int run_all() {
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    st().done.clear();
    const long before = st().failures;
    for (int run = 0; run < 1000; ++run) {
      st().entered = false;
      st().pending = false;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        ++st().failures;
        std::printf("%s:%d: TEST CASE '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
      }
      if (!st().pending) break;
    }
    if (st().failures != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | failed: %d | assertions: %ld | failed: %ld\n",
              registry().size(), failed_cases, st().checks, st().failures);
  return st().failures == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                            \
  static void DOCTEST_UNIQUE(doctest_fn_)();                                       \
  [[maybe_unused]] static const int DOCTEST_UNIQUE(doctest_reg_) =                 \
      doctest::detail::reg(name, __FILE__, __LINE__, &DOCTEST_UNIQUE(doctest_fn_)); \
  static void DOCTEST_UNIQUE(doctest_fn_)()

#define SUBCASE(name) \
  if (const doctest::detail::Subcase DOCTEST_UNIQUE(doctest_sc_){name, __FILE__, __LINE__})

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                             \
  do {                                                                                           \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                     \
    doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);           \
    if (!doctest_ok_) throw doctest::detail::RequireAbort{};                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    bool doctest_ok_ = false;                                                           \
    try {                                                                               \
      expr;                                                                             \
    } catch (const __VA_ARGS__&) {                                                      \
      doctest_ok_ = true;                                                               \
    } catch (...) {                                                                     \
    }                                                                                   \
    doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                           \
  do {                                                                                \
    bool doctest_ok_ = true;                                                          \
    try {                                                                             \
      expr;                                                                           \
    } catch (...) {                                                                   \
      doctest_ok_ = false;                                                            \
    }                                                                                 \
    doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_MESSAGE(cond, msg) \
  doctest::detail::report(static_cast<bool>(cond), "CHECK_MESSAGE", #cond, __FILE__, __LINE__)
#define CAPTURE(x) \
  const doctest::detail::Capture DOCTEST_UNIQUE(doctest_cap_)(std::string(#x " := ") + doctest::detail::to_str(x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
