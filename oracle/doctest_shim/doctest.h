// From-scratch, minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
// Supports what the reference's proj/tests/test_tsdf_integrator.cpp and
// proj/tests/test_voxel_store.cpp use: TEST_CASE, SUBCASE (with doctest's
// re-execution semantics: the whole test body re-runs once per leaf subcase, so
// locals declared before a SUBCASE are fresh for each one), CHECK, REQUIRE,
// CHECK_THROWS, CHECK_THROWS_AS and doctest::Approx(...).epsilon(...).
// Approx follows doctest's documented rule:
//   |a - b| < eps * (scale + max(|a|, |b|)), eps = 100 * FLT_EPSILON, scale = 1.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !operator==(rhs, lhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

namespace detail {

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

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

// Subcase re-execution state (single and nested levels).
struct SubcaseState {
  std::set<std::string> done;       // leaf paths fully executed
  std::vector<std::string> stack;   // current path
  bool entered_new = false;         // a not-yet-done subcase was entered this run
  std::set<std::string> seen_children;  // paths that turned out to have children this run
};

inline SubcaseState& sub() {
  static SubcaseState s;
  return s;
}

inline long long& checks() { static long long c = 0; return c; }
inline long long& failures() { static long long f = 0; return f; }
inline const char*& current_test() { static const char* t = ""; return t; }

inline void report(bool ok, const char* expr, const char* file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    std::string path;
    for (const auto& s : sub().stack) path += " / " + s;
    std::fprintf(stderr, "%s:%d: FAILED [%s%s]: %s\n", file, line, current_test(), path.c_str(),
                 expr);
  }
}

class SubcaseGuard {
 public:
  SubcaseGuard(const char* name, const char* file, int line) {
    SubcaseState& s = sub();
    std::string key = std::string(file) + ":" + std::to_string(line) + ":" + name;
    std::string full;
    for (const auto& p : s.stack) full += p + "|";
    full += key;
    if (s.entered_new || s.done.count(full)) {
      entered_ = false;
      return;
    }
    entered_ = true;
    s.entered_new = true;
    s.stack.push_back(key);
    full_ = full;
  }
  ~SubcaseGuard() {
    if (!entered_) return;
    sub().stack.pop_back();
    sub().done.insert(full_);
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
  std::string full_;
};

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    current_test() = tc.name;
    sub() = SubcaseState{};
    const long long before = failures();
    for (int run = 0; run < 100000; ++run) {
      sub().entered_new = false;
      sub().stack.clear();
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++failures();
        std::fprintf(stderr, "%s:%d: [%s] unexpected exception: %s\n", tc.file, tc.line, tc.name,
                     e.what());
      }
      if (!sub().entered_new) break;
    }
    if (failures() != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | failed: %d | assertions: %lld | failed: %lld\n",
              registry().size(), failed_cases, checks(), failures());
  return failures() == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(p) DOCTEST_CAT(p, __LINE__)

#define TEST_CASE(name)                                                                  \
  static void DOCTEST_ANON(doctest_fn_)();                                               \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__, \
                                                                 &DOCTEST_ANON(doctest_fn_)); \
  static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) \
  if (const ::doctest::detail::SubcaseGuard DOCTEST_ANON(doctest_sc_){name, __FILE__, __LINE__})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                             \
  do {                                                                           \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                     \
    ::doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);    \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                  \
  } while (0)
#define CHECK_THROWS(...)                                                          \
  do {                                                                             \
    bool doctest_threw_ = false;                                                   \
    try { (void)(__VA_ARGS__); } catch (...) { doctest_threw_ = true; }            \
    ::doctest::detail::report(doctest_threw_, "throws: " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                 \
  do {                                                                             \
    bool doctest_threw_ = false;                                                   \
    try { (void)(expr); } catch (const __VA_ARGS__&) { doctest_threw_ = true; } catch (...) {} \
    ::doctest::detail::report(doctest_threw_, "throws as " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                         \
  do {                                                                             \
    bool doctest_ok_ = true;                                                       \
    try { (void)(__VA_ARGS__); } catch (...) { doctest_ok_ = false; }              \
    ::doctest::detail::report(doctest_ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
