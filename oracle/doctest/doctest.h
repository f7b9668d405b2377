// Minimal doctest-compatible test shim (test infrastructure only).
//
// The reference vendors doctest under proj/vendor/, which is git-ignored and
// absent (proj/.gitignore:2). This header implements just the subset its
// gen+inf unit tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, doctest::Approx with .epsilon) so that
// proj/tests/test_genfuse.cpp and proj/tests/test_numerics.cpp can be compiled
// unchanged against either the reference library or this repo's library
// (oracle/Makefile targets `reftests-ref` and `reftests-b200`).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};

namespace detail {
struct Case { const char* name; void (*fn)(); const char* file; int line; };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
inline int& assertions() { static int a = 0; return a; }
struct Registrar { Registrar(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); } };
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++assertions();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  if (fatal) throw RequireFailed{};
}
inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    const int before = failures();
    try { c.fn(); } catch (const RequireFailed&) {
    } catch (const std::exception& e) { ++failures(); std::fprintf(stderr, "%s: exception: %s\n", c.name, e.what()); }
    if (failures() != before) { ++failed_cases; std::fprintf(stderr, "[case failed] %s\n", c.name); }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, assertions(), failures());
  return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                              \
  static void fn();                                                                          \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);  \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                          \
  do {                                                                                       \
    bool doctest_ok_ = false;                                                                \
    try { (void)(expr); } catch (const type&) { doctest_ok_ = true; } catch (...) {}         \
    ::doctest::detail::report(doctest_ok_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
