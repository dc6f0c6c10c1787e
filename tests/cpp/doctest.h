// Minimal doctest-compatible test harness (the vendored doctest is absent
// from the reference, proj/.gitignore:2).  Implements exactly what the
// reference's unit tests use: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, FAIL, INFO and doctest::Approx, with a main() that runs
// every registered case and exits non-zero on any failed check.
//
// Test infrastructure only (used to run /root/reference/proj/tests/*.cpp
// unmodified against the device-backed shim, tests/cpp/b200_shim.cpp).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
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
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct AbortCase {};

inline int& failed_checks() {
  static int n = 0;
  return n;
}
inline int& total_checks() {
  static int n = 0;
  return n;
}
inline const char*& current_case() {
  static const char* c = "";
  return c;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
  ++total_checks();
  if (ok) return;
  ++failed_checks();
  std::printf("%s:%d: FAILED %s( %s ) in TEST_CASE \"%s\"\n", file, line, kind, expr, current_case());
  if (fatal) throw AbortCase{};
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)

#define TEST_CASE(name)                                                                       \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                         \
  static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                    \
      name, &DOCTEST_CAT(doctest_case_, __LINE__), __FILE__, __LINE__);                       \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define DOCTEST_EVAL(kind, fatal, negate, ...)                                                \
  do {                                                                                        \
    bool doctest_ok = false;                                                                  \
    try {                                                                                     \
      doctest_ok = static_cast<bool>(__VA_ARGS__) != (negate);                                \
    } catch (const ::doctest::detail::AbortCase&) {                                           \
      throw;                                                                                  \
    } catch (const std::exception& doctest_e) {                                               \
      std::printf("  unexpected exception: %s\n", doctest_e.what());                          \
    }                                                                                         \
    ::doctest::detail::report(doctest_ok, kind, #__VA_ARGS__, __FILE__, __LINE__, fatal);     \
  } while (0)

#define CHECK(...) DOCTEST_EVAL("CHECK", false, false, __VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_EVAL("CHECK_FALSE", false, true, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_EVAL("REQUIRE", true, false, __VA_ARGS__)

#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                        \
    bool doctest_thrown = false;                                                              \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const __VA_ARGS__&) {                                                            \
      doctest_thrown = true;                                                                  \
    } catch (...) {                                                                           \
    }                                                                                         \
    ::doctest::detail::report(doctest_thrown, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__, false); \
  } while (0)

#define FAIL(msg) ::doctest::detail::report(false, "FAIL", msg, __FILE__, __LINE__, true)
#define INFO(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
  }
  int cases = 0, failed_cases = 0;
  for (const auto& tc : ::doctest::detail::registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ++cases;
    const int before = ::doctest::detail::failed_checks();
    ::doctest::detail::current_case() = tc.name;
    try {
      tc.fn();
    } catch (const ::doctest::detail::AbortCase&) {
    } catch (const std::exception& e) {
      std::printf("%s:%d: TEST_CASE \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
      ++::doctest::detail::failed_checks();
    }
    if (::doctest::detail::failed_checks() != before) ++failed_cases;
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases, failed_cases);
  std::printf("[doctest] assertions: %d | %d failed\n", ::doctest::detail::total_checks(),
              ::doctest::detail::failed_checks());
  std::printf("[doctest] Status: %s!\n", failed_cases ? "FAILURE" : "SUCCESS");
  return failed_cases ? 1 : 0;
}
#endif
