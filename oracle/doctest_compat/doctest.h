// doctest_compat/doctest.h -- a minimal, independently written header that
// implements the subset of the doctest API the reference test suites use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, INFO,
// doctest::Approx).  The reference tree gitignores its vendored doctest
// (proj/.gitignore:2), so the suites are compiled against this instead.
//
// TEST INFRASTRUCTURE ONLY (oracle/Makefile targets ref-tests, ref-tests-cuda).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

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

struct Stats {
  long checks = 0;
  long failed_checks = 0;
  bool current_failed = false;
  const char* current_name = "";
};

inline Stats& stats() {
  static Stats s;
  return s;
}

inline std::vector<std::string>& info_stack() {
  static std::vector<std::string> v;
  return v;
}

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back(TestCase{name, fn, file, line});
  }
};

struct RequireFailure {};

inline bool record(bool ok, const char* kind, const char* expr, const char* file, int line) {
  Stats& s = stats();
  ++s.checks;
  if (!ok) {
    ++s.failed_checks;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in test case \"%s\"\n", file, line, kind, expr,
                 s.current_name);
    for (const auto& m : info_stack()) std::fprintf(stderr, "  with context: %s\n", m.c_str());
  }
  return ok;
}

struct InfoScope {
  explicit InfoScope(std::string msg) { info_stack().push_back(std::move(msg)); }
  ~InfoScope() { info_stack().pop_back(); }
};

// doctest's comparison: |lhs - rhs| < eps * (scale + max(|lhs|, |rhs|)),
// default eps = 100 * float epsilon, scale = 1
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
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100;
  double scale_ = 1.0;
};

inline int run(int argc, char** argv) {
  std::string filter;
  for (int k = 1; k < argc; ++k) {
    std::string a = argv[k];
    if (a.rfind("-tc=", 0) == 0) filter = a.substr(4);
  }
  int cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    if (!filter.empty() && std::string(tc.name).find(filter) == std::string::npos) continue;
    ++cases;
    Stats& s = stats();
    s.current_failed = false;
    s.current_name = tc.name;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      s.current_failed = true;
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name,
                   e.what());
    } catch (...) {
      s.current_failed = true;
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw an unknown exception\n", tc.file,
                   tc.line, tc.name);
    }
    info_stack().clear();
    if (s.current_failed) ++failed_cases;
  }
  const Stats& s = stats();
  std::printf("[doctest-compat] test cases: %d | %d passed | %d failed\n", cases,
              cases - failed_cases, failed_cases);
  std::printf("[doctest-compat] assertions: %ld | %ld passed | %ld failed\n", s.checks,
              s.checks - s.failed_checks, s.failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(prefix) DOCTEST_CAT(prefix, __LINE__)

#define TEST_CASE(name)                                                              \
  static void DOCTEST_ANON(doctest_case_fn_)();                                      \
  static doctest::Registrar DOCTEST_ANON(doctest_case_reg_)(                         \
      name, &DOCTEST_ANON(doctest_case_fn_), __FILE__, __LINE__);                    \
  static void DOCTEST_ANON(doctest_case_fn_)()

#define CHECK(...) doctest::record(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  doctest::record(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    if (!doctest::record(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, \
                         __LINE__))                                                       \
      throw doctest::RequireFailure{};                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                          \
  do {                                                                      \
    bool doctest_threw_ = false;                                            \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const __VA_ARGS__&) {                                          \
      doctest_threw_ = true;                                                \
    } catch (...) {                                                         \
    }                                                                       \
    doctest::record(doctest_threw_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define INFO(...)                                                             \
  doctest::InfoScope DOCTEST_ANON(doctest_info_)([&] {                        \
    std::ostringstream doctest_os_;                                           \
    doctest_os_ << __VA_ARGS__;                                               \
    return doctest_os_.str();                                                 \
  }())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::run(argc, argv); }
#endif
