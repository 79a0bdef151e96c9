// catch_amalgamated.hpp — TEST INFRASTRUCTURE ONLY.
//
// A minimal stand-in for the part of the Catch2 v3 API that the reference's unit tests
// (/root/reference/proj/tests/test_*.cpp) use — TEST_CASE, CHECK/REQUIRE(_FALSE),
// CHECK_THROWS_AS/_WITH, FAIL, Catch::Approx (epsilon/margin/scale), and
// Catch::Matchers::ContainsSubstring — so that the reference's own test suite can be compiled
// here (Catch2 is not installed) and run against the reference built on the Eigen-subset shim
// (oracle/ref/Makefile, oracle/_ref/ref_tests). Written for this repository; not Catch2 code.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

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
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct State {
  int checks = 0, failed_checks = 0;
  bool current_failed = false;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireFailure {};

inline void report(bool ok, const char* what, const char* file, int line, bool fatal) {
  ++state().checks;
  if (ok) return;
  ++state().failed_checks;
  state().current_failed = true;
  std::fprintf(stderr, "  FAILED %s at %s:%d\n", what, file, line);
  if (fatal) throw RequireFailure{};
}

class Approx {
 public:
  explicit Approx(double v) : value_(v), eps_(std::numeric_limits<float>::epsilon() * 100.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool equals(double other) const {
    const double d = std::fabs(other - value_);
    if (d <= margin_) return true;
    return d <= eps_ * (scale_ + (std::isinf(value_) ? 0.0 : std::fabs(value_)));
  }
  friend bool operator==(double a, const Approx& b) { return b.equals(a); }
  friend bool operator==(const Approx& a, double b) { return a.equals(b); }
  friend bool operator!=(double a, const Approx& b) { return !b.equals(a); }
  friend bool operator!=(const Approx& a, double b) { return !a.equals(b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.value_ || b.equals(a); }
  friend bool operator>=(double a, const Approx& b) { return a > b.value_ || b.equals(a); }

 private:
  double value_, eps_, margin_ = 0.0, scale_ = 0.0;
};

namespace Matchers {
struct ContainsSubstring {
  std::string s;
  explicit ContainsSubstring(std::string x) : s(std::move(x)) {}
  bool match(const std::string& msg) const { return msg.find(s) != std::string::npos; }
};
}  // namespace Matchers

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& t : registry()) {
    state().current_failed = false;
    try {
      t.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "  unexpected exception: %s\n", e.what());
      state().current_failed = true;
    }
    std::printf("%s %s (%s:%d)\n", state().current_failed ? "FAIL" : "PASS", t.name, t.file, t.line);
    failed_cases += state().current_failed ? 1 : 0;
  }
  std::printf("test cases: %zu, failed: %d; checks: %d, failed: %d\n", registry().size(), failed_cases,
              state().checks, state().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace Catch

#define CATCH_CAT2(a, b) a##b
#define CATCH_CAT(a, b) CATCH_CAT2(a, b)
#define TEST_CASE(name, ...)                                                                         \
  static void CATCH_CAT(catch_test_, __LINE__)();                                                    \
  static ::Catch::Registrar CATCH_CAT(catch_reg_, __LINE__)(name, __FILE__, __LINE__,                \
                                                            &CATCH_CAT(catch_test_, __LINE__));      \
  static void CATCH_CAT(catch_test_, __LINE__)()
#define CHECK(...) ::Catch::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::Catch::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) ::Catch::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE_FALSE(...) ::Catch::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg)                                                                                    \
  do {                                                                                               \
    std::ostringstream catch_os_;                                                                    \
    catch_os_ << msg;                                                                                \
    ::Catch::report(false, catch_os_.str().c_str(), __FILE__, __LINE__, true);                       \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                                  \
  do {                                                                                               \
    bool catch_ok_ = false;                                                                          \
    try {                                                                                            \
      static_cast<void>(expr);                                                                       \
    } catch (const type&) {                                                                          \
      catch_ok_ = true;                                                                              \
    } catch (...) {                                                                                  \
    }                                                                                                \
    ::Catch::report(catch_ok_, #expr " throws " #type, __FILE__, __LINE__, false);                   \
  } while (0)
#define CHECK_THROWS_WITH(expr, matcher)                                                             \
  do {                                                                                               \
    bool catch_ok_ = false;                                                                          \
    try {                                                                                            \
      static_cast<void>(expr);                                                                       \
    } catch (const std::exception& catch_e_) {                                                       \
      catch_ok_ = (matcher).match(catch_e_.what());                                                  \
    } catch (...) {                                                                                  \
    }                                                                                                \
    ::Catch::report(catch_ok_, #expr " throws with " #matcher, __FILE__, __LINE__, false);           \
  } while (0)
