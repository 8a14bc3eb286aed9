// Minimal Catch2-compatible test harness (our own, ~150 lines) so the
// reference's Catch2 unit tests (R/tests/test_*.cpp) compile UNMODIFIED
// against this repo's drop-in texforge:: headers. It implements only what
// those tests use: TEST_CASE, CHECK/CHECK_FALSE/REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH, CHECK_NOTHROW, CHECK_THAT, FAIL, Catch::Approx
// (epsilon/margin) and Catch::Matchers::ContainsSubstring.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace Catch {

struct TestCase {
  const char* name;
  void (*fn)();
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};

inline int& check_failures() {
  static int n = 0;
  return n;
}
inline int& check_count() {
  static int n = 0;
  return n;
}
inline const char*& current_test() {
  static const char* t = "";
  return t;
}
inline void report(bool ok, const char* what, const char* file, int line, const std::string& extra = "") {
  ++check_count();
  if (ok) return;
  ++check_failures();
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s%s%s\n", file, line, current_test(), what,
               extra.empty() ? "" : " -- ", extra.c_str());
}

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) { return a.equals(lhs); }
  friend bool operator==(const Approx& a, double rhs) { return a.equals(rhs); }
  friend bool operator!=(double lhs, const Approx& a) { return !a.equals(lhs); }

 private:
  bool equals(double x) const {
    const double diff = std::fabs(x - value_);
    if (diff <= margin_) return true;
    return diff <= eps_ * std::fabs(std::isinf(value_) ? 0.0 : value_);
  }
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100.0;
  double margin_ = 0.0;
};

namespace Matchers {
struct ContainsSubstring {
  std::string needle;
  explicit ContainsSubstring(std::string s) : needle(std::move(s)) {}
  bool match(const std::string& s) const { return s.find(needle) != std::string::npos; }
};
}  // namespace Matchers

}  // namespace Catch

#define CATCH_CAT2(a, b) a##b
#define CATCH_CAT(a, b) CATCH_CAT2(a, b)
#define TEST_CASE(name, ...)                                                                  \
  static void CATCH_CAT(catch_test_, __LINE__)();                                             \
  static ::Catch::Registrar CATCH_CAT(catch_reg_, __LINE__)(name, &CATCH_CAT(catch_test_, __LINE__)); \
  static void CATCH_CAT(catch_test_, __LINE__)()

#define CHECK(...) ::Catch::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::Catch::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                           \
  do {                                                                         \
    const bool catch_ok_ = static_cast<bool>(__VA_ARGS__);                     \
    ::Catch::report(catch_ok_, #__VA_ARGS__, __FILE__, __LINE__);              \
    if (!catch_ok_) throw ::Catch::RequireFailed{};                            \
  } while (0)
#define FAIL(msg)                                                              \
  do {                                                                         \
    ::Catch::report(false, "FAIL", __FILE__, __LINE__, msg);                   \
    throw ::Catch::RequireFailed{};                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                             \
  do {                                                                         \
    bool catch_ok_ = false;                                                    \
    std::string catch_msg_ = "nothing thrown";                                 \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                             \
      catch_ok_ = true;                                                        \
    } catch (const std::exception& e) {                                        \
      catch_msg_ = std::string("other exception: ") + e.what();               \
    } catch (...) {                                                            \
      catch_msg_ = "unknown exception";                                        \
    }                                                                          \
    ::Catch::report(catch_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, catch_ok_ ? "" : catch_msg_); \
  } while (0)
#define CHECK_THROWS_WITH(expr, matcher)                                       \
  do {                                                                         \
    bool catch_ok_ = false;                                                    \
    std::string catch_msg_ = "nothing thrown";                                 \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const std::exception& e) {                                        \
      catch_msg_ = e.what();                                                   \
      catch_ok_ = (matcher).match(catch_msg_);                                 \
    }                                                                          \
    ::Catch::report(catch_ok_, #expr " throws with " #matcher, __FILE__, __LINE__, catch_ok_ ? "" : catch_msg_); \
  } while (0)
#define CHECK_NOTHROW(...)                                                     \
  do {                                                                         \
    bool catch_ok_ = true;                                                     \
    std::string catch_msg_;                                                    \
    try {                                                                      \
      (void)(__VA_ARGS__);                                                     \
    } catch (const std::exception& e) {                                        \
      catch_ok_ = false;                                                       \
      catch_msg_ = e.what();                                                   \
    }                                                                          \
    ::Catch::report(catch_ok_, #__VA_ARGS__ " does not throw", __FILE__, __LINE__, catch_msg_); \
  } while (0)
#define CHECK_THAT(arg, matcher) \
  ::Catch::report((matcher).match(std::string(arg)), #arg " matches " #matcher, __FILE__, __LINE__, std::string(arg))
