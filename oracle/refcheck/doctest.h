// Minimal doctest-API stand-in (TEST INFRASTRUCTURE; the reference's
// vendor/doctest is not shipped, proj/.gitignore:2).  Implements what the
// reference's hot-path tests use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS
// and doctest::Approx (default epsilon 100 * FLT_EPSILON, scale 1, as doctest
// 2.x).  SURVEY.md Appendix B.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
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
  bool eq(double lhs) const {
    return std::fabs(lhs - value_) < eps_ * (scale_ + std::fmax(std::fabs(lhs), std::fabs(value_)));
  }
  friend bool operator==(double l, const Approx& r) { return r.eq(l); }
  friend bool operator==(const Approx& l, double r) { return l.eq(r); }
  friend bool operator!=(double l, const Approx& r) { return !r.eq(l); }
  friend bool operator!=(const Approx& l, double r) { return !l.eq(r); }
  friend bool operator<=(double l, const Approx& r) { return l < r.value_ || r.eq(l); }
  friend bool operator<=(const Approx& l, double r) { return l.value_ < r || l.eq(r); }
  friend bool operator>=(double l, const Approx& r) { return l > r.value_ || r.eq(l); }
  friend bool operator>=(const Approx& l, double r) { return l.value_ > r || l.eq(r); }
  friend bool operator<(double l, const Approx& r) { return l < r.value_ && !r.eq(l); }
  friend bool operator<(const Approx& l, double r) { return l.value_ < r && !l.eq(r); }
  friend bool operator>(double l, const Approx& r) { return l > r.value_ && !r.eq(l); }
  friend bool operator>(const Approx& l, double r) { return l.value_ > r && !l.eq(r); }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

namespace detail {
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
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
struct RequireFailed {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline long& assertions() {
  static long a = 0;
  return a;
}
inline void report(const char* file, int line, const char* what, const char* expr) {
  ++failures();
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, what, expr);
}
}  // namespace detail

inline int run(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
  int cases = 0, failed = 0;
  for (const auto& c : detail::registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    const int before = detail::failures();
    try {
      c.fn();
    } catch (const detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++detail::failures();
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
    }
    if (detail::failures() != before) {
      ++failed;
      std::fprintf(stderr, "  in TEST CASE \"%s\"\n", c.name);
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", cases, cases - failed, failed);
  std::printf("[doctest] assertions: %ld | %ld passed | %d failed\n", detail::assertions(),
              detail::assertions() - detail::failures(), detail::failures());
  return failed ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                    \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                      \
  static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                 \
      name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_case_, __LINE__));                    \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define CHECK(...)                                                                         \
  do {                                                                                     \
    ++::doctest::detail::assertions();                                                     \
    if (!(__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, "CHECK", #__VA_ARGS__); \
  } while (0)
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    ++::doctest::detail::assertions();                                                     \
    if (!(__VA_ARGS__)) {                                                                  \
      ::doctest::detail::report(__FILE__, __LINE__, "REQUIRE", #__VA_ARGS__);              \
      throw ::doctest::detail::RequireFailed{};                                            \
    }                                                                                      \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, type)                                                        \
  do {                                                                                     \
    ++::doctest::detail::assertions();                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const type&) {                                                                \
      doctest_ok_ = true;                                                                  \
    } catch (...) {                                                                        \
    }                                                                                      \
    if (!doctest_ok_) ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::run(argc, argv); }
#endif
