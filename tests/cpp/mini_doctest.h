// The few doctest macros the reference's tests use (TEST_CASE, SUBCASE,
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, doctest::Approx), so the
// omega = 32 variants of its cases read like the originals.  vendor/doctest.h
// is absent from the reference tree; this is test tooling only.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace mini {
struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Register {
  Register(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline void fail(const char* expr, const char* file, int line, bool fatal) {
  std::printf("  %s:%d: CHECK failed: %s\n", file, line, expr);
  ++failures();
  if (fatal) throw RequireFailed{};
}
inline int run_all() {
  int bad_cases = 0;
  for (const Case& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("  unexpected exception: %s\n", e.what());
      ++failures();
    }
    const bool ok = failures() == before;
    bad_cases += !ok;
    std::printf("[%s] %s\n", ok ? "ok" : "FAILED", c.name);
  }
  std::printf("%zu cases, %d failed\n", registry().size(), bad_cases);
  return bad_cases ? 1 : 0;
}
}  // namespace mini

namespace doctest {
struct Approx {
  double v, eps = 1e-5;
  explicit Approx(double value) : v(value) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::abs(a - b.v) <= b.eps * (1.0 + std::max(std::abs(a), std::abs(b.v)));
  }
};
}  // namespace doctest

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name)                                                                 \
  static void MINI_CAT(mini_case_, __LINE__)();                                         \
  static mini::Register MINI_CAT(mini_reg_, __LINE__)(name, &MINI_CAT(mini_case_, __LINE__)); \
  static void MINI_CAT(mini_case_, __LINE__)()
#define SUBCASE(name) if (true)
#define CHECK(e) ((e) ? (void)0 : mini::fail(#e, __FILE__, __LINE__, false))
#define CHECK_FALSE(e) ((!(e)) ? (void)0 : mini::fail("!(" #e ")", __FILE__, __LINE__, false))
#define REQUIRE(e) ((e) ? (void)0 : mini::fail(#e, __FILE__, __LINE__, true))
#define CHECK_THROWS_AS(e, T)                                          \
  do {                                                                 \
    bool thrown_ = false;                                              \
    try {                                                              \
      (void)(e);                                                       \
    } catch (const T&) {                                               \
      thrown_ = true;                                                  \
    } catch (...) {                                                    \
    }                                                                  \
    if (!thrown_) mini::fail(#e " throws " #T, __FILE__, __LINE__, false); \
  } while (0)
