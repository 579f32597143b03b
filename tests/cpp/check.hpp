// Minimal test macros for the C++ host suites (the reference uses doctest,
// which is not in this image; only CHECK / CHECK_THROWS / SKIP are needed).
#pragma once

#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace ffcheck {

struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int n = 0;
  return n;
}
inline int& checks() {
  static int n = 0;
  return n;
}
struct Register {
  Register(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
struct Skip {
  std::string why;
};

inline int run_all() {
  int failed_cases = 0, skipped = 0;
  for (const Case& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const Skip& s) {
      std::printf("SKIP %s: %s\n", c.name, s.why.c_str());
      ++skipped;
      continue;
    } catch (const std::exception& e) {
      std::printf("FAIL %s: unexpected exception: %s\n", c.name, e.what());
      ++failures();
    }
    if (failures() != before) {
      ++failed_cases;
      std::printf("FAIL %s\n", c.name);
    } else {
      std::printf("ok   %s\n", c.name);
    }
  }
  std::printf("%zu cases, %d failed, %d skipped, %d checks\n", registry().size(), failed_cases, skipped, checks());
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace ffcheck

#define FF_CAT2(a, b) a##b
#define FF_CAT(a, b) FF_CAT2(a, b)
#define TEST_CASE(name)                                                         \
  static void FF_CAT(ff_case_, __LINE__)();                                     \
  static ffcheck::Register FF_CAT(ff_reg_, __LINE__)(name, FF_CAT(ff_case_, __LINE__)); \
  static void FF_CAT(ff_case_, __LINE__)()
#define CHECK(cond)                                                             \
  do {                                                                          \
    ++ffcheck::checks();                                                        \
    if (!(cond)) {                                                              \
      ++ffcheck::failures();                                                    \
      std::printf("  %s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond);    \
    }                                                                           \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                             \
  do {                                                                          \
    ++ffcheck::checks();                                                        \
    bool thrown_ = false;                                                       \
    try {                                                                       \
      (void)(expr);                                                             \
    } catch (const type&) {                                                     \
      thrown_ = true;                                                           \
    } catch (...) {                                                             \
    }                                                                           \
    if (!thrown_) {                                                             \
      ++ffcheck::failures();                                                    \
      std::printf("  %s:%d: %s did not throw %s\n", __FILE__, __LINE__, #expr, #type); \
    }                                                                           \
  } while (0)
#define SKIP(why) throw ffcheck::Skip{why}
