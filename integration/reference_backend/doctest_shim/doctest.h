// doctest.h -- a minimal stand-in for the doctest test framework (not in
// this image), implementing only what the reference's unit tests use:
// TEST_CASE, CHECK, CHECK_FALSE, CHECK_THROWS_AS, REQUIRE, CAPTURE and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  It lets proj/tests/test_lookup.cpp,
// test_oracle.cpp and test_tables.cpp compile and run unchanged against a
// roster with the cuda backend registered (integration/reference_backend).
// Written for this repository; not the doctest library's source.
#pragma once
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace mini_doctest {

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

struct State {
  long checks = 0, failures = 0;
  bool case_failed = false;
  std::vector<std::function<std::string()>> captures;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* macro, const char* expr, const char* file, int line, bool fatal) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  s.case_failed = true;
  std::printf("%s:%d: ERROR: %s( %s ) failed\n", file, line, macro, expr);
  for (auto& c : s.captures) std::printf("  with %s\n", c().c_str());
  if (fatal) throw RequireFailed{};
}

template <class T>
struct Capture {
  const char* name;
  const T& value;
  Capture(const char* n, const T& v) : name(n), value(v) {
    state().captures.push_back([this] {
      std::ostringstream o;
      o << name << " := " << value;
      return o.str();
    });
  }
  ~Capture() { state().captures.pop_back(); }
};

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    state().case_failed = false;
    state().captures.clear();
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("%s:%d: ERROR: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
      state().case_failed = true;
    }
    if (state().case_failed) ++failed_cases;
    std::printf("[%s] %s\n", state().case_failed ? "FAIL" : " ok ", c.name);
  }
  std::printf("test cases: %zu | %zu passed | %d failed; assertions: %ld | %ld failed\n", registry().size(),
              registry().size() - failed_cases, failed_cases, state().checks, state().failures);
  return failed_cases ? 1 : 0;
}

}  // namespace mini_doctest

#define MD_CAT2(a, b) a##b
#define MD_CAT(a, b) MD_CAT2(a, b)
#define MD_TEST_CASE_IMPL(fn, name)                                                           \
  static void fn();                                                                           \
  static mini_doctest::Registrar MD_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);             \
  static void fn()
#define TEST_CASE(name) MD_TEST_CASE_IMPL(MD_CAT(md_test_, __COUNTER__), name)
#define CHECK(...) mini_doctest::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  mini_doctest::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
  mini_doctest::report(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                                   \
  do {                                                                                               \
    bool md_thrown = false;                                                                          \
    try {                                                                                            \
      (void)(expr);                                                                                  \
    } catch (const __VA_ARGS__&) {                                                                   \
      md_thrown = true;                                                                              \
    } catch (...) {                                                                                  \
    }                                                                                                \
    mini_doctest::report(md_thrown, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define CAPTURE(x) mini_doctest::Capture<std::decay_t<decltype(x)>> MD_CAT(md_capture_, __COUNTER__)(#x, x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return mini_doctest::run_all(); }
#endif
