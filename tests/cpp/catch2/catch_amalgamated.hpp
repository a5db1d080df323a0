// Minimal Catch2-v3-compatible test harness (TEST_CASE, CHECK, REQUIRE,
// CHECK_FALSE, CHECK_THROWS_AS, REQUIRE_THROWS_AS, CHECK_NOTHROW, FAIL, INFO).
// The Catch2 amalgamation the reference expects (proj/.gitignore:2) is not
// vendored and there is no network, so this stand-in lets the reference's own
// test files (proj/tests/test_seq.cpp, test_parallel.cpp) and this repo's C++
// parity tests compile unchanged. Link with tests/cpp/catch_main.cpp.
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {
struct TestCase { const char* name; void (*fn)(); const char* file; int line; };
inline std::vector<TestCase>& registry() { static std::vector<TestCase> r; return r; }
struct Registrar { Registrar(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); } };
struct AbortTest {};
struct State { long checks = 0, failures = 0; bool case_failed = false; std::string info; };
inline State& state() { static State s; return s; }
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  State& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED: %s%s%s\n", file, line, expr, s.info.empty() ? "" : "  [", s.info.empty() ? "" : (s.info + "]").c_str());
    if (fatal) throw AbortTest{};
  }
}
}  // namespace catch_shim

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                                   \
  static void CATCH_SHIM_CAT(catch_shim_test_, __LINE__)();                                    \
  static catch_shim::Registrar CATCH_SHIM_CAT(catch_shim_reg_, __LINE__)(                      \
      name, &CATCH_SHIM_CAT(catch_shim_test_, __LINE__), __FILE__, __LINE__);                   \
  static void CATCH_SHIM_CAT(catch_shim_test_, __LINE__)()
#define CATCH_SHIM_CHECK(expr, fatal)                                                          \
  do {                                                                                         \
    bool catch_shim_ok = false;                                                                \
    try { catch_shim_ok = static_cast<bool>(expr); } catch (const std::exception& e) {         \
      std::fprintf(stderr, "unexpected exception: %s\n", e.what()); }                          \
    catch_shim::report(catch_shim_ok, #expr, __FILE__, __LINE__, fatal);                       \
  } while (0)
#define CHECK(...) CATCH_SHIM_CHECK((__VA_ARGS__), false)
#define REQUIRE(...) CATCH_SHIM_CHECK((__VA_ARGS__), true)
#define CHECK_FALSE(...) CATCH_SHIM_CHECK(!(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) CATCH_SHIM_CHECK(!(__VA_ARGS__), true)
#define CATCH_SHIM_THROWS_AS(expr, type, fatal)                                                \
  do {                                                                                         \
    bool catch_shim_ok = false;                                                                \
    try { static_cast<void>(expr); } catch (const type&) { catch_shim_ok = true; } catch (...) {} \
    catch_shim::report(catch_shim_ok, #expr " throws " #type, __FILE__, __LINE__, fatal);      \
  } while (0)
#define CHECK_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS(expr, type, false)
#define REQUIRE_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS(expr, type, true)
#define CHECK_NOTHROW(expr)                                                                    \
  do {                                                                                         \
    bool catch_shim_ok = true;                                                                 \
    try { static_cast<void>(expr); } catch (...) { catch_shim_ok = false; }                    \
    catch_shim::report(catch_shim_ok, #expr " does not throw", __FILE__, __LINE__, false);     \
  } while (0)
#define FAIL(msg) catch_shim::report(false, msg, __FILE__, __LINE__, true)
#define INFO(...)                                                                              \
  do { std::ostringstream catch_shim_os; catch_shim_os << __VA_ARGS__;                         \
       catch_shim::state().info = catch_shim_os.str(); } while (0)
