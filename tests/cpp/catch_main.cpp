// Runner for the Catch2 stand-in: `prog [substring]` runs matching TEST_CASEs
// and prints one "ok|FAIL <name>" line per case plus a summary; exit 1 on failure.
#include <catch2/catch_amalgamated.hpp>
#include <cstring>

int main(int argc, char** argv) {
  std::setvbuf(stdout, nullptr, _IOLBF, 0);
  const char* filter = argc > 1 ? argv[1] : nullptr;
  long cases = 0, failed_cases = 0;
  for (const auto& tc : catch_shim::registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    auto& s = catch_shim::state();
    s.case_failed = false;
    s.info.clear();
    ++cases;
    try {
      tc.fn();
    } catch (const catch_shim::AbortTest&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: unexpected exception in '%s': %s\n", tc.file, tc.line, tc.name, e.what());
      s.case_failed = true;
      ++s.failures;
    }
    if (s.case_failed) ++failed_cases;
    std::printf("%s %s\n", s.case_failed ? "FAIL" : "ok", tc.name);
  }
  auto& s = catch_shim::state();
  std::printf("test cases: %ld | %ld passed | %ld failed ; assertions: %ld | %ld failed\n", cases,
              cases - failed_cases, failed_cases, s.checks, s.failures);
  return failed_cases ? 1 : 0;
}
