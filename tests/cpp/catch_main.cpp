// Runner for the Catch2-compatible shim: runs every registered TEST_CASE,
// prints one line per case and a summary; exit code = failed case count.
#include <cstdio>
#include <cstring>
#include <exception>

#include "catch2/catch_amalgamated.hpp"

int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int failed_cases = 0, run = 0;
  for (const auto& tc : Catch::registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ++run;
    Catch::current_test() = tc.name;
    const int before = Catch::check_failures();
    bool threw = false;
    try {
      tc.fn();
    } catch (const Catch::RequireFailed&) {
    } catch (const std::exception& e) {
      threw = true;
      std::fprintf(stderr, "FAILED in \"%s\": unexpected exception: %s\n", tc.name, e.what());
    } catch (...) {
      threw = true;
      std::fprintf(stderr, "FAILED in \"%s\": unexpected non-std exception\n", tc.name);
    }
    const bool ok = !threw && Catch::check_failures() == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
  }
  std::printf("test cases: %d run, %d failed; checks: %d run, %d failed\n", run, failed_cases,
              Catch::check_count(), Catch::check_failures());
  return failed_cases;
}
