// main() for the GoogleTest shim -- TEST INFRASTRUCTURE ONLY.
#include <gtest/gtest.h>

#include <cstdio>
#include <exception>

int main() {
  int passed = 0, failed = 0;
  for (const auto& c : gshim::registry()) {
    gshim::current_failed() = false;
    try {
      c.fn();
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s.%s: uncaught exception: %s\n", c.suite, c.name, e.what());
      gshim::current_failed() = true;
    }
    if (gshim::current_failed()) {
      ++failed;
      std::printf("[  FAILED  ] %s.%s\n", c.suite, c.name);
    } else {
      ++passed;
      std::printf("[       OK ] %s.%s\n", c.suite, c.name);
    }
  }
  std::printf("[==========] %d passed, %d failed\n", passed, failed);
  return failed == 0 ? 0 : 1;
}
