// TEST INFRASTRUCTURE ONLY — main() for the mini-gtest harness (oracle/shim/gtest/gtest.h).
#include <gtest/gtest.h>

#include <cstring>

int main(int argc, char** argv) {
  std::string filter;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
  }
  int passed = 0, failed = 0;
  std::vector<std::string> failures;
  for (auto& t : testing::internal::registry()) {
    std::string full = t.suite + "." + t.name;
    if (!filter.empty() && full.rfind(filter, 0) != 0) continue;
    testing::internal::current_failed() = false;
    std::cout << "[ RUN      ] " << full << std::endl;
    try {
      t.fn();
    } catch (const std::exception& e) {
      std::cerr << "uncaught exception: " << e.what() << "\n";
      testing::internal::current_failed() = true;
    } catch (...) {
      std::cerr << "uncaught non-std exception\n";
      testing::internal::current_failed() = true;
    }
    if (testing::internal::current_failed()) {
      ++failed;
      failures.push_back(full);
      std::cout << "[  FAILED  ] " << full << std::endl;
    } else {
      ++passed;
      std::cout << "[       OK ] " << full << std::endl;
    }
  }
  std::cout << "[==========] " << passed << " passed, " << failed << " failed" << std::endl;
  for (auto& f : failures) std::cout << "[  FAILED  ] " << f << std::endl;
  return failed == 0 ? 0 : 1;
}
