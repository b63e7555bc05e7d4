// TEST INFRASTRUCTURE ONLY — part of the parity oracle under oracle/.
//
// A minimal GoogleTest-compatible harness so that the reference's own unit
// and acceptance suites (`/root/reference/proj/tests/*.cpp`) compile and run
// unmodified against the oracle build. GTest is not installed in this image.
// Supported surface (exactly what those suites use): TEST, EXPECT_/ASSERT_
// {EQ,NE,LT,LE,GT,GE,TRUE,FALSE}, EXPECT_THROW, EXPECT_NO_THROW, streamed
// failure messages, testing::TempDir(), and a --gtest_filter=Suite.Name
// prefix filter in the bundled main.
#pragma once

#include <cstdlib>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

inline std::string TempDir() {
  const char* t = std::getenv("TEST_TMPDIR");
  return t ? std::string(t) : std::string("/tmp");
}

namespace internal {

struct TestInfo {
  std::string suite, name;
  std::function<void()> fn;
};

inline std::vector<TestInfo>& registry() {
  static std::vector<TestInfo> r;
  return r;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}

struct Registrar {
  Registrar(const char* suite, const char* name, std::function<void()> fn) {
    registry().push_back({suite, name, std::move(fn)});
  }
};

template <class T, class = void>
struct Printable : std::false_type {};
template <class T>
struct Printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <class T>
std::string show(const T& v) {
  if constexpr (Printable<T>::value) {
    std::ostringstream os;
    os << v;
    return os.str();
  } else {
    return "<unprintable>";
  }
}

// Collects a streamed message and reports the failure when destroyed.
class Failure {
 public:
  Failure(const char* file, int line, std::string what) : file_(file), line_(line), what_(std::move(what)) {}
  Failure(const Failure&) = delete;
  ~Failure() {
    current_failed() = true;
    std::cerr << file_ << ":" << line_ << ": Failure\n" << what_;
    std::string m = msg_.str();
    if (!m.empty()) std::cerr << "\n  " << m;
    std::cerr << "\n";
  }
  template <class T>
  Failure& operator<<(const T& v) {
    msg_ << v;
    return *this;
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
  std::ostringstream msg_;
};

// `return AssertReturn() = Failure(...) << ...;` ends a void test body.
struct AssertReturn {
  void operator=(const Failure&) const {}
};

struct CheckResult {
  bool ok;
  std::string what;
  explicit operator bool() const { return ok; }
};

template <class A, class B, class Op>
CheckResult cmp(const A& a, const B& b, const char* ea, const char* eb, const char* op, Op f) {
  if (f(a, b)) return {true, {}};
  std::ostringstream os;
  os << "Expected: (" << ea << ") " << op << " (" << eb << "), actual: " << show(a) << " vs "
     << show(b);
  return {false, os.str()};
}

inline CheckResult truth(bool v, const char* e, bool want) {
  if (v == want) return {true, {}};
  return {false, std::string("Value of: ") + e + "\n  Expected: " + (want ? "true" : "false")};
}

}  // namespace internal
}  // namespace testing

#define MGT_CONCAT2(a, b) a##b
#define MGT_CONCAT(a, b) MGT_CONCAT2(a, b)

#define TEST(suite, name)                                                           \
  static void MGT_CONCAT(mgt_test_##suite##_, name)();                              \
  static ::testing::internal::Registrar MGT_CONCAT(mgt_reg_##suite##_, name)(       \
      #suite, #name, &MGT_CONCAT(mgt_test_##suite##_, name));                       \
  static void MGT_CONCAT(mgt_test_##suite##_, name)()

#define MGT_EXPECT(res)                                                              \
  if (auto mgt_r = (res)) {                                                          \
  } else                                                                             \
    ::testing::internal::Failure(__FILE__, __LINE__, mgt_r.what)

#define MGT_ASSERT(res)                                                              \
  if (auto mgt_r = (res)) {                                                          \
  } else                                                                             \
    return ::testing::internal::AssertReturn() =                                     \
               ::testing::internal::Failure(__FILE__, __LINE__, mgt_r.what)

#define MGT_CMP(a, b, op)                                                            \
  ::testing::internal::cmp((a), (b), #a, #b, #op,                                    \
                           [](const auto& x, const auto& y) { return bool(x op y); })

#define EXPECT_EQ(a, b) MGT_EXPECT(MGT_CMP(a, b, ==))
#define EXPECT_NE(a, b) MGT_EXPECT(MGT_CMP(a, b, !=))
#define EXPECT_LT(a, b) MGT_EXPECT(MGT_CMP(a, b, <))
#define EXPECT_LE(a, b) MGT_EXPECT(MGT_CMP(a, b, <=))
#define EXPECT_GT(a, b) MGT_EXPECT(MGT_CMP(a, b, >))
#define EXPECT_GE(a, b) MGT_EXPECT(MGT_CMP(a, b, >=))
#define ASSERT_EQ(a, b) MGT_ASSERT(MGT_CMP(a, b, ==))
#define ASSERT_NE(a, b) MGT_ASSERT(MGT_CMP(a, b, !=))
#define ASSERT_LT(a, b) MGT_ASSERT(MGT_CMP(a, b, <))
#define ASSERT_LE(a, b) MGT_ASSERT(MGT_CMP(a, b, <=))
#define ASSERT_GT(a, b) MGT_ASSERT(MGT_CMP(a, b, >))
#define ASSERT_GE(a, b) MGT_ASSERT(MGT_CMP(a, b, >=))
#define EXPECT_TRUE(c) MGT_EXPECT(::testing::internal::truth(bool(c), #c, true))
#define EXPECT_FALSE(c) MGT_EXPECT(::testing::internal::truth(bool(c), #c, false))
#define ASSERT_TRUE(c) MGT_ASSERT(::testing::internal::truth(bool(c), #c, true))
#define ASSERT_FALSE(c) MGT_ASSERT(::testing::internal::truth(bool(c), #c, false))

#define FAIL()                                                                       \
  return ::testing::internal::AssertReturn() =                                       \
             ::testing::internal::Failure(__FILE__, __LINE__, "Failed")
#define ADD_FAILURE() ::testing::internal::Failure(__FILE__, __LINE__, "Failed")
#define SUCCEED() \
  if (true) {     \
  } else          \
    ::testing::internal::Failure(__FILE__, __LINE__, "")

#define EXPECT_THROW(stmt, exc)                                                      \
  MGT_EXPECT(([&]() -> ::testing::internal::CheckResult {                            \
    try {                                                                            \
      stmt;                                                                          \
    } catch (const exc&) {                                                           \
      return {true, {}};                                                             \
    } catch (...) {                                                                  \
      return {false, "Expected: " #stmt " throws " #exc "; it threw another type"};  \
    }                                                                                \
    return {false, "Expected: " #stmt " throws " #exc "; it threw nothing"};         \
  })())

#define EXPECT_NO_THROW(stmt)                                                        \
  MGT_EXPECT(([&]() -> ::testing::internal::CheckResult {                            \
    try {                                                                            \
      stmt;                                                                          \
    } catch (const std::exception& e) {                                              \
      return {false, std::string("Expected no throw from " #stmt "; got: ") + e.what()}; \
    } catch (...) {                                                                  \
      return {false, "Expected no throw from " #stmt};                               \
    }                                                                                \
    return {true, {}};                                                               \
  })())
