// Minimal GoogleTest-compatible harness (TEST, EXPECT_* / ASSERT_*, streamed
// failure messages, a main that runs every registered test), so the
// reference's own gtest suites compile and run against the CUDA-backed
// mirror without GoogleTest, which this image does not have.  Test
// infrastructure only.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace mini_gtest {

struct TestCase {
  const char* suite;
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}

struct Registrar {
  Registrar(const char* suite, const char* name, void (*fn)()) { registry().push_back({suite, name, fn}); }
};

template <typename T, typename = void>
struct printable : std::false_type {};
template <typename T>
struct printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <typename T>
std::string show(const T& v) {
  if constexpr (printable<T>::value) {
    std::ostringstream o;
    o << v;
    return o.str();
  } else {
    return "<value>";
  }
}

// Collects the streamed message; reports on destruction of the assignment.
struct Message {
  std::ostringstream os;
  template <typename T>
  Message& operator<<(const T& v) {
    if constexpr (printable<T>::value) os << v;
    return *this;
  }
};

struct Failure {
  const char* file;
  int line;
  std::string what;
  // `Failure(...) = Message() << ...` prints once the message is complete.
  void operator=(const Message& m) const {
    current_failed() = true;
    std::printf("%s:%d: Failure\n  %s\n  %s\n", file, line, what.c_str(), m.os.str().c_str());
  }
};

template <typename A, typename B>
std::string cmp_text(const char* op, const char* ea, const char* eb, const A& a, const B& b) {
  return std::string("Expected: (") + ea + ") " + op + " (" + eb + "), actual: " + show(a) + " vs " + show(b);
}

// --gtest_filter=A.*:B.c (':'-separated patterns, '*' wildcard), as GoogleTest.
inline bool glob_match(const char* p, const char* s) {
  if (*p == '\0') return *s == '\0';
  if (*p == '*') return glob_match(p + 1, s) || (*s && glob_match(p, s + 1));
  return *s == *p && glob_match(p + 1, s + 1);
}
inline bool selected(const std::string& filter, const std::string& name) {
  if (filter.empty()) return true;
  std::size_t b = 0;
  while (b <= filter.size()) {
    const std::size_t e = filter.find(':', b);
    const std::string pat = filter.substr(b, e == std::string::npos ? std::string::npos : e - b);
    if (glob_match(pat.c_str(), name.c_str())) return true;
    if (e == std::string::npos) break;
    b = e + 1;
  }
  return false;
}

inline int run_all(const std::string& filter = "") {
  int failed = 0;
  std::size_t ran = 0;
  for (const auto& t : registry()) {
    if (!selected(filter, std::string(t.suite) + "." + t.name)) continue;
    ++ran;
    current_failed() = false;
    std::printf("[ RUN      ] %s.%s\n", t.suite, t.name);
    try {
      t.fn();
    } catch (const std::exception& e) {
      current_failed() = true;
      std::printf("  uncaught exception: %s\n", e.what());
    } catch (...) {
      current_failed() = true;
      std::printf("  uncaught exception\n");
    }
    std::printf("%s %s.%s\n", current_failed() ? "[  FAILED  ]" : "[       OK ]", t.suite, t.name);
    failed += current_failed() ? 1 : 0;
  }
  std::printf("[==========] %zu tests, %zu passed, %d failed\n", ran, ran - static_cast<std::size_t>(failed),
              failed);
  return failed ? 1 : 0;
}

}  // namespace mini_gtest

#define TEST(suite, name)                                                                 \
  static void suite##_##name##_body();                                                    \
  static ::mini_gtest::Registrar suite##_##name##_reg(#suite, #name, &suite##_##name##_body); \
  static void suite##_##name##_body()

#define MG_CHECK_(cond, text, on_fail) \
  if (cond) {                          \
  } else                               \
    on_fail ::mini_gtest::Failure{__FILE__, __LINE__, text} = ::mini_gtest::Message()

#define MG_CMP_(op, a, b, on_fail)                                                              \
  MG_CHECK_(((a)op(b)), ::mini_gtest::cmp_text(#op, #a, #b, (a), (b)), on_fail)

#define EXPECT_TRUE(c) MG_CHECK_(static_cast<bool>(c), std::string("Expected true: ") + #c, )
#define EXPECT_FALSE(c) MG_CHECK_(!static_cast<bool>(c), std::string("Expected false: ") + #c, )
#define ASSERT_TRUE(c) MG_CHECK_(static_cast<bool>(c), std::string("Expected true: ") + #c, return)
#define ASSERT_FALSE(c) MG_CHECK_(!static_cast<bool>(c), std::string("Expected false: ") + #c, return)
#define EXPECT_EQ(a, b) MG_CMP_(==, a, b, )
#define EXPECT_NE(a, b) MG_CMP_(!=, a, b, )
#define EXPECT_LT(a, b) MG_CMP_(<, a, b, )
#define EXPECT_LE(a, b) MG_CMP_(<=, a, b, )
#define EXPECT_GT(a, b) MG_CMP_(>, a, b, )
#define EXPECT_GE(a, b) MG_CMP_(>=, a, b, )
#define ASSERT_EQ(a, b) MG_CMP_(==, a, b, return)
#define ASSERT_NE(a, b) MG_CMP_(!=, a, b, return)
#define ASSERT_LT(a, b) MG_CMP_(<, a, b, return)
#define ASSERT_LE(a, b) MG_CMP_(<=, a, b, return)
#define ASSERT_GT(a, b) MG_CMP_(>, a, b, return)
#define ASSERT_GE(a, b) MG_CMP_(>=, a, b, return)
#define EXPECT_NEAR(a, b, tol) \
  MG_CHECK_(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= (tol), \
            ::mini_gtest::cmp_text("~=", #a, #b, (a), (b)), )
#define ASSERT_NEAR(a, b, tol) \
  MG_CHECK_(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= (tol), \
            ::mini_gtest::cmp_text("~=", #a, #b, (a), (b)), return)
#define EXPECT_FLOAT_EQ(a, b) EXPECT_EQ(static_cast<float>(a), static_cast<float>(b))
#define MG_THROW_(stmt, exc, on_fail)                                   \
  MG_CHECK_(([&]() -> bool {                                            \
              try {                                                     \
                stmt;                                                   \
              } catch (const exc&) {                                    \
                return true;                                            \
              } catch (...) {                                           \
                return false;                                           \
              }                                                         \
              return false;                                             \
            }()),                                                       \
            std::string("Expected ") + #stmt + " to throw " + #exc, on_fail)
#define EXPECT_THROW(stmt, exc) MG_THROW_(stmt, exc, )
#define ASSERT_THROW(stmt, exc) MG_THROW_(stmt, exc, return)
#define MG_NOTHROW_(stmt, on_fail)                                      \
  MG_CHECK_(([&]() -> bool {                                            \
              try {                                                     \
                stmt;                                                   \
              } catch (...) {                                           \
                return false;                                           \
              }                                                         \
              return true;                                              \
            }()),                                                       \
            std::string("Expected no throw: ") + #stmt, on_fail)
#define EXPECT_NO_THROW(stmt) MG_NOTHROW_(stmt, )
#define ASSERT_NO_THROW(stmt) MG_NOTHROW_(stmt, return)

int main(int argc, char** argv) {
  std::string filter;
  for (int i = 1; i < argc; ++i)
    if (std::string(argv[i]).rfind("--gtest_filter=", 0) == 0) filter = std::string(argv[i]).substr(15);
  return ::mini_gtest::run_all(filter);
}
