// Minimal GoogleTest-compatible harness (TEST, EXPECT_*/ASSERT_*, streaming
// messages) so the reference's own unit tests (proj/tests/test_*.cpp) can be
// compiled, unmodified, against the B200 drop-in (include/lsp/*.hpp).
// GoogleTest itself is not installed in this image.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

struct TestCase {
  std::string suite, name;
  std::function<void()> fn;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, std::function<void()> f) {
    registry().push_back({s, n, std::move(f)});
  }
};

struct AssertFatal {};

// Collects the streamed message; reports on destruction when failed.
class Check {
 public:
  Check(bool ok, const char* file, int line, const std::string& what, bool fatal)
      : ok_(ok), file_(file), line_(line), what_(what), fatal_(fatal) {}
  template <typename T>
  Check& operator<<(const T& v) {
    if (!ok_) msg_ << v;
    return *this;
  }
  ~Check() noexcept(false) {
    if (ok_) return;
    ++failures();
    std::cout << file_ << ":" << line_ << ": Failure\n  " << what_;
    const std::string m = msg_.str();
    if (!m.empty()) std::cout << "\n  " << m;
    std::cout << std::endl;
    if (fatal_ && !std::uncaught_exceptions()) throw AssertFatal{};
  }

 private:
  bool ok_;
  const char* file_;
  int line_;
  std::string what_;
  bool fatal_;
  std::ostringstream msg_;
};

template <typename T, typename = void>
struct Streamable : std::false_type {};
template <typename T>
struct Streamable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <typename T>
void print(std::ostream& s, const T& v) {
  if constexpr (Streamable<T>::value) {
    s << v;
  } else {
    s << "<value>";
  }
}
template <typename T>
void print(std::ostream& s, const std::vector<T>& v) {
  s << "{";
  for (size_t i = 0; i < v.size() && i < 16; ++i) {
    if (i) s << ", ";
    print(s, v[i]);
  }
  if (v.size() > 16) s << ", ...";
  s << "}";
}

template <typename A, typename B>
std::string describe(const char* op, const char* ea, const char* eb, const A& a, const B& b) {
  std::ostringstream s;
  s.precision(17);
  s << "Expected: (" << ea << ") " << op << " (" << eb << "), actual: ";
  print(s, a);
  s << " vs ";
  print(s, b);
  return s.str();
}

inline bool double_eq(double a, double b) {  // within 4 ulps, like gtest
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  int64_t ia, ib;
  std::memcpy(&ia, &a, 8);
  std::memcpy(&ib, &b, 8);
  if ((ia < 0) != (ib < 0)) return false;
  const int64_t d = ia > ib ? ia - ib : ib - ia;
  return d <= 4;
}

}  // namespace testing

#define LSPT_CAT2(a, b) a##b
#define LSPT_CAT(a, b) LSPT_CAT2(a, b)

#define TEST(suite, name)                                                           \
  static void LSPT_CAT(lspt_##suite##_, name)();                                    \
  static ::testing::Registrar LSPT_CAT(lspt_reg_##suite##_, name)(                  \
      #suite, #name, &LSPT_CAT(lspt_##suite##_, name));                             \
  static void LSPT_CAT(lspt_##suite##_, name)()

#define LSPT_CMP(op, a, b, fatal)                                                    \
  ::testing::Check(((a)op(b)), __FILE__, __LINE__,                                   \
                   ::testing::describe(#op, #a, #b, (a), (b)), fatal)

#define EXPECT_EQ(a, b) LSPT_CMP(==, a, b, false)
#define EXPECT_NE(a, b) LSPT_CMP(!=, a, b, false)
#define EXPECT_LT(a, b) LSPT_CMP(<, a, b, false)
#define EXPECT_LE(a, b) LSPT_CMP(<=, a, b, false)
#define EXPECT_GT(a, b) LSPT_CMP(>, a, b, false)
#define EXPECT_GE(a, b) LSPT_CMP(>=, a, b, false)
#define ASSERT_EQ(a, b) LSPT_CMP(==, a, b, true)
#define ASSERT_NE(a, b) LSPT_CMP(!=, a, b, true)
#define ASSERT_LT(a, b) LSPT_CMP(<, a, b, true)
#define ASSERT_LE(a, b) LSPT_CMP(<=, a, b, true)
#define ASSERT_GT(a, b) LSPT_CMP(>, a, b, true)
#define ASSERT_GE(a, b) LSPT_CMP(>=, a, b, true)
#define EXPECT_TRUE(c) ::testing::Check(static_cast<bool>(c), __FILE__, __LINE__, "Expected true: " #c, false)
#define EXPECT_FALSE(c) ::testing::Check(!static_cast<bool>(c), __FILE__, __LINE__, "Expected false: " #c, false)
#define ASSERT_TRUE(c) ::testing::Check(static_cast<bool>(c), __FILE__, __LINE__, "Expected true: " #c, true)
#define ASSERT_FALSE(c) ::testing::Check(!static_cast<bool>(c), __FILE__, __LINE__, "Expected false: " #c, true)
#define EXPECT_NEAR(a, b, tol)                                                          \
  ::testing::Check(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= (tol), \
                   __FILE__, __LINE__, ::testing::describe("~=", #a, #b, (a), (b)), false)
#define ASSERT_NEAR(a, b, tol)                                                          \
  ::testing::Check(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= (tol), \
                   __FILE__, __LINE__, ::testing::describe("~=", #a, #b, (a), (b)), true)
#define EXPECT_DOUBLE_EQ(a, b)                                                            \
  ::testing::Check(::testing::double_eq((a), (b)), __FILE__, __LINE__,                    \
                   ::testing::describe("==(4ulp)", #a, #b, (a), (b)), false)
#define LSPT_THROW(stmt, exc, fatal)                                                     \
  do {                                                                                   \
    bool lspt_ok = false;                                                                \
    try {                                                                                \
      stmt;                                                                              \
    } catch (const exc&) {                                                               \
      lspt_ok = true;                                                                    \
    } catch (...) {                                                                      \
    }                                                                                    \
    ::testing::Check(lspt_ok, __FILE__, __LINE__, "Expected " #stmt " to throw " #exc, fatal); \
  } while (0)
#define EXPECT_THROW(stmt, exc) LSPT_THROW(stmt, exc, false)
#define ASSERT_THROW(stmt, exc) LSPT_THROW(stmt, exc, true)
#define EXPECT_NO_THROW(stmt)                                                            \
  do {                                                                                   \
    bool lspt_ok = true;                                                                 \
    try {                                                                                \
      stmt;                                                                              \
    } catch (...) {                                                                      \
      lspt_ok = false;                                                                   \
    }                                                                                    \
    ::testing::Check(lspt_ok, __FILE__, __LINE__, "Expected no throw: " #stmt, false);   \
  } while (0)

// Test runner (link exactly one TU with LSPT_MAIN defined, or use main.cpp).
namespace testing {
inline int run_all() {
  int failed_tests = 0;
  for (auto& t : registry()) {
    const int before = failures();
    std::cout << "[ RUN      ] " << t.suite << "." << t.name << std::endl;
    try {
      t.fn();
    } catch (const AssertFatal&) {
    } catch (const std::exception& e) {
      ++failures();
      std::cout << "  uncaught exception: " << e.what() << std::endl;
    }
    const bool ok = failures() == before;
    if (!ok) ++failed_tests;
    std::cout << (ok ? "[       OK ] " : "[  FAILED  ] ") << t.suite << "." << t.name << std::endl;
  }
  std::cout << "[==========] " << registry().size() << " tests, " << failed_tests << " failed"
            << std::endl;
  return failed_tests == 0 ? 0 : 1;
}
}  // namespace testing
