// TEST INFRASTRUCTURE — a minimal GoogleTest-compatible shim (GTest is not in this image). It covers
// exactly what the reference's suite (proj/tests) uses: TEST / TEST_F, ::testing::Test with SetUp /
// TearDown / HasFailure, testing::TempDir, EXPECT_ / ASSERT_ {TRUE, FALSE, EQ, NE, LT, LE, GT, GE,
// NEAR, DOUBLE_EQ, THROW, NO_THROW}, ADD_FAILURE / FAIL, streamed messages, and a main() with
// --gtest_filter=POS[-NEG] (':'-separated wildcards). Not product code.
#ifndef MINI_GTEST_H
#define MINI_GTEST_H

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

class Message {
 public:
  template <class T>
  Message& operator<<(const T& v) {
    if constexpr (requires(std::ostream& o) { o << v; }) os_ << v;
    return *this;
  }
  std::string str() const { return os_.str(); }

 private:
  std::ostringstream os_;
};

namespace internal {

struct State {
  bool failed = false;
  int n_failures = 0;
  static State& get() {
    static State s;
    return s;
  }
};

inline void report(const char* file, int line, const std::string& what) {
  State::get().failed = true;
  ++State::get().n_failures;
  std::printf("%s:%d: Failure\n%s\n", file, line, what.c_str());
}

struct AssertHelper {
  const char* file;
  int line;
  std::string msg;
  AssertHelper(const char* f, int l, std::string m) : file(f), line(l), msg(std::move(m)) {}
  void operator=(const Message& m) const {
    const std::string extra = m.str();
    report(file, line, extra.empty() ? msg : msg + "\n" + extra);
  }
};

template <class T>
std::string show(const T& v) {
  if constexpr (requires(std::ostream& o) { o << v; }) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
  } else {
    return "<unprintable>";
  }
}

struct Result {
  bool ok;
  std::string msg;
};

#define MINI_GTEST_CMP_FN(NAME, OP)                                                                  \
  template <class A, class B>                                                                        \
  Result NAME(const char* ea, const char* eb, const A& a, const B& b) {                             \
    if (a OP b) return {true, {}};                                                                   \
    return {false, std::string("Expected: (") + ea + ") " #OP " (" + eb + "), actual: " + show(a) + \
                       " vs " + show(b)};                                                            \
  }
#pragma GCC diagnostic push
#pragma GCC diagnostic ignored "-Wsign-compare"
MINI_GTEST_CMP_FN(CmpEQ, ==)
MINI_GTEST_CMP_FN(CmpNE, !=)
MINI_GTEST_CMP_FN(CmpLT, <)
MINI_GTEST_CMP_FN(CmpLE, <=)
MINI_GTEST_CMP_FN(CmpGT, >)
MINI_GTEST_CMP_FN(CmpGE, >=)
#pragma GCC diagnostic pop

inline Result CmpNear(const char* ea, const char* eb, const char* et, double a, double b, double tol) {
  if (std::abs(a - b) <= tol) return {true, {}};
  return {false, std::string("The difference between ") + ea + " and " + eb + " is " + show(std::abs(a - b)) +
                     ", which exceeds " + et + " (" + show(tol) + "); " + show(a) + " vs " + show(b)};
}

inline Result CmpDoubleEq(const char* ea, const char* eb, double a, double b) {  // within 4 ULPs
  auto key = [](double x) {
    std::int64_t i;
    std::memcpy(&i, &x, 8);
    return i < 0 ? std::numeric_limits<std::int64_t>::min() - i : i;
  };
  if (a == b) return {true, {}};
  if (!std::isnan(a) && !std::isnan(b)) {
    const std::int64_t ka = key(a), kb = key(b);
    const std::uint64_t d = ka > kb ? static_cast<std::uint64_t>(ka) - static_cast<std::uint64_t>(kb)
                                    : static_cast<std::uint64_t>(kb) - static_cast<std::uint64_t>(ka);
    if (d <= 4) return {true, {}};
  }
  return {false, std::string("Expected equality (4 ULPs) of ") + ea + " and " + eb + ": " + show(a) + " vs " + show(b)};
}

}  // namespace internal

class Test {
 public:
  virtual ~Test() = default;
  virtual void SetUp() {}
  virtual void TearDown() {}
  virtual void TestBody() = 0;
  static bool HasFailure() { return internal::State::get().failed; }
};

inline std::string TempDir() {
  const char* t = std::getenv("TMPDIR");
  std::string d = t && *t ? t : "/tmp";
  if (d.back() != '/') d += '/';
  return d;
}

namespace internal {

struct TestInfo {
  std::string suite, name;
  std::function<Test*()> make;
};

inline std::vector<TestInfo>& registry() {
  static std::vector<TestInfo> r;
  return r;
}

struct Registrar {
  Registrar(const char* s, const char* n, std::function<Test*()> f) { registry().push_back({s, n, std::move(f)}); }
};

inline bool wild(const char* p, const char* s) {
  if (*p == 0) return *s == 0;
  if (*p == '*') return wild(p + 1, s) || (*s && wild(p, s + 1));
  if (*p == '?') return *s && wild(p + 1, s + 1);
  return *p == *s && wild(p + 1, s + 1);
}

inline bool any_match(const std::string& pats, const std::string& full) {
  std::size_t a = 0;
  while (a <= pats.size()) {
    std::size_t b = pats.find(':', a);
    if (b == std::string::npos) b = pats.size();
    if (b > a && wild(pats.substr(a, b - a).c_str(), full.c_str())) return true;
    a = b + 1;
  }
  return false;
}

inline int run_all(int argc, char** argv) {
  std::string pos = "*", neg;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--gtest_filter=", 0) == 0) {
      std::string f = a.substr(15);
      const auto d = f.find('-');
      pos = d == std::string::npos ? f : f.substr(0, d);
      neg = d == std::string::npos ? "" : f.substr(d + 1);
      if (pos.empty()) pos = "*";
    }
  }
  int run = 0;
  std::vector<std::string> failed;
  for (const TestInfo& t : registry()) {
    const std::string full = t.suite + "." + t.name;
    if (!any_match(pos, full) || (!neg.empty() && any_match(neg, full))) continue;
    ++run;
    State::get().failed = false;
    std::printf("[ RUN      ] %s\n", full.c_str());
    std::fflush(stdout);
    Test* obj = nullptr;
    try {
      obj = t.make();
      obj->SetUp();
      if (!State::get().failed) obj->TestBody();
      obj->TearDown();
    } catch (const std::exception& e) {
      report(__FILE__, __LINE__, std::string("uncaught exception: ") + e.what());
    } catch (...) {
      report(__FILE__, __LINE__, "uncaught non-standard exception");
    }
    delete obj;
    if (State::get().failed) failed.push_back(full);
    std::printf("%s %s\n", State::get().failed ? "[  FAILED  ]" : "[       OK ]", full.c_str());
    std::fflush(stdout);
  }
  std::printf("[==========] %d tests ran.\n[  PASSED  ] %d tests.\n", run, run - static_cast<int>(failed.size()));
  for (const auto& f : failed) std::printf("[  FAILED  ] %s\n", f.c_str());
  std::fflush(stdout);
  return failed.empty() ? 0 : 1;
}

}  // namespace internal
}  // namespace testing

#define MINI_GTEST_CLASS_(s, n) s##_##n##_Test
#define MINI_GTEST_DEFINE_(s, n, base)                                                                   \
  class MINI_GTEST_CLASS_(s, n) : public base {                                                          \
   public:                                                                                               \
    void TestBody() override;                                                                            \
  };                                                                                                     \
  static ::testing::internal::Registrar s##_##n##_registrar_(#s, #n, []() -> ::testing::Test* {          \
    return new MINI_GTEST_CLASS_(s, n);                                                                  \
  });                                                                                                    \
  void MINI_GTEST_CLASS_(s, n)::TestBody()

#define TEST(s, n) MINI_GTEST_DEFINE_(s, n, ::testing::Test)
#define TEST_F(f, n) MINI_GTEST_DEFINE_(f, n, f)

#define MINI_GTEST_CHECK_(expr, ret)                \
  if (auto mini_r_ = (expr); mini_r_.ok)            \
    ;                                               \
  else                                              \
    ret ::testing::internal::AssertHelper(__FILE__, __LINE__, mini_r_.msg) = ::testing::Message()

#define MINI_GTEST_BOOL_(cond, text, ret) \
  MINI_GTEST_CHECK_((::testing::internal::Result{static_cast<bool>(cond), text}), ret)

#define EXPECT_TRUE(c) MINI_GTEST_BOOL_(c, "Value of: " #c "\n  Actual: false", )
#define EXPECT_FALSE(c) MINI_GTEST_BOOL_(!(c), "Value of: " #c "\n  Actual: true", )
#define ASSERT_TRUE(c) MINI_GTEST_BOOL_(c, "Value of: " #c "\n  Actual: false", return)
#define ASSERT_FALSE(c) MINI_GTEST_BOOL_(!(c), "Value of: " #c "\n  Actual: true", return)

#define EXPECT_EQ(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpEQ(#a, #b, a, b), )
#define EXPECT_NE(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpNE(#a, #b, a, b), )
#define EXPECT_LT(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpLT(#a, #b, a, b), )
#define EXPECT_LE(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpLE(#a, #b, a, b), )
#define EXPECT_GT(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpGT(#a, #b, a, b), )
#define EXPECT_GE(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpGE(#a, #b, a, b), )
#define ASSERT_EQ(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpEQ(#a, #b, a, b), return)
#define ASSERT_NE(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpNE(#a, #b, a, b), return)
#define ASSERT_LT(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpLT(#a, #b, a, b), return)
#define ASSERT_LE(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpLE(#a, #b, a, b), return)
#define ASSERT_GT(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpGT(#a, #b, a, b), return)
#define ASSERT_GE(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpGE(#a, #b, a, b), return)

#define EXPECT_NEAR(a, b, t) MINI_GTEST_CHECK_(::testing::internal::CmpNear(#a, #b, #t, a, b, t), )
#define ASSERT_NEAR(a, b, t) MINI_GTEST_CHECK_(::testing::internal::CmpNear(#a, #b, #t, a, b, t), return)
#define EXPECT_DOUBLE_EQ(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpDoubleEq(#a, #b, a, b), )
#define ASSERT_DOUBLE_EQ(a, b) MINI_GTEST_CHECK_(::testing::internal::CmpDoubleEq(#a, #b, a, b), return)

#define MINI_GTEST_THROW_(stmt, type, ret)                                                             \
  MINI_GTEST_CHECK_(([&]() -> ::testing::internal::Result {                                            \
                      try {                                                                            \
                        stmt;                                                                          \
                      } catch (const type&) {                                                          \
                        return {true, {}};                                                             \
                      } catch (const std::exception& e) {                                              \
                        return {false, std::string("Expected: " #stmt " throws " #type                 \
                                                   ".\n  Actual: it throws a different type: ") +      \
                                           e.what()};                                                  \
                      } catch (...) {                                                                  \
                        return {false, "Expected: " #stmt " throws " #type ".\n  Actual: other type"}; \
                      }                                                                                \
                      return {false, "Expected: " #stmt " throws " #type ".\n  Actual: it throws nothing"}; \
                    }()),                                                                              \
                    ret)
#define EXPECT_THROW(stmt, type) MINI_GTEST_THROW_(stmt, type, )
#define ASSERT_THROW(stmt, type) MINI_GTEST_THROW_(stmt, type, return)

#define MINI_GTEST_NO_THROW_(stmt, ret)                                                             \
  MINI_GTEST_CHECK_(([&]() -> ::testing::internal::Result {                                         \
                      try {                                                                         \
                        stmt;                                                                       \
                      } catch (const std::exception& e) {                                           \
                        return {false, std::string("Expected: " #stmt " does not throw.\n  Actual: ") + \
                                           e.what()};                                               \
                      } catch (...) {                                                               \
                        return {false, "Expected: " #stmt " does not throw."};                      \
                      }                                                                             \
                      return {true, {}};                                                            \
                    }()),                                                                           \
                    ret)
#define EXPECT_NO_THROW(stmt) MINI_GTEST_NO_THROW_(stmt, )
#define ASSERT_NO_THROW(stmt) MINI_GTEST_NO_THROW_(stmt, return)

#define ADD_FAILURE() MINI_GTEST_BOOL_(false, "Failed", )
#define FAIL() MINI_GTEST_BOOL_(false, "Failed", return)
#define SUCCEED() static_cast<void>(0)

#endif  // MINI_GTEST_H
