// Minimal GoogleTest-compatible shim (TEST test infrastructure only).
//
// GoogleTest is not installed in this image and there is no network, so the
// reference's unit suites (/root/reference/proj/tests/*_test.cpp) are
// compiled against this header instead. It implements exactly the subset
// those suites use: TEST, EXPECT_/ASSERT_ {EQ,NE,LT,LE,GT,GE,TRUE,FALSE},
// EXPECT_NEAR, EXPECT_DOUBLE_EQ, EXPECT_STREQ, EXPECT_THROW,
// EXPECT_NO_THROW, `<< message` streaming, and a main() that runs every
// registered test and returns non-zero on any failure.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace gtest_shim {

struct Registry {
  struct Case {
    std::string name;
    std::function<void()> body;
  };
  std::vector<Case> cases;
  int failures_in_case = 0;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

struct Registrar {
  Registrar(const char* suite, const char* name, void (*fn)()) {
    Registry::get().cases.push_back({std::string(suite) + "." + name, fn});
  }
};

class Message {
 public:
  template <typename T>
  Message& operator<<(const T& v) {
    os_ << v;
    return *this;
  }
  std::string str() const { return os_.str(); }

 private:
  std::ostringstream os_;
};

class Failure {
 public:
  Failure(const char* file, int line, const char* what)
      : file_(file), line_(line), what_(what) {}
  // `return Failure(...) = Message() << ...;` -> records and yields void.
  void operator=(const Message& m) const {
    ++Registry::get().failures_in_case;
    std::printf("%s:%d: Failure: %s %s\n", file_, line_, what_,
                m.str().c_str());
  }

 private:
  const char* file_;
  int line_;
  const char* what_;
};

inline bool double_eq(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  auto biased = [](double x) {
    std::uint64_t u;
    std::memcpy(&u, &x, sizeof u);
    const std::uint64_t sign = std::uint64_t{1} << 63;
    return (u & sign) ? ~u + 1 : u | sign;
  };
  const std::uint64_t x = biased(a), y = biased(b);
  return (x > y ? x - y : y - x) <= 4;
}

template <typename F>
bool throws_nothing(F&& f) {
  try {
    f();
    return true;
  } catch (...) {
    return false;
  }
}

}  // namespace gtest_shim

#define GSHIM_CAT2(a, b) a##b
#define GSHIM_CAT(a, b) GSHIM_CAT2(a, b)

#define TEST(suite, name)                                                  \
  static void GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, GSHIM_CAT(_, name)))(); \
  static ::gtest_shim::Registrar GSHIM_CAT(                                \
      gshim_reg_, GSHIM_CAT(suite, GSHIM_CAT(_, name)))(                   \
      #suite, #name, &GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, GSHIM_CAT(_, name)))); \
  static void GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, GSHIM_CAT(_, name)))()

#define GSHIM_CHECK(cond, text, on_fail) \
  if (cond)                              \
    ;                                    \
  else                                   \
    on_fail ::gtest_shim::Failure(__FILE__, __LINE__, text) = ::gtest_shim::Message()

#define GSHIM_EXPECT(cond, text) GSHIM_CHECK(cond, text, )
#define GSHIM_ASSERT(cond, text) GSHIM_CHECK(cond, text, return)

#define EXPECT_TRUE(c) GSHIM_EXPECT(static_cast<bool>(c), "EXPECT_TRUE(" #c ")")
#define EXPECT_FALSE(c) GSHIM_EXPECT(!static_cast<bool>(c), "EXPECT_FALSE(" #c ")")
#define ASSERT_TRUE(c) GSHIM_ASSERT(static_cast<bool>(c), "ASSERT_TRUE(" #c ")")
#define ASSERT_FALSE(c) GSHIM_ASSERT(!static_cast<bool>(c), "ASSERT_FALSE(" #c ")")

#define EXPECT_EQ(a, b) GSHIM_EXPECT((a) == (b), "EXPECT_EQ(" #a ", " #b ")")
#define EXPECT_NE(a, b) GSHIM_EXPECT((a) != (b), "EXPECT_NE(" #a ", " #b ")")
#define EXPECT_LT(a, b) GSHIM_EXPECT((a) < (b), "EXPECT_LT(" #a ", " #b ")")
#define EXPECT_LE(a, b) GSHIM_EXPECT((a) <= (b), "EXPECT_LE(" #a ", " #b ")")
#define EXPECT_GT(a, b) GSHIM_EXPECT((a) > (b), "EXPECT_GT(" #a ", " #b ")")
#define EXPECT_GE(a, b) GSHIM_EXPECT((a) >= (b), "EXPECT_GE(" #a ", " #b ")")
#define ASSERT_EQ(a, b) GSHIM_ASSERT((a) == (b), "ASSERT_EQ(" #a ", " #b ")")
#define ASSERT_NE(a, b) GSHIM_ASSERT((a) != (b), "ASSERT_NE(" #a ", " #b ")")
#define ASSERT_LT(a, b) GSHIM_ASSERT((a) < (b), "ASSERT_LT(" #a ", " #b ")")
#define ASSERT_LE(a, b) GSHIM_ASSERT((a) <= (b), "ASSERT_LE(" #a ", " #b ")")
#define ASSERT_GT(a, b) GSHIM_ASSERT((a) > (b), "ASSERT_GT(" #a ", " #b ")")
#define ASSERT_GE(a, b) GSHIM_ASSERT((a) >= (b), "ASSERT_GE(" #a ", " #b ")")

#define EXPECT_NEAR(a, b, tol) \
  GSHIM_EXPECT(std::fabs((a) - (b)) <= (tol), "EXPECT_NEAR(" #a ", " #b ", " #tol ")")
#define EXPECT_DOUBLE_EQ(a, b) \
  GSHIM_EXPECT(::gtest_shim::double_eq((a), (b)), "EXPECT_DOUBLE_EQ(" #a ", " #b ")")
#define EXPECT_STREQ(a, b) \
  GSHIM_EXPECT(std::strcmp((a), (b)) == 0, "EXPECT_STREQ(" #a ", " #b ")")

#define EXPECT_THROW(stmt, type)                                          \
  GSHIM_EXPECT(([&]() -> bool {                                           \
                 try {                                                    \
                   stmt;                                                  \
                 } catch (const type&) {                                  \
                   return true;                                           \
                 } catch (...) {                                          \
                   return false;                                          \
                 }                                                        \
                 return false;                                            \
               }()),                                                      \
               "EXPECT_THROW(" #stmt ", " #type ")")
#define EXPECT_NO_THROW(stmt)                                               \
  GSHIM_EXPECT(::gtest_shim::throws_nothing([&]() { stmt; }),              \
               "EXPECT_NO_THROW(" #stmt ")")

int main(int, char**) {
  auto& reg = ::gtest_shim::Registry::get();
  int failed = 0;
  for (auto& c : reg.cases) {
    reg.failures_in_case = 0;
    try {
      c.body();
    } catch (const std::exception& e) {
      std::printf("uncaught exception: %s\n", e.what());
      ++reg.failures_in_case;
    }
    std::printf("[%s] %s\n", reg.failures_in_case ? "  FAILED  " : "       OK ",
                c.name.c_str());
    failed += reg.failures_in_case ? 1 : 0;
  }
  std::printf("%zu tests, %d failed\n", reg.cases.size(), failed);
  return failed ? 1 : 0;
}
