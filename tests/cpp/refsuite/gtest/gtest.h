// Minimal GoogleTest-compatible shim (GTest is not installed in this image):
// TEST, EXPECT_/ASSERT_ {EQ, NE, LT, LE, GT, GE, TRUE, FALSE, THROW, NO_THROW,
// DOUBLE_EQ, NEAR}
// with `<<` messages, and a main() that runs every registered test and
// exits with the number of failed tests. Enough to compile the reference's
// own unit suites unmodified against the B200 library (tests/cpp/refsuite).
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace gshim {

struct Registry {
  struct Case {
    std::string suite, name;
    std::function<void()> fn;
  };
  std::vector<Case> cases;
  bool current_failed = false;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

struct Registrar {
  Registrar(const char* suite, const char* name, std::function<void()> fn) {
    Registry::get().cases.push_back({suite, name, std::move(fn)});
  }
};

// Collects a `<<` message; reports the failure when destroyed (EXPECT) or
// when assigned to an AssertReturn (ASSERT, which then returns).
class Message {
 public:
  Message(const char* file, int line, std::string what) : file_(file), line_(line), what_(std::move(what)) {}
  Message(const Message&) = delete;
  template <class T>
  Message& operator<<(const T& v) {
    os_ << v;
    return *this;
  }
  ~Message() {
    Registry::get().current_failed = true;
    std::cerr << file_ << ":" << line_ << ": Failure: " << what_;
    const std::string extra = os_.str();
    if (!extra.empty()) std::cerr << "\n  " << extra;
    std::cerr << std::endl;
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
  std::ostringstream os_;
};

struct AssertReturn {
  void operator=(const Message&) const {}
};

template <class A, class B>
std::string eq_text(const char* ea, const char* eb, const A&, const B&) {
  return std::string("expected ") + ea + " == " + eb;
}

}  // namespace gshim

#define GSHIM_CAT2(a, b) a##b
#define GSHIM_CAT(a, b) GSHIM_CAT2(a, b)
#define TEST(suite, name)                                                                         \
  static void GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, GSHIM_CAT(_, name)))();                     \
  static ::gshim::Registrar GSHIM_CAT(gshim_reg_, GSHIM_CAT(suite, GSHIM_CAT(_, name)))(          \
      #suite, #name, &GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, GSHIM_CAT(_, name))));               \
  static void GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, GSHIM_CAT(_, name)))()

#define GSHIM_EXPECT(cond, text) \
  if (cond)                      \
    ;                            \
  else                           \
    ::gshim::Message(__FILE__, __LINE__, text)
#define GSHIM_ASSERT(cond, text) \
  if (cond)                      \
    ;                            \
  else                           \
    return ::gshim::AssertReturn() = ::gshim::Message(__FILE__, __LINE__, text)

#define EXPECT_TRUE(c) GSHIM_EXPECT(static_cast<bool>(c), "expected true: " #c)
#define EXPECT_FALSE(c) GSHIM_EXPECT(!static_cast<bool>(c), "expected false: " #c)
#define EXPECT_EQ(a, b) GSHIM_EXPECT((a) == (b), "expected " #a " == " #b)
#define EXPECT_NE(a, b) GSHIM_EXPECT((a) != (b), "expected " #a " != " #b)
#define EXPECT_DOUBLE_EQ(a, b) \
  GSHIM_EXPECT(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= 1e-12 * std::fabs(static_cast<double>(b)) + 1e-300, "expected " #a " ~= " #b)
#define ASSERT_TRUE(c) GSHIM_ASSERT(static_cast<bool>(c), "expected true: " #c)
#define ASSERT_FALSE(c) GSHIM_ASSERT(!static_cast<bool>(c), "expected false: " #c)
#define ASSERT_EQ(a, b) GSHIM_ASSERT((a) == (b), "expected " #a " == " #b)
#define ASSERT_NE(a, b) GSHIM_ASSERT((a) != (b), "expected " #a " != " #b)

#define EXPECT_THROW(stmt, ex)                                                        \
  GSHIM_EXPECT(([&]() -> bool {                                                       \
                 try {                                                                \
                   stmt;                                                              \
                 } catch (const ex&) {                                                \
                   return true;                                                       \
                 } catch (...) {                                                      \
                   return false;                                                      \
                 }                                                                    \
                 return false;                                                        \
               })(),                                                                  \
               "expected " #stmt " to throw " #ex)
#define EXPECT_NO_THROW(stmt)                                                         \
  GSHIM_EXPECT(([&]() -> bool {                                                       \
                 try {                                                                \
                   stmt;                                                              \
                 } catch (...) {                                                      \
                   return false;                                                      \
                 }                                                                    \
                 return true;                                                         \
               })(),                                                                  \
               "expected " #stmt " not to throw")
#define EXPECT_LT(a, b) GSHIM_EXPECT((a) < (b), "expected " #a " < " #b)
#define EXPECT_LE(a, b) GSHIM_EXPECT((a) <= (b), "expected " #a " <= " #b)
#define EXPECT_GT(a, b) GSHIM_EXPECT((a) > (b), "expected " #a " > " #b)
#define EXPECT_GE(a, b) GSHIM_EXPECT((a) >= (b), "expected " #a " >= " #b)
#define ASSERT_LT(a, b) GSHIM_ASSERT((a) < (b), "expected " #a " < " #b)
#define ASSERT_LE(a, b) GSHIM_ASSERT((a) <= (b), "expected " #a " <= " #b)
#define ASSERT_GT(a, b) GSHIM_ASSERT((a) > (b), "expected " #a " > " #b)
#define ASSERT_GE(a, b) GSHIM_ASSERT((a) >= (b), "expected " #a " >= " #b)
#define EXPECT_NEAR(a, b, tol) \
  GSHIM_EXPECT(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= static_cast<double>(tol), \
               "expected |" #a " - " #b "| <= " #tol)
#define ASSERT_NEAR(a, b, tol) \
  GSHIM_ASSERT(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= static_cast<double>(tol), \
               "expected |" #a " - " #b "| <= " #tol)
#define ASSERT_THROW(stmt, ex) EXPECT_THROW(stmt, ex)
#define ASSERT_NO_THROW(stmt) EXPECT_NO_THROW(stmt)

int main() {
  auto& r = ::gshim::Registry::get();
  int failed = 0;
  for (auto& c : r.cases) {
    r.current_failed = false;
    try {
      c.fn();
    } catch (const std::exception& e) {
      r.current_failed = true;
      std::cerr << "uncaught exception: " << e.what() << std::endl;
    }
    std::printf("[ %s ] %s.%s\n", r.current_failed ? "FAILED" : "    OK", c.suite.c_str(), c.name.c_str());
    failed += r.current_failed ? 1 : 0;
  }
  std::printf("%zu tests, %d failed\n", r.cases.size(), failed);
  return failed;
}
