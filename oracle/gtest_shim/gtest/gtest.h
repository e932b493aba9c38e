// Minimal GoogleTest-compatible shim -- TEST INFRASTRUCTURE ONLY.
// GTest is not installed in this image; this header lets oracle/Makefile
// build the reference's own test files (/root/reference/proj/tests/*.cpp,
// compiled in place, not copied) to show the reference passes its suite
// on this host before it is used as the parity oracle.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace gshim {
struct Case { const char* suite; const char* name; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
inline bool& current_failed() { static bool b = false; return b; }
struct Reg { Reg(const char* s, const char* n, void (*f)()) { registry().push_back({s, n, f}); } };
struct Msg {
  std::ostringstream os;
  bool fatal;
  const char* file; int line;
  bool active;
  Msg(bool act, bool fat, const char* f, int l) : fatal(fat), file(f), line(l), active(act) {}
  template <class T> Msg& operator<<(const T& v) { if (active) os << v; return *this; }
  ~Msg() {
    if (active) {
      std::fprintf(stderr, "%s:%d: failure %s\n", file, line, os.str().c_str());
      current_failed() = true;
    }
  }
};
struct FatalReturn { void operator=(const Msg&) {} };
}  // namespace gshim

namespace testing { using gshim::Msg; }

#define TEST(S, N) \
  static void S##_##N##_body(); \
  static gshim::Reg S##_##N##_reg(#S, #N, &S##_##N##_body); \
  static void S##_##N##_body()

#define GSHIM_CHECK(cond, fatal, text) \
  if (bool gshim_ok_ = (cond); gshim_ok_) {} else \
    return_if_fatal_##fatal gshim::Msg(true, fatal, __FILE__, __LINE__) << text << " "

#define return_if_fatal_true return gshim::FatalReturn() =
#define return_if_fatal_false

#define EXPECT_TRUE(c) GSHIM_CHECK((c), false, "EXPECT_TRUE(" #c ")")
#define EXPECT_FALSE(c) GSHIM_CHECK(!(c), false, "EXPECT_FALSE(" #c ")")
#define ASSERT_TRUE(c) GSHIM_CHECK((c), true, "ASSERT_TRUE(" #c ")")
#define ASSERT_FALSE(c) GSHIM_CHECK(!(c), true, "ASSERT_FALSE(" #c ")")
#define EXPECT_EQ(a, b) GSHIM_CHECK((a) == (b), false, "EXPECT_EQ(" #a ", " #b ")")
#define ASSERT_EQ(a, b) GSHIM_CHECK((a) == (b), true, "ASSERT_EQ(" #a ", " #b ")")
#define EXPECT_NE(a, b) GSHIM_CHECK((a) != (b), false, "EXPECT_NE(" #a ", " #b ")")
#define EXPECT_LT(a, b) GSHIM_CHECK((a) < (b), false, "EXPECT_LT(" #a ", " #b ")")
#define ASSERT_LT(a, b) GSHIM_CHECK((a) < (b), true, "ASSERT_LT(" #a ", " #b ")")
#define EXPECT_GE(a, b) GSHIM_CHECK((a) >= (b), false, "EXPECT_GE(" #a ", " #b ")")
#define ASSERT_GE(a, b) GSHIM_CHECK((a) >= (b), true, "ASSERT_GE(" #a ", " #b ")")
#define EXPECT_NEAR(a, b, t) GSHIM_CHECK(std::fabs(double(a) - double(b)) <= double(t), false, "EXPECT_NEAR(" #a ", " #b ")")
#define EXPECT_DOUBLE_EQ(a, b) \
  GSHIM_CHECK(std::fabs(double(a) - double(b)) <= 4 * 2.220446049250313e-16 * std::fmax(std::fabs(double(a)), std::fabs(double(b))), false, "EXPECT_DOUBLE_EQ(" #a ", " #b ")")
#define EXPECT_THROW(stmt, ex) \
  { bool gshim_thrown_ = false; try { stmt; } catch (const ex&) { gshim_thrown_ = true; } catch (...) {} \
    EXPECT_TRUE(gshim_thrown_) << "EXPECT_THROW(" #stmt ")"; }
#define EXPECT_NO_THROW(stmt) \
  { bool gshim_thrown_ = false; try { stmt; } catch (...) { gshim_thrown_ = true; } \
    EXPECT_FALSE(gshim_thrown_) << "EXPECT_NO_THROW(" #stmt ")"; }
#define FAIL() return gshim::FatalReturn() = gshim::Msg(true, true, __FILE__, __LINE__) << "FAIL "
