// Minimal GoogleTest-compatible harness (TEST, EXPECT_*/ASSERT_*, streamed messages, main)
// used to compile the reference's own unit-test sources against the B200 lowprec shim
// (tests/reftests/build.sh). GoogleTest itself is not installed in this image.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace gt {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct Message {
  std::ostringstream s;
  template <class T>
  Message& operator<<(const T& v) {
    s << v;
    return *this;
  }
};
struct Helper {
  const char* file;
  int line;
  const char* text;
  void operator=(const Message& m) const {
    ++failures();
    std::fprintf(stderr, "%s:%d: Failure: %s %s\n", file, line, text, m.s.str().c_str());
  }
};
inline bool double_eq(double a, double b) {  // within 4 ULPs, like ::testing::DoubleLE
  if (a == b) return true;
  if (std::isnan(a) || std::isnan(b)) return false;
  int64_t ia, ib;
  std::memcpy(&ia, &a, 8);
  std::memcpy(&ib, &b, 8);
  if ((ia < 0) != (ib < 0)) return false;
  const int64_t d = ia > ib ? ia - ib : ib - ia;
  return d <= 4;
}
}  // namespace gt

#define GT_CHECK_(cond, text) \
  if (cond)                   \
    ;                         \
  else                        \
    ::gt::Helper{__FILE__, __LINE__, text} = ::gt::Message()
#define GT_FATAL_(cond, text) \
  if (cond)                   \
    ;                         \
  else                        \
    return ::gt::Helper{__FILE__, __LINE__, text} = ::gt::Message()

#define EXPECT_TRUE(c) GT_CHECK_((c), "EXPECT_TRUE(" #c ")")
#define EXPECT_FALSE(c) GT_CHECK_(!(c), "EXPECT_FALSE(" #c ")")
#define EXPECT_EQ(a, b) GT_CHECK_((a) == (b), "EXPECT_EQ(" #a ", " #b ")")
#define EXPECT_NE(a, b) GT_CHECK_((a) != (b), "EXPECT_NE(" #a ", " #b ")")
#define EXPECT_LT(a, b) GT_CHECK_((a) < (b), "EXPECT_LT(" #a ", " #b ")")
#define EXPECT_LE(a, b) GT_CHECK_((a) <= (b), "EXPECT_LE(" #a ", " #b ")")
#define EXPECT_GT(a, b) GT_CHECK_((a) > (b), "EXPECT_GT(" #a ", " #b ")")
#define EXPECT_GE(a, b) GT_CHECK_((a) >= (b), "EXPECT_GE(" #a ", " #b ")")
#define EXPECT_NEAR(a, b, t) GT_CHECK_(std::fabs(double(a) - double(b)) <= double(t), "EXPECT_NEAR(" #a ", " #b ")")
#define EXPECT_DOUBLE_EQ(a, b) GT_CHECK_(::gt::double_eq(double(a), double(b)), "EXPECT_DOUBLE_EQ(" #a ", " #b ")")
#define ASSERT_TRUE(c) GT_FATAL_((c), "ASSERT_TRUE(" #c ")")
#define ASSERT_EQ(a, b) GT_FATAL_((a) == (b), "ASSERT_EQ(" #a ", " #b ")")
#define ASSERT_LE(a, b) GT_FATAL_((a) <= (b), "ASSERT_LE(" #a ", " #b ")")
#define ASSERT_GE(a, b) GT_FATAL_((a) >= (b), "ASSERT_GE(" #a ", " #b ")")
#define ASSERT_DOUBLE_EQ(a, b) GT_FATAL_(::gt::double_eq(double(a), double(b)), "ASSERT_DOUBLE_EQ(" #a ", " #b ")")
#define EXPECT_THROW(stmt, exc)                                          \
  do {                                                                   \
    bool gt_caught_ = false;                                             \
    try {                                                                \
      stmt;                                                              \
    } catch (const exc&) {                                               \
      gt_caught_ = true;                                                 \
    } catch (...) {                                                      \
    }                                                                    \
    GT_CHECK_(gt_caught_, "EXPECT_THROW(" #stmt ", " #exc ")");          \
  } while (0)

#define TEST(S, N)                                             \
  static void gt_##S##_##N();                                  \
  static ::gt::Reg gt_reg_##S##_##N(#S "." #N, &gt_##S##_##N); \
  static void gt_##S##_##N()

inline int gt_run_all() {
  int failed = 0;
  for (const auto& c : ::gt::registry()) {
    const int before = ::gt::failures();
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++::gt::failures();
      std::fprintf(stderr, "%s: uncaught exception: %s\n", c.name, e.what());
    }
    const bool ok = ::gt::failures() == before;
    std::printf("[ %s ] %s\n", ok ? "    OK" : "FAILED", c.name);
    failed += ok ? 0 : 1;
  }
  std::printf("%zu tests, %d failed\n", ::gt::registry().size(), failed);
  return failed ? 1 : 0;
}
