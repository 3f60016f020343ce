// gtest.h -- a minimal stand-in for GoogleTest (not installed in this image)
// covering exactly what the reference's test suite uses: TEST, the
// EXPECT_/ASSERT_ comparison family, EXPECT_DOUBLE_EQ (4 ULPs),
// EXPECT_THROW / EXPECT_NO_THROW, FAIL(), streamed failure messages and a
// main() with --gtest_filter.  It lets /root/reference/proj/tests/*.cpp
// compile unchanged against the B200 drop-in (tests/cpp/refsuite/).
#pragma once
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace gtest_shim {

struct Case {
  const char* suite;
  const char* name;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

inline int& failures_in_case() {
  static int f = 0;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, void (*fn)()) { registry().push_back({s, n, fn}); }
};

template <class T, class = void>
struct streamable : std::false_type {};
template <class T>
struct streamable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <class T>
std::string show(const T& v) {
  std::ostringstream os;
  if constexpr (std::is_enum_v<T>) {
    os << static_cast<long long>(static_cast<std::underlying_type_t<T>>(v));
  } else if constexpr (std::is_floating_point_v<T>) {
    os.precision(17);
    os << v;
  } else if constexpr (std::is_same_v<T, unsigned char> || std::is_same_v<T, signed char>) {
    os << static_cast<int>(v);
  } else if constexpr (streamable<T>::value) {
    os << v;
  } else {
    os << "<" << sizeof(T) << "-byte object>";
  }
  return os.str();
}

struct Result {
  bool ok;
  std::string text;
};

class Message {
 public:
  template <class T>
  Message& operator<<(const T& v) {
    os_ << v;
    return *this;
  }
  std::string str() const { return os_.str(); }

 private:
  std::ostringstream os_;
};

class Reporter {
 public:
  Reporter(const char* file, int line, std::string text) : file_(file), line_(line), text_(std::move(text)) {}
  void operator=(const Message& m) const {
    ++failures_in_case();
    std::cout << file_ << ":" << line_ << ": Failure\n" << text_;
    const std::string extra = m.str();
    if (!extra.empty()) std::cout << "\n" << extra;
    std::cout << std::endl;
  }

 private:
  const char* file_;
  int line_;
  std::string text_;
};

#define GTS_CMP_(name, op)                                                                                 \
  template <class A, class B>                                                                           \
  Result name(const char* ea, const char* eb, const A& a, const B& b) {                                \
    if (a op b) return {true, ""};                                                                      \
    return {false, std::string("Expected: (") + ea + ") " #op " (" + eb + "), actual: " + show(a) +     \
                       " vs " + show(b)};                                                               \
  }
#if defined(__GNUC__)
#pragma GCC diagnostic push
#pragma GCC diagnostic ignored "-Wsign-compare"
#endif
GTS_CMP_(cmp_eq, ==)
GTS_CMP_(cmp_ne, !=)
GTS_CMP_(cmp_lt, <)
GTS_CMP_(cmp_le, <=)
GTS_CMP_(cmp_gt, >)
GTS_CMP_(cmp_ge, >=)
#if defined(__GNUC__)
#pragma GCC diagnostic pop
#endif
#undef GTS_CMP_

inline Result cmp_bool(const char* e, bool v, bool want) {
  if (v == want) return {true, ""};
  return {false, std::string("Value of: ") + e + "\n  Actual: " + (v ? "true" : "false") +
                     "\nExpected: " + (want ? "true" : "false")};
}

// GoogleTest's AlmostEquals: within 4 units in the last place.
inline Result cmp_double_eq(const char* ea, const char* eb, double a, double b) {
  auto biased = [](double x) {
    std::uint64_t u;
    std::memcpy(&u, &x, 8);
    const std::uint64_t sign = 1ull << 63;
    return (u & sign) ? ~u + 1 : u | sign;
  };
  bool ok = false;
  if (!std::isnan(a) && !std::isnan(b)) {
    const std::uint64_t x = biased(a), y = biased(b);
    ok = (x >= y ? x - y : y - x) <= 4;
  }
  if (ok) return {true, ""};
  return {false, std::string("Expected equality (4 ULPs) of ") + ea + " and " + eb + ", actual: " + show(a) +
                     " vs " + show(b)};
}

inline bool name_matches(const std::string& pat, const std::string& s) {  // '*' and '?' globs, ':' alternatives
  size_t start = 0;
  while (true) {
    const size_t end = pat.find(':', start);
    const std::string p = pat.substr(start, end == std::string::npos ? std::string::npos : end - start);
    std::function<bool(size_t, size_t)> m = [&](size_t i, size_t j) -> bool {
      if (i == p.size()) return j == s.size();
      if (p[i] == '*') return m(i + 1, j) || (j < s.size() && m(i, j + 1));
      return j < s.size() && (p[i] == '?' || p[i] == s[j]) && m(i + 1, j + 1);
    };
    if (m(0, 0)) return true;
    if (end == std::string::npos) return false;
    start = end + 1;
  }
}

inline int run_all(int argc, char** argv) {
  std::string filter = "*";
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
  int run = 0, failed = 0;
  std::vector<std::string> failed_names;
  for (const Case& c : registry()) {
    const std::string full = std::string(c.suite) + "." + c.name;
    if (!name_matches(filter, full)) continue;
    ++run;
    failures_in_case() = 0;
    std::cout << "[ RUN      ] " << full << std::endl;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++failures_in_case();
      std::cout << "unexpected exception: " << e.what() << std::endl;
    } catch (...) {
      ++failures_in_case();
      std::cout << "unexpected non-std exception" << std::endl;
    }
    if (failures_in_case()) {
      ++failed;
      failed_names.push_back(full);
      std::cout << "[  FAILED  ] " << full << std::endl;
    } else {
      std::cout << "[       OK ] " << full << std::endl;
    }
  }
  std::cout << "[==========] " << run << " tests ran.\n[  PASSED  ] " << (run - failed) << " tests." << std::endl;
  for (const auto& n : failed_names) std::cout << "[  FAILED  ] " << n << std::endl;
  return failed ? 1 : 0;
}

}  // namespace gtest_shim

#define TEST(suite, name)                                                                        \
  static void gts_##suite##_##name();                                                            \
  static ::gtest_shim::Registrar gts_reg_##suite##_##name(#suite, #name, &gts_##suite##_##name); \
  static void gts_##suite##_##name()

#define GTS_CHECK_(res, on_fail)                                  \
  if (::gtest_shim::Result gts_r_ = (res); gts_r_.ok) {           \
  } else                                                          \
    on_fail ::gtest_shim::Reporter(__FILE__, __LINE__, gts_r_.text) = ::gtest_shim::Message()

#define GTS_NONFATAL_
#define GTS_FATAL_ return

#define EXPECT_EQ(a, b) GTS_CHECK_(::gtest_shim::cmp_eq(#a, #b, (a), (b)), GTS_NONFATAL_)
#define EXPECT_NE(a, b) GTS_CHECK_(::gtest_shim::cmp_ne(#a, #b, (a), (b)), GTS_NONFATAL_)
#define EXPECT_LT(a, b) GTS_CHECK_(::gtest_shim::cmp_lt(#a, #b, (a), (b)), GTS_NONFATAL_)
#define EXPECT_LE(a, b) GTS_CHECK_(::gtest_shim::cmp_le(#a, #b, (a), (b)), GTS_NONFATAL_)
#define EXPECT_GT(a, b) GTS_CHECK_(::gtest_shim::cmp_gt(#a, #b, (a), (b)), GTS_NONFATAL_)
#define EXPECT_GE(a, b) GTS_CHECK_(::gtest_shim::cmp_ge(#a, #b, (a), (b)), GTS_NONFATAL_)
#define EXPECT_TRUE(c) GTS_CHECK_(::gtest_shim::cmp_bool(#c, static_cast<bool>(c), true), GTS_NONFATAL_)
#define EXPECT_FALSE(c) GTS_CHECK_(::gtest_shim::cmp_bool(#c, static_cast<bool>(c), false), GTS_NONFATAL_)
#define EXPECT_DOUBLE_EQ(a, b) GTS_CHECK_(::gtest_shim::cmp_double_eq(#a, #b, (a), (b)), GTS_NONFATAL_)
#define ASSERT_EQ(a, b) GTS_CHECK_(::gtest_shim::cmp_eq(#a, #b, (a), (b)), GTS_FATAL_)
#define ASSERT_NE(a, b) GTS_CHECK_(::gtest_shim::cmp_ne(#a, #b, (a), (b)), GTS_FATAL_)
#define ASSERT_LT(a, b) GTS_CHECK_(::gtest_shim::cmp_lt(#a, #b, (a), (b)), GTS_FATAL_)
#define ASSERT_LE(a, b) GTS_CHECK_(::gtest_shim::cmp_le(#a, #b, (a), (b)), GTS_FATAL_)
#define ASSERT_GT(a, b) GTS_CHECK_(::gtest_shim::cmp_gt(#a, #b, (a), (b)), GTS_FATAL_)
#define ASSERT_GE(a, b) GTS_CHECK_(::gtest_shim::cmp_ge(#a, #b, (a), (b)), GTS_FATAL_)
#define ASSERT_TRUE(c) GTS_CHECK_(::gtest_shim::cmp_bool(#c, static_cast<bool>(c), true), GTS_FATAL_)
#define ASSERT_FALSE(c) GTS_CHECK_(::gtest_shim::cmp_bool(#c, static_cast<bool>(c), false), GTS_FATAL_)

#define GTS_THROWS_(stmt, T)                                                                 \
  [&]() -> ::gtest_shim::Result {                                                            \
    try {                                                                                    \
      stmt;                                                                                  \
    } catch (const T&) {                                                                     \
      return {true, ""};                                                                     \
    } catch (const std::exception& e) {                                                      \
      return {false, std::string("Expected: " #stmt " throws " #T ", actual: threw ") + e.what()}; \
    } catch (...) {                                                                          \
      return {false, "Expected: " #stmt " throws " #T ", actual: threw a different type"};  \
    }                                                                                        \
    return {false, "Expected: " #stmt " throws " #T ", actual: it throws nothing"};         \
  }()
#define GTS_NO_THROW_(stmt)                                                                  \
  [&]() -> ::gtest_shim::Result {                                                            \
    try {                                                                                    \
      stmt;                                                                                  \
    } catch (const std::exception& e) {                                                      \
      return {false, std::string("Expected: " #stmt " doesn't throw, actual: ") + e.what()}; \
    } catch (...) {                                                                          \
      return {false, "Expected: " #stmt " doesn't throw, actual: it throws"};               \
    }                                                                                        \
    return {true, ""};                                                                       \
  }()
#define EXPECT_THROW(stmt, T) GTS_CHECK_(GTS_THROWS_(stmt, T), GTS_NONFATAL_)
#define ASSERT_THROW(stmt, T) GTS_CHECK_(GTS_THROWS_(stmt, T), GTS_FATAL_)
#define EXPECT_NO_THROW(stmt) GTS_CHECK_(GTS_NO_THROW_(stmt), GTS_NONFATAL_)
#define ASSERT_NO_THROW(stmt) GTS_CHECK_(GTS_NO_THROW_(stmt), GTS_FATAL_)
#define FAIL() GTS_CHECK_((::gtest_shim::Result{false, "Failed"}), GTS_FATAL_)
#define ADD_FAILURE() GTS_CHECK_((::gtest_shim::Result{false, "Failed"}), GTS_NONFATAL_)
#define SUCCEED() \
  do {            \
  } while (0)
