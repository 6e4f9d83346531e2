// doctest-subset shim — TEST INFRASTRUCTURE ONLY (runs the reference's own unit tests
// against oracle/_ref). The reference expects doctest in `vendor/` (proj/CMakeLists.txt:16),
// which is not shipped. This implements the macros those tests use with doctest's
// semantics: SUBCASE re-entry (one leaf per run), REQUIRE aborts the test case,
// CHECK_THROWS_WITH_AS compares what() exactly, Approx uses doctest's formula.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value)
      : m_epsilon(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), m_scale(1.0),
        m_value(value) {}
  Approx& epsilon(double e) {
    m_epsilon = e;
    return *this;
  }
  Approx& scale(double s) {
    m_scale = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.m_value) <
           rhs.m_epsilon * (rhs.m_scale + std::max<double>(std::fabs(lhs), std::fabs(rhs.m_value)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !operator==(rhs, lhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.m_value || lhs == rhs; }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.m_value || lhs == rhs; }
  friend bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.m_value && lhs != rhs; }
  friend bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.m_value && lhs != rhs; }

 private:
  double m_epsilon, m_scale, m_value;
};

namespace detail {

struct TestAbort {};

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

struct State {
  std::vector<TestCase> cases;
  // subcase traversal (doctest's algorithm)
  std::vector<std::string> stack;
  std::set<std::vector<std::string>> passed;
  size_t current_max_level = 0;
  bool should_reenter = false;
  // accounting
  long asserts = 0, asserts_failed = 0;
  bool case_failed = false;
  const TestCase* current = nullptr;
};

inline State& state() {
  static State s;
  return s;
}

inline int reg(const char* name, const char* file, int line, void (*fn)()) {
  state().cases.push_back({name, file, line, fn});
  return 0;
}

inline void report_fail(const char* file, int line, const std::string& what) {
  State& s = state();
  ++s.asserts_failed;
  s.case_failed = true;
  std::string path;
  for (const auto& p : s.stack) path += " / " + p;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\"%s: %s\n", file, line,
               s.current ? s.current->name : "?", path.c_str(), what.c_str());
}

inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
  ++state().asserts;
  if (!ok) {
    report_fail(file, line, std::string(require ? "REQUIRE( " : "CHECK( ") + expr + " )");
    if (require) throw TestAbort{};
  }
}

class Subcase {
 public:
  Subcase(const char* name) {
    State& s = state();
    if (s.stack.size() < s.current_max_level) {
      s.should_reenter = true;
      return;
    }
    s.stack.push_back(name);
    if (s.passed.count(s.stack) != 0) {
      s.stack.pop_back();
      return;
    }
    s.current_max_level = s.stack.size();
    m_entered = true;
  }
  ~Subcase() {
    if (m_entered) {
      State& s = state();
      if (!s.should_reenter) s.passed.insert(s.stack);
      s.stack.pop_back();
    }
  }
  Subcase(const Subcase&) = delete;
  operator bool() const { return m_entered; }

 private:
  bool m_entered = false;
};

inline int run_all(int argc, char** argv) {
  State& s = state();
  std::string filter;
  std::vector<std::string> exclude;  // -tce=<substring>, repeatable
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "--tc=", 5) == 0) filter = argv[i] + 5;
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
    if (std::strncmp(argv[i], "--tce=", 6) == 0) exclude.emplace_back(argv[i] + 6);
    if (std::strncmp(argv[i], "-tce=", 5) == 0) exclude.emplace_back(argv[i] + 5);
  }
  int ran = 0, failed = 0;
  for (const TestCase& tc : s.cases) {
    if (!filter.empty() && std::string(tc.name).find(filter) == std::string::npos) continue;
    bool skip = false;
    for (const std::string& x : exclude) skip = skip || std::string(tc.name).find(x) != std::string::npos;
    if (skip) continue;
    ++ran;
    s.current = &tc;
    s.case_failed = false;
    s.passed.clear();
    do {
      s.stack.clear();
      s.current_max_level = 0;
      s.should_reenter = false;
      try {
        tc.fn();
      } catch (const TestAbort&) {
      } catch (const std::exception& e) {
        report_fail(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        report_fail(tc.file, tc.line, "unexpected unknown exception");
      }
    } while (s.should_reenter);
    if (s.case_failed) ++failed;
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", ran, ran - failed, failed);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", s.asserts,
              s.asserts - s.asserts_failed, s.asserts_failed);
  return failed == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, regv, name)                                                 \
  static void fn();                                                                     \
  static const int regv = doctest::detail::reg(name, __FILE__, __LINE__, &fn);          \
  static void fn()
#define TEST_CASE(name) \
  DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_fn_, __COUNTER__), DOCTEST_CAT(doctest_reg_, __COUNTER__), name)
#define SUBCASE(name) \
  if (const doctest::detail::Subcase& DOCTEST_CAT(doctest_sc_, __COUNTER__) = doctest::detail::Subcase(name))

#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) doctest::detail::check(!(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) doctest::detail::check(!(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", true)

#define DOCTEST_THROWS_IMPL(expr, msg, T, require)                                              \
  do {                                                                                          \
    bool doctest_ok = false;                                                                    \
    std::string doctest_got = "no exception";                                                   \
    try {                                                                                       \
      static_cast<void>(expr);                                                                  \
    } catch (const T& e) {                                                                      \
      const char* doctest_want = msg;                                                           \
      doctest_ok = doctest_want == nullptr || std::string(e.what()) == doctest_want;            \
      doctest_got = std::string("what()=\"") + e.what() + "\"";                                 \
    } catch (const std::exception& e) {                                                         \
      doctest_got = std::string("other exception: ") + e.what();                                \
    } catch (...) {                                                                             \
      doctest_got = "unknown exception";                                                        \
    }                                                                                           \
    ++doctest::detail::state().asserts;                                                         \
    if (!doctest_ok) {                                                                          \
      doctest::detail::report_fail(__FILE__, __LINE__,                                          \
                                   std::string("THROWS( " #expr " ) as " #T ": ") + doctest_got); \
      if (require) throw doctest::detail::TestAbort{};                                          \
    }                                                                                           \
  } while (0)

#define CHECK_THROWS_AS(expr, T) DOCTEST_THROWS_IMPL(expr, (const char*)nullptr, T, false)
#define CHECK_THROWS_WITH_AS(expr, msg, T) DOCTEST_THROWS_IMPL(expr, msg, T, false)
#define REQUIRE_THROWS_AS(expr, T) DOCTEST_THROWS_IMPL(expr, (const char*)nullptr, T, true)
#define CHECK_THROWS(expr) DOCTEST_THROWS_IMPL(expr, (const char*)nullptr, std::exception, false)
#define CHECK_NOTHROW(expr)                                                                    \
  do {                                                                                         \
    ++doctest::detail::state().asserts;                                                        \
    try {                                                                                      \
      static_cast<void>(expr);                                                                 \
    } catch (const std::exception& e) {                                                        \
      doctest::detail::report_fail(__FILE__, __LINE__,                                         \
                                   std::string("NOTHROW( " #expr " ): ") + e.what());          \
    }                                                                                          \
  } while (0)

#define INFO(...)                 \
  do {                            \
    std::ostringstream doctest_os; \
    doctest_os << __VA_ARGS__;    \
  } while (0)
#define CAPTURE(x) INFO(#x " := " << (x))
#define MESSAGE(...)                                              \
  do {                                                            \
    std::ostringstream doctest_os;                                \
    doctest_os << __VA_ARGS__;                                    \
    std::printf("%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, doctest_os.str().c_str()); \
  } while (0)
#define FAIL_CHECK(...)                                                         \
  do {                                                                          \
    std::ostringstream doctest_os;                                              \
    doctest_os << __VA_ARGS__;                                                  \
    doctest::detail::report_fail(__FILE__, __LINE__, "FAIL_CHECK: " + doctest_os.str()); \
  } while (0)
#define FAIL(...)                                                         \
  do {                                                                    \
    std::ostringstream doctest_os;                                        \
    doctest_os << __VA_ARGS__;                                            \
    doctest::detail::report_fail(__FILE__, __LINE__, "FAIL: " + doctest_os.str()); \
    throw doctest::detail::TestAbort{};                                   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
