// Minimal Catch2-v3-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) include
// <catch2/catch_amalgamated.hpp>, which is not vendored there or in this image.  This shim
// implements the subset they use — TEST_CASE, SECTION (with Catch's re-entry semantics: each
// run of a test case executes one not-yet-finished leaf section, until none is left), CHECK /
// REQUIRE / CHECK_FALSE / REQUIRE_FALSE, CHECK_THROWS / CHECK_THROWS_AS / CHECK_THROWS_WITH
// with Catch::Matchers::ContainsSubstring, scoped INFO messages and Catch::Approx — so those
// files compile UNMODIFIED against this repository's ppsim headers and libamdp.so
// (tests/cpp/Makefile, tests/test_reference_cpp_suites.py).
//
// One translation unit per binary must `#define CATCH_SHIM_MAIN` before including this header
// (tests/cpp/catch_main.cpp); it defines main(), which runs every registered test case and
// exits with the number of failed test cases.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestCase {
  std::string name;
  std::function<void()> fn;
  const char* file;
  int line;
};

struct RunState {
  std::vector<TestCase> cases;
  std::vector<std::string> info;   // active INFO messages
  std::vector<std::string> path;   // entered section path, "" = test case body
  std::set<std::string> done;      // finished section paths of the current test case
  bool finished_one = false;       // a section body completed during this run
  int pending = 0;                 // sections skipped this run that still have to run
  long assertions = 0, failures = 0;
  bool case_failed = false;
};
inline RunState& state() {
  static RunState s;
  return s;
}

struct AbortTest {};  // REQUIRE failure: ends the current run of the test case

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    state().cases.push_back({name, fn, file, line});
  }
};

inline void report(bool ok, const char* macro, const char* expr, const char* file, int line, bool fatal,
                   const std::string& extra = "") {
  RunState& s = state();
  ++s.assertions;
  if (ok) return;
  ++s.failures;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s(%s)%s\n", file, line, macro, expr, extra.c_str());
  for (const auto& m : s.info) std::fprintf(stderr, "    with message: %s\n", m.c_str());
  if (fatal) throw AbortTest{};
}

// SECTION("name"): entered when not finished and no other section has completed in this run.
class Section {
 public:
  explicit Section(const std::string& name) {
    RunState& s = state();
    path_ = (s.path.empty() ? std::string() : s.path.back()) + "/" + name;
    if (s.done.count(path_)) return;
    if (s.finished_one) {
      ++s.pending;
      return;
    }
    entered_ = true;
    pending_before_ = s.pending;
    s.path.push_back(path_);
  }
  ~Section() {
    if (!entered_) return;
    RunState& s = state();
    s.path.pop_back();
    // an exception (REQUIRE failure) also ends the section: it is not re-run
    if (s.pending == pending_before_ || std::uncaught_exceptions() > 0) s.done.insert(path_);
    s.finished_one = true;
  }
  explicit operator bool() const { return entered_; }

 private:
  std::string path_;
  bool entered_ = false;
  int pending_before_ = 0;
};

class ScopedInfo {
 public:
  explicit ScopedInfo(const std::string& m) { state().info.push_back(m); }
  ~ScopedInfo() { state().info.pop_back(); }
};

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  friend bool operator==(double x, const Approx& a) {
    const double d = std::fabs(x - a.v_);
    return d <= a.margin_ || d <= a.eps_ * (1.0 + std::fabs(std::isinf(a.v_) ? 0.0 : a.v_));
  }
  friend bool operator==(const Approx& a, double x) { return x == a; }
  friend bool operator!=(double x, const Approx& a) { return !(x == a); }
  friend bool operator!=(const Approx& a, double x) { return !(x == a); }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double margin_ = 0.0;
};

namespace Matchers {
struct ContainsSubstring {
  std::string needle;
  explicit ContainsSubstring(std::string n) : needle(std::move(n)) {}
  bool match(const std::string& s) const { return s.find(needle) != std::string::npos; }
  std::string describe() const { return "contains \"" + needle + "\""; }
};
}  // namespace Matchers

inline bool message_matches(const std::string& what, const Matchers::ContainsSubstring& m) { return m.match(what); }
inline bool message_matches(const std::string& what, const std::string& exact) { return what == exact; }
inline bool message_matches(const std::string& what, const char* exact) { return what == exact; }

inline int run_all() {
  RunState& s = state();
  int failed_cases = 0;
  for (const TestCase& tc : s.cases) {
    s.done.clear();
    s.case_failed = false;
    for (int run = 0; run < 10000; ++run) {
      s.finished_one = false;
      s.pending = 0;
      s.path.clear();
      s.info.clear();
      try {
        tc.fn();
      } catch (const AbortTest&) {
      } catch (const std::exception& e) {
        report(false, "unexpected exception", e.what(), tc.file, tc.line, false);
      } catch (...) {
        report(false, "unexpected exception", "(non-std)", tc.file, tc.line, false);
      }
      if (s.pending == 0) break;
    }
    if (s.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "test case FAILED: %s\n", tc.name.c_str());
    }
  }
  std::printf("test cases: %zu | %zu passed | %d failed\nassertions: %ld | %ld passed | %ld failed\n", s.cases.size(),
              s.cases.size() - static_cast<size_t>(failed_cases), failed_cases, s.assertions,
              s.assertions - s.failures, s.failures);
  return failed_cases;
}

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_UNIQUE(p) CATCH_SHIM_CAT(p, __COUNTER__)

#define CATCH_SHIM_TEST_CASE2(fn, name, ...)                                   \
  static void fn();                                                           \
  static const ::Catch::Registrar CATCH_SHIM_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(...) CATCH_SHIM_TEST_CASE2(CATCH_SHIM_UNIQUE(catch_shim_test_), __VA_ARGS__, "")

#define SECTION(...) if (const ::Catch::Section CATCH_SHIM_UNIQUE(catch_shim_section_){std::string(__VA_ARGS__)})

#define INFO(msg)                                                                   \
  const ::Catch::ScopedInfo CATCH_SHIM_UNIQUE(catch_shim_info_)(                    \
      static_cast<const std::ostringstream&>(std::ostringstream() << msg).str())

#define CATCH_SHIM_CHECK(macro, fatal, negate, ...)                                                  \
  do {                                                                                                \
    bool catch_shim_ok = false;                                                                       \
    std::string catch_shim_extra;                                                                     \
    try {                                                                                             \
      catch_shim_ok = static_cast<bool>(__VA_ARGS__) != (negate);                                     \
    } catch (const std::exception& e) {                                                               \
      catch_shim_extra = std::string(" threw ") + e.what();                                           \
    } catch (...) {                                                                                   \
      catch_shim_extra = " threw";                                                                    \
    }                                                                                                 \
    ::Catch::report(catch_shim_ok, macro, #__VA_ARGS__, __FILE__, __LINE__, fatal, catch_shim_extra); \
  } while (false)

#define CHECK(...) CATCH_SHIM_CHECK("CHECK", false, false, __VA_ARGS__)
#define REQUIRE(...) CATCH_SHIM_CHECK("REQUIRE", true, false, __VA_ARGS__)
#define CHECK_FALSE(...) CATCH_SHIM_CHECK("CHECK_FALSE", false, true, __VA_ARGS__)
#define REQUIRE_FALSE(...) CATCH_SHIM_CHECK("REQUIRE_FALSE", true, true, __VA_ARGS__)

#define CATCH_SHIM_THROWS(macro, fatal, expr)                                            \
  do {                                                                                   \
    bool catch_shim_threw = false;                                                       \
    try {                                                                                \
      static_cast<void>(expr);                                                           \
    } catch (...) {                                                                      \
      catch_shim_threw = true;                                                           \
    }                                                                                    \
    ::Catch::report(catch_shim_threw, macro, #expr, __FILE__, __LINE__, fatal, " did not throw"); \
  } while (false)
#define CHECK_THROWS(expr) CATCH_SHIM_THROWS("CHECK_THROWS", false, expr)
#define REQUIRE_THROWS(expr) CATCH_SHIM_THROWS("REQUIRE_THROWS", true, expr)

#define CATCH_SHIM_THROWS_AS(macro, fatal, expr, type)                                   \
  do {                                                                                   \
    bool catch_shim_ok = false;                                                          \
    std::string catch_shim_extra = " did not throw";                                     \
    try {                                                                                \
      static_cast<void>(expr);                                                           \
    } catch (const type&) {                                                              \
      catch_shim_ok = true;                                                              \
    } catch (const std::exception& e) {                                                  \
      catch_shim_extra = std::string(" threw another type: ") + e.what();                \
    } catch (...) {                                                                      \
      catch_shim_extra = " threw another type";                                          \
    }                                                                                    \
    ::Catch::report(catch_shim_ok, macro, #expr ", " #type, __FILE__, __LINE__, fatal, catch_shim_extra); \
  } while (false)
#define CHECK_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS("CHECK_THROWS_AS", false, expr, type)
#define REQUIRE_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS("REQUIRE_THROWS_AS", true, expr, type)

#define CATCH_SHIM_THROWS_WITH(macro, fatal, expr, matcher)                              \
  do {                                                                                   \
    bool catch_shim_ok = false;                                                          \
    std::string catch_shim_extra = " did not throw";                                     \
    try {                                                                                \
      static_cast<void>(expr);                                                           \
    } catch (const std::exception& e) {                                                  \
      catch_shim_ok = ::Catch::message_matches(e.what(), matcher);                       \
      catch_shim_extra = std::string(" message: ") + e.what();                           \
    } catch (...) {                                                                      \
      catch_shim_extra = " threw a non-std exception";                                   \
    }                                                                                    \
    ::Catch::report(catch_shim_ok, macro, #expr ", " #matcher, __FILE__, __LINE__, fatal, catch_shim_extra); \
  } while (false)
#define CHECK_THROWS_WITH(expr, matcher) CATCH_SHIM_THROWS_WITH("CHECK_THROWS_WITH", false, expr, matcher)
#define REQUIRE_THROWS_WITH(expr, matcher) CATCH_SHIM_THROWS_WITH("REQUIRE_THROWS_WITH", true, expr, matcher)

#ifdef CATCH_SHIM_MAIN
int main() { return ::Catch::run_all(); }
#endif
