// Self-test of the Catch2 shim: failures must be counted, REQUIRE must stop a run, and
// SECTIONs must re-enter with Catch's semantics (each leaf once, the enclosing code once per
// leaf).  tests/test_reference_cpp_suites.py checks the exact output.
#include <catch2/catch_amalgamated.hpp>

#include <stdexcept>
#include <string>

static std::string trace;

TEST_CASE("sections run each leaf once") {
  trace += "[";
  SECTION("a") {
    trace += "a";
    SECTION("a1") { trace += "1"; }
    SECTION("a2") { trace += "2"; }
  }
  SECTION("b") { trace += "b"; }
  trace += "]";
}

TEST_CASE("trace of the previous case") { CHECK(trace == "[a1][a2][b]"); }

TEST_CASE("a failing check is counted and the case continues") {
  CHECK(1 + 1 == 3);
  CHECK_FALSE(false);
  CHECK_THROWS_AS(throw std::invalid_argument("x"), std::invalid_argument);
  CHECK_THROWS_WITH(throw std::runtime_error("dependency cycle: a"), Catch::Matchers::ContainsSubstring("cycle"));
  CHECK(0.1 + 0.2 == Catch::Approx(0.3));
}

TEST_CASE("require stops the run") {
  REQUIRE(false);
  CHECK(false);  // not reached
}
