// Self-test of tests/cpp/doctest_shim/doctest.h: subcase re-run semantics,
// failure reporting and the exit code (tests/test_dropin.py).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <stdexcept>
#include <string>

static std::string trace;

TEST_CASE("subcases run once per leaf") {
    trace += "[";
    SUBCASE("a") {
        trace += "a";
        SUBCASE("a1") { trace += "1"; }
        SUBCASE("a2") { trace += "2"; }
    }
    SUBCASE("b") { trace += "b"; }
    trace += "]";
}

TEST_CASE("trace is complete") { CHECK(trace == "[a1][a2][b]"); }

TEST_CASE("approx and throws") {
    CHECK(1.0 == doctest::Approx(1.0 + 1e-9));
    CHECK(1.0 != doctest::Approx(1.1));
    CHECK(2.0 == doctest::Approx(2.0 + 1e-15).epsilon(1e-14));
    CHECK_THROWS_AS(throw std::runtime_error("x"), std::runtime_error);
}

TEST_CASE("a failing check is reported") { CHECK(1 + 1 == 3); }
