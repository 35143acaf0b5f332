// Self-test of the doctest-compatible shim (tests/cpp/doctest_shim/doctest.h):
// Approx tolerances, SUBCASE re-runs, REQUIRE aborts, CHECK_THROWS_AS and the
// exit status.  Cases named "bad*" must fail; run with -tce=bad* they are
// skipped and the binary must exit 0.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <stdexcept>
#include <vector>

static std::vector<int> order_seen;

TEST_CASE("approx semantics") {
    CHECK(1.0 == doctest::Approx(1.0 + 1e-6));            // default eps = 100 * FLT_EPSILON
    CHECK(1.0 != doctest::Approx(1.0 + 1e-3));
    CHECK(1.0 == doctest::Approx(1.0 + 1e-13).epsilon(1e-12));
    CHECK(1.0 != doctest::Approx(1.0 + 1e-11).epsilon(1e-12));
    CHECK(0.0 == doctest::Approx(1e-13).epsilon(1e-12));   // the scale (1) term
}

TEST_CASE("subcases run once each with the shared prefix") {
    order_seen.push_back(0);
    SUBCASE("first") { order_seen.push_back(1); }
    SUBCASE("second") { order_seen.push_back(2); }
}

TEST_CASE("subcase bookkeeping") {
    // runs after the test above (registration order)
    CHECK(order_seen == std::vector<int>{0, 1, 0, 2});
}

TEST_CASE("throws as") {
    CHECK_THROWS_AS(throw std::invalid_argument("x"), std::invalid_argument);
    CHECK_THROWS_AS(throw std::runtime_error("y"), std::runtime_error);
}

TEST_CASE("bad check") { CHECK(1 == 2); }

TEST_CASE("bad require aborts") {
    REQUIRE(false);
    order_seen.push_back(99);  // never reached
}

TEST_CASE("bad exception escapes") { throw std::runtime_error("boom"); }

TEST_CASE("bad throws as wrong type") { CHECK_THROWS_AS(throw std::runtime_error("z"), std::invalid_argument); }
