// main() of the Catch2 shim (catch2/catch_amalgamated.hpp): runs every registered test case.
#define CATCH_SHIM_MAIN
#include <catch2/catch_amalgamated.hpp>
