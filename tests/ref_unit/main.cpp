// Entry point for the reference unit tests compiled with the Catch2-API shim.
#include <catch_amalgamated.hpp>

int main() { return catchshim::run_all() == 0 ? 0 : 1; }
