// Runs the reference's own unit tests (tests/test_*.cpp, compiled into this binary by
// oracle/ref/Makefile against the Eigen-subset and Catch2-subset shims). TEST INFRASTRUCTURE ONLY.
#include "catch_amalgamated.hpp"
int main() { return Catch::run_all(); }
