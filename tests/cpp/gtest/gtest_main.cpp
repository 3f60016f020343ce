// main() of the GoogleTest stand-in (tests/cpp/gtest/gtest.h).
#include "gtest/gtest.h"

int main(int argc, char** argv) { return gtest_shim::run_all(argc, argv); }
