// TEST INFRASTRUCTURE — gtest_main for the mini GoogleTest shim.
#include <gtest/gtest.h>

int main(int argc, char** argv) { return ::testing::internal::run_all(argc, argv); }
