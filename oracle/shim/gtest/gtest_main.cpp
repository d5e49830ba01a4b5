// ORACLE TEST INFRASTRUCTURE: main() for the GTest-subset shim.
#include <gtest/gtest.h>
int main(int argc, char** argv) { return ::testing::RunAllTests(argc, argv); }
