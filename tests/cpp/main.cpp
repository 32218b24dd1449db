// Runner for the reference unit tests compiled against the B200 drop-in.
#include "gtest/gtest.h"
int main() { return testing::run_all(); }
