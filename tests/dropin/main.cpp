// Entry point of the drop-in test binary: the reference's unit tests
// (test_quant / test_qgemm / test_balance) linked against libdtq_dropin.so.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
