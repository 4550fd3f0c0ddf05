// Entry point for the reference doctest suites built by oracle/Makefile
// (stands in for proj/tests/doctest_main.cpp).  TEST INFRASTRUCTURE ONLY.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
