// Runner for the reference's own test sources compiled against the B200 drop-in.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>
