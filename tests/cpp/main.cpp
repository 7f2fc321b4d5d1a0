// Runner for the reference unit suites compiled against the B200 façade.
#include "doctest.h"

int main() { return doctest::run_all(); }
