/* TEST INFRASTRUCTURE ONLY: prototype shim so the reference's own sources
 * (/root/reference/proj/src/oracle.cpp, proj/tests/*.cpp) compile against the
 * image's runtime libgmp.so.10 without development headers. */
#pragma once
#include "../mpfr_shim.h"
