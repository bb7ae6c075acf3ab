/* TEST INFRASTRUCTURE ONLY: prototype shim so the reference's own sources
 * compile against the image's runtime libmpfr.so.6 (MPFR 4.2.1) without
 * development headers. Adds the few macros the reference uses on top of
 * oracle/mpfr_shim.h. */
#pragma once
#include <climits>
#include "../mpfr_shim.h"
extern "C" {
int mpfr_cmp_d(mpfr_srcptr, double);
int mpfr_cmp_ui_2exp(mpfr_srcptr, unsigned long, mpfr_exp_t);
int mpfr_sub_ui(mpfr_ptr, mpfr_srcptr, unsigned long, mpfr_rnd_t);
int mpfr_sqr(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
}
#define mpfr_cmp_ui(b, i) mpfr_cmp_ui_2exp((b), (i), 0)
#define MPFR_DECL_INIT(_x, _p)                                              \
  mp_limb_t __gmpfr_local_tab_##_x[((_p) - 1) / 64 + 1];                   \
  __mpfr_struct _x[1] = {{(_p), 1, (mpfr_exp_t)(1 - LONG_MAX), __gmpfr_local_tab_##_x}}
