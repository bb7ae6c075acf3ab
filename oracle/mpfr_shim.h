/* TEST INFRASTRUCTURE ONLY — part of the CPU oracle, never linked into the
 * product library.
 *
 * Prototype-only declarations for the MPFR 4.2.1 / GMP 6.3.0 runtime that
 * ships in this image (/lib/x86_64-linux-gnu/libmpfr.so.6, libgmp.so.10)
 * without development headers. The reference links the same two libraries
 * (ref: proj/CMakeLists.txt:26-27). Only the handful of entry points the
 * oracle calls are declared; the struct layouts are the documented public
 * layouts of mpfr.h / gmp.h for LP64.
 */
#ifndef CRVEC_ORACLE_MPFR_SHIM_H
#define CRVEC_ORACLE_MPFR_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned long mp_limb_t;
typedef long mpfr_prec_t;
typedef int mpfr_sign_t;
typedef long mpfr_exp_t;

typedef struct {
  mpfr_prec_t _mpfr_prec;
  mpfr_sign_t _mpfr_sign;
  mpfr_exp_t _mpfr_exp;
  mp_limb_t *_mpfr_d;
} __mpfr_struct;
typedef __mpfr_struct mpfr_t[1];
typedef __mpfr_struct *mpfr_ptr;
typedef const __mpfr_struct *mpfr_srcptr;

typedef enum { MPFR_RNDN = 0, MPFR_RNDZ, MPFR_RNDU, MPFR_RNDD, MPFR_RNDA } mpfr_rnd_t;

typedef struct {
  int _mp_alloc;
  int _mp_size;
  mp_limb_t *_mp_d;
} __mpz_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpz_struct *mpz_ptr;
typedef const __mpz_struct *mpz_srcptr;

void mpfr_init2(mpfr_ptr, mpfr_prec_t);
void mpfr_clear(mpfr_ptr);
void mpfr_set_prec(mpfr_ptr, mpfr_prec_t);
mpfr_prec_t mpfr_get_prec(mpfr_srcptr);
int mpfr_set(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_set_d(mpfr_ptr, double, mpfr_rnd_t);
int mpfr_set_flt(mpfr_ptr, float, mpfr_rnd_t);
int mpfr_set_ui_2exp(mpfr_ptr, unsigned long, mpfr_exp_t, mpfr_rnd_t);
double mpfr_get_d(mpfr_srcptr, mpfr_rnd_t);
float mpfr_get_flt(mpfr_srcptr, mpfr_rnd_t);
mpfr_exp_t mpfr_get_z_2exp(mpz_ptr, mpfr_srcptr);
int mpfr_sgn(mpfr_srcptr);
int mpfr_zero_p(mpfr_srcptr);
int mpfr_nan_p(mpfr_srcptr);
int mpfr_inf_p(mpfr_srcptr);
mpfr_exp_t mpfr_get_exp(mpfr_srcptr);
int mpfr_abs(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_neg(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_add(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_sub(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_mul(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_div(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_mul_2si(mpfr_ptr, mpfr_srcptr, long, mpfr_rnd_t);
int mpfr_div_2si(mpfr_ptr, mpfr_srcptr, long, mpfr_rnd_t);
int mpfr_add_d(mpfr_ptr, mpfr_srcptr, double, mpfr_rnd_t);
int mpfr_cmp(mpfr_srcptr, mpfr_srcptr);
int mpfr_const_pi(mpfr_ptr, mpfr_rnd_t);
void mpfr_free_cache(void);
mpfr_exp_t mpfr_get_emin(void);
mpfr_exp_t mpfr_get_emax(void);
int mpfr_set_emin(mpfr_exp_t);
int mpfr_set_emax(mpfr_exp_t);
int mpfr_check_range(mpfr_ptr, int, mpfr_rnd_t);
int mpfr_subnormalize(mpfr_ptr, int, mpfr_rnd_t);

int mpfr_exp(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_exp2(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_exp10(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_expm1(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_log(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_log2(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_log10(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_log1p(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_sin(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_cos(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_tan(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_asin(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_acos(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_atan(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_sinh(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_cosh(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_tanh(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_rec_sqrt(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);

void __gmpz_init(mpz_ptr);
void __gmpz_clear(mpz_ptr);
void __gmpz_abs(mpz_ptr, mpz_srcptr);
unsigned long __gmpz_scan1(mpz_srcptr, unsigned long);
void __gmpz_fdiv_q_2exp(mpz_ptr, mpz_srcptr, unsigned long);
unsigned long __gmpz_get_ui(mpz_srcptr);
unsigned long __gmpz_sizeinbase(mpz_srcptr, int);
#define mpz_init __gmpz_init
#define mpz_clear __gmpz_clear
#define mpz_abs __gmpz_abs
#define mpz_scan1 __gmpz_scan1
#define mpz_fdiv_q_2exp __gmpz_fdiv_q_2exp
#define mpz_get_ui __gmpz_get_ui
#define mpz_sizeinbase __gmpz_sizeinbase

#ifdef __cplusplus
}
#endif
#endif
