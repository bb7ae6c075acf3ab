/* crvec.h — C ABI of the B200-native correctly rounded (CR) vector math library.
 *
 * Drop-in array boundary for the paper's CR functions (arxiv 2605.15547,
 * "Correctly Rounded Functions For Vector Applications"). The reference's
 * public surface is C++ templates over lane batches; each entry point below
 * replaces one of them with an array-in/array-out call:
 *
 *   crvec_exp2f / crvec_exp2f_dev  <- template cr_exp2f<W>(Batch<float,W>, RoundingMode, Backend)
 *                                     and cr_exp2f_scalar(float, RoundingMode)
 *                                     (ref: proj/include/crvec/kernels_f32.hpp:27-35,
 *                                      proj/src/kernels_f32.cpp:170-181)
 *   crvec_log2f / crvec_log2f_dev  <- cr_log2f<W>, cr_log2f_scalar
 *                                     (ref: proj/include/crvec/kernels_f32.hpp:30-35,
 *                                      proj/src/kernels_f32.cpp:171,183-191)
 *   crvec_<fn>f for the other 17 binary32 functions of ref: PAPER.md:49
 *                                     (no reference code; same contract)
 *   crvec_exp2 / crvec_log (+ _dev) <- cr_exp2<W>, cr_log<W>, cr_exp2_scalar, cr_log_scalar,
 *                                     cr_exp2_counted / cr_log_counted with FastPathStats
 *                                     (ref: proj/include/crvec/kernels_f64.hpp:58-81)
 *   crvec_sweep_f32                <- exhaustive_f32 of the verify module
 *                                     (ref: SPEC.md:250-258; proj/src/verify.cpp:1 is a stub)
 *
 * Conventions (ref: proj/include/crvec/fpbits.hpp:13-18, SPEC.md "[OP] cr_exp2f"):
 *   - rounding modes are numbered as the reference's RoundingMode;
 *   - every bit pattern is accepted; specials are values, never errors:
 *     NaN in -> quiet(x) (payload and sign kept), invalid -> +qNaN 0x7FC00000;
 *   - return 0 on success or a negative CRVEC_E* code; no exceptions cross
 *     the ABI; there is no CPU fallback: without a usable CUDA device every
 *     entry point returns CRVEC_ENODEV;
 *   - host-pointer calls are synchronous; _dev calls take device pointers
 *     and a cudaStream_t (passed as void*, NULL = default stream) and are
 *     stream-ordered; in-place (x == y) is allowed; any alignment accepted.
 *   - reentrant: the library keeps per device a mutex-guarded staging
 *     workspace for the host-pointer calls (see crvec_workspace_bytes) and
 *     device-side counters; host-pointer calls on one device are serialised,
 *     calls on different devices run concurrently; _dev calls take no lock.
 */
#ifndef CRVEC_H
#define CRVEC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CRVEC_RNE = 0, /* RoundingMode::NearestEven */
  CRVEC_RZ = 1,  /* RoundingMode::TowardZero */
  CRVEC_RU = 2,  /* RoundingMode::TowardPositive */
  CRVEC_RD = 3   /* RoundingMode::TowardNegative */
} crvec_mode_t;

/* Function ids; the first three follow the reference FuncId order
 * (ref: proj/include/crvec/oracle.hpp:21). */
typedef enum {
  CRVEC_FN_EXP2F = 0, CRVEC_FN_LOGF = 1, CRVEC_FN_LOG2F = 2, CRVEC_FN_EXPF = 3,
  CRVEC_FN_EXP10F = 4, CRVEC_FN_EXPM1F = 5, CRVEC_FN_LOG10F = 6, CRVEC_FN_LOG1PF = 7,
  CRVEC_FN_SINF = 8, CRVEC_FN_COSF = 9, CRVEC_FN_TANF = 10, CRVEC_FN_ASINF = 11,
  CRVEC_FN_ACOSF = 12, CRVEC_FN_ATANF = 13, CRVEC_FN_SINHF = 14, CRVEC_FN_COSHF = 15,
  CRVEC_FN_TANHF = 16, CRVEC_FN_RSQRTF = 17, CRVEC_FN_SINCOSF = 18,
  CRVEC_FN_COUNT = 19
} crvec_fn_t;

#define CRVEC_OK 0
#define CRVEC_EINVAL (-1)  /* bad mode / function id / null pointer with n > 0 */
#define CRVEC_ECUDA (-2)   /* CUDA runtime error (see crvec_last_cuda_error) */
#define CRVEC_ENOMEM (-3)  /* device allocation failed */
#define CRVEC_ENODEV (-4)  /* no usable sm_100 device */

/* Fast-path accounting, mirrors FastPathStats (ref: proj/include/crvec/kernels_f64.hpp:72-81)
 * extended with the accurate-path tiers of this implementation. */
typedef struct {
  uint64_t lanes;              /* elements evaluated */
  uint64_t fast_undecided;     /* lanes whose fast-path rounding test failed */
  uint64_t accurate_undecided; /* fp64: lanes whose accurate-path test also failed */
  uint64_t host_callouts;      /* fp64: lanes resolved by the counted last resort */
} crvec_stats_t;

/* ---- binary32, host pointers (synchronous) ---- */
int crvec_expf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_exp2f(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_exp10f(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_expm1f(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_logf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_log2f(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_log10f(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_log1pf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_sinf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_cosf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_tanf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_asinf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_acosf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_atanf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_sinhf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_coshf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_tanhf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_rsqrtf(const float *x, float *y, size_t n, crvec_mode_t mode);
int crvec_sincosf(const float *x, float *s, float *c, size_t n, crvec_mode_t mode);

/* ---- binary32, device pointers (stream-ordered) ---- */
int crvec_expf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_exp2f_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_exp10f_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_expm1f_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_logf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_log2f_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_log10f_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_log1pf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_sinf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_cosf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_tanf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_asinf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_acosf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_atanf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_sinhf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_coshf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_tanhf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_rsqrtf_dev(const float *x, float *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_sincosf_dev(const float *x, float *s, float *c, size_t n, crvec_mode_t mode, void *stream);

/* Generic forms (y2 used by CRVEC_FN_SINCOSF only). */
int crvec_eval_f32(crvec_fn_t fn, const float *x, float *y, float *y2, size_t n, crvec_mode_t mode);
int crvec_eval_f32_dev(crvec_fn_t fn, const float *x, float *y, float *y2, size_t n,
                       crvec_mode_t mode, void *stream);

/* ---- binary64 exp2 / log (fast path + ballot-compacted accurate path) ---- */
int crvec_exp2(const double *x, double *y, size_t n, crvec_mode_t mode, crvec_stats_t *stats);
int crvec_log(const double *x, double *y, size_t n, crvec_mode_t mode, crvec_stats_t *stats);
int crvec_exp2_dev(const double *x, double *y, size_t n, crvec_mode_t mode, void *stream);
int crvec_log_dev(const double *x, double *y, size_t n, crvec_mode_t mode, void *stream);
/* Verification entry point: every non-special lane through the binary64
 * accurate path (fn 0 = exp2, 1 = log); device pointers. */
int crvec_f64_accurate_dev(int fn, const double *x, double *y, size_t n, crvec_mode_t mode,
                           void *stream);

/* Host-pointer callout: every lane through the binary64 accurate path (fn 0 =
 * exp2, 1 = log). Replaces the reference's scalar MPFR fallback
 * callout(FuncId, double, RoundingMode) (ref: proj/include/crvec/kernels_f64.hpp:58-59,
 * proj/src/kernels_f64.cpp:78-80). */
int crvec_callout_f64(int fn, const double *x, double *y, size_t n, crvec_mode_t mode);

/* The reference's Ziv straddle test over n lanes (ref: proj/include/crvec/kernels_f64.hpp:27-56,
 * proj/src/kernels_f64.cpp:63-76 round_test_lane): per lane, bound
 * b = (eps_rel[i] |hi[i]| + eps_abs[i]) (1 + 2^-30) + 2^-1000; value[i] = (hi + lo - b) * 2^scale[i]
 * rounded exactly to binary64 in `mode` (normal, subnormal or overflowing);
 * decided[i] = 1 iff (hi + lo + b) * 2^scale[i] rounds to the same value.
 * scale / eps_rel / eps_abs may be NULL (all zero). Host pointers; evaluated on the GPU. */
int crvec_round_test_f64(const double *hi, const double *lo, const int64_t *scale,
                         const double *eps_rel, const double *eps_abs, crvec_mode_t mode,
                         double *value, unsigned char *decided, size_t n);

/* ---- exhaustive binary32 sweep (verify) ----
 * For chunks [chunk_lo, chunk_hi) of 2^20 bit patterns (chunk c = patterns
 * c<<20 .. (c<<20)+2^20-1), adds into hashes[(c - chunk_lo)*4 + mode]
 *   sum_p mix64(((uint64)out_mode(p) << 32) | p)   (mod 2^64)
 * for all four modes at once; for CRVEC_FN_SINCOSF, hashes2 receives the cos
 * outputs' hashes. hashes / hashes2 / counters are DEVICE pointers and must be
 * zeroed by the caller (the sweep accumulates). counters[0] += fast-path
 * lanes sent to the accurate path. force_accurate: 0 = the sweep kernels'
 * fast path + accurate fallback; 1 routes every non-special lane through the
 * accurate path (self-check of that path); 3 runs the PRODUCT map kernels (the
 * crvec_<fn>f_dev path, with its streaming template, rare-path form and
 * shape) over the chunks' patterns in all four modes and hashes their outputs
 * the same way (stream-ordered device workspace of 512-768 MiB); 4 does the
 * same with relatively misaligned input / output arrays, i.e. through the
 * element kernel that serves unaligned calls. */
int crvec_sweep_f32(crvec_fn_t fn, uint32_t chunk_lo, uint32_t chunk_hi, uint64_t *hashes,
                    uint64_t *hashes2, uint64_t *counters, int force_accurate, void *stream);

/* ---- hard-case screen (GPU worst-case finder) ----
 * Evaluates every pattern of chunks [chunk_lo, chunk_hi) on the double-double
 * path and appends inputs whose value lies within rel_threshold (relative) of a
 * binary32 rounding boundary: out_bits / out_dist (device, capacity entries),
 * *count (device, caller-zeroed) = total candidates found. The GPU analogue of
 * the reference's hardest_case_search (ref: proj/src/oracle.cpp:565-580); the
 * exact ranking is then confirmed by the oracle's boundary distance. */
int crvec_hardcase_scan_f32(crvec_fn_t fn, uint32_t chunk_lo, uint32_t chunk_hi, double rel_threshold,
                            uint32_t *out_bits, double *out_dist, uint64_t capacity,
                            uint64_t *count, void *stream);

/* ---- host-path workspace ----
 * The host-pointer calls stage data through per-device device buffers
 * (4 pipeline slots x {input, output[, second output for sincosf]} x up to
 * 64 MiB), allocated on first use and kept for later calls. */
int crvec_workspace_release(void);    /* free the current device's staging buffers */
size_t crvec_workspace_bytes(void);   /* bytes currently held on the current device */

/* Binary64 hard-case screen: for the n inputs x (device), the fast-path value
 * of exp2 (fn 0) or log (fn 1) and its distance to the nearest binary64 rounding
 * boundary relative to the value; main-range inputs closer than rel_threshold
 * are appended to out_x / out_dist (device, capacity entries), *count (device,
 * caller-zeroed) = candidates found. Seeds the binary64 hard set whose exact
 * ranking uses the reference's boundary_distance_f64 (ref: proj/src/oracle.cpp:502-563). */
int crvec_hardcase_scan_f64(int fn, const double *x, size_t n, double rel_threshold, double *out_x,
                            double *out_dist, uint64_t capacity, uint64_t *count, void *stream);

/* ---- accounting / errors ---- */
int crvec_stats_get(crvec_stats_t *out);   /* cumulative since load / last reset */
int crvec_stats_reset(void);
const char *crvec_strerror(int code);
const char *crvec_last_cuda_error(void);
const char *crvec_version(void);
int crvec_fn_count(void);
const char *crvec_fn_name(crvec_fn_t fn);

#ifdef __cplusplus
}
#endif
#endif /* CRVEC_H */
