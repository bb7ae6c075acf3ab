// C ABI (include/crvec.h): argument checking, dispatch to the per-(function,
// mode) kernels, the pipelined host-pointer path, device counters.
//
// There is no CPU fallback anywhere: without an sm_100 device every entry
// point returns CRVEC_ENODEV.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "crvec.h"
#include "crvec_kernels.cuh"

namespace crvec {
void register_exp(FnEntry *t);
void register_log(FnEntry *t);
void register_trig(FnEntry *t);
void register_atrig(FnEntry *t);
int f64_dispatch(int fn, const double *x, double *y, size_t n, int mode, cudaStream_t s,
                 unsigned long long *ctr);
int f64_accurate_dispatch(int fn, const double *x, double *y, size_t n, int mode, cudaStream_t s,
                          unsigned long long *ctr);
int hardscan64_dispatch(int fn, const double *x, size_t n, double thr, double *ox, double *od,
                        unsigned long long cap, unsigned long long *count, cudaStream_t s);
int round_test_dispatch(const double *hi, const double *lo, const long long *scale,
                        const double *eps_rel, const double *eps_abs, int mode, double *val,
                        unsigned char *decided, size_t n, cudaStream_t s);
}  // namespace crvec

using namespace crvec;

namespace {

constexpr int kMaxDev = 16;
// Host-path pipeline chunk: 64 MiB of input per chunk (2^24 binary32 or 2^23
// binary64 elements; measured binary32: 2^21 10.3, 2^22 11.1, 2^24 11.4 Gelem/s).
constexpr size_t kChunkBytes = size_t(64) << 20;
constexpr int kPipe = 4;  // host path streams / staging sets

FnEntry g_table[CRVEC_FN_COUNT];
std::once_flag g_table_once;
std::atomic<uint64_t> g_lanes{0};
thread_local char g_err[256] = "";

struct Dev {
  std::atomic<bool> init{false};
  std::mutex mu;  // guards initialisation and this device's host-path staging
  int status = CRVEC_ENODEV;
  unsigned long long *counters = nullptr;  // [0] lanes (unused), [1] fast_undecided, [2] acc, [3] host
  // host-path staging: x, y and (sincosf only) the second output per pipe slot
  void *buf[kPipe][3] = {};
  size_t buf_bytes = 0;
  bool buf_y2 = false;
  cudaStream_t st[kPipe] = {};
};
Dev g_dev[kMaxDev];

int cuda_fail(cudaError_t e) {
  std::snprintf(g_err, sizeof(g_err), "%s", cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? CRVEC_ENOMEM : CRVEC_ECUDA;
}

// Current device, initialised on first use (sm_100 required). Each device's
// state is initialised once under its own mutex (double-checked on an atomic).
int device(Dev **out) {
  std::call_once(g_table_once, [] {
    register_exp(g_table);
    register_log(g_table);
    register_trig(g_table);
    register_atrig(g_table);
  });
  int d = 0;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess || d < 0 || d >= kMaxDev) {
    std::snprintf(g_err, sizeof(g_err), "no CUDA device: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return CRVEC_ENODEV;
  }
  Dev &D = g_dev[d];
  if (!D.init.load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lk(D.mu);
    if (!D.init.load(std::memory_order_relaxed)) {
      cudaDeviceProp p;
      e = cudaGetDeviceProperties(&p, d);
      if (e != cudaSuccess || p.major != 10) {
        std::snprintf(g_err, sizeof(g_err), "device %d is not sm_100 (cc %d.%d)", d,
                      e == cudaSuccess ? p.major : -1, e == cudaSuccess ? p.minor : -1);
        D.status = CRVEC_ENODEV;
      } else if ((e = cudaMalloc(&D.counters, 4 * sizeof(unsigned long long))) != cudaSuccess ||
                 (e = cudaMemset(D.counters, 0, 4 * sizeof(unsigned long long))) != cudaSuccess) {
        D.status = cuda_fail(e);
      } else {
        D.status = CRVEC_OK;
      }
      D.init.store(true, std::memory_order_release);
    }
  }
  *out = &D;
  return D.status;
}

int check_args(int fn, const void *x, const void *y, const void *y2, size_t n, int mode) {
  if (fn < 0 || fn >= CRVEC_FN_COUNT || mode < 0 || mode > 3) return CRVEC_EINVAL;
  if (n && (!x || !y)) return CRVEC_EINVAL;
  if (n && fn == CRVEC_FN_SINCOSF && !y2) return CRVEC_EINVAL;
  return CRVEC_OK;
}

int launch(Dev *D, int fn, const float *x, float *y, float *y2, size_t n, int mode,
           cudaStream_t s) {
  if (!n) return CRVEC_OK;
  g_lanes += n;
  cudaError_t e = g_table[fn].map[mode](x, y, y2, n, s, D->counters + 1);
  return e == cudaSuccess ? CRVEC_OK : cuda_fail(e);
}

void free_staging(Dev *D) {
  for (auto &b : D->buf)
    for (auto &p : b)
      if (p) { cudaFree(p); p = nullptr; }
  D->buf_bytes = 0;
  D->buf_y2 = false;
}

// Staging for the host path (caller holds D->mu): per pipe slot an input and
// an output buffer of `bytes`, plus a second output for sincosf.
int ensure_staging(Dev *D, size_t bytes, bool y2) {
  if (D->buf_bytes >= bytes && (D->buf_y2 || !y2)) return CRVEC_OK;
  if (D->buf_bytes < bytes) bytes = bytes > D->buf_bytes ? bytes : D->buf_bytes;
  y2 = y2 || D->buf_y2;
  free_staging(D);
  for (auto &b : D->buf)
    for (int j = 0; j < (y2 ? 3 : 2); ++j) {
      cudaError_t e = cudaMalloc(&b[j], bytes);
      if (e != cudaSuccess) { free_staging(D); return cuda_fail(e); }
    }
  for (auto &s : D->st)
    if (!s) {
      cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_fail(e);
    }
  D->buf_bytes = bytes;
  D->buf_y2 = y2;
  return CRVEC_OK;
}

// Host-pointer path: chunks rotate over kPipe streams (each with its own
// staging buffers) so H2D copies, kernels and D2H copies of different chunks
// overlap and both copy engines stay busy (fully when the host buffers are
// pinned; with two streams an H2D would wait behind its stream's D2H).
// Serialised per device (the staging is per device); calls on different
// devices run concurrently.
template <class T, class Launch>
int host_pipeline(Dev *D, const T *x, T *y, T *y2, size_t n, Launch &&lf) {
  std::lock_guard<std::mutex> lk(D->mu);
  const size_t kChunk = kChunkBytes / sizeof(T);
  size_t chunk = n < kChunk ? n : kChunk;
  int rc = ensure_staging(D, chunk * sizeof(T), y2 != nullptr);
  if (rc) return rc;
  size_t i = 0;
  for (size_t off = 0; off < n; off += chunk, ++i) {
    size_t cnt = n - off < chunk ? n - off : chunk;
    int k = (int)(i % kPipe);
    cudaStream_t s = D->st[k];
    T *dx = (T *)D->buf[k][0], *dy = (T *)D->buf[k][1], *dy2 = (T *)D->buf[k][2];
    cudaError_t e = cudaMemcpyAsync(dx, x + off, cnt * sizeof(T), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e);
    rc = lf(dx, dy, y2 ? dy2 : nullptr, cnt, s);
    if (rc) return rc;
    e = cudaMemcpyAsync(y + off, dy, cnt * sizeof(T), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && y2)
      e = cudaMemcpyAsync(y2 + off, dy2, cnt * sizeof(T), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  for (auto s : D->st) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  return CRVEC_OK;
}

// ---- map-kernel sweep (force mode 3): the PRODUCT map kernels over every
// pattern of a chunk range, in all four modes, hashed like the sweep kernels
// (the sweep kernels share the function code but not the streaming template,
// the rare-path forms or the kernel shapes; this run covers those too).
__global__ void k_iota(uint32_t *x, uint32_t first, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[i] = first + i;
}
// one block per 4096 patterns (256 blocks per 2^20 chunk): h[chunk*4 + mode] +=
// sum mix64((y << 32) | p)
__global__ void __launch_bounds__(crvec::kThreads) k_hash_chunks(const uint32_t *y, uint32_t first,
                                                                 uint64_t *h, int mode) {
  const uint32_t i0 = blockIdx.x * (uint32_t)crvec::kSweepPerBlock;
  uint64_t acc[1] = {0};
  for (int j = 0; j < crvec::kSweepPerThread; ++j) {
    const uint32_t i = i0 + j * crvec::kThreads + threadIdx.x;
    acc[0] += crvec::mix64(((uint64_t)y[i] << 32) | (uint64_t)(first + i));
  }
  crvec::block_add<1>(acc, h + 4ull * (blockIdx.x / crvec::kSweepBlocksPerChunk) + mode);
}

// misaligned = true: the input sits one float past a 256-byte boundary and
// the outputs on one, so the arrays are relatively misaligned and the whole
// range runs the element kernel (k_map_scalar) instead of the vector kernel.
int map_sweep(Dev *D, int fn, uint32_t chunk_lo, uint32_t chunk_hi, uint64_t *h, uint64_t *h2,
              cudaStream_t s, bool misaligned = false) {
  constexpr uint32_t kBlockChunks = 64;  // 2^26 patterns (256 MiB) per pass
  const uint32_t cap = kBlockChunks << 20;
  uint32_t *xbuf = nullptr, *y = nullptr, *y2 = nullptr;
  cudaError_t e = cudaMallocAsync((void **)&xbuf, 4ull * cap + 256, s);
  uint32_t *x = xbuf + (misaligned ? 1 : 0);
  if (e == cudaSuccess) e = cudaMallocAsync((void **)&y, 4ull * cap, s);
  if (e == cudaSuccess && h2) e = cudaMallocAsync((void **)&y2, 4ull * cap, s);
  int rc = e == cudaSuccess ? CRVEC_OK : cuda_fail(e);
  for (uint32_t c = chunk_lo; rc == CRVEC_OK && c < chunk_hi; c += kBlockChunks) {
    const uint32_t nc = chunk_hi - c < kBlockChunks ? chunk_hi - c : kBlockChunks;
    const uint32_t n = nc << 20, first = c << 20;
    k_iota<<<1184, 256, 0, s>>>(x, first, n);
    for (int m = 0; m < 4 && rc == CRVEC_OK; ++m) {
      rc = launch(D, fn, (const float *)x, (float *)y, (float *)y2, n, m, s);
      if (rc) break;
      const unsigned blocks = nc * crvec::kSweepBlocksPerChunk;
      k_hash_chunks<<<blocks, crvec::kThreads, 0, s>>>(y, first, h + 4ull * (c - chunk_lo), m);
      if (h2) k_hash_chunks<<<blocks, crvec::kThreads, 0, s>>>(y2, first, h2 + 4ull * (c - chunk_lo), m);
      e = cudaGetLastError();
      if (e != cudaSuccess) rc = cuda_fail(e);
    }
  }
  if (xbuf) cudaFreeAsync(xbuf, s);
  if (y) cudaFreeAsync(y, s);
  if (y2) cudaFreeAsync(y2, s);
  return rc;
}

}  // namespace

extern "C" {

int crvec_eval_f32_dev(crvec_fn_t fn, const float *x, float *y, float *y2, size_t n,
                       crvec_mode_t mode, void *stream) {
  int rc = check_args(fn, x, y, y2, n, mode);
  if (rc) return rc;
  Dev *D;
  if ((rc = device(&D))) return rc;
  return launch(D, fn, x, y, y2, n, mode, (cudaStream_t)stream);
}

int crvec_eval_f32(crvec_fn_t fn, const float *x, float *y, float *y2, size_t n,
                   crvec_mode_t mode) {
  int rc = check_args(fn, x, y, y2, n, mode);
  if (rc || !n) return rc;
  Dev *D;
  if ((rc = device(&D))) return rc;
  return host_pipeline<float>(D, x, y, fn == CRVEC_FN_SINCOSF ? y2 : nullptr, n,
                              [&](const float *dx, float *dy, float *dy2, size_t cnt,
                                  cudaStream_t s) { return launch(D, fn, dx, dy, dy2, cnt, mode, s); });
}

#define CRVEC_DEF(name, id)                                                                 \
  int crvec_##name(const float *x, float *y, size_t n, crvec_mode_t m) {                    \
    return crvec_eval_f32(id, x, y, nullptr, n, m);                                         \
  }                                                                                         \
  int crvec_##name##_dev(const float *x, float *y, size_t n, crvec_mode_t m, void *s) {     \
    return crvec_eval_f32_dev(id, x, y, nullptr, n, m, s);                                  \
  }
CRVEC_DEF(expf, CRVEC_FN_EXPF)
CRVEC_DEF(exp2f, CRVEC_FN_EXP2F)
CRVEC_DEF(exp10f, CRVEC_FN_EXP10F)
CRVEC_DEF(expm1f, CRVEC_FN_EXPM1F)
CRVEC_DEF(logf, CRVEC_FN_LOGF)
CRVEC_DEF(log2f, CRVEC_FN_LOG2F)
CRVEC_DEF(log10f, CRVEC_FN_LOG10F)
CRVEC_DEF(log1pf, CRVEC_FN_LOG1PF)
CRVEC_DEF(sinf, CRVEC_FN_SINF)
CRVEC_DEF(cosf, CRVEC_FN_COSF)
CRVEC_DEF(tanf, CRVEC_FN_TANF)
CRVEC_DEF(asinf, CRVEC_FN_ASINF)
CRVEC_DEF(acosf, CRVEC_FN_ACOSF)
CRVEC_DEF(atanf, CRVEC_FN_ATANF)
CRVEC_DEF(sinhf, CRVEC_FN_SINHF)
CRVEC_DEF(coshf, CRVEC_FN_COSHF)
CRVEC_DEF(tanhf, CRVEC_FN_TANHF)
CRVEC_DEF(rsqrtf, CRVEC_FN_RSQRTF)
#undef CRVEC_DEF

int crvec_sincosf(const float *x, float *s, float *c, size_t n, crvec_mode_t m) {
  return crvec_eval_f32(CRVEC_FN_SINCOSF, x, s, c, n, m);
}
int crvec_sincosf_dev(const float *x, float *s, float *c, size_t n, crvec_mode_t m, void *st) {
  return crvec_eval_f32_dev(CRVEC_FN_SINCOSF, x, s, c, n, m, st);
}

#ifdef CRVEC_WITH_F64
// ---- binary64 ----
static int eval_f64(int fn, const double *x, double *y, size_t n, int mode, crvec_stats_t *stats) {
  if (mode < 0 || mode > 3 || (n && (!x || !y))) return CRVEC_EINVAL;
  if (!n) return CRVEC_OK;
  Dev *D;
  int rc = device(&D);
  if (rc) return rc;
  unsigned long long before[4] = {0, 0, 0, 0}, after[4] = {0, 0, 0, 0};
  if (stats) cudaMemcpy(before, D->counters, sizeof(before), cudaMemcpyDeviceToHost);
  g_lanes += n;
  rc = host_pipeline<double>(D, x, y, nullptr, n,
                             [&](const double *dx, double *dy, double *, size_t cnt, cudaStream_t s) {
                               return f64_dispatch(fn, dx, dy, cnt, mode, s, D->counters);
                             });
  if (rc) return rc;
  if (stats) {
    cudaMemcpy(after, D->counters, sizeof(after), cudaMemcpyDeviceToHost);
    stats->lanes = n;
    stats->fast_undecided = after[1] - before[1];
    stats->accurate_undecided = after[2] - before[2];
    stats->host_callouts = after[3] - before[3];
  }
  return CRVEC_OK;
}
static int eval_f64_dev(int fn, const double *x, double *y, size_t n, int mode, void *stream) {
  if (mode < 0 || mode > 3 || (n && (!x || !y))) return CRVEC_EINVAL;
  if (!n) return CRVEC_OK;
  Dev *D;
  int rc = device(&D);
  if (rc) return rc;
  g_lanes += n;
  return f64_dispatch(fn, x, y, n, mode, (cudaStream_t)stream, D->counters);
}
int crvec_exp2(const double *x, double *y, size_t n, crvec_mode_t m, crvec_stats_t *st) {
  return eval_f64(0, x, y, n, m, st);
}
int crvec_log(const double *x, double *y, size_t n, crvec_mode_t m, crvec_stats_t *st) {
  return eval_f64(1, x, y, n, m, st);
}
int crvec_exp2_dev(const double *x, double *y, size_t n, crvec_mode_t m, void *s) {
  return eval_f64_dev(0, x, y, n, m, s);
}
int crvec_log_dev(const double *x, double *y, size_t n, crvec_mode_t m, void *s) {
  return eval_f64_dev(1, x, y, n, m, s);
}
int crvec_f64_accurate_dev(int fn, const double *x, double *y, size_t n, crvec_mode_t m,
                           void *stream) {
  if (fn < 0 || fn > 1 || m < 0 || m > 3 || (n && (!x || !y))) return CRVEC_EINVAL;
  Dev *D;
  int rc = device(&D);
  if (rc) return rc;
  return f64_accurate_dispatch(fn, x, y, n, m, (cudaStream_t)stream, D->counters + 1) ? CRVEC_ECUDA
                                                                                       : CRVEC_OK;
}

int crvec_hardcase_scan_f64(int fn, const double *x, size_t n, double rel_threshold, double *out_x,
                            double *out_dist, uint64_t capacity, uint64_t *count, void *stream) {
  if (fn < 0 || fn > 1 || !count || (n && !x) || (capacity && (!out_x || !out_dist))) return CRVEC_EINVAL;
  Dev *D;
  int rc = device(&D);
  if (rc) return rc;
  return hardscan64_dispatch(fn, x, n, rel_threshold, out_x, out_dist, (unsigned long long)capacity,
                             (unsigned long long *)count, (cudaStream_t)stream)
             ? CRVEC_ECUDA : CRVEC_OK;
}

// Host-pointer callout: every lane through the binary64 accurate path (the
// GPU replacement of the reference's scalar MPFR callout).
int crvec_callout_f64(int fn, const double *x, double *y, size_t n, crvec_mode_t m) {
  if (fn < 0 || fn > 1 || m < 0 || m > 3 || (n && (!x || !y))) return CRVEC_EINVAL;
  if (!n) return CRVEC_OK;
  Dev *D;
  int rc = device(&D);
  if (rc) return rc;
  return host_pipeline<double>(D, x, y, nullptr, n,
                               [&](const double *dx, double *dy, double *, size_t cnt, cudaStream_t s) {
                                 return f64_accurate_dispatch(fn, dx, dy, cnt, m, s, D->counters + 1)
                                            ? CRVEC_ECUDA : CRVEC_OK;
                               });
}

int crvec_round_test_f64(const double *hi, const double *lo, const int64_t *scale,
                         const double *eps_rel, const double *eps_abs, crvec_mode_t m, double *value,
                         unsigned char *decided, size_t n) {
  if (m < 0 || m > 3 || (n && (!hi || !lo || !value || !decided))) return CRVEC_EINVAL;
  if (!n) return CRVEC_OK;
  Dev *D;
  int rc = device(&D);
  if (rc) return rc;
  cudaStream_t s = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_fail(e);
  // one device block: hi, lo, value, scale, eps_rel, eps_abs (8 B each), decided (1 B)
  const size_t b8 = n * 8;
  char *buf = nullptr;
  e = cudaMallocAsync((void **)&buf, 6 * b8 + n, s);
  if (e == cudaSuccess) {
    double *dh = (double *)buf, *dl = dh + n, *dv = dl + n;
    long long *dsc = scale ? (long long *)(dv + n) : nullptr;
    double *der = eps_rel ? dv + 2 * n : nullptr, *dea = eps_abs ? dv + 3 * n : nullptr;
    unsigned char *dd = (unsigned char *)(dv + 4 * n);
    auto h2d = [&](void *d, const void *h) {
      return h ? cudaMemcpyAsync(d, h, b8, cudaMemcpyHostToDevice, s) : cudaSuccess;
    };
    if ((e = h2d(dh, hi)) == cudaSuccess && (e = h2d(dl, lo)) == cudaSuccess &&
        (e = h2d(dsc, scale)) == cudaSuccess && (e = h2d(der, eps_rel)) == cudaSuccess &&
        (e = h2d(dea, eps_abs)) == cudaSuccess) {
      if (round_test_dispatch(dh, dl, dsc, der, dea, m, dv, dd, n, s)) e = cudaGetLastError();
      if (e == cudaSuccess && (e = cudaMemcpyAsync(value, dv, b8, cudaMemcpyDeviceToHost, s)) == cudaSuccess)
        e = cudaMemcpyAsync(decided, dd, n, cudaMemcpyDeviceToHost, s);
    }
    cudaFreeAsync(buf, s);
  }
  cudaError_t e2 = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (e == cudaSuccess) e = e2;
  return e == cudaSuccess ? CRVEC_OK : cuda_fail(e);
}

#endif

// ---- sweep ----
int crvec_sweep_f32(crvec_fn_t fn, uint32_t chunk_lo, uint32_t chunk_hi, uint64_t *hashes,
                    uint64_t *hashes2, uint64_t *counters, int force_accurate, void *stream) {
  if (fn < 0 || fn >= CRVEC_FN_COUNT || chunk_hi > 4096 || chunk_lo >= chunk_hi || !hashes ||
      !counters || (fn == CRVEC_FN_SINCOSF && !hashes2))
    return CRVEC_EINVAL;
  Dev *D;
  int rc = device(&D);
  if (rc) return rc;
  if (force_accurate == 3 || force_accurate == 4)
    return map_sweep(D, fn, chunk_lo, chunk_hi, hashes, fn == CRVEC_FN_SINCOSF ? hashes2 : nullptr,
                     (cudaStream_t)stream, force_accurate == 4);
  cudaError_t e = g_table[fn].sweep(chunk_lo, chunk_hi, hashes, hashes2, force_accurate,
                                    (cudaStream_t)stream, (unsigned long long *)counters);
  return e == cudaSuccess ? CRVEC_OK : cuda_fail(e);
}

// ---- hard-case screen ----
int crvec_hardcase_scan_f32(crvec_fn_t fn, uint32_t chunk_lo, uint32_t chunk_hi, double rel_threshold,
                            uint32_t *out_bits, double *out_dist, uint64_t capacity,
                            uint64_t *count, void *stream) {
  if (fn < 0 || fn >= CRVEC_FN_COUNT || fn == CRVEC_FN_SINCOSF || chunk_hi > 4096 ||
      chunk_lo >= chunk_hi || !count || (capacity && (!out_bits || !out_dist)))
    return CRVEC_EINVAL;
  Dev *D;
  int rc = device(&D);
  if (rc) return rc;
  cudaError_t e = g_table[fn].scan(chunk_lo, chunk_hi, rel_threshold, out_bits, out_dist,
                                   (unsigned long long)capacity, (unsigned long long *)count,
                                   (cudaStream_t)stream);
  return e == cudaSuccess ? CRVEC_OK : cuda_fail(e);
}

// ---- workspace ----
int crvec_workspace_release(void) {
  Dev *D;
  int rc = device(&D);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(D->mu);
  for (auto s : D->st)
    if (s) cudaStreamSynchronize(s);
  free_staging(D);
  return CRVEC_OK;
}
size_t crvec_workspace_bytes(void) {
  Dev *D;
  if (device(&D)) return 0;
  std::lock_guard<std::mutex> lk(D->mu);
  return D->buf_bytes * kPipe * (D->buf_y2 ? 3 : 2);
}

// ---- accounting ----
int crvec_stats_get(crvec_stats_t *out) {
  if (!out) return CRVEC_EINVAL;
  Dev *D;
  int rc = device(&D);
  if (rc) return rc;
  unsigned long long c[4];
  cudaError_t e = cudaMemcpy(c, D->counters, sizeof(c), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e);
  out->lanes = g_lanes.load();
  out->fast_undecided = c[1];
  out->accurate_undecided = c[2];
  out->host_callouts = c[3];
  return CRVEC_OK;
}
int crvec_stats_reset(void) {
  Dev *D;
  int rc = device(&D);
  if (rc) return rc;
  g_lanes = 0;
  cudaError_t e = cudaMemset(D->counters, 0, 4 * sizeof(unsigned long long));
  return e == cudaSuccess ? CRVEC_OK : cuda_fail(e);
}

const char *crvec_strerror(int code) {
  switch (code) {
    case CRVEC_OK: return "ok";
    case CRVEC_EINVAL: return "invalid argument";
    case CRVEC_ECUDA: return "CUDA runtime error";
    case CRVEC_ENOMEM: return "device allocation failed";
    case CRVEC_ENODEV: return "no usable sm_100 CUDA device";
  }
  return "unknown error";
}
const char *crvec_last_cuda_error(void) { return g_err; }
const char *crvec_version(void) { return "crvec-b200 0.1 (sm_100a)"; }
int crvec_fn_count(void) { return CRVEC_FN_COUNT; }
const char *crvec_fn_name(crvec_fn_t fn) {
  static const char *names[CRVEC_FN_COUNT] = {
      "exp2f", "logf",  "log2f", "expf",  "exp10f", "expm1f", "log10f", "log1pf", "sinf", "cosf",
      "tanf",  "asinf", "acosf", "atanf", "sinhf",  "coshf",  "tanhf",  "rsqrtf", "sincosf"};
  return (fn >= 0 && fn < CRVEC_FN_COUNT) ? names[fn] : "?";
}

}  // extern "C"
