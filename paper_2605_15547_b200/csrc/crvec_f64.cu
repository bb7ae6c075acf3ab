// Binary64 exp2 / log kernels: double-double fast path + Ziv round test in
// registers; undecided lanes are compacted per warp with __ballot_sync into a
// shared-memory side queue and evaluated by FULL warps on the 256-bit
// fixed-point accurate path, so a rare hard case never serialises the warp's
// fast path (ref: "an entire packed vector computation is
// disrupted when one element requires the accurate path").
#include <cuda_runtime.h>

#include "crvec_fns_f64.cuh"

namespace crvec {

constexpr int kT64 = 256;
constexpr int kW64 = kT64 / 32;
// Kernel shape per function (measured, profiles/r01/f64_shapes.txt): double2
// per lane per step, __launch_bounds__ min blocks per SM, grid waves.
template <int FN> struct F64Shape;
// dist = prefetch distance in loop steps; measured per function (profiles/r01/f64_shapes.txt)
#ifndef CRVEC_LOG64_SHAPE
#define CRVEC_LOG64_SHAPE nv = 2, minb = 3, waves = 1, dist = 1
#endif
template <> struct F64Shape<0> { static constexpr int nv = 1, minb = 4, waves = 4, dist = 2; };  // exp2
template <> struct F64Shape<1> { static constexpr int CRVEC_LOG64_SHAPE; };                      // log
constexpr int kF64MaxNV = 2;
constexpr int kQ = 32 + 32 * 2 * kF64MaxNV;  // per-warp queue capacity: < 32 left + one step

struct F64Queue {
  double x[kQ];
  unsigned long long idx[kQ];
};

// Shared-memory copy of the function's fast-path tables (exp2: 2 KB, log: 12 KB).
template <int FN>
__device__ __forceinline__ void load_tables(F64Tab &T) {
  if (FN == 0) {
    for (int i = threadIdx.x; i < 64; i += kT64) {
      T.ta[i] = Pair64{EXP2D_A_HI[i], EXP2D_A_LO[i]};
      T.tb[i] = Pair64{EXP2D_B_HI[i], EXP2D_B_LO[i]};
    }
  } else {
    for (int i = threadIdx.x; i < 512; i += kT64) {
      T.lc[i] = Pair64{LOGD5_C[i], LOGD5_LT_HI[i]};
      T.lll[i] = LOGD5_LT_LO[i];
    }
  }
  __syncthreads();
}

template <int FN, int M>
__device__ __noinline__ double accurate(double x, int *und) {
  return FN == 0 ? exp2d_accurate<M>(x, und) : logd_accurate<M>(x, und);
}

// Drain `cnt` (<= 32) queue entries starting at `from`: one entry per lane.
// The entry is first re-run through the rule-complete fast path (specials,
// exact integers, subnormal arguments); what it cannot decide goes to the
// accurate path. ctr[0] counts lanes sent to the accurate path, ctr[1] the
// ones it could not decide either.
template <int FN, int M>
__device__ __forceinline__ void drain(F64Queue &q, int from, int cnt, const F64Tab &T, double *y,
                                      unsigned long long *ctr) {
  int lane = threadIdx.x & 31;
  int und = 0;
  bool acc = false;
  if (lane < cnt) {
    double xv = q.x[from + lane];
    unsigned long long i = q.idx[from + lane];
    F64Out r = FN == 0 ? exp2d_fast<M>(xv, T) : logd_fast<M>(xv, T);
    if (!r.decided) {
      acc = true;
      r.y = accurate<FN, M>(xv, &und);
    }
    y[i] = r.y;
  }
  unsigned ma = __ballot_sync(0xffffffffu, acc), mu = __ballot_sync(0xffffffffu, und);
  if (lane == 0 && ma) atomicAdd(ctr, (unsigned long long)__popc(ma));
  if (lane == 0 && mu) atomicAdd(ctr + 1, (unsigned long long)__popc(mu));
}

// One step: NE = 2*NV doubles per lane (NV double2 per lane, 32 lanes apart
// so each warp access is 512 B contiguous), fast path + round test, stores,
// then the undecided lanes are appended to the warp's side queue; a full
// queue (32) is drained by the whole warp on the accurate path.
template <int FN, int M, int NV>
__device__ __forceinline__ void f64_step(const double2 *__restrict__ x2, double2 *__restrict__ y2,
                                         const double *x, double *y, uint32_t n2, uint64_t n, uint32_t base,
                                         uint32_t stride, const double2 (&cur)[NV],
                                         double2 (&nxt)[NV], const F64Tab &T, F64Queue &q,
                                         int &qn,
                                         unsigned long long *ctr) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const uint32_t in = base + F64Shape<FN>::dist * stride + 32 * k;
    if (in < n2) nxt[k] = __ldcs(x2 + in);  // n is even: every slot holds two doubles
  }
  double xv[2 * NV];
  F64Out r[2 * NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    xv[2 * k] = cur[k].x;
    xv[2 * k + 1] = cur[k].y;
  }
#pragma unroll
  for (int e = 0; e < 2 * NV; ++e)
    r[e] = FN == 0 ? exp2d_main_path<M>(xv[e], T) : logd_main_path<M>(xv[e], T);
  unsigned und = 0;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const uint32_t i = base + 32 * k;
    if (i < n2) {
      __stcs(y2 + i, make_double2(r[2 * k].y, r[2 * k + 1].y));
      und |= (unsigned)(!r[2 * k].decided) << (2 * k);
      und |= (unsigned)(!r[2 * k + 1].decided) << (2 * k + 1);
    }
  }
  // compact undecided lanes into the warp's side queue
  if (__any_sync(0xffffffffu, und != 0)) {
#pragma unroll
    for (int e = 0; e < 2 * NV; ++e) {
      const bool u = (und >> e) & 1u;
      const unsigned m = __ballot_sync(0xffffffffu, u);
      if (u) {
        const int p = qn + __popc(m & lt);
        q.x[p] = xv[e];
        q.idx[p] = 2ull * (base + 32 * (e >> 1)) + (e & 1);
      }
      qn += __popc(m);
    }
    __syncwarp();
    while (qn >= 32) {  // a full warp of hard lanes: evaluate together
      drain<FN, M>(q, qn - 32, 32, T, y, ctr);
      qn -= 32;
      __syncwarp();
    }
  }
}

template <int FN, int M>
__global__ void __launch_bounds__(kT64, F64Shape<FN>::minb) k_f64(const double *x, double *y, uint64_t n,
                                                 unsigned long long *ctr) {
  constexpr int NV = F64Shape<FN>::nv;
  __shared__ F64Tab T;
  __shared__ F64Queue Q[kW64];
  load_tables<FN>(T);
  F64Queue &q = Q[threadIdx.x >> 5];
  const uint32_t lane = threadIdx.x & 31;
  int qn = 0;  // warp-uniform queue length
  // 16-byte aligned x / y and an even n (the launcher guarantees both)
  const double2 *x2 = reinterpret_cast<const double2 *>(x);
  double2 *y2 = reinterpret_cast<double2 *>(y);
  const uint32_t n2 = (uint32_t)((n + 1) / 2);
  const uint32_t stride = gridDim.x * (uint32_t)(kT64 * NV);
  uint32_t base = ((blockIdx.x * kT64 + threadIdx.x) >> 5) * (32 * NV) + lane;
  double2 va[NV], vb[NV], vc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    va[k] = make_double2(1.0, 1.0);
    vb[k] = va[k];
    vc[k] = va[k];
    const uint32_t i = base + 32 * k;
    if (i < n2) va[k] = __ldcs(x2 + i);
    if (F64Shape<FN>::dist == 2 && i + stride < n2) vb[k] = __ldcs(x2 + i + stride);
  }
  if constexpr (F64Shape<FN>::dist == 2) {
    // three register buffers rotated: loads run two steps ahead (the binary64
    // kernels stream 16 B per element and are memory-latency bound)
    while (base - lane < n2) {
      f64_step<FN, M, NV>(x2, y2, x, y, n2, n, base, stride, va, vc, T, q, qn, ctr);
      base += stride;
      if (base - lane >= n2) break;
      f64_step<FN, M, NV>(x2, y2, x, y, n2, n, base, stride, vb, va, T, q, qn, ctr);
      base += stride;
      if (base - lane >= n2) break;
      f64_step<FN, M, NV>(x2, y2, x, y, n2, n, base, stride, vc, vb, T, q, qn, ctr);
      base += stride;
    }
  } else {
    while (base - lane < n2) {
      f64_step<FN, M, NV>(x2, y2, x, y, n2, n, base, stride, va, vb, T, q, qn, ctr);
      base += stride;
      if (base - lane >= n2) break;
      f64_step<FN, M, NV>(x2, y2, x, y, n2, n, base, stride, vb, va, T, q, qn, ctr);
      base += stride;
    }
  }
  __syncwarp();
  if (qn) drain<FN, M>(q, 0, qn, T, y, ctr);
}

// Any alignment: one element per thread (fast path, accurate path inline).
template <int FN, int M>
__global__ void __launch_bounds__(kT64) k_f64_scalar(const double *x, double *y, uint64_t n,
                                                     unsigned long long *ctr) {
  __shared__ F64Tab T;
  load_tables<FN>(T);
  for (uint64_t i = (uint64_t)blockIdx.x * kT64 + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kT64) {
    const double xv = x[i];
    F64Out r = FN == 0 ? exp2d_fast<M>(xv, T) : logd_fast<M>(xv, T);
    if (!r.decided) {
      int und = 0;
      atomicAdd(ctr, 1ull);
      r.y = accurate<FN, M>(xv, &und);
      if (und) atomicAdd(ctr + 1, 1ull);
    }
    y[i] = r.y;
  }
}

template <int FN, int M>
cudaError_t launch64(const double *x, double *y, uint64_t n, cudaStream_t s,
                     unsigned long long *ctr) {
  static int maxb = [] {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_f64<FN, M>, kT64, 0);
    return sms * (per > 0 ? per : 1);
  }();
  if (!n) return cudaSuccess;
  const uintptr_t ax = (uintptr_t)x & 15, ay = (uintptr_t)y & 15;
  if (ax != ay || (ax & 7)) {  // no common 16-byte alignment: element kernel
    uint64_t blocks = (n + kT64 - 1) / kT64;
    if (blocks > (uint64_t)maxb) blocks = maxb;
    k_f64_scalar<FN, M><<<(unsigned)blocks, kT64, 0, s>>>(x, y, n, ctr);
    return cudaGetLastError();
  }
  uint64_t head = ax ? 1 : 0;  // one element until both are 16-byte aligned
  if (head) k_f64_scalar<FN, M><<<1, kT64, 0, s>>>(x, y, 1, ctr);
  // 32-bit double2 slot indices: launches of at most 2^32 doubles
  constexpr uint64_t kMax = uint64_t(1) << 32;
  const uint64_t body = (n - head) & ~uint64_t(1);  // even count for the double2 kernel
  if (head + body < n) k_f64_scalar<FN, M><<<1, kT64, 0, s>>>(x + n - 1, y + n - 1, 1, ctr);
  for (uint64_t off = head; off < head + body; off += kMax) {
    const uint64_t m = head + body - off < kMax ? head + body - off : kMax;
    constexpr int NV = F64Shape<FN>::nv;
    uint64_t blocks = ((m + 1) / 2 + kT64 * NV - 1) / (kT64 * NV);
    if (blocks > F64Shape<FN>::waves * (uint64_t)maxb) blocks = F64Shape<FN>::waves * (uint64_t)maxb;
    k_f64<FN, M><<<(unsigned)(blocks ? blocks : 1), kT64, 0, s>>>(x + off, y + off, m, ctr);
  }
  return cudaGetLastError();
}

// Verification: every lane through the accurate path (one lane per thread).
template <int FN, int M>
__global__ void __launch_bounds__(kT64) k_f64_accurate(const double *x, double *y, uint64_t n,
                                                       unsigned long long *ctr) {
  uint64_t i = (uint64_t)blockIdx.x * kT64 + threadIdx.x;
  int und = 0;
  if (i < n) {
    double xv = x[i];
    F64Tab *T = nullptr;
    (void)T;
    bool special;
    if (FN == 0) special = xv != xv || xv >= 1024.0 || xv <= -1075.0 || xv == floor(xv) || dabs(xv) <= 0x1p-55;
    else special = xv != xv || xv <= 0.0 || xv == INFINITY || xv == 1.0;
    if (special) {
      // specials / exact / rule lanes have no accurate-path form: fast path
      __shared__ F64Tab Ts;  // unused by the special branches
      y[i] = FN == 0 ? exp2d_fast<M>(xv, Ts).y : logd_fast<M>(xv, Ts).y;
    } else {
      y[i] = accurate<FN, M>(xv, &und);
    }
  }
  if (und) atomicAdd(ctr + 1, 1ull);
}

int f64_accurate_dispatch(int fn, const double *x, double *y, size_t n, int mode, cudaStream_t s,
                          unsigned long long *ctr) {
  using K = void (*)(const double *, double *, uint64_t, unsigned long long *);
  static const K tab[2][4] = {
      {k_f64_accurate<0, RNE>, k_f64_accurate<0, RZ>, k_f64_accurate<0, RU>, k_f64_accurate<0, RD>},
      {k_f64_accurate<1, RNE>, k_f64_accurate<1, RZ>, k_f64_accurate<1, RU>, k_f64_accurate<1, RD>}};
  if (fn < 0 || fn > 1 || mode < 0 || mode > 3) return -1;
  if (!n) return 0;
  tab[fn][mode]<<<(unsigned)((n + kT64 - 1) / kT64), kT64, 0, s>>>(x, y, n, ctr);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// ------------------------------------------------------ hard-case screen ----
// Binary64 worst-case screen: the fast-path value
// of every input's main-range evaluation and its distance to the nearest
// binary64 rounding boundary (representable value or midpoint, any mode),
// relative to the value; inputs closer than `thr` are appended. The ranking is
// then confirmed with the reference's boundary_distance_f64 (MPFR).
__device__ __forceinline__ double boundary_rel_distance64(DD v) {
  const double h = v.hi;
  if (!(dabs(h) < INFINITY) || h == 0.0) return 1.0;
  const uint64_t hb = d2u(dabs(h));
  // h itself is a boundary; the next ones on the side of lo are h +- ulp/2,
  // or ulp/4 below a power of two (the binade below is twice as dense)
  double half = u2d(hb & 0x7FF0000000000000ull) * 0x1p-53;
  if ((hb & 0xFFFFFFFFFFFFFull) == 0 && (v.lo < 0.0) == (h > 0.0)) half *= 0.5;
  const double al = dabs(v.lo);
  return fmin(al, dabs(half - al)) / dabs(h);
}

template <int FN>
__global__ void __launch_bounds__(kT64) k_hardscan64(const double *x, uint64_t n, double thr,
                                                     double *ox, double *od, unsigned long long cap,
                                                     unsigned long long *count) {
  __shared__ F64Tab T;
  load_tables<FN>(T);
  for (uint64_t i = (uint64_t)blockIdx.x * kT64 + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kT64) {
    const double xv = x[i];
    bool main;
    DD V;
    if (FN == 0) {
      main = exp2d_main(xv) && xv < 1024.0 && xv >= -1022.0 && xv != floor(xv);
      V = exp2d_value(main ? xv : 0.5, T).V;
    } else {
      const uint64_t xb = d2u(xv);
      main = xb - 0x0010000000000000ull < 0x7FE0000000000000ull && xv != 1.0;
      V = logd_value(main ? xv : 2.0, 0, T).V;
    }
    if (main) {
      const double d = boundary_rel_distance64(fast_two_sum(V.hi, V.lo));  // normalised pair
      if (d < thr) {
        const unsigned long long k = atomicAdd(count, 1ull);
        if (k < cap) {
          ox[k] = xv;
          od[k] = d;
        }
      }
    }
  }
}

int hardscan64_dispatch(int fn, const double *x, size_t n, double thr, double *ox, double *od,
                        unsigned long long cap, unsigned long long *count, cudaStream_t s) {
  if (fn < 0 || fn > 1) return -1;
  if (!n) return 0;
  uint64_t blocks = (n + kT64 - 1) / kT64;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  if (fn == 0) k_hardscan64<0><<<(unsigned)blocks, kT64, 0, s>>>(x, n, thr, ox, od, cap, count);
  else k_hardscan64<1><<<(unsigned)blocks, kT64, 0, s>>>(x, n, thr, ox, od, cap, count);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// ------------------------------------------------- reference round test ----
// The reference's Ziv straddle test as a standalone batch operation
// (ref: proj/src/kernels_f64.cpp:63-76 round_test_lane, kernels_f64.hpp:27-56):
// bound b = RN(RN(eps_rel |hi| + eps_abs) (1 + 2^-30) + 2^-1000), the two ends
// fast_two_sum(hi, lo -+ b) are rounded EXACTLY after scaling by 2^scale
// (normal, subnormal and overflowing results alike) in the requested mode,
// and the lane is decided iff both ends round to the same binary64. The kernels
// use the cheaper in-register form round_test64() (no scale, b precomputed);
// this one serves the C++ compatibility surface (round_test<W>).

// Round sign * mant * 2^(E - 63) (mant bit 63 set; `sticky`: nonzero bits
// below mant) to binary64 in mode M, subnormals and overflow included.
template <int M>
__device__ __forceinline__ double round_parts64(bool neg, int E, uint64_t mant, bool sticky) {
  const uint64_t sgn = neg ? 0x8000000000000000ull : 0ull;
  const bool to_inf = M == RNE || (M == RU && !neg) || (M == RD && neg);
  if (E > 1023) return u2d(sgn | (to_inf ? 0x7FF0000000000000ull : 0x7FEFFFFFFFFFFFFFull));
  const int sh = E >= -1022 ? 11 : 11 + (-1022 - E);  // bits dropped below the kept significand
  uint64_t kept;
  bool rb, st;
  if (sh >= 65) {
    kept = 0; rb = false; st = sticky || mant != 0;
  } else if (sh == 64) {
    kept = 0; rb = (mant >> 63) != 0; st = sticky || (mant << 1) != 0;
  } else {
    kept = mant >> sh;
    rb = ((mant >> (sh - 1)) & 1u) != 0;
    st = sticky || (mant & ((1ull << (sh - 1)) - 1u)) != 0;
  }
  const bool inexact = rb || st;
  bool up;
  if (M == RNE) up = rb && (st || (kept & 1u));
  else if (M == RZ) up = false;
  else if (M == RU) up = !neg && inexact;
  else up = neg && inexact;
  kept += up ? 1u : 0u;
  if (E >= -1022) {
    if (kept >> 53) { kept >>= 1; ++E; }
    if (E > 1023) return u2d(sgn | (to_inf ? 0x7FF0000000000000ull : 0x7FEFFFFFFFFFFFFFull));
    return u2d(sgn | ((uint64_t)(E + 1023) << 52) | (kept & 0xFFFFFFFFFFFFFull));
  }
  return u2d(sgn | kept);  // subnormal (a carry to 2^52 encodes the least normal)
}

// Exact rounding of (s + e) * 2^n, s normal, |e| <= ulp(s)/2: s's significand
// in a 72-bit window (19 guard bits), e added in guard-lsb units; the bits of
// e below the window only set the sticky flag.
template <int M>
__device__ __forceinline__ double round_pair_scaled(double s, double e, long long n) {
  const uint64_t bs = d2u(s);
  const bool neg = (bs >> 63) != 0;
  const int es = (int)((bs >> 52) & 0x7FF) - 1023;
  const unsigned __int128 M53 = (bs & 0xFFFFFFFFFFFFFull) | 0x10000000000000ull;
  unsigned __int128 m = M53 << 19;  // value = m * 2^(es - 71)
  bool sticky = false;
  if (e != 0.0) {
    const double w = ldexp(e, 71 - es);  // exact: e's bits above 2^(es-71)
    const double aw = fabs(w);
    const uint64_t whole = (uint64_t)aw;
    const bool frac = aw != (double)whole;
    if ((e < 0.0) != neg) {
      m -= whole;
      m -= frac ? 1u : 0u;
    } else {
      m += whole;
    }
    sticky = frac;
  }
  const uint64_t hi = (uint64_t)(m >> 64), lo = (uint64_t)m;
  const int msb = hi ? 64 + 63 - __clzll((long long)hi) : 63 - __clzll((long long)lo);
  const int drop = msb - 63;
  uint64_t mant;
  if (drop > 0) {
    sticky = sticky || (lo & ((1ull << drop) - 1u)) != 0;
    mant = (uint64_t)(m >> drop);
  } else {
    mant = lo << (-drop);
  }
  const long long E = (long long)es - 71 + msb + n;
  const int Ec = E > 2000 ? 2000 : (E < -2000 ? -2000 : (int)E);
  return round_parts64<M>(neg, Ec, mant, sticky);
}

template <int M>
__global__ void __launch_bounds__(kT64) k_round_test(const double *hi, const double *lo,
                                                     const long long *scale, const double *eps_rel,
                                                     const double *eps_abs, double *val,
                                                     unsigned char *decided, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * kT64 + threadIdx.x;
  if (i >= n) return;
  const double h = hi[i], l = lo[i];
  const long long sc = scale ? scale[i] : 0;
  double b = fma_(eps_rel ? eps_rel[i] : 0.0, dabs(h), eps_abs ? eps_abs[i] : 0.0);
  b = add_(mul_(b, 1.0 + 0x1p-30), 0x1p-1000);  // absorb the bound's own rounding
  const DD le = fast_two_sum(h, sub_(l, b)), he = fast_two_sum(h, add_(l, b));
  const double rl = round_pair_scaled<M>(le.hi, le.lo, sc);
  const double rh = round_pair_scaled<M>(he.hi, he.lo, sc);
  val[i] = rl;
  decided[i] = d2u(rl) == d2u(rh);
}

int round_test_dispatch(const double *hi, const double *lo, const long long *scale,
                        const double *eps_rel, const double *eps_abs, int mode, double *val,
                        unsigned char *decided, size_t n, cudaStream_t s) {
  using K = void (*)(const double *, const double *, const long long *, const double *, const double *,
                     double *, unsigned char *, uint64_t);
  static const K tab[4] = {k_round_test<RNE>, k_round_test<RZ>, k_round_test<RU>, k_round_test<RD>};
  if (mode < 0 || mode > 3) return -1;
  if (!n) return 0;
  tab[mode]<<<(unsigned)((n + kT64 - 1) / kT64), kT64, 0, s>>>(hi, lo, scale, eps_rel, eps_abs, val,
                                                              decided, n);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// ctr: [1] fast_undecided, [2] accurate_undecided (device counters of the API)
int f64_dispatch(int fn, const double *x, double *y, size_t n, int mode, cudaStream_t s,
                 unsigned long long *ctr) {
  using L = cudaError_t (*)(const double *, double *, uint64_t, cudaStream_t, unsigned long long *);
  static const L tab[2][4] = {
      {launch64<0, RNE>, launch64<0, RZ>, launch64<0, RU>, launch64<0, RD>},
      {launch64<1, RNE>, launch64<1, RZ>, launch64<1, RU>, launch64<1, RD>}};
  if (fn < 0 || fn > 1 || mode < 0 || mode > 3) return -1;
  cudaError_t e = tab[fn][mode](x, y, n, s, ctr + 1);
  return e == cudaSuccess ? 0 : -2;
}

}  // namespace crvec
