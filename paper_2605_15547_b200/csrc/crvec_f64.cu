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
constexpr int kQ = 128;  // per-warp queue capacity

struct F64Queue {
  double x[kQ];
  unsigned long long idx[kQ];
};

template <int FN, int M>
__device__ __noinline__ double accurate(double x, int *und) {
  return FN == 0 ? exp2d_accurate<M>(x, und) : logd_accurate<M>(x, und);
}

// Drain `cnt` (<= 32) queue entries starting at `from`: one entry per lane.
template <int FN, int M>
__device__ __forceinline__ void drain(F64Queue &q, int from, int cnt, double *y,
                                      unsigned long long *ctr) {
  int lane = threadIdx.x & 31;
  int und = 0;
  if (lane < cnt) {
    double xv = q.x[from + lane];
    unsigned long long i = q.idx[from + lane];
    y[i] = accurate<FN, M>(xv, &und);
  }
  unsigned m = __ballot_sync(0xffffffffu, und);
  if (lane == 0 && m) atomicAdd(ctr + 1, (unsigned long long)__popc(m));
}

template <int FN, int M>
__global__ void __launch_bounds__(kT64) k_f64(const double *x, double *y, uint64_t n,
                                              unsigned long long *ctr) {
  __shared__ F64Tab T;
  __shared__ F64Queue Q[kW64];
  for (int i = threadIdx.x; i < 16; i += kT64) {
    T.t1h[i] = EXP2D_T1_HI[i]; T.t1l[i] = EXP2D_T1_LO[i];
    T.t2h[i] = EXP2D_T2_HI[i]; T.t2l[i] = EXP2D_T2_LO[i];
    T.t3h[i] = EXP2D_T3_HI[i]; T.t3l[i] = EXP2D_T3_LO[i];
  }
  for (int i = threadIdx.x; i < 128; i += kT64) {
    T.lc[i] = LOGD_C[i]; T.llh[i] = LOGD_LT_HI[i]; T.lll[i] = LOGD_LT_LO[i];
  }
  __syncthreads();
  F64Queue &q = Q[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int qn = 0;  // warp-uniform queue length
  unsigned long long nfast = 0;
  const uint64_t warp = ((uint64_t)blockIdx.x * kT64 + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * kT64) >> 5;
  const uint64_t n2 = (n + 1) / 2;  // double2 slots
  const bool vec = (((uintptr_t)x | (uintptr_t)y) & 15) == 0;
  // register double buffer: the next slot's two doubles are requested before
  // this slot is computed
  auto load2 = [&](uint64_t slot) {
    uint64_t j = 2 * slot;
    double2 t = make_double2(1.0, 1.0);
    if (vec && j + 1 < n) {
      t = __ldcs((const double2 *)(x + j));
    } else {
      if (j < n) t.x = x[j];
      if (j + 1 < n) t.y = x[j + 1];
    }
    return t;
  };
  const uint64_t stride = nwarps * 32;
  double2 cur = load2(warp * 32 + lane);
  for (uint64_t base = warp * 32; base < n2; base += stride) {
    uint64_t s = base + lane;
    uint64_t i0 = 2 * s;
    double2 nxt = load2(s + stride);
    double xv[2] = {cur.x, cur.y};
    cur = nxt;
    bool v0 = i0 < n, v1 = i0 + 1 < n;
    F64Out r[2];
#pragma unroll
    for (int e = 0; e < 2; ++e)
      r[e] = FN == 0 ? exp2d_fast<M>(xv[e], T) : logd_fast<M>(xv[e], T);
    bool und0 = v0 && !r[0].decided, und1 = v1 && !r[1].decided;
    if (vec && v1) {
      __stcs((double2 *)(y + i0), make_double2(r[0].y, r[1].y));
    } else {
      if (v0) y[i0] = r[0].y;
      if (v1) y[i0 + 1] = r[1].y;
    }
    // compact undecided lanes into the warp's side queue
    unsigned m0 = __ballot_sync(0xffffffffu, und0);
    unsigned m1 = __ballot_sync(0xffffffffu, und1);
    if (m0 | m1) {
      if (und0) { int p = qn + __popc(m0 & lt); q.x[p] = xv[0]; q.idx[p] = i0; }
      qn += __popc(m0);
      if (und1) { int p = qn + __popc(m1 & lt); q.x[p] = xv[1]; q.idx[p] = i0 + 1; }
      qn += __popc(m1);
      nfast += __popc(m0) + __popc(m1);
      __syncwarp();
      while (qn >= 32) {  // a full warp of hard lanes: evaluate together
        drain<FN, M>(q, qn - 32, 32, y, ctr);
        qn -= 32;
        __syncwarp();
      }
    }
  }
  __syncwarp();
  if (qn) drain<FN, M>(q, 0, qn, y, ctr);
  if (lane == 0 && nfast) atomicAdd(ctr, nfast);
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
  uint64_t slots = (n + 1) / 2;
  uint64_t blocks = (slots + kT64 - 1) / kT64;
  if (blocks > (uint64_t)maxb) blocks = maxb;
  if (!blocks) blocks = 1;
  k_f64<FN, M><<<(unsigned)blocks, kT64, 0, s>>>(x, y, n, ctr);
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
