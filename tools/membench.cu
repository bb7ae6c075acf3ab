// Developer microbenchmark: streaming-template variants for the binary32 map
// kernels, on an identity op (memory ceiling) and on logf (real work).
//   A  float4 per lane, register prefetch of the next float4   (current)
//   B  2 x float4 per lane per iteration, both loads issued first
//   C  B + register prefetch of the next 2 x float4
//   T  TMA bulk (cp.async.bulk + mbarrier) 4-stage smem pipeline, 4 elem/lane
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -I include tools/membench.cu -o membench
#include <algorithm>
#include <cstdio>
#include <vector>

#include "../paper_2605_15547_b200/csrc/crvec_kernels.cuh"

using namespace crvec;

struct FnIdent {
  static constexpr uint32_t E = 8;
  struct Regs {};
  CR_F static void load(Regs &) {}
  CR_F static Fast fast(float x, const Regs &) { return Fast{f2d(x), false}; }
  template <int M>
  CR_F static uint32_t special(float x) { return f2u(x); }
  CR_F static DD slow(float x) { return DD{f2d(x), 0.0}; }
};

template <class F, int NV, bool PF>
__global__ void __launch_bounds__(256) k_var(const float4 *x, float4 *y, uint64_t n4,
                                             unsigned long long *ctr) {
  typename F::Regs R;
  F::load(R);
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * 256) >> 5;
  const uint64_t stride = nwarps * 32 * NV;
  const float4 ones = make_float4(1.f, 1.f, 1.f, 1.f);
  uint64_t base = warp * 32 * NV;
  float4 v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    uint64_t i = base + k * 32 + lane;
    v[k] = (PF && i < n4) ? ld_stream(x + i) : ones;
  }
  for (; base < n4; base += stride) {
    float4 vn[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      uint64_t i = base + k * 32 + lane;
      if (PF) {
        uint64_t in = i + stride;
        vn[k] = in < n4 ? ld_stream(x + in) : ones;
      } else {
        v[k] = i < n4 ? ld_stream(x + i) : ones;
      }
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      uint64_t i = base + k * 32 + lane;
      float xs[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
      uint32_t ys[4];
      eval_lanes<F, RNE, 4>(xs, ys, R, nullptr, ctr);
      if (i < n4) st_stream(y + i, make_float4(u2f(ys[0]), u2f(ys[1]), u2f(ys[2]), u2f(ys[3])));
    }
    if (PF) {
#pragma unroll
      for (int k = 0; k < NV; ++k) v[k] = vn[k];
    }
  }
}

template <class F, int NV, int MINB>
__global__ void __launch_bounds__(256, MINB) k_lb(const float4 *x, float4 *y, uint64_t n4,
                                                  unsigned long long *ctr) {
  typename F::Regs R;
  F::load(R);
  PHBlock *sh = ph_storage<F>();
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * 256) >> 5;
  const uint64_t stride = nwarps * 32 * NV;
  const float4 ones = make_float4(1.f, 1.f, 1.f, 1.f);
  uint64_t base = warp * 32 * NV;
  float4 v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = base + 32 * k + lane < n4 ? ld_stream(x + base + 32 * k + lane) : ones;
  for (; base < n4; base += stride) {
    float4 nx[NV];
    float xs[4 * NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      uint64_t in = base + 32 * k + lane + stride;
      nx[k] = in < n4 ? ld_stream(x + in) : ones;
      xs[4 * k] = v[k].x; xs[4 * k + 1] = v[k].y; xs[4 * k + 2] = v[k].z; xs[4 * k + 3] = v[k].w;
    }
    uint32_t ys[4 * NV];
    eval_lanes<F, RNE, 4 * NV>(xs, ys, R, sh, ctr);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      uint64_t i = base + 32 * k + lane;
      if (i < n4) st_stream(y + i, make_float4(u2f(ys[4 * k]), u2f(ys[4 * k + 1]), u2f(ys[4 * k + 2]), u2f(ys[4 * k + 3])));
      v[k] = nx[k];
    }
  }
}

// ---- TMA bulk pipeline -------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned phase) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(phase));
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, uint64_t *b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b))
      : "memory");
}

template <class F, int ST>
__global__ void __launch_bounds__(256) k_tma(const float4 *x, float4 *y, uint64_t n4,
                                             unsigned long long *ctr) {
  __shared__ alignas(128) float4 buf[ST][256];
  __shared__ uint64_t bar[ST];
  typename F::Regs R;
  F::load(R);
  uint64_t ntiles = n4 / 256;  // n4 multiple of 256 in this benchmark
  if (threadIdx.x == 0)
    for (int s = 0; s < ST; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint64_t t0 = blockIdx.x, tstride = gridDim.x;
  if (threadIdx.x == 0)
    for (int s = 0; s < ST; ++s) {
      uint64_t t = t0 + s * tstride;
      if (t < ntiles) {
        mbar_expect(&bar[s], 4096);
        bulk_load(buf[s], x + t * 256, 4096, &bar[s]);
      }
    }
  unsigned phase[ST];
  for (int s = 0; s < ST; ++s) phase[s] = 0;
  int s = 0;
  for (uint64_t t = t0, it = 0; t < ntiles; t += tstride, ++it) {
    mbar_wait(&bar[s], phase[s]);
    phase[s] ^= 1;
    float4 v = buf[s][threadIdx.x];
    __syncthreads();  // everyone has read stage s
    if (threadIdx.x == 0) {
      uint64_t tn = t + (uint64_t)ST * tstride;
      if (tn < ntiles) {
        mbar_expect(&bar[s], 4096);
        bulk_load(buf[s], x + tn * 256, 4096, &bar[s]);
      }
    }
    float xs[4] = {v.x, v.y, v.z, v.w};
    uint32_t ys[4];
    eval_lanes<F, RNE, 4>(xs, ys, R, nullptr, ctr);
    st_stream(y + t * 256 + threadIdx.x, make_float4(u2f(ys[0]), u2f(ys[1]), u2f(ys[2]), u2f(ys[3])));
    s = (s + 1) % ST;
  }
}

template <class K>
float timeit(K kern, int blocks, const float4 *x, float4 *y, uint64_t n4, unsigned long long *c,
             size_t smem = 0) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) kern<<<blocks, 256, smem>>>(x, y, n4, c);
  std::vector<float> ts;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(a);
    kern<<<blocks, 256, smem>>>(x, y, n4, c);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
  return ts[3];
}

template <class K>
int occ(K k) {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0);
  return per;
}

int main() {
  uint64_t n = 1ull << 28, n4 = n / 4;
  float *x, *y;
  unsigned long long *c;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&y, n * 4);
  cudaMalloc(&c, 64);
  // positive finite inputs (log domain)
  std::vector<float> h(1 << 20);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 0.5f + (float)i / (1 << 19);
  for (uint64_t off = 0; off < n; off += h.size()) cudaMemcpy(x + off, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  const float4 *x4 = (const float4 *)x;
  float4 *y4 = (float4 *)y;
  int sms = 148;
  auto rep = [&](const char *name, float ms, int per) {
    printf("%-28s %7.3f ms  %7.1f GB/s  %6.1f Gelem/s  occ %d blk/SM\n", name, ms, 8.0 * n / ms / 1e6,
           n / ms / 1e6, per);
  };
#define RUNV(F, NV, PF)                                                              \
  {                                                                                  \
    auto k = k_var<F, NV, PF>;                                                       \
    int per = occ(k);                                                                \
    for (int mult : {1, 2, 4}) {                                                     \
      char nm[64];                                                                   \
      snprintf(nm, 64, #F " NV=%d PF=%d g=%dx", NV, PF, mult);                      \
      rep(nm, timeit(k, sms * per * mult, x4, y4, n4, c), per);                      \
    }                                                                                \
  }
#define RUNLB(F, NV, MB)                                                             \
  {                                                                                  \
    auto k = k_lb<F, NV, MB>;                                                        \
    int per = occ(k);                                                                \
    char nm[64];                                                                     \
    snprintf(nm, 64, #F " NV=%d minB=%d", NV, MB);                                   \
    rep(nm, timeit(k, sms * per * 4, x4, y4, n4, c), per);                           \
  }
  RUNLB(FnLog, 2, 1) RUNLB(FnLog, 2, 3) RUNLB(FnLog, 2, 4) RUNLB(FnLog, 1, 4) RUNLB(FnLog, 1, 5) RUNLB(FnLog, 3, 2) RUNLB(FnLog, 3, 3)
  RUNLB(FnLog1p, 2, 1) RUNLB(FnLog1p, 2, 3) RUNLB(FnLog1p, 2, 4) RUNLB(FnLog1p, 1, 4)
  RUNLB(FnExp, 2, 1) RUNLB(FnExp, 2, 3) RUNLB(FnExp, 2, 4) RUNLB(FnExp, 1, 4)
  RUNLB(FnSin, 2, 1) RUNLB(FnSin, 2, 2) RUNLB(FnSin, 2, 3) RUNLB(FnSin, 1, 4)
  RUNLB(FnAsin, 2, 1) RUNLB(FnAsin, 2, 3) RUNLB(FnAsin, 1, 4)
  // plain cudaMemcpy D2D for reference
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaMemcpy(y, x, n * 4, cudaMemcpyDeviceToDevice);
    cudaEventRecord(a);
    cudaMemcpy(y, x, n * 4, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    rep("cudaMemcpy D2D", ms, 0);
  }
  return 0;
}
