// Developer microbenchmark: sustained DFMA throughput of one B200 (the FP64
// roofline for the binary64 kernels; MEASURED_PEAKS.json has no fp64 entry).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64peak tools/fp64peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double *out, int iters, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 1e-12);  // 8 independent chains
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += a[i];
  if (t == 12345.0) out[0] = t;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double *o;
  cudaMalloc(&o, 8);
  const int iters = 1 << 14, threads = 256, blocks = sms * 8;
  k<<<blocks, threads>>>(o, 64, 0.999999);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k<<<blocks, threads>>>(o, iters, 0.999999);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  double dfma = (double)blocks * threads * iters * 8;
  printf("{\"sms\": %d, \"dfma_per_s\": %.4e, \"fp64_tflops\": %.2f, \"dfma_per_sm_per_clk_at_1965MHz\": %.1f}\n", sms,
         dfma / (best * 1e-3), 2 * dfma / (best * 1e-3) / 1e12, dfma / (best * 1e-3) / sms / 1.965e9);
  return 0;
}
