// Seed accuracy of the fp64 MUFU approximations the fast paths start from
// (rcp.approx.ftz.f64 -> MUFU.RCP64H, rsqrt.approx.ftz.f64 -> MUFU.RSQ64H):
// max |e| with e = 1 - x r (rcp) and e = 1 - x y^2 (rsqrt) over every
// 20-bit high mantissa pattern x low words x exponents. div_fast /
// sqrt_fast truncate their series after e^2 (error ~e^3), which needs
// |e| < 2^-18.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_probe.cu -o /tmp/mufu_probe
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cstring>

__device__ double rcp_a(double x) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ double rsq_a(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }

__device__ unsigned long long g_max[2];

__global__ void probe(int exp_lo, int nexp) {
  uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;  // 20-bit high mantissa
  if (m >= (1u << 20)) return;
  double wr = 0, ws = 0;
  for (int ei = 0; ei < nexp; ++ei) {
    for (int l = 0; l < 4; ++l) {
      uint32_t lo = l == 0 ? 0u : (l == 1 ? 0xFFFFFFFFu : (m * 2654435761u) ^ (ei * 40503u + l));
      uint32_t hi = ((uint32_t)(1023 + exp_lo + ei) << 20) | m;
      double x = __hiloint2double((int)hi, (int)lo);
      double r = rcp_a(x);
      double er = fabs(__fma_rn(-x, r, 1.0));
      double y = rsq_a(x);
      double es = fabs(__fma_rn(-x * y, y, 1.0));  // x*y rounded: ~2^-53 extra
      wr = fmax(wr, er);
      ws = fmax(ws, es);
    }
  }
  atomicMax(&g_max[0], (unsigned long long)__double_as_longlong(wr));
  atomicMax(&g_max[1], (unsigned long long)__double_as_longlong(ws));
}

int main() {
  unsigned long long z[2] = {0, 0}, h[2];
  cudaMemcpyToSymbol(g_max, z, sizeof z);
  probe<<<(1 << 20) / 256, 256>>>(-40, 80);
  cudaMemcpyFromSymbol(h, g_max, sizeof h);
  double r, s;
  memcpy(&r, &h[0], 8);
  memcpy(&s, &h[1], 8);
  printf("rcp.approx.ftz.f64   max |1 - x r|   = %.3e = 2^%.2f\n", r, log2(r));
  printf("rsqrt.approx.ftz.f64 max |1 - x y^2| = %.3e = 2^%.2f\n", s, log2(s));
  printf("series truncation: rcp e^3 = 2^%.2f, sqrt 5e^3/16 = 2^%.2f\n", 3 * log2(r), 3 * log2(s) + log2(5.0 / 16));
  return cudaGetLastError() != cudaSuccess;
}
