// Accuracy probe of the FP64 reciprocal used by the fast P2P path:
// MUFU.RCP64H seed (rcp.approx.ftz.f64), after one quadratic Newton step
// (2 DFMA) and after the cubic step (3 DFMA) the kernel uses.  Max relative
// error over r^2 spanning the magnitudes the near field sees.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ double relerr(double a, double ref) { return fabs(a - ref) / fabs(ref); }

__global__ void probe(double* out, uint64_t n, uint64_t seed) {
  double m0 = 0, m1 = 0, m2 = 0;
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint64_t h = (i + seed) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    const double u = double(h >> 11) * (1.0 / 9007199254740992.0);
    const double x = exp2(-40.0 + 42.0 * u);  // r^2 in [2^-40, 4)
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double ref = 1.0 / x;
    const double e = fma(-x, y, 1.0);
    const double yq = fma(y, e, y);
    const double yc = fma(y, fma(e, e, e), y);
    m0 = fmax(m0, relerr(y, ref));
    m1 = fmax(m1, relerr(yq, ref));
    m2 = fmax(m2, relerr(yc, ref));
  }
  atomicMax((unsigned long long*)&out[0], __double_as_longlong(m0));
  atomicMax((unsigned long long*)&out[1], __double_as_longlong(m1));
  atomicMax((unsigned long long*)&out[2], __double_as_longlong(m2));
}

int main() {
  double* d;
  cudaMalloc(&d, 24);
  cudaMemset(d, 0, 24);
  probe<<<148 * 8, 256>>>(d, 1ull << 30, 12345);
  double h[3];
  cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  std::printf("rcp.approx.f64 seed max rel err %.3e (2^%.2f)\n", h[0], std::log2(h[0]));
  std::printf("1 quadratic Newton (2 DFMA)  %.3e (2^%.2f)\n", h[1], std::log2(h[1]));
  std::printf("1 cubic Newton (3 DFMA)      %.3e (2^%.2f)\n", h[2], std::log2(h[2]));
  return 0;
}
