// Accuracy of a fast FP64 1/sqrt: rsqrt.approx.ftz.f64 seed + one third-order
// Newton step, against the correctly rounded 1/__dsqrt_rn (ulps), over
// 2^24 random positive doubles spanning 1e-300 .. 1e300 and [0.5, 2].
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);          // 1 - x y^2
  return fma(y, e * fma(0.375, e, 0.5), y);        // y (1 + e/2 + 3e^2/8)
}

__global__ void k(uint64_t seed, int n, double* maxulp, double* maxulp_sqrt, int mode) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t z = seed + (uint64_t)i * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  double u = (z >> 11) * (1.0 / 9007199254740992.0);
  double x = mode == 0 ? exp2(-996.0 + 1992.0 * u) : 0.5 + 1.5 * u;
  double r = rsqrt_fast(x), ref = 1.0 / __dsqrt_rn(x);
  double ulp = fabs(r - ref) / (fabs(ref) * 2.220446049250313e-16);
  double s = x * r, sref = __dsqrt_rn(x);
  double ulps = fabs(s - sref) / (sref * 2.220446049250313e-16);
  atomicMax((unsigned long long*)maxulp, __double_as_longlong(ulp));
  atomicMax((unsigned long long*)maxulp_sqrt, __double_as_longlong(ulps));
}

int main() {
  double *m;
  cudaMalloc(&m, 16);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(m, 0, 16);
    const int n = 1 << 24;
    k<<<n / 256, 256>>>(12345 + mode, n, m, m + 1, mode);
    double h[2];
    cudaMemcpy(h, m, 16, cudaMemcpyDeviceToHost);
    printf("%s: max rel err rsqrt %.3f ulp, x*rsqrt vs sqrt %.3f ulp\n",
           mode == 0 ? "x in [1e-300, 1e300]" : "x in [0.5, 2]", h[0], h[1]);
  }
  return 0;
}
