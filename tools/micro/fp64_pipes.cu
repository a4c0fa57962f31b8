// Microbenchmark: FP64 throughput of DFMA (vector pipe) vs DMMA
// (mma.sync m8n8k4 / m16n8k16 f64 tensor pipe) on sm_100a, and both
// interleaved (are the pipes independent?).  nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>

template <int NDFMA, int NDMMA>
__global__ void k_mix(double* out, int iters, double s) {
  double a[8], acc[8];
  for (int i = 0; i < 8; ++i) { a[i] = s * (threadIdx.x + i); acc[i] = 0.0; }
  double ma = s * threadIdx.x, mb = s + threadIdx.x;
  double d[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < NDFMA; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fma(a[i], s, acc[i]);
    }
#pragma unroll
    for (int r = 0; r < NDMMA; ++r) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[q][0]), "+d"(d[q][1]) : "d"(ma), "d"(mb));
    }
  }
  double t = 0;
  for (int i = 0; i < 8; ++i) t += acc[i];
  for (int q = 0; q < 4; ++q) t += d[q][0] + d[q][1];
  if (t == 1.2345) out[0] = t;
}

template <int NDFMA, int NDMMA>
void run(const char* name, int blocks, int threads, int iters) {
  double* o;
  cudaMalloc(&o, 8);
  k_mix<NDFMA, NDMMA><<<blocks, threads>>>(o, 10, 1.0000001);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mix<NDFMA, NDMMA><<<blocks, threads>>>(o, iters, 1.0000001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double warps = (double)blocks * threads / 32;
  double fl_fma = warps * 32 * 8.0 * NDFMA * iters * 2;
  double fl_mma = warps * 4.0 * NDMMA * iters * (8 * 8 * 4 * 2);
  printf("%-28s %8.3f ms  DFMA %6.2f TF/s  DMMA %6.2f TF/s  total %6.2f TF/s\n", name, ms,
         fl_fma / ms / 1e9, fl_mma / ms / 1e9, (fl_fma + fl_mma) / ms / 1e9);
  cudaFree(o);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int B = sms * 4, T = 256, I = 4000;
  run<4, 0>("dfma only", B, T, I);
  run<0, 4>("dmma m8n8k4 only", B, T, I);
  run<4, 4>("dfma + dmma interleaved", B, T, I);
  run<4, 1>("dfma + 1/4 dmma", B, T, I);
  run<1, 4>("1/4 dfma + dmma", B, T, I);
  return 0;
}
