// Microbenchmark: latency of a dependent mma.sync.m8n8k4.f64 chain and the
// throughput with G independent chains per warp, W warps per SM (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int G>
__global__ void chain(double* out, int iters, double s, long long* cyc) {
  double ma = s * threadIdx.x, mb = s + threadIdx.x;
  double d[G][2];
  for (int g = 0; g < G; ++g) d[g][0] = d[g][1] = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int g = 0; g < G; ++g)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[g][0]), "+d"(d[g][1]) : "d"(ma), "d"(mb));
  }
  long long t1 = clock64();
  double t = 0;
  for (int g = 0; g < G; ++g) t += d[g][0] + d[g][1];
  if (t == 1.2345) out[0] = t;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int G>
void run(int sms, int warps_per_sm, int iters) {
  double* o;
  long long* cyc;
  cudaMalloc(&o, 8);
  cudaMalloc(&cyc, 8);
  const int blocks = warps_per_sm == 1 ? 1 : sms * warps_per_sm / 4, threads = warps_per_sm == 1 ? 32 : 128;
  chain<G><<<blocks, threads>>>(o, 10, 1.0000001, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  chain<G><<<blocks, threads>>>(o, iters, 1.0000001, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double fl = (double)blocks * threads / 32 * G * iters * 512.0;
  printf("G=%d chains/warp, %3d warps/SM%s: %7.1f clk per dependent step, %6.2f TF/s\n", G,
         warps_per_sm == 1 ? 1 : warps_per_sm, warps_per_sm == 1 ? " (1 warp total)" : "",
         (double)c / iters, fl / ms / 1e9);
  cudaFree(o);
  cudaFree(cyc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1>(sms, 1, 20000);
  run<2>(sms, 1, 20000);
  run<4>(sms, 1, 20000);
  run<8>(sms, 1, 20000);
  for (int w : {4, 8, 16, 32}) {
    run<1>(sms, w, 20000);
    run<2>(sms, w, 20000);
    run<4>(sms, w, 10000);
  }
  return 0;
}
