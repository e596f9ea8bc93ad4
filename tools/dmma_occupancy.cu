// DMMA.8x8x4 throughput vs. warps per SM sub-partition and independent
// accumulator chains per warp (is 2 warps x 16 chains enough to saturate?),
// plus the dependent-chain latency. Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
double run(int sms, int warps_per_sm, int iters, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_loop<CHAINS><<<sms, 32 * warps_per_sm>>>(d, 10, 1.0);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  dmma_loop<CHAINS><<<sms, 32 * warps_per_sm>>>(d, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return (double)sms * warps_per_sm * iters * CHAINS * 512.0 / (ms * 1e-3) / 1e12;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  cudaMalloc(&d, 64);
  printf("{\"sms\": %d", sms);
  const int wps[] = {4, 8, 12, 16};
  for (int w : wps) {
    printf(", \"w%d_c4\": %.2f", w, run<4>(sms, w, 20000, d));
    printf(", \"w%d_c8\": %.2f", w, run<8>(sms, w, 10000, d));
    printf(", \"w%d_c16\": %.2f", w, run<16>(sms, w, 5000, d));
  }
  // latency: one warp per SM, one chain
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    dmma_loop<1><<<1, 32>>>(d, 10, 1.0);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    dmma_loop<1><<<1, 32>>>(d, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"latency_ns\": %.2f", ms * 1e6 / iters);
  }
  printf("}\n");
  return 0;
}
