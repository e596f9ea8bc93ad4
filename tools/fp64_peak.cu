// FP64 peak microbenchmark for B200 (sm_100a): DMMA.8x8x4 (mma.sync m8n8k4 f64)
// and DFMA throughput, timed with CUDA events. Prints one JSON line.
// This measures the roofline denominator the inversion kernels are reported against.
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 0.999999;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void log_probe(double* out) {
  // device log on the values the reference's exact-power KATs use
  double g = 0.3, y = 0.3 * 0.3;
  out[0] = log(y) / log(g);
  out[1] = log(0.1) / log(0.1);
  out[2] = log(0.5) / log(0.5);
  out[3] = y;
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* d; CK(cudaMalloc(&d, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256;
  double best_dmma = 0, best_dfma = 0;
  for (int blocks_per_sm = 1; blocks_per_sm <= 4; blocks_per_sm *= 2) {
    int blocks = sms * blocks_per_sm;
    int iters = 4000;
    dmma_loop<8><<<blocks, threads>>>(d, 100, 1.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) dmma_loop<8><<<blocks, threads>>>(d, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5.0 * blocks * (threads / 32) * (double)iters * 8 * 512;
    double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best_dmma) best_dmma = tf;
    fprintf(stderr, "dmma blocks/sm=%d  %.2f TFLOP/s\n", blocks_per_sm, tf);

    dfma_loop<8><<<blocks, threads>>>(d, 100, 1.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) dfma_loop<8><<<blocks, threads>>>(d, iters * 4, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 5.0 * blocks * threads * (double)iters * 4 * 8 * 2;
    tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best_dfma) best_dfma = tf;
    fprintf(stderr, "dfma blocks/sm=%d  %.2f TFLOP/s\n", blocks_per_sm, tf);
  }
  // sustained DMMA: ~3 s of back-to-back launches
  int blocks = sms * 2;
  cudaEventRecord(e0);
  int reps = 0; float ms = 0;
  while (ms < 3000.f) {
    for (int r = 0; r < 10; ++r) dmma_loop<8><<<blocks, threads>>>(d, 4000, 1.0);
    reps += 10;
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  }
  double sustained = (double)reps * blocks * (threads / 32) * 4000.0 * 8 * 512 / (ms * 1e-3) / 1e12;
  log_probe<<<1, 1>>>(d);
  double h[4]; CK(cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost));
  printf("{\"dmma_tflops_burst\": %.3f, \"dmma_tflops_sustained\": %.3f, \"dfma_tflops_burst\": %.3f, \"sms\": %d, "
         "\"log_0p09_over_log_0p3\": %.17g, \"log_ratio_0p1\": %.17g, \"log_ratio_0p5\": %.17g}\n",
         best_dmma, sustained, best_dfma, sms, h[0], h[1], h[2]);
  return 0;
}
