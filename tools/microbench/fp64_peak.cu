// FP64 peak microbenchmark: DFMA (CUDA cores) vs DMMA (mma.sync f64 tensor path).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
  #pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

template <int SHAPE>
__global__ void dmma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b0 = 0.5, b1 = 0.25;
  double c[8][4];
  #pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a0), "d"(b0));
      } else if (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b0));
      } else {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(a0), "d"(a1), "d"(b0), "d"(b1));
      }
    }
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

// Sustained DMMA rate: back-to-back launches for ~seconds s (power-capped
// clocks under a long load, the denominator for a kernel timed inside a
// long step); prints the rate of each 0.5 s window and the SM clock.
static int sustained(double seconds) {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * 8, iters = 20000;
  const double flops_per_launch = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
  dmma_kernel<0><<<blocks, threads>>>(d, 100);
  cudaDeviceSynchronize();
  double total_ms = 0, best = 0, last = 0;
  while (total_ms < seconds * 1e3) {
    cudaEventRecord(e0);
    int n = 0;
    float ms = 0;
    while (ms < 500.f) {
      dmma_kernel<0><<<blocks, threads>>>(d, iters);
      ++n;
      if (n % 8 == 0) { cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); }
    }
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    last = flops_per_launch * n / ms / 1e9;
    best = last > best ? last : best;
    total_ms += ms;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("sustained DMMA m8n8k4 t=%.1f s: %.2f TFLOP/s\n", total_ms / 1e3, last);
  }
  printf("sustained DMMA m8n8k4 over %.1f s: last window %.2f TFLOP/s, best %.2f\n", total_ms / 1e3, last, best);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1) return sustained(atof(argv[1]));
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads);
    int iters = 20000;
    dfma_kernel<<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("DFMA threads=%d: %.2f TFLOP/s (%.3f ms)\n", threads, flops / ms / 1e9, ms);
  }
  auto run = [&](auto kern, const char* name, double flop_per_mma) {
    for (int threads : {128, 256, 512}) {
      int blocks = sms * (1024 / threads);
      int iters = 20000;
      kern<<<blocks, threads>>>(d, 100);
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = flop_per_mma * 8 * iters * (double)blocks * (threads / 32);
      printf("%s threads=%d: %.2f TFLOP/s (%.3f ms) err=%s\n", name, threads, flops / ms / 1e9, ms,
             cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(dmma_kernel<0>, "DMMA m8n8k4", 2.0 * 8 * 8 * 4);
  run(dmma_kernel<1>, "DMMA m16n8k4", 2.0 * 16 * 8 * 4);
  run(dmma_kernel<2>, "DMMA m16n8k8", 2.0 * 16 * 8 * 8);
  return 0;
}
