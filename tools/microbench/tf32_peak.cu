// Legacy mma.sync tensor throughput on sm_100a: tf32 m16n8k8 and bf16 m16n8k16 (f32 accumulate).
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void mma_kernel(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 7, b1 = 9;
  float c[8][4];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (K == 8)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5f) out[0] = s;
}
int main() {
  float* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int threads : {128, 256, 512}) {
    int blocks = sms * (1024 / threads), iters = 20000;
    mma_kernel<8><<<blocks, threads>>>(d, 100);
    cudaEventRecord(e0); mma_kernel<8><<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("TF32 m16n8k8 threads=%d: %.1f TFLOP/s\n", threads, 2.0 * 16 * 8 * 8 * 8 * iters * (double)blocks * (threads / 32) / ms / 1e9);
    mma_kernel<16><<<blocks, threads>>>(d, 100);
    cudaEventRecord(e0); mma_kernel<16><<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("BF16 m16n8k16 threads=%d: %.1f TFLOP/s %s\n", threads, 2.0 * 16 * 8 * 16 * 8 * iters * (double)blocks * (threads / 32) / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
}
