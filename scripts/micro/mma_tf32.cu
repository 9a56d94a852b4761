// Microbenchmark: legacy warp-level mma.sync m16n8k8 TF32 throughput on sm_100a
// (decides whether the r >= 8 projection can use it; scripts/micro, not product code).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kb(float* out, int iters) {  // bf16 m16n8k16 for comparison
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w : {4, 8, 16}) {
    int iters = 4096;
    k<<<148 * 4, w * 32>>>(d, iters);
    cudaEventRecord(e0);
    k<<<148 * 4, w * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * w * 148 * 4;
    printf("tf32 mma.sync m16n8k8: warps/CTA %d: %.1f TFLOP/s\n", w, flops / ms / 1e9);
    kb<<<148 * 4, w * 32>>>(d, iters);
    cudaEventRecord(e0);
    kb<<<148 * 4, w * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * w * 148 * 4;
    printf("bf16 mma.sync m16n8k16: warps/CTA %d: %.1f TFLOP/s\n", w, flops / ms / 1e9);
  }
  return 0;
}
