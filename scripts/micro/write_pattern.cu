// Write-only HBM bandwidth vs store pattern (n x m fp32 matrix, m = 1024):
//  P1 rows: each warp stores 512 B contiguous per instruction, whole rows in order
//  P2 tile-col: 128x128 tiles; a warp instruction stores 128 B (32 cols) of ONE row,
//     thread = column, 32 rows per warp in sequence (the tcgen05 decode's D^T epilogue)
//  P3 tile-row: 128x128 tiles; a warp instruction stores a whole 512 B tile row
//  P4 tile-col with 32-row tiles
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_pattern write_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void p1(float* g, long n, int m) {
  const long total4 = n * (long)m / 4;
  float4* g4 = reinterpret_cast<float4*>(g);
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total4; i += (long)gridDim.x * blockDim.x)
    __stcs(g4 + i, make_float4(1.f, 2.f, 3.f, 4.f));
}
// persistent: CTA c takes tiles c, c + grid, ...; 4 warps; tile = TR rows x 128 cols
template <int TR>
__global__ void p2(float* g, long n, int m) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long nrb = (n + TR - 1) / TR, nct = m / 128;
  for (long t = blockIdx.x; t < nrb * nct; t += gridDim.x) {
    const long rb = (t / nct) * TR, c0 = (t % nct) * 128;
    const long col = c0 + 32 * warp + lane;
    for (int i = 0; i < TR; ++i) {
      const long row = rb + i;
      if (row < n) __stcs(g + row * m + col, (float)i);
    }
  }
}
__global__ void p3(float* g, long n, int m) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long nrb = (n + 127) / 128, nct = m / 128;
  for (long t = blockIdx.x; t < nrb * nct; t += gridDim.x) {
    const long rb = (t / nct) * 128, c0 = (t % nct) * 128;
    for (int i = warp; i < 128; i += 4) {
      const long row = rb + i;
      if (row < n) __stcs(reinterpret_cast<float4*>(g + row * m + c0) + lane, make_float4(1.f, 2.f, 3.f, 4.f));
    }
  }
}

int main() {
  const long n = 327680;
  const int m = 1024;  // 1.34 GB
  float* g;
  cudaMalloc(&g, n * (long)m * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 10;
    printf("%-34s %.4f ms  %.0f GB/s  (%s)\n", name, ms, n * (double)m * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run("P1 rows, 512B/instr, 148x8 CTAs", [&] { p1<<<148 * 8, 256>>>(g, n, m); });
  run("P2 tile-col 128-row tiles, 148x1", [&] { p2<128><<<148, 128>>>(g, n, m); });
  run("P2 tile-col 128-row tiles, 148x4", [&] { p2<128><<<148 * 4, 128>>>(g, n, m); });
  run("P4 tile-col 32-row tiles, 148x1", [&] { p2<32><<<148, 128>>>(g, n, m); });
  run("P4 tile-col 32-row tiles, 148x4", [&] { p2<32><<<148 * 4, 128>>>(g, n, m); });
  run("P3 tile-row 512B/instr, 148x1", [&] { p3<<<148, 128>>>(g, n, m); });
  run("P3 tile-row 512B/instr, 148x4", [&] { p3<<<148 * 4, 128>>>(g, n, m); });
  return 0;
}
