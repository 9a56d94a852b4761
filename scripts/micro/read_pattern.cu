// Read-read-write HBM streaming vs access pattern (K1's traffic: read M, S;
// write S), n x m fp32, m = 1024, through TMA into shared memory:
//   A  1-D bulk copies of whole-row tiles (8 rows = 32 KB contiguous per tensor)
//   B  2-D tensor boxes of 32 cols x 128 rows (128 B per row), TMA store back
//   C  3-D boxes {32, 4, 128} over [rows][m/32][32]: 512 B contiguous per row
// One persistent CTA per SM, 4-stage ring, one producer thread, consumers just
// release the stage (no compute). Prints GB/s of algorithmic traffic (12 B/elem).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_pattern read_pattern.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(n)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b))); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t d;
  do { asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(d) : "r"(s32(b)), "r"(ph)); } while (!d);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t n, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(dst)), "l"(src), "r"(n), "r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(s32(src)), "r"(n) : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* m, int c, int r, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(s32(dst)), "l"(m), "r"(c), "r"(r), "r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void tma2_st(const CUtensorMap* m, const void* src, int c, int r) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(c), "r"(r), "r"(s32(src)) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, int c, int b, int r, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(s32(dst)), "l"(m), "r"(c), "r"(b), "r"(r), "r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void tma3_st(const CUtensorMap* m, const void* src, int c, int b, int r) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(m), "r"(c), "r"(b), "r"(r), "r"(s32(src)) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

constexpr int NS = 3, TB = 32768;  // stage: M tile + S tile of 32 KB each
template <int MODE>
__global__ void __launch_bounds__(64, 1) kern(const float* M, float* S, long n, int m, const __grid_constant__ CUtensorMap mM,
                                             const __grid_constant__ CUtensorMap mS) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* base = raw + ((1024 - (s32(raw) & 1023)) & 1023);
  __shared__ uint64_t full[NS], empty[NS];
  if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 32); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  // tiles: MODE 0: 8 whole rows (32 KB); MODE 1: 128 rows x 64 cols (2 boxes); MODE 2: 128 rows x 64 cols via one 3-D box {32, 2, 128}
  const long ntiles = MODE == 0 ? n / 8 : (n / 128) * (m / 64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    int st = 0; uint32_t ph = 0; int pend = -1;
    for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(&empty[st], ph ^ 1);
      unsigned char* dm = base + st * 2 * TB; unsigned char* ds = dm + TB;
      mbar_tx(&full[st], 2 * TB);
      if (MODE == 0) { bulk_g2s(dm, M + t * 8 * m, TB, &full[st]); bulk_g2s(ds, S + t * 8 * m, TB, &full[st]); }
      else {
        const long rb = (t / (m / 64)) * 128; const int c0 = (int)(t % (m / 64)) * 64;
        if (MODE == 1) { for (int b = 0; b < 2; ++b) { tma2(dm + b * 16384, &mM, c0 + 32 * b, (int)rb, &full[st]); tma2(ds + b * 16384, &mS, c0 + 32 * b, (int)rb, &full[st]); } }
        else { tma3(dm, &mM, 0, c0 / 32, (int)rb, &full[st]); tma3(ds, &mS, 0, c0 / 32, (int)rb, &full[st]); }
      }
      if (++st == NS) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    int st = 0; uint32_t ph = 0; int pend = -1;
    for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(&full[st], ph);
      unsigned char* ds = base + st * 2 * TB + TB;
      if (lane == 0) {
        if (MODE == 0) bulk_s2g(S + t * 8 * m, ds, TB);
        else {
          const long rb = (t / (m / 64)) * 128; const int c0 = (int)(t % (m / 64)) * 64;
          if (MODE == 1) { for (int b = 0; b < 2; ++b) tma2_st(&mS, ds + b * 16384, c0 + 32 * b, (int)rb); }
          else tma3_st(&mS, ds, 0, c0 / 32, (int)rb);
        }
        commit();
        if (pend >= 0) { wait_read1(); }
      }
      __syncwarp();
      if (pend >= 0) mbar_arrive(&empty[pend]);
      pend = st;
      if (++st == NS) { st = 0; ph ^= 1; }
    }
    if (lane == 0) wait_all();
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long n = 327680; const int m = 1024;
  float *M, *S;
  cudaMalloc(&M, n * m * 4); cudaMalloc(&S, n * m * 4);
  cudaMemset(M, 0, n * m * 4); cudaMemset(S, 0, n * m * 4);
  EncFn enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m2[2], m3[2];
  for (int k = 0; k < 2; ++k) {
    void* p = k ? (void*)S : (void*)M;
    cuuint64_t d2[2] = {(cuuint64_t)m, (cuuint64_t)n}, s2[1] = {(cuuint64_t)m * 4}; cuuint32_t b2[2] = {32, 128}, e2[2] = {1, 1};
    enc(&m2[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t d3[3] = {32, (cuuint64_t)m / 32, (cuuint64_t)n}, s3[2] = {128, (cuuint64_t)m * 4}; cuuint32_t b3[3] = {32, 2, 128}, e3[3] = {1, 1, 1};
    enc(&m3[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  const int smem = NS * 2 * TB + 1024;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto kfn, const CUtensorMap& x, const CUtensorMap& y) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int w = 0; w < 3; ++w) kfn<<<148, 64, smem>>>(M, S, n, m, x, y);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) kfn<<<148, 64, smem>>>(M, S, n, m, x, y);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("%-40s %.4f ms  %.0f GB/s  (%s)\n", name, ms, 12.0 * n * m / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run("A 1-D bulk, 8 whole rows (32 KB)", kern<0>, m2[0], m2[1]);
  run("B 2-D boxes 32x128 (128 B/row), x2", kern<1>, m2[0], m2[1]);
  run("C 3-D box {32,2,128} (256 B/row)", kern<2>, m3[0], m3[1]);
  return 0;
}
