// Bring-up check of the tcgen05 kind::tf32 MMA used by k_tc5.cu: one CTA,
// A (128 x K) and B (128 x K) in MN-major 128B-swizzled atoms, D = A B^T in
// TMEM, read back with tcgen05.ld 32x32b, compared with a host GEMM.
// nvcc -gencode arch=compute_100a,code=sm_100a -o umma_tf32_test umma_tf32_test.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int KG>
__device__ __forceinline__ uint32_t atom_off(int mn, int k) {
  return (uint32_t)((mn >> 5) * (KG * 1024) + (k >> 3) * 1024 + (k & 7) * 128 + ((((mn & 31) >> 2) ^ (k & 7)) << 4) + (mn & 3) * 4);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint64_t mode) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (mode << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int amaj, int bmaj) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t done;
  do {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(s32(b)), "r"(ph));
  } while (!done);
}

template <int K, int VAR>
__global__ void kern(const float* A, const float* B, float* D, uint32_t* info) {
  constexpr int KG = K / 8;
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* base = raw + ((1024u - (s32(raw) & 1023u)) & 1023u);
  unsigned char* sA = base;
  unsigned char* sB = base + 128 * K * 4;
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int idx = tid; idx < 128 * K; idx += blockDim.x) {
    const int i = idx % 128, k = idx / 128;
    if (VAR == 4) {  // K-major SW128, K = 32 tf32 per 128 B row
      const uint32_t o = (i / 8) * 1024 + (i % 8) * 128 + ((((k / 4) ^ (i % 8))) << 4) + (k % 4) * 4;
      *reinterpret_cast<float*>(sA + o) = A[i * K + k];
      *reinterpret_cast<float*>(sB + o) = B[i * K + k];
    } else if (VAR == 5) {  // K-major SW128 bf16, 64 per row (K = 32 used)
      const uint32_t o = (i / 8) * 1024 + (i % 8) * 128 + ((((k / 8) ^ (i % 8))) << 4) + (k % 8) * 2;
      *reinterpret_cast<__nv_bfloat16*>(sA + o) = __float2bfloat16(A[i * K + k]);
      *reinterpret_cast<__nv_bfloat16*>(sB + o) = __float2bfloat16(B[i * K + k]);
    } else if (VAR == 6 || VAR == 7) {  // MN-major SW128 with 32-byte atoms (layout type 1)
      const uint32_t o = (i / 32) * (K * 128) + (k / 4) * 512 + (k % 4) * 128 + ((((i % 32) / 8) ^ (k % 4)) << 5) + (i % 8) * 4;
      *reinterpret_cast<float*>(sA + o) = A[i * K + k];
      *reinterpret_cast<float*>(sB + o) = B[i * K + k];
    } else {
      *reinterpret_cast<float*>(sA + atom_off<KG>(i, k)) = A[i * K + k];
      *reinterpret_cast<float*>(sB + atom_off<KG>(i, k)) = B[i * K + k];
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(s32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tm;
  if (tid == 0) {
    info[0] = tb;
    const uint32_t ID = idesc(128, 128, 1, 1);
    for (int kg = 0; kg < KG; ++kg) {
      uint64_t a, b;
      if (VAR == 0) { a = sdesc(s32(sA) + kg * 1024, KG * 1024, 1024, 2); b = sdesc(s32(sB) + kg * 1024, KG * 1024, 1024, 2); }
      else { a = sdesc(s32(sA) + kg * 1024, 1024, KG * 1024, 2); b = sdesc(s32(sB) + kg * 1024, 1024, KG * 1024, 2); }
      uint32_t acc = kg > 0;
      if (VAR == 2) {
        a = sdesc(s32(sA) + kg * 1024, KG * 1024, 1024, 2); b = sdesc(s32(sB) + kg * 1024, KG * 1024, 1024, 2);
        uint32_t z = 0;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n}" ::"r"(tb), "l"(a), "l"(b), "r"(ID), "r"(acc), "r"(z));
      } else if (VAR == 6) {
        a = sdesc(s32(sA) + kg * 1024, K * 128, 512, 1); b = sdesc(s32(sB) + kg * 1024, K * 128, 512, 1);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tb), "l"(a), "l"(b), "r"(ID), "r"(acc));
      } else if (VAR == 7) {  // same, LBO/SBO swapped
        a = sdesc(s32(sA) + kg * 1024, 512, K * 128, 1); b = sdesc(s32(sB) + kg * 1024, 512, K * 128, 1);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tb), "l"(a), "l"(b), "r"(ID), "r"(acc));
      } else if (VAR == 4) {
        a = sdesc(s32(sA) + kg * 32, 16, 1024, 2); b = sdesc(s32(sB) + kg * 32, 16, 1024, 2);
        const uint32_t IDK = idesc(128, 128, 0, 0);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tb), "l"(a), "l"(b), "r"(IDK), "r"(acc));
      } else if (VAR == 5) {
        if (kg < KG / 2) {
          a = sdesc(s32(sA) + kg * 32, 16, 1024, 2); b = sdesc(s32(sB) + kg * 32, 16, 1024, 2);
          const uint32_t IDB = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tb), "l"(a), "l"(b), "r"(IDB), "r"(acc));
        }
      } else if (VAR != 3) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tb), "l"(a), "l"(b), "r"(ID), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&bar)));
  }
  if (VAR != 3) mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (VAR == 3 && warp < 4) {
    for (int j = 0; j < 128; ++j) {
      uint32_t x = __float_as_uint((float)(1000 * (32 * warp + lane) + j));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tb + ((uint32_t)(32 * warp) << 16) + j), "r"(x));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  if (warp < 4) {
    for (int j = 0; j < 4; ++j) {
      uint32_t v[32];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(tb + ((uint32_t)(32 * warp) << 16) + 32 * j));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int c = 0; c < 32; ++c) D[(32 * warp + lane) * 128 + 32 * j + c] = __uint_as_float(v[c]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb));
}

template <int K, int VAR>
int run() {
  std::vector<float> A(128 * K), B(128 * K), D(128 * 128), R(128 * 128);
  for (int i = 0; i < 128; ++i)
    for (int k = 0; k < K; ++k) {
      A[i * K + k] = (float)((i * 7 + k * 3) % 11 - 5);
      B[i * K + k] = (float)((i * 5 + k * 13) % 9 - 4);
    }
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
      R[i * 128 + j] = (float)s;
    }
  float *dA, *dB, *dD;
  uint32_t* dI;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dI, 64);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  const int smem = 2 * 128 * K * 4 + 1024;
  cudaFuncSetAttribute(kern<K, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<K, VAR><<<1, 128, smem>>>(dA, dB, dD, dI);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  double maxerr = 0;
  for (int i = 0; i < 128 * 128; ++i) {
    const double d = fabs(D[i] - R[i]);
    if (d > 1e-3) ++bad;
    if (d > maxerr) maxerr = d;
  }
  uint32_t info[4];
  cudaMemcpy(info, dI, 16, cudaMemcpyDeviceToHost);
  if (VAR == 3) { printf("st/ld roundtrip: D[0][0..2]=%g %g %g D[37][50]=%g (expect 0 1 2 37050) tb=%u\n", D[0], D[1], D[2], D[37*128+50], info[0]); return 0; }
  printf("tb=%u K=%d var=%d err=%s bad=%d/%d maxerr=%g  D[0][0..3]=%g %g %g %g  R=%g %g %g %g  D[37][50]=%g R=%g\n", info[0], K, VAR,
         cudaGetErrorString(e), bad, 128 * 128, maxerr, D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3], D[37 * 128 + 50],
         R[37 * 128 + 50]);
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dI);
  return bad;
}

int main() {
  run<8, 3>();

  run<8, 6>();
  run<8, 7>();
  run<16, 6>();
  run<16, 7>();
  run<32, 6>();
  run<32, 7>();
  return 0;
}
