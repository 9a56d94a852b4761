// Device helpers shared by the sm_100a kernels.
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>
#include "acp_internal.h"

namespace acp {

// Streaming 128-bit global accesses: M and E are touched once per kernel, so
// they bypass L1 retention (ld.global.cs / st.global.cs) and leave L1 to the
// r-column factors, which every row of a layer re-reads.
__device__ __forceinline__ float4 ld_cs4(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st_cs4(float* p, float4 v) {
  __stcs(reinterpret_cast<float4*>(p), v);
}
// Factor loads: read-only for the whole kernel, L1-cached.
__device__ __forceinline__ float4 ld_f4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float f4dot(float4 a, float4 b) {
  return fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, a.w * b.w)));
}
__device__ __forceinline__ void f4fma(float4& acc, float s, float4 q) {
  acc.x = fmaf(s, q.x, acc.x);
  acc.y = fmaf(s, q.y, acc.y);
  acc.z = fmaf(s, q.z, acc.z);
  acc.w = fmaf(s, q.w, acc.w);
}
__device__ __forceinline__ float4 f4scale(float4 a, float s) {
  return make_float4(a.x * s, a.y * s, a.z * s, a.w * s);
}

// splitmix64 and the counter-based N(0,1) of DESIGN.md "Counter-based
// generator" (the oracle implements the same definition independently).
__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t column_key(uint64_t seed, uint64_t tag, uint64_t layer,
                                               uint64_t step, uint64_t col) {
  uint64_t k = sm64(seed);
  k = sm64(k ^ tag);
  k = sm64(k ^ layer);
  k = sm64(k ^ step);
  return sm64(k ^ col);
}
__device__ __forceinline__ float gaussian_at(uint64_t key, uint64_t i) {
  const uint64_t a = sm64(key ^ (2ull * i));
  const uint64_t b = sm64(key ^ (2ull * i + 1ull));
  const double u1 = (double)((a >> 11) + 1ull) * 0x1p-53;
  const double u2 = (double)(b >> 11) * 0x1p-53;
  const double z = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
  return (float)z;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Bounded spin (device-side waits on flags other CTAs publish): a broken
// epoch / counter traps after 10 s instead of hanging the GPU.
constexpr uint64_t kSpinLimitNs = 10000000000ull;

// Host: launch `kern` on `s`; cooperative = the CTAs of the grid wait on each
// other (NVLS barriers), so ask for guaranteed co-residency
// (cudaLaunchAttributeCooperative: the launch fails instead of deadlocking
// when the grid cannot be resident at once; valid inside graph capture).
template <class... KArgs, class... Args>
inline cudaError_t launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t s, bool cooperative, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cooperative ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// mbarrier / async-copy helpers (k_stream.cu, k_tc.cu)
__device__ __forceinline__ uint32_t s32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(s32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(done)
      : "r"(s32(b)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(s32(dst)),
      "l"(src), "r"(bytes), "r"(s32(bar)), "l"(policy)
      : "memory");
}
// 4-byte async copy global -> shared (LDGSTS); src_bytes = 0 zero-fills
__device__ __forceinline__ void cp_async4(float* dst, const float* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
// arrive on `bar` once all of this thread's prior cp.async have landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(s32(bar)) : "memory");
}
// 16-byte async copy global -> shared (L2 only); src_bytes = 0 zero-fills
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}

// ---- tensor-map TMA (k_tc.cu, k_tc5.cu) ----
// 2-D tensor-map TMA load (box at column c0, row r0) completing on `bar`
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int r0,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(s32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(s32(bar)), "l"(policy)
      : "memory");
}
// L2 prefetch of a tensor-map box (no shared memory, no completion): keeps
// more HBM reads in flight than the shared-memory ring can hold
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int r0) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(r0)
               : "memory");
}
// L2 prefetch of `bytes` (multiple of 16) at a 16-byte-aligned address
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tmap_acquire(const CUtensorMap* map) {
  asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(
                   reinterpret_cast<uint64_t>(map))
               : "memory");
}

// 2-D tensor-map TMA store of a shared-memory box (bulk group; the caller
// commits and waits for the shared-memory read before reusing the buffer)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int r0) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(r0), "r"(s32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Warm L1 with the descriptors a CTA's work segments refer to (segment,
// LayerDesc, gradient pointer), one round trip for all of them: each segment
// otherwise starts with a chain of dependent loads (segment -> layer ->
// gradient pointer), which dominated models with many small layers.
template <class Seg>
__device__ __forceinline__ void prefetch_segs(const Tables& t, const Seg* segs, int sb, int se) {
  for (int i = sb + (int)threadIdx.x; i < se; i += (int)blockDim.x) {
    const int layer = segs[i].layer;
    const char* L = reinterpret_cast<const char*>(t.layers + layer);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(L));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(L + 128));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(L + sizeof(LayerDesc) - 1));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(t.grads + layer));
  }
}

// A run of consecutive vector (1-D) segments starting at s. Short segments
// are spread over the warps (warp w takes every nwarps-th one, lanes stride
// its elements), so the run's small tensors are in flight together instead
// of costing one memory round trip each; long ones (>= 64 elements per warp)
// use the whole CTA. f(seg, layer, first, stride) walks elements
// [row0 + first, row1) with the given stride. Returns the index of the first
// non-vector segment.
template <class Seg, class F>
__device__ __forceinline__ int vector_run(const Tables& t, const Seg* segs, int s, int se, int warp,
                                          int nwarps, F&& f) {
  const int lane = threadIdx.x & 31, nt = 32 * nwarps;
  int e = s, k = 0;
  for (; e < se; ++e) {
    const Seg sg = segs[e];
    const LayerDesc& L = t.layers[sg.layer];
    if (L.mat) break;
    if (sg.row1 - sg.row0 >= 64 * nwarps) {
      f(sg, L, (int)threadIdx.x, nt);
    } else {
      if (k == warp) f(sg, L, lane, 32);
      if (++k == nwarps) k = 0;
    }
  }
  return e;
}

constexpr int kTagQ0 = 1, kTagDegenerate = 2, kTagNoReuse = 3;

// 3xTF32: x = hi + lo with hi = x rounded to TF32 (10-bit
// mantissa, round half away from zero on the bit pattern) and lo = x - hi
// (exact); the tensor core reads lo truncated to TF32, an error below
// 2^-21 |x|. A product a*b is taken as ah*bh + ah*bl + al*bh, which keeps
// fp32-class accuracy at TF32 MMA rate.
__device__ __forceinline__ uint32_t tf32_hi(float x) {
  return (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
}
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = tf32_hi(x);
  lo = __float_as_uint(x - __uint_as_float(hi));
}
// D += A B, m16n8k8, TF32 inputs, fp32 accumulate (warp-level tensor-core MMA).
// Fragments (g = lane / 4, t = lane % 4): a0 (g, t), a1 (g + 8, t), a2 (g, t + 4),
// a3 (g + 8, t + 4); b0 (k = t, n = g), b1 (k = t + 4, n = g); d0 (g, 2t),
// d1 (g, 2t + 1), d2 (g + 8, 2t), d3 (g + 8, 2t + 1).
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 3xTF32 product accumulate
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                     uint32_t bh0, uint32_t bh1, uint32_t bl0, uint32_t bl1) {
  mma_tf32(d, al, bh0, bh1);
  mma_tf32(d, ah, bl0, bl1);
  mma_tf32(d, ah, bh0, bh1);
}

}  // namespace acp
