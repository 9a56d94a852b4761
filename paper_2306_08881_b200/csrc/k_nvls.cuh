// NVLS all-reduce fused into a decode kernel's prologue:
// the decode of parity p first sums fused buffer p over the ranks IN THE
// SWITCH (multimem.ld_reduce + multimem.st), then decodes -- one kernel for
// "all-reduce -> decode". Needs the whole grid resident (the plan caps decode
// grids at one wave) and the symmetric region of acp_attach_symmetric.
#pragma once
#include "k_common.cuh"

namespace acp {

__device__ __forceinline__ void nv_st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t nv_ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t nv_ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void nv_wait_ge(const uint32_t* p, uint32_t target, bool sys) {
  const uint64_t t0 = globaltimer_ns();
  while ((int)((sys ? nv_ld_acquire_sys(p) : nv_ld_acquire_gpu(p)) - target) < 0) {
    __nanosleep(64);
    if (globaltimer_ns() - t0 > kSpinLimitNs) __trap();  // never hang the GPU
  }
}

// Every CTA of the grid on every rank arrives; the last CTA of this rank
// trades flags with the other ranks, then releases its grid.
__device__ __forceinline__ void nv_grid_barrier(const NvlsArgs& a, FusedSync* fs, uint32_t target, int row) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t arrived = atomicAdd(&fs->gcount, 1u) + 1u;
    if (arrived == target * gridDim.x) {
      const int slot = row * kNvlsMaxCtas * kNvlsMaxRanks;
      __threadfence_system();
      for (int p = 0; p < a.world; ++p) nv_st_release_sys(a.peer_flags[p] + slot + a.rank, target);
      for (int p = 0; p < a.world; ++p) nv_wait_ge(a.my_flags + slot + p, target, true);
      __threadfence();
      atomicExch(&fs->release, target);
    }
    nv_wait_ge(&fs->release, target, false);
  }
  __syncthreads();
}

// Sum buffer `parity` over the ranks: this rank reduces a 1/p slice, every
// rank receives the result through the multicast store.
__device__ __forceinline__ void nvls_fused_reduce(const Tables& t, int parity) {
  const NvlsArgs& a = *t.nv;
  FusedSync* fs = t.fsync + parity;
  __shared__ uint32_t nv_epoch_sh;
  if (threadIdx.x == 0) nv_epoch_sh = *reinterpret_cast<volatile uint32_t*>(&fs->epoch);
  __syncthreads();
  const uint32_t e = nv_epoch_sh;
  const int world = a.world, rank = a.rank;
  const int row = 2 + 2 * parity;          // flag rows per parity (epochs are per parity)
  nv_grid_barrier(a, fs, 2u * e + 1u, row);  // every rank's fused buffer is complete
  const int64_t n4 = a.n_buf[parity] / 4;
  const int64_t per = (n4 + world - 1) / world;
  const int64_t b = (int64_t)rank * per, end = (b + per < n4) ? b + per : n4;
  float* base = a.mc_buf[parity];
  for (int64_t i = b + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < end;
       i += (int64_t)gridDim.x * blockDim.x) {
    float* p = base + 4 * i;
    float x, y, z, w;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(x), "=f"(y), "=f"(z), "=f"(w)
                 : "l"(p)
                 : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(x), "f"(y),
                 "f"(z), "f"(w)
                 : "memory");
  }
  nv_grid_barrier(a, fs, 2u * e + 2u, row + 1);  // every slice is summed everywhere
  if (blockIdx.x == 0 && threadIdx.x == 0) fs->epoch = e + 1u;  // all CTAs read e at entry
  // the decode reads the summed buffer through TMA / cp.async.bulk (async
  // proxy) as well as plain loads: order the generic-proxy multimem writes
  // before them
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

}  // namespace acp
