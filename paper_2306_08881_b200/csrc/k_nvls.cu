// NVLS all-reduce of a fused-buffer range: the P / Q fused
// buffers live in symmetric memory bound to an NVLink-SHARP multicast object;
// each rank reduces a 1/p slice of the range IN THE SWITCH
// (multimem.ld_reduce.add) and writes the sum back to every rank with one
// multicast store (multimem.st). Replaces the per-bucket ncclAllReduce of
// P:223 / P:228 for world_size > 1: one small kernel per compute group, no
// NCCL launch, no ring / tree protocol.
//
// Cross-rank ordering: CTA c of every rank meets CTA c of every other rank
// at an entry barrier (all ranks' projections of the range are done) and an
// exit barrier (all slices are reduced) through flags in the symmetric flag
// region (st.release.sys / ld.acquire.sys; epochs from a per-CTA launch
// counter, so nothing is ever reset and CUDA-graph replays stay valid).
#include "k_common.cuh"

namespace acp {
namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// flags: [2 barriers][kNvlsMaxCtas][kNvlsMaxRanks] uint32 per rank
__device__ void cross_rank_barrier(const NvlsArgs& a, int which, uint32_t epoch) {
  const int slot = (which * kNvlsMaxCtas + blockIdx.x) * kNvlsMaxRanks;
  if ((int)threadIdx.x < a.world) {
    const int p = threadIdx.x;
    __threadfence_system();
    st_release_sys(a.peer_flags[p] + slot + a.rank, epoch);
    // a peer that never arrives (crashed rank, mismatched launch sequence)
    // must not hang the GPU: trap after 10 s, which fails the stream loudly
    const uint64_t t0 = globaltimer_ns();
    while ((int)(ld_acquire_sys(a.my_flags + slot + p) - epoch) < 0) {
      __nanosleep(32);
      if (globaltimer_ns() - t0 > 10000000000ull) __trap();
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(512) nvls_allreduce_kernel(NvlsArgs a, int64_t off, int64_t cnt) {
  __shared__ uint32_t epoch_sh;
  if (threadIdx.x == 0) epoch_sh = ++a.epoch[blockIdx.x];
  __syncthreads();
  const uint32_t epoch = epoch_sh;
  cross_rank_barrier(a, 0, epoch);
  // this rank's slice of the range, in float4 units (ranges are 16-byte aligned)
  const int64_t n4 = cnt / 4;
  const int64_t per = (n4 + a.world - 1) / a.world;
  const int64_t b = (int64_t)a.rank * per, e = (b + per < n4) ? b + per : n4;
  float* base = a.mc + off;
  for (int64_t i = b + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e;
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
  cross_rank_barrier(a, 1, epoch);
}

}  // namespace

cudaError_t launch_nvls_allreduce(const NvlsArgs& a, int64_t off, int64_t cnt, cudaStream_t s) {
  if (cnt <= 0) return cudaSuccess;
  const int64_t per4 = (cnt / 4 + a.world - 1) / a.world;
  int grid = (int)std::min<int64_t>(kNvlsMaxCtas, std::max<int64_t>(1, (per4 + 511) / 512));
  // CTA c of every rank meets CTA c of every other rank: co-resident grid
  return launch_kernel(nvls_allreduce_kernel, dim3(grid), dim3(512), 0, s, true, a, off, cnt);
}

}  // namespace acp
