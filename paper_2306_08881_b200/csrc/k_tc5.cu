// K3 decodes for r >= 8 on the 5th-generation tensor cores (tcgen05 + TMEM):
//
//   mode 2, P-step (Alg. 2):  grad = (scale * P_agg) Q_orth^T
//   mode 3, Q-step (Alg. 2):  grad = scale * (P_orth Q_agg^T)
//
// A rank-r product per output element is a GEMM with a tiny K (= R8, the rank
// padded to 8) and a write-only output stream: 4 B of HBM per element, which
// is what bounds it. The tensor-core work is 3xTF32 (x = hi + lo, DESIGN.md
// §6b): D = A_lo B_hi + A_hi B_lo + A_hi B_hi, accumulated in TMEM by
// `tcgen05.mma.kind::tf32` (M = 128 rows, N = 128 columns, K = 8 per
// instruction, both operands MN-major in shared memory). MN-major TF32
// operands take the "128B swizzle with 32-byte atoms" layout (UMMA layout
// type 1: 4 K-rows of 128 B, 32-byte chunk c of row k stored at c ^ (k % 4));
// the plain 128B swizzle reads as zeros for 32-bit MN-major operands
// (scripts/micro/umma_tf32_test.cu). TMA writes that layout itself
// (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).
//
// CTA (one per SM, persistent over its host-planned segments), warp roles:
//   warp 0     producer: TMA boxes of the column factor (R8 x 32 floats,
//              SWIZZLE_128B_ATOM_32B = the MN-major UMMA tf32 layout) into a
//              ring of NS stages
//   warp 1     MMA issuer (one thread) + TMEM owner (2 x 128 accumulator
//              columns, double-buffered)
//   warps 2-5  epilogue: tcgen05.ld (thread = row = TMEM lane) -> registers ->
//              swizzled shared staging box (32 rows x 32 columns) -> TMA store
//              (the TMA engine writes whole lines: no partial-sector stores)
//   warp 6     A converter: the row factor (k-major P slot, coalesced loads
//              batched 16 deep) split into hi / lo in the atom layout, running
//              ahead of the MMA by up to two row blocks; vectors (unpack)
//   warp 7     B converter: the column factor split in place when it arrives
//              raw (mode 3) or gathered without TMA (m % 4 != 0)
// Synchronisation: mbarriers (full / ready / empty per B stage, full / empty
// per A buffer, full / empty per TMEM accumulator); tcgen05.commit arrives on
// the MMA-side ones.
//
// Rows: segments are whole 128-row tiles except at a layer's end (plan align);
// the TMA store clips at the tensor's edge. Layers whose column factor or
// gradient cannot take TMA (m % 4 != 0, unaligned gradient) use the gathered
// B path and per-element stores from registers.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "k_common.cuh"
#include "k_nvls.cuh"

namespace acp {
namespace {

constexpr int kT5M = 128;        // rows per tile (MMA M, TMEM lanes)
constexpr int kT5N = 128;        // columns per tile (MMA N): 4 boxes of 32
constexpr int kT5Threads = 256;
constexpr int kT5OutBufs = 4;    // staging boxes per epilogue warp (two pairs)
constexpr int kT5TmemCols = 512; // up to 4 accumulators x 128 columns

template <int R8>
struct T5 {
  static constexpr int KG = R8 / 8;              // MMA K-steps (K = 8)
  static constexpr int ATOM_MN = R8 * 128;       // bytes between 32-wide MN blocks (LBO)
  static constexpr int A_BYTES = kT5M * R8 * 4;  // one operand array (hi or lo)
  static constexpr int B_BYTES = kT5N * R8 * 4;
  static constexpr int NS = R8 >= 32 ? 3 : 4;    // column-factor stages
  static constexpr int A_OFF = 0;                                  // [2 buf][hi, lo]
  static constexpr int B_OFF = A_OFF + 4 * A_BYTES;                // [NS][hi, lo]
  static constexpr int O_OFF = B_OFF + NS * 2 * B_BYTES;           // [4 warps][bufs][4 KB]
  static constexpr int BAR_OFF = O_OFF + 4 * kT5OutBufs * 4096;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;                // + barriers + align slack
};

// byte offset of element (mn, k) of an MN-major operand in the
// [mn/32][k][32] layout with 128B / 32-byte-atom swizzle (32-byte chunk
// XOR k % 4; K-rows of 128 B, groups of 4 rows = 512 B)
template <int R8>
__device__ __forceinline__ uint32_t atom_off(int mn, int k) {
  return (uint32_t)((mn >> 5) * T5<R8>::ATOM_MN + (k >> 2) * 512 + (k & 3) * 128 +
                    ((((mn & 31) >> 3) ^ (k & 3)) << 5) + (mn & 7) * 4);
}

// UMMA shared-memory descriptor: SWIZZLE_128B_BASE32B (layout type 1),
// MN-major (LBO = stride of the 32-element MN blocks, SBO = stride of the
// 4-deep K groups), Blackwell descriptor version 1
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (1ull << 61);
}
// instruction descriptor: D fp32, A / B tf32, both MN-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void umma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// arrive on `bar` when every tcgen05 operation this thread issued so far is done
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// grad[i] = scale * slot[i], i in [i0, i1), by one warp: 16 loads in flight
// per lane (the slot is 16-byte aligned; float4 when the gradient is too)
__device__ __forceinline__ void vec_unpack(float* grad, const float* slot, int64_t i0, int64_t i1, float scale,
                                           bool fused, int lane) {
  constexpr int kB = 16;
  int64_t i = i0;
  if (((reinterpret_cast<uintptr_t>(grad) & 15u) == 0) && (i0 & 3) == 0) {
    const int64_t n4 = (i1 - i0) >> 2;
    const float4* s4 = reinterpret_cast<const float4*>(slot + i0);
    float4* g4 = reinterpret_cast<float4*>(grad + i0);
    for (int64_t b = 0; b < n4; b += 32 * kB) {
      float4 v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int64_t j = b + 32 * u + lane;
        if (j < n4) v[u] = fused ? __ldcg(s4 + j) : __ldg(s4 + j);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int64_t j = b + 32 * u + lane;
        if (j < n4) g4[j] = make_float4(v[u].x * scale, v[u].y * scale, v[u].z * scale, v[u].w * scale);
      }
    }
    i = i0 + 4 * n4;
  }
  for (int64_t b = i; b < i1; b += 32 * kB) {
    float v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int64_t j = b + 32 * u + lane;
      if (j < i1) v[u] = fused ? __ldcg(slot + j) : __ldg(slot + j);
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int64_t j = b + 32 * u + lane;
      if (j < i1) grad[j] = v[u] * scale;
    }
  }
}

struct T5Bars {
  uint64_t* bfull;   // [NS] producer (TMA complete_tx or plain arrive)
  uint64_t* bready;  // [NS] B converter warp (32 arrivals)
  uint64_t* bempty;  // [NS] MMA commit
  uint64_t* afull;   // [2] A converter warp (32 arrivals)
  uint64_t* aempty;  // [2] MMA commit
  uint64_t* tfull;   // [2] MMA commit
  uint64_t* tempty;  // [2] epilogue warps (4 arrivals)
  uint32_t* tmem;    // TMEM base written by tcgen05.alloc
};

// Iteration state shared by every role: row blocks (A buffers) and tiles
// (B stages, TMEM accumulators) are numbered in the same order everywhere.
struct T5Iter {
  uint32_t a_it = 0, t_it = 0;
};

template <int MODE, int R8>
__global__ void __launch_bounds__(kT5Threads, 1)
tc5_decode_kernel(Tables t, const TcSeg* __restrict__ segs, const int32_t* __restrict__ cta_begin, float scale,
                  int dbg) {
  using G = T5<R8>;
  constexpr int NS = G::NS;
  extern __shared__ __align__(1024) unsigned char t5_raw[];
  unsigned char* base = t5_raw + ((1024u - (s32(t5_raw) & 1023u)) & 1023u);
  const uint32_t sbase = s32(base);
  T5Bars b;
  {
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + G::BAR_OFF);
    b.bfull = bars;
    b.bready = bars + NS;
    b.bempty = bars + 2 * NS;
    b.afull = bars + 3 * NS;
    b.aempty = b.afull + 2;
    b.tfull = b.aempty + 2;
    b.tempty = b.tfull + 4;
    b.tmem = reinterpret_cast<uint32_t*>(b.tempty + 4);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&b.bfull[i], 1);
      mbar_init(&b.bready[i], 32);
      mbar_init(&b.bempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b.afull[i], 32);
      mbar_init(&b.aempty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&b.tfull[i], 1);
      mbar_init(&b.tempty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(b.tmem)),
                 "r"(kT5TmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *b.tmem;
  __shared__ unsigned long long dbg_t[8];
  const unsigned long long t_start = globaltimer_ns();
  const int sb = cta_begin[blockIdx.x], se = cta_begin[blockIdx.x + 1];
  prefetch_segs(t, segs, sb, se);
  // NVLS (NEXT-3): sum this parity's fused buffer over the ranks first
  if (t.nvls_fused) nvls_fused_reduce(t, MODE == 2 ? 0 : 1);
  T5Iter it;
  const int nacc = (dbg & 32) ? 4 : 2;

  if (warp == 0) {
    // ---------------- producer: column-factor boxes ----------------
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      for (int si = sb; si < se; ++si) {
        const TcSeg s = segs[si];
        const LayerDesc& L = t.layers[s.layer];
        if (!L.mat) continue;
        const int64_t m = L.m;
        const bool tma = (m % 4) == 0;
        const CUtensorMap* maps = t.tmaps + kTmapsPerLayer * (int64_t)s.layer;
        if (tma) {
          tmap_acquire(maps + (MODE == 2 ? 10 : 12));
          if (MODE == 2) tmap_acquire(maps + 11);
        }
        for (int64_t rb = s.row0; rb < s.row1; rb += kT5M) {
          for (int64_t c0 = 0; c0 < m; c0 += kT5N, ++it.t_it) {
            const int stage = it.t_it % NS;
            const uint32_t ph = (it.t_it / NS) & 1u;
            mbar_wait(&b.bempty[stage], ph ^ 1u);
            unsigned char* dB = base + G::B_OFF + stage * 2 * G::B_BYTES;
            if (tma && !(dbg & 8)) {
              const int nbox = (int)((m - c0 + 31) / 32) < 4 ? (int)((m - c0 + 31) / 32) : 4;
              const uint32_t box = R8 * 32 * 4;
              mbar_arrive_tx(&b.bfull[stage], (MODE == 2 ? 2u : 1u) * box * (uint32_t)nbox);
              for (int nb = 0; nb < nbox; ++nb) {
                if (MODE == 2) {
                  tma_load_2d(dB + nb * G::ATOM_MN, maps + 10, (int)c0 + 32 * nb, 0, &b.bfull[stage], pol);
                  tma_load_2d(dB + G::B_BYTES + nb * G::ATOM_MN, maps + 11, (int)c0 + 32 * nb, 0, &b.bfull[stage],
                              pol);
                } else {
                  tma_load_2d(dB + nb * G::ATOM_MN, maps + 12, (int)c0 + 32 * nb, 0, &b.bfull[stage], pol);
                }
              }
            } else {
              mbar_arrive(&b.bfull[stage]);  // converters gather B themselves
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t ID = idesc_tf32(kT5M, kT5N);
      for (int si = sb; si < se; ++si) {
        const TcSeg s = segs[si];
        const LayerDesc& L = t.layers[s.layer];
        if (!L.mat) continue;
        const int64_t m = L.m;
        for (int64_t rb = s.row0; rb < s.row1; rb += kT5M, ++it.a_it) {
          const int ab = it.a_it & 1;
          mbar_wait(&b.afull[ab], (it.a_it >> 1) & 1u);
          const uint32_t aH = sbase + G::A_OFF + ab * 2 * G::A_BYTES, aL = aH + G::A_BYTES;
          for (int64_t c0 = 0; c0 < m; c0 += kT5N, ++it.t_it) {
            const int stage = it.t_it % NS;
            const int acc = it.t_it % nacc;
            mbar_wait(&b.bready[stage], (it.t_it / NS) & 1u);
            mbar_wait(&b.tempty[acc], ((it.t_it / nacc) & 1u) ^ 1u);
            tc_fence_after();
            const uint32_t bH = sbase + G::B_OFF + stage * 2 * G::B_BYTES, bL = bH + G::B_BYTES;
            const uint32_t d = tbase + (uint32_t)(acc * kT5N);
#pragma unroll
            for (int kg = 0; kg < G::KG; ++kg) {
              if (dbg & 2) break;
              const uint32_t ko = kg * 1024;
              const uint64_t ah = sdesc(aH + ko, G::ATOM_MN, 512), al = sdesc(aL + ko, G::ATOM_MN, 512);
              const uint64_t bh = sdesc(bH + ko, G::ATOM_MN, 512), bl = sdesc(bL + ko, G::ATOM_MN, 512);
              // small terms first (the tensor core truncates while accumulating)
              umma_tf32(d, al, bh, ID, kg > 0 ? 1u : 0u);
              umma_tf32(d, ah, bl, ID, 1u);
              umma_tf32(d, ah, bh, ID, 1u);
            }
            umma_commit(&b.bempty[stage]);  // B stage free once these MMAs are done
            umma_commit(&b.tfull[acc]);     // accumulator ready for the epilogue
          }
          umma_commit(&b.aempty[ab]);
        }
      }
    }
  } else if (warp < 6) {
    // ---------------- epilogue: TMEM -> registers -> smem box -> TMA store ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int ew = warp - 2;
    unsigned char* obox = base + G::O_OFF + ew * kT5OutBufs * 4096;
    int nstore = 0;
    for (int si = sb; si < se; ++si) {
      const TcSeg s = segs[si];
      const LayerDesc& L = t.layers[s.layer];
      if (!L.mat) continue;
      const int64_t m = L.m;
      float* grad = t.grads[s.layer];
      const bool tma_out = (m % 4) == 0 && ((reinterpret_cast<uintptr_t>(grad) & 15u) == 0);
      const CUtensorMap* gmap = t.tmaps + kTmapsPerLayer * (int64_t)s.layer + 9;
      if (tma_out && lane == 0) tmap_acquire(gmap);
      for (int64_t rb = s.row0; rb < s.row1; rb += kT5M) {
        const int64_t r0w = rb + 32 * q;  // this warp's 32 rows
        const int64_t row = r0w + lane;
        // whole box inside the segment, or clipped by the tensor's edge
        const bool box_tma = tma_out && (r0w + 32 <= s.row1 || s.row1 == L.n);
        for (int64_t c0 = 0; c0 < m; c0 += kT5N, ++it.t_it) {
          const int acc = it.t_it % nacc;
          mbar_wait(&b.tfull[acc], (it.t_it / nacc) & 1u);
          tc_fence_after();
          // two 32-column chunks per half-step: both TMEM loads in flight, one
          // wait, one proxy fence and one bulk group for the pair
          const int nh = (int)(((m - c0) < kT5N ? (m - c0) : kT5N) + 63) / 64;
#pragma unroll 1
          for (int h = 0; h < nh; ++h) {
            const int64_t ca = c0 + 64 * h, cb = ca + 32;
            const bool has_b = cb < m;  // warp-uniform
            uint32_t va[32], vb[32];
            const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * kT5N + 64 * h);
            if (!(dbg & 16)) {
              tmem_ld32_nowait(ta, va);
              if (has_b) tmem_ld32_nowait(ta + 32, vb);
              tmem_wait_ld();
            }
            if (h == nh - 1) {  // accumulator drained: the MMA may refill it now
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&b.tempty[acc]);
            }
            if (MODE == 3) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                va[i] = __float_as_uint(__uint_as_float(va[i]) * scale);
                vb[i] = __float_as_uint(__uint_as_float(vb[i]) * scale);
              }
            }
            if (r0w >= s.row1 || (dbg & 1)) continue;  // rows past the segment (layer end): nothing to store
            if (box_tma) {
              unsigned char* oa = obox + (nstore % kT5OutBufs) * 4096;
              unsigned char* ob = obox + ((nstore + 1) % kT5OutBufs) * 4096;
              if (lane == 0) bulk_wait_read<kT5OutBufs / 2 - 1>();  // the pair's boxes are free again
              __syncwarp();
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const int o = lane * 128 + ((c ^ (lane & 7)) << 4);
                *reinterpret_cast<uint4*>(oa + o) = make_uint4(va[4 * c], va[4 * c + 1], va[4 * c + 2], va[4 * c + 3]);
                if (has_b)
                  *reinterpret_cast<uint4*>(ob + o) = make_uint4(vb[4 * c], vb[4 * c + 1], vb[4 * c + 2], vb[4 * c + 3]);
              }
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(gmap, oa, (int)ca, (int)r0w);
                if (has_b) tma_store_2d(gmap, ob, (int)cb, (int)r0w);
                bulk_commit();
              }
              nstore += 2;
            } else if (row < s.row1) {
              float* g = grad + row * m;
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                if (ca + i < m) g[ca + i] = __uint_as_float(va[i]);
                if (cb + i < m) g[cb + i] = __uint_as_float(vb[i]);
              }
            }
          }
        }
      }
    }
    if (lane == 0) bulk_wait_all();
  } else {
    // ---------------- converters ----------------
    // warp 6: the row factor (A) of every row block, running ahead of the MMA
    //         by up to the two A buffers; loads batched 16 deep per lane
    // warp 7: column-factor stages (split in place / gather) and vectors
    if (warp == 6) {
      for (int si = sb; si < se; ++si) {
        const TcSeg s = segs[si];
        const LayerDesc& L = t.layers[s.layer];
        if (!L.mat) {  // vectors: unpack from the parity's buffer
          vec_unpack(t.grads[s.layer], (MODE == 2 ? t.pbuf + L.p_off : t.qbuf + L.q_off), s.row0, s.row1,
                     scale, t.nvls_fused != 0, lane);
          continue;
        }
        const int64_t n = L.n;
        const int r = L.r;
        const float* P = t.pbuf + L.p_off;  // k-major [r][n]: P_agg (mode 2) / P_orth (mode 3)
        const float sA = MODE == 2 ? scale : 1.f;
        for (int64_t rb = s.row0; rb < s.row1; rb += kT5M, ++it.a_it) {
          const int ab = it.a_it & 1;
          mbar_wait(&b.aempty[ab], ((it.a_it >> 1) & 1u) ^ 1u);
          unsigned char* aH = base + G::A_OFF + ab * 2 * G::A_BYTES;
          constexpr int kB = 16;  // loads in flight per lane
#pragma unroll 1
          for (int i0 = 0; i0 < ((dbg & 4) ? 0 : kT5M * R8); i0 += 32 * kB) {
            float x[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u) {
              const int idx = i0 + 32 * u + lane;
              const int i = idx & (kT5M - 1), k = idx >> 7;
              const int64_t row = rb + i;
              x[u] = (k < r && row < s.row1) ? __ldcg(P + (int64_t)k * n + row) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < kB; ++u) {
              const int idx = i0 + 32 * u + lane;
              const int i = idx & (kT5M - 1), k = idx >> 7;
              uint32_t hi, lo;
              split_tf32(x[u] * sA, hi, lo);
              const uint32_t o = atom_off<R8>(i, k);
              *reinterpret_cast<uint32_t*>(aH + o) = hi;
              *reinterpret_cast<uint32_t*>(aH + G::A_BYTES + o) = lo;
            }
          }
          fence_async_smem();
          mbar_arrive(&b.afull[ab]);
        }
      }
    } else {
      for (int si = sb; si < se; ++si) {
        const TcSeg s = segs[si];
        const LayerDesc& L = t.layers[s.layer];
        if (!L.mat) continue;  // vectors: the A converter warp
        const int64_t m = L.m;
        const int r = L.r;
        const bool tma = (m % 4) == 0;
        for (int64_t rb = s.row0; rb < s.row1; rb += kT5M) {
          for (int64_t c0 = 0; c0 < m; c0 += kT5N, ++it.t_it) {
            const int stage = it.t_it % NS;
            mbar_wait(&b.bfull[stage], (it.t_it / NS) & 1u);
            unsigned char* bH = base + G::B_OFF + stage * 2 * G::B_BYTES;
            if (!tma) {  // gather B (k-major source, columns c0 + cl)
              const float* src = MODE == 2 ? t.qsplit + L.qs_off : t.qbuf + L.q_off;
              for (int idx = lane; idx < kT5N * R8; idx += 32) {
                const int cl = idx & (kT5N - 1), k = idx >> 7;
                const int64_t col = c0 + cl;
                const bool ok = col < m && k < (MODE == 2 ? R8 : r);
                uint32_t hi, lo;
                if (MODE == 2) {
                  hi = ok ? __float_as_uint(src[(int64_t)k * m + col]) : 0u;
                  lo = ok ? __float_as_uint(src[((int64_t)R8 + k) * m + col]) : 0u;
                } else {
                  const float x = ok ? (t.nvls_fused ? __ldcg(src + (int64_t)k * m + col) : src[(int64_t)k * m + col]) : 0.f;
                  split_tf32(x, hi, lo);
                }
                const uint32_t o = atom_off<R8>(cl, k);
                *reinterpret_cast<uint32_t*>(bH + o) = hi;
                *reinterpret_cast<uint32_t*>(bH + G::B_BYTES + o) = lo;
              }
              fence_async_smem();
            } else if (MODE == 3) {  // TMA brought the raw aggregated Q: split in place
#pragma unroll 4
              for (int idx = lane; idx < kT5N * R8 / 4; idx += 32) {
                uint4* ph = reinterpret_cast<uint4*>(bH) + idx;
                uint4* pl = reinterpret_cast<uint4*>(bH + G::B_BYTES) + idx;
                const uint4 x = *ph;
                uint4 h, l;
                split_tf32(__uint_as_float(x.x), h.x, l.x);
                split_tf32(__uint_as_float(x.y), h.y, l.y);
                split_tf32(__uint_as_float(x.z), h.z, l.z);
                split_tf32(__uint_as_float(x.w), h.w, l.w);
                *ph = h;
                *pl = l;
              }
              fence_async_smem();
            }
            mbar_arrive(&b.bready[stage]);
          }
        }
      }
    }
  }
  if ((dbg & 64) && lane == 0) dbg_t[warp] = globaltimer_ns() - t_start;
  tc_fence_before();
  __syncthreads();
  if ((dbg & 64) && threadIdx.x == 0)
    printf("tc5 cta %d segs %d tiles %u | role ns: prod %llu mma %llu epi %llu %llu %llu %llu convA %llu convB %llu\n",
           blockIdx.x, se - sb, it.t_it, dbg_t[0], dbg_t[1], dbg_t[2], dbg_t[3], dbg_t[4], dbg_t[5], dbg_t[6], dbg_t[7]);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(kT5TmemCols)
                 : "memory");
  }
}

}  // namespace

size_t tc5_smem_bytes(int r8) {
  switch (r8) {
    case 8: return T5<8>::SMEM;
    case 16: return T5<16>::SMEM;
    case 32: return T5<32>::SMEM;
    default: return 0;
  }
}

cudaError_t launch_tc5_decode(int mode, int r8, const Tables& t, const TcSeg* segs, const int32_t* cb,
                              int ncta, float scale, cudaStream_t st) {
  if (ncta <= 0) return cudaSuccess;
  const size_t smem = tc5_smem_bytes(r8);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern));
    if (e != cudaSuccess) return e;
    // the NVLS-fused prologue barriers the whole grid (k_nvls.cuh): cooperative
    static const int dbg = std::getenv("ACP_TC5_DBG") ? std::atoi(std::getenv("ACP_TC5_DBG")) : 0;
    return launch_kernel(kern, dim3(ncta), dim3(kT5Threads), smem, st, t.nvls_fused != 0, t, segs, cb, scale, dbg);
  };
  switch (mode * 100 + r8) {
    case 208: return go(tc5_decode_kernel<2, 8>);
    case 216: return go(tc5_decode_kernel<2, 16>);
    case 232: return go(tc5_decode_kernel<2, 32>);
    case 308: return go(tc5_decode_kernel<3, 8>);
    case 316: return go(tc5_decode_kernel<3, 16>);
    case 332: return go(tc5_decode_kernel<3, 32>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace acp
