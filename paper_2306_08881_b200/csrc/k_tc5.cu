// K3 decodes for r >= 8 on the 5th-generation tensor cores (tcgen05 + TMEM):
//
//   mode 2, P-step (Alg. 2):  grad = (scale * P_agg) Q_orth^T
//   mode 3, Q-step (Alg. 2):  grad = scale * (P_orth Q_agg^T)
//
// A rank-r product per output element is a GEMM with a tiny K (= R8, the rank
// padded to 8) and a write-only output stream: 4 B of HBM per element, which
// is what bounds it. The tensor-core work is 3xTF32 (x = hi + lo, DESIGN.md
// §6b): D^T = Q_lo P_hi^T + Q_hi P_lo^T + Q_hi P_hi^T, accumulated in TMEM by
// `tcgen05.mma.kind::tf32` (M = 128 output columns, N = 128 output rows, K = 8
// per instruction, both operands MN-major in shared memory). MN-major TF32
// operands take the "128B swizzle with 32-byte atoms" layout (UMMA layout
// type 1: 4 K-rows of 128 B, 32-byte chunk c of row k stored at c ^ (k % 4));
// the plain 128B swizzle reads as zeros for 32-bit MN-major operands
// (scripts/micro/umma_tf32_test.cu). TMA writes that layout itself
// (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).
//
// Work items are 128-row blocks of a layer (and chunks of 1-D tensors),
// handed out DYNAMICALLY: one CTA per SM fetches the next item from a global
// counter (largest layers first), so no SM idles while another still holds a
// statically assigned tail. CTA warp roles:
//   warp 0      fetcher (atomic item counter -> ring of item slots in shared
//               memory) + producer: TMA boxes of the column factor (R8 x 32
//               floats, SWIZZLE_128B_ATOM_32B) into a ring of NS stages
//   warp 1      TMEM owner (4 x 128 accumulator columns) + MMA issuer (one thread)
//   warps 2-17  epilogue, four per TMEM lane quarter, 32 rows each: TMEM holds
//               D^T (lane = output column), so a 32x32b tcgen05.ld gives each
//               thread 32 rows of ONE output column and every warp store is a
//               whole 128-byte row segment, straight from registers (any m, any
//               alignment). Sixteen warps keep enough 4-byte stores in flight
//               to saturate HBM writes (scripts/micro/write_pattern.cu: four
//               warps per SM of this pattern reach 3.1 TB/s, sixteen 6.3 TB/s)
//   warp 18     A converter: the row factor (k-major P slot) of every block
//               via 4-byte cp.async (no alignment needed), the next block's
//               loads in flight while the current one is split in place into
//               hi / lo; 1-D tensors (unpack)
//   warp 19     B converter: the column factor split in place when it arrives
//               raw (mode 3) or gathered without TMA (m % 4 != 0)
// Synchronisation: mbarriers (item ring full / empty; column-factor stage full
// / ready / empty; A buffer raw / full / empty; accumulator full / empty);
// tcgen05.commit arrives on the MMA-side ones.
#include <cuda.h>

#include "k_common.cuh"
#include "k_nvls.cuh"
#include "k_umma.cuh"

namespace acp {
namespace {

constexpr int kT5M = 128;         // output rows per item / tile (MMA N, TMEM columns)
constexpr int kT5N = 128;         // output columns per tile (MMA M, TMEM lanes): 4 boxes of 32
constexpr int kT5EpiWarps = 16;   // 4 per TMEM lane quarter, one 32-row chunk each
constexpr int kT5Threads = 32 * (4 + kT5EpiWarps);
constexpr int kT5Acc = 4;         // TMEM accumulators
constexpr int kT5TmemCols = kT5Acc * kT5M;
constexpr int kT5Ring = 8;        // item slots
constexpr int kT5WarpA = 2 + kT5EpiWarps, kT5WarpB = kT5WarpA + 1;
// consumers of an item slot: MMA thread, epilogue warps, A and B converters
constexpr int kT5SlotReaders = 1 + kT5EpiWarps + 2;

template <int R8>
struct T5 {
  static constexpr int KG = R8 / 8;              // MMA K-steps (K = 8)
  static constexpr int ATOM_MN = R8 * 128;       // bytes between 32-wide MN blocks (LBO)
  static constexpr int A_BYTES = kT5M * R8 * 4;  // one operand array (hi or lo)
  static constexpr int B_BYTES = kT5N * R8 * 4;
  static constexpr int NS = R8 >= 32 ? 4 : 6;    // column-factor stages
  static constexpr int A_OFF = 0;                                  // [2 buf][hi, lo]
  static constexpr int B_OFF = A_OFF + 4 * A_BYTES;                // [NS][hi, lo]
  static constexpr int BAR_OFF = B_OFF + NS * 2 * B_BYTES;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;                // + barriers / ring + align slack
};

// byte offset of element (mn, k) of an MN-major operand in the
// [mn/32][k][32] layout with 128B / 32-byte-atom swizzle (32-byte chunk
// XOR k % 4; K-rows of 128 B, groups of 4 rows = 512 B)
template <int R8>
__device__ __forceinline__ uint32_t atom_off(int mn, int k) {
  return (uint32_t)((mn >> 5) * T5<R8>::ATOM_MN + (k >> 2) * 512 + (k & 3) * 128 +
                    ((((mn & 31) >> 3) ^ (k & 3)) << 5) + (mn & 7) * 4);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return umma_sdesc(saddr, lbo, sbo, kLayoutSw128Atom32);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) { return umma_idesc_tf32(M, N, 1, 1); }

// grad[i] = scale * slot[i], i in [i0, i1), by one warp: 8 loads in flight
// per lane (the slot is 16-byte aligned; float4 when the gradient is too)
__device__ __forceinline__ void vec_unpack(float* grad, const float* slot, int64_t i0, int64_t i1, float scale,
                                           bool fused, int lane) {
  constexpr int kB = 8;
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

// in-place 3xTF32 split of `bytes` of raw fp32 at h: h <- hi, l <- lo (one warp)
__device__ __forceinline__ void split_inplace(unsigned char* h, unsigned char* l, int bytes, float s, int lane) {
#pragma unroll 4
  for (int idx = lane; idx < bytes / 16; idx += 32) {
    uint4* ph = reinterpret_cast<uint4*>(h) + idx;
    uint4* pl = reinterpret_cast<uint4*>(l) + idx;
    const uint4 x = *ph;
    uint4 a, c;
    split_tf32(__uint_as_float(x.x) * s, a.x, c.x);
    split_tf32(__uint_as_float(x.y) * s, a.y, c.y);
    split_tf32(__uint_as_float(x.z) * s, a.z, c.z);
    split_tf32(__uint_as_float(x.w) * s, a.w, c.w);
    *ph = a;
    *pl = c;
  }
}

struct T5Bars {
  uint64_t* sfull;   // [kT5Ring] item slot written (fetcher)
  uint64_t* sempty;  // [kT5Ring] item slot consumed (kT5SlotReaders arrivals)
  uint64_t* bfull;   // [NS] producer (TMA complete_tx or plain arrive)
  uint64_t* bready;  // [NS] B converter warp (32 arrivals)
  uint64_t* bempty;  // [NS] MMA commit
  uint64_t* araw;    // [2] A converter's raw cp.async loads (32 noinc arrivals)
  uint64_t* afull;   // [2] A converter warp (32 arrivals)
  uint64_t* aempty;  // [2] MMA commit
  uint64_t* tfull;   // [kT5Acc] MMA commit
  uint64_t* tempty;  // [kT5Acc] epilogue warps (kT5EpiWarps arrivals)
  int32_t* ring;     // [kT5Ring] item index (-1: no more work)
  uint32_t* tmem;    // TMEM base written by tcgen05.alloc
};

// Consumer view of the item ring: item number c (0, 1, ...) of this CTA.
__device__ __forceinline__ int ring_read(const T5Bars& b, uint32_t c) { return acp::ring_read(b.sfull, b.ring, kT5Ring, c); }

template <int MODE, int R8>
__global__ void __launch_bounds__(kT5Threads, 1)
tc5_decode_kernel(Tables t, const TcSeg* __restrict__ items, int nitems, int32_t* __restrict__ sched,
                  float scale) {
  using G = T5<R8>;
  constexpr int NS = G::NS;
  extern __shared__ __align__(1024) unsigned char t5_raw[];
  unsigned char* base = t5_raw + ((1024u - (s32(t5_raw) & 1023u)) & 1023u);
  const uint32_t sbase = s32(base);
  T5Bars b;
  {
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + G::BAR_OFF);
    b.sfull = bars;
    b.sempty = b.sfull + kT5Ring;
    b.bfull = b.sempty + kT5Ring;
    b.bready = b.bfull + NS;
    b.bempty = b.bready + NS;
    b.araw = b.bempty + NS;
    b.afull = b.araw + 2;
    b.aempty = b.afull + 2;
    b.tfull = b.aempty + 2;
    b.tempty = b.tfull + kT5Acc;
    b.ring = reinterpret_cast<int32_t*>(b.tempty + kT5Acc);
    b.tmem = reinterpret_cast<uint32_t*>(b.ring + kT5Ring);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kT5Ring; ++i) {
      mbar_init(&b.sfull[i], 1);
      mbar_init(&b.sempty[i], kT5SlotReaders);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&b.bfull[i], 1);
      mbar_init(&b.bready[i], 32);
      mbar_init(&b.bempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b.araw[i], 32);
      mbar_init(&b.afull[i], 32);
      mbar_init(&b.aempty[i], 1);
    }
    for (int i = 0; i < kT5Acc; ++i) {
      mbar_init(&b.tfull[i], 1);
      mbar_init(&b.tempty[i], kT5EpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    tmem_alloc(b.tmem, kT5TmemCols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *b.tmem;
  // NVLS (NEXT-3): sum this parity's fused buffer over the ranks first
  if (t.nvls_fused) nvls_fused_reduce(t, MODE == 2 ? 0 : 1);

  if (warp == 0) {
    // ---------------- fetcher + producer ----------------
    if (lane == 0) {
      uint32_t f = 0;
      auto fetch = [&]() -> int {
        const int slot = f % kT5Ring;
        mbar_wait(&b.sempty[slot], ((f / kT5Ring) & 1u) ^ 1u);
        int it = atomicAdd(sched, 1);
        if (it >= nitems) it = -1;
        *reinterpret_cast<volatile int32_t*>(b.ring + slot) = it;
        mbar_arrive(&b.sfull[slot]);  // release: the slot write is visible to its waiters
        ++f;
        return it;
      };
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      uint32_t t_it = 0;
      int cur = fetch();
      int nxt = cur >= 0 ? fetch() : -1;  // one item ahead (the A converter prefetches it)
      while (cur >= 0) {
        const TcSeg s = items[cur];
        const LayerDesc& L = t.layers[s.layer];
        if (L.mat) {
          const int64_t m = L.m;
          const bool tma = (m % 4) == 0;
          const CUtensorMap* maps = t.tmaps + kTmapsPerLayer * (int64_t)s.layer;
          if (tma) {
            tmap_acquire(maps + (MODE == 2 ? 10 : 12));
            if (MODE == 2) tmap_acquire(maps + 11);
          }
          for (int64_t c0 = 0; c0 < m; c0 += kT5N, ++t_it) {
            const int stage = t_it % NS;
            mbar_wait(&b.bempty[stage], ((t_it / NS) & 1u) ^ 1u);
            unsigned char* dB = base + G::B_OFF + stage * 2 * G::B_BYTES;
            if (tma) {
              const int nbox = (int)((m - c0 + 31) / 32) < 4 ? (int)((m - c0 + 31) / 32) : 4;
              const uint32_t box = R8 * 32 * 4;
              mbar_arrive_tx(&b.bfull[stage], (MODE == 2 ? 2u : 1u) * box * (uint32_t)nbox);
              for (int nb = 0; nb < nbox; ++nb) {
                if (MODE == 2) {
                  tma_load_2d(dB + nb * G::ATOM_MN, maps + 10, (int)c0 + 32 * nb, 0, &b.bfull[stage], pol);
                  tma_load_2d(dB + G::B_BYTES + nb * G::ATOM_MN, maps + 11, (int)c0 + 32 * nb, 0,
                              &b.bfull[stage], pol);
                } else {
                  tma_load_2d(dB + nb * G::ATOM_MN, maps + 12, (int)c0 + 32 * nb, 0, &b.bfull[stage], pol);
                }
              }
            } else {
              mbar_arrive(&b.bfull[stage]);  // the B converter gathers it
            }
          }
        }
        cur = nxt;
        nxt = cur >= 0 ? fetch() : -1;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t ID = idesc_tf32(kT5N, kT5M);
      uint32_t a_it = 0, t_it = 0;
      for (uint32_t c = 0;; ++c) {
        const int cur = ring_read(b, c);
        if (cur < 0) break;
        const TcSeg s = items[cur];
        const LayerDesc& L = t.layers[s.layer];
        if (L.mat) {
          const int64_t m = L.m;
          const int ab = a_it & 1;
          mbar_wait(&b.afull[ab], (a_it >> 1) & 1u);
          const uint32_t aH = sbase + G::A_OFF + ab * 2 * G::A_BYTES, aL = aH + G::A_BYTES;
          for (int64_t c0 = 0; c0 < m; c0 += kT5N, ++t_it) {
            const int stage = t_it % NS;
            const int acc = t_it % kT5Acc;
            mbar_wait(&b.bready[stage], (t_it / NS) & 1u);
            mbar_wait(&b.tempty[acc], ((t_it / kT5Acc) & 1u) ^ 1u);
            tc_fence_after();
            const uint32_t bH = sbase + G::B_OFF + stage * 2 * G::B_BYTES, bL = bH + G::B_BYTES;
            const uint32_t d = tbase + (uint32_t)(acc * kT5M);
#pragma unroll
            for (int kg = 0; kg < G::KG; ++kg) {
              const uint32_t ko = kg * 1024;
              const uint64_t ah = sdesc(aH + ko, G::ATOM_MN, 512), al = sdesc(aL + ko, G::ATOM_MN, 512);
              const uint64_t bh = sdesc(bH + ko, G::ATOM_MN, 512), bl = sdesc(bL + ko, G::ATOM_MN, 512);
              // D^T = Q_panel P_block^T: the column factor is the M side (TMEM
              // lane = output column), the row factor the N side (TMEM column
              // = output row). Small terms first (the tensor core truncates
              // while accumulating).
              umma_tf32(d, bh, al, ID, kg > 0 ? 1u : 0u);
              umma_tf32(d, bl, ah, ID, 1u);
              umma_tf32(d, bh, ah, ID, 1u);
            }
            umma_commit(&b.bempty[stage]);  // B stage free once these MMAs are done
            umma_commit(&b.tfull[acc]);     // accumulator ready for the epilogue
          }
          umma_commit(&b.aempty[ab]);
          ++a_it;
        }
        mbar_arrive(&b.sempty[c % kT5Ring]);
      }
    }
  } else if (warp < kT5WarpA) {
    // ---------------- epilogue: TMEM -> registers -> coalesced stores ----------------
    const int q = warp & 3;           // TMEM lane quarter this warp may access (32 output columns)
    const int jc = (warp - 2) >> 2;   // which 32 of the block's 128 rows
    uint32_t t_it = 0;
    for (uint32_t c = 0;; ++c) {
      const int cur = ring_read(b, c);
      if (cur < 0) break;
      const TcSeg s = items[cur];
      const LayerDesc& L = t.layers[s.layer];
      if (L.mat) {
        const int64_t m = L.m;
        float* grad = t.grads[s.layer];
        const int nrow = (int)(s.row1 - s.row0);
        const int na = nrow - 32 * jc < 32 ? nrow - 32 * jc : 32;  // this warp's rows (<= 0: none)
        for (int64_t c0 = 0; c0 < m; c0 += kT5N, ++t_it) {
          const int acc = t_it % kT5Acc;
          mbar_wait(&b.tfull[acc], (t_it / kT5Acc) & 1u);
          tc_fence_after();
          uint32_t v[32];
          if (na > 0) {
            tmem_ld_x32(tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * kT5M + 32 * jc), v);
            tmem_wait_ld();
          }
          // this warp's part of the accumulator is drained: the MMA may refill
          // it once every epilogue warp has arrived
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&b.tempty[acc]);
          const int64_t col = c0 + 32 * q + lane;
          if (na <= 0 || col >= m) continue;
          float* g = grad + (s.row0 + 32 * jc) * m + col;
          const float sc = MODE == 3 ? scale : 1.f;
          if (na == 32) {
#pragma unroll
            for (int i = 0; i < 32; ++i) __stcs(g + (int64_t)i * m, __uint_as_float(v[i]) * sc);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < na) __stcs(g + (int64_t)i * m, __uint_as_float(v[i]) * sc);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&b.sempty[c % kT5Ring]);
    }
  } else if (warp == kT5WarpA) {
    // ---------------- A converter (+ 1-D tensors) ----------------
    // the raw P rows of block i+1 are in flight (4-byte cp.async into the hi
    // array's atom positions, zero-filled beyond r / the block) while block i
    // is split in place into hi / lo
    auto issue = [&](const TcSeg& s, int ab) {
      const LayerDesc& L = t.layers[s.layer];
      const int64_t n = L.n;
      const int r = L.r;
      const float* P = t.pbuf + L.p_off;  // k-major [r][n]: P_agg (mode 2) / P_orth (mode 3)
      unsigned char* aH = base + G::A_OFF + ab * 2 * G::A_BYTES;
#pragma unroll 8
      for (int idx = lane; idx < kT5M * R8; idx += 32) {
        const int i = idx & (kT5M - 1), k = idx >> 7;
        const int64_t row = s.row0 + i;
        const bool ok = k < r && row < s.row1;
        cp_async4(reinterpret_cast<float*>(aH + atom_off<R8>(i, k)), ok ? P + (int64_t)k * n + row : P,
                  ok ? 4u : 0u);
      }
      cp_async_arrive(&b.araw[ab]);
    };
    const float sA = MODE == 2 ? scale : 1.f;
    uint32_t a_it = 0;  // matrix blocks issued so far
    uint32_t c = 0;
    int cur = ring_read(b, 0);
    bool cur_issued = false;
    while (cur >= 0) {
      const TcSeg s = items[cur];
      const LayerDesc& L = t.layers[s.layer];
      if (!L.mat) {
        vec_unpack(t.grads[s.layer], (MODE == 2 ? t.pbuf + L.p_off : t.qbuf + L.q_off), s.row0, s.row1, scale,
                   t.nvls_fused != 0, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&b.sempty[c % kT5Ring]);
        cur = ring_read(b, ++c);
        cur_issued = false;
        continue;
      }
      const uint32_t my = cur_issued ? a_it - 1 : a_it;  // this block's A sequence number
      if (!cur_issued) {
        mbar_wait(&b.aempty[my & 1], ((my >> 1) & 1u) ^ 1u);
        issue(s, my & 1);
        ++a_it;
      }
      // prefetch: the next matrix block's raw loads before this block's split
      const int nxt = ring_read(b, c + 1);
      bool nxt_issued = false;
      if (nxt >= 0 && t.layers[items[nxt].layer].mat) {
        mbar_wait(&b.aempty[a_it & 1], ((a_it >> 1) & 1u) ^ 1u);
        issue(items[nxt], a_it & 1);
        ++a_it;
        nxt_issued = true;
      }
      const int ab = my & 1;
      mbar_wait(&b.araw[ab], (my >> 1) & 1u);
      unsigned char* aH = base + G::A_OFF + ab * 2 * G::A_BYTES;
      split_inplace(aH, aH + G::A_BYTES, G::A_BYTES, sA, lane);
      fence_async_smem();
      mbar_arrive(&b.afull[ab]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&b.sempty[c % kT5Ring]);
      ++c;
      cur = nxt;
      cur_issued = nxt_issued;
    }
  } else {
    // ---------------- B converter ----------------
    uint32_t t_it = 0;
    for (uint32_t c = 0;; ++c) {
      const int cur = ring_read(b, c);
      if (cur < 0) break;
      const TcSeg s = items[cur];
      const LayerDesc& L = t.layers[s.layer];
      if (L.mat) {
        const int64_t m = L.m;
        const int r = L.r;
        const bool tma = (m % 4) == 0;
        for (int64_t c0 = 0; c0 < m; c0 += kT5N, ++t_it) {
          const int stage = t_it % NS;
          mbar_wait(&b.bfull[stage], (t_it / NS) & 1u);
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
                const float x =
                    ok ? (t.nvls_fused ? __ldcg(src + (int64_t)k * m + col) : src[(int64_t)k * m + col]) : 0.f;
                split_tf32(x, hi, lo);
              }
              const uint32_t o = atom_off<R8>(cl, k);
              *reinterpret_cast<uint32_t*>(bH + o) = hi;
              *reinterpret_cast<uint32_t*>(bH + G::B_BYTES + o) = lo;
            }
            fence_async_smem();
          } else if (MODE == 3) {  // TMA brought the raw aggregated Q: split in place
            split_inplace(bH, bH + G::B_BYTES, G::B_BYTES, 1.f, lane);
            fence_async_smem();
          }
          mbar_arrive(&b.bready[stage]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&b.sempty[c % kT5Ring]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, kT5TmemCols);
  }
  sched_rearm(sched);
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

cudaError_t launch_tc5_decode(int mode, int r8, const Tables& t, const TcSeg* items, int nitems, int32_t* sched,
                              int ncta, float scale, cudaStream_t st) {
  if (ncta <= 0 || nitems <= 0) return cudaSuccess;
  const size_t smem = tc5_smem_bytes(r8);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern));
    if (e != cudaSuccess) return e;
    // the NVLS-fused prologue barriers the whole grid (k_nvls.cuh): cooperative
    return launch_kernel(kern, dim3(ncta), dim3(kT5Threads), smem, st, t.nvls_fused != 0, t, items, nitems, sched,
                         scale);
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
