// K1, P-step, on the 5th-generation tensor cores (tcgen05 + TMEM): the same
// double-deferred step as k_tc.cu's mode 0 (Alg. 2
// with the Q-step's residual applied on the fly):
//
//   x = M + S - P_orth Q_loc^T ;  S <- x ;  P_loc = x Q_orth   (-> P slot, P_loc split)
//
// Per 128-row block (a dynamically fetched work item) and 32-column tile:
//   * TMA: the M and S tiles (32 x 128 boxes, SWIZZLE_128B = the K-major UMMA
//     atom), the tile's Q_orth panel (K-major, 128B swizzle) and Q_loc panel
//     (MN-major, 128B swizzle with 32-byte atoms), and once per block the
//     P_orth rows (K-major, swizzle = row bytes: 32 / 64 / 128 B);
//   * MMA 1 (tcgen05, 3xTF32): corr = P_orth Q_loc^T -> TMEM (128 x 32);
//   * converter warps (thread = row): x = M + S - corr from shared memory and
//     TMEM; x goes back into the S tile (TMA-stored to global by the storer
//     warp) and its hi / lo split into the M tile / a third tile -- which is
//     exactly the K-major A operand layout of
//   * MMA 2: P_part = x Q_orth (128 x R8) into one of two TMEM partials; the
//     converters add every tile's partial to fp32 registers (round to nearest:
//     the tensor core truncates while accumulating, so chains stay one tile
//     long, 12 MMAs) and write P_loc at the end of the block.
// 12 B / element of HBM (read M, S; write S), like the mma.sync kernel; the
// rank-r products are tensor-core work. CTA roles: warp 0 fetcher + TMA
// producer, warp 1 TMEM owner + MMA issuer, warps 2-9 converters (two per
// TMEM lane quarter = warp % 4, 16 columns each), warp 10 S-tile TMA storer +
// 1-D tensors (pack).
#include <cuda.h>

#include "k_common.cuh"
#include "k_umma.cuh"

namespace acp {
namespace {

constexpr int kK1M = 128;         // rows per block (MMA M, TMEM lanes)
constexpr int kK1N = 32;          // columns per tile (one 128-byte box)
constexpr int kK1Conv = 8;        // converter warps: 2 per TMEM lane quarter, 16 columns each
constexpr int kK1Threads = 32 * (3 + kK1Conv);  // + producer, MMA, storer
constexpr int kK1WarpStore = 2 + kK1Conv;
constexpr int kK1Ring = 8;        // item slots
constexpr int kK1SlotReaders = 1 + kK1Conv + 1;  // MMA thread, converter warps, storer warp
constexpr int kK1TmemCols = 128;  // corr 2 x 32 at [0, 64); P partials 2 x PN at [64, 64 + 2 PN)

template <int R8>
struct K1 {
  static constexpr int KG = R8 / 8;
  static constexpr int TILE = kK1M * kK1N * 4;        // 16 KB: 128 rows x 32 columns
  static constexpr int FBOX = R8 * kK1N * 4;          // factor box: R8 rows x 32 columns
  static constexpr int STAGE = 3 * TILE + 4 * FBOX;   // M (-> x_hi), S (-> x), x_lo, Qo hi/lo, Ql hi/lo
  static constexpr int NS = R8 >= 16 ? 3 : 4;
  static constexpr int PO = kK1M * R8 * 4;            // P_orth rows of a block (hi or lo)
  static constexpr int NPO = R8 >= 32 ? 1 : 2;        // P_orth buffers
  static constexpr int PO_OFF = NS * STAGE;           // [NPO buffers][hi, lo]
  static constexpr int BAR_OFF = PO_OFF + NPO * 2 * PO;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;
  static constexpr uint32_t PO_LAYOUT = R8 == 8 ? kLayoutSw32 : (R8 == 16 ? kLayoutSw64 : kLayoutSw128);
  // MMA 2 width: N >= 16 for M = 128 (at R8 = 8 the extra 8 columns read the
  // next factor box and are ignored)
  static constexpr int PN = R8 < 16 ? 16 : R8;
  // stage sub-buffers (byte offsets inside a stage)
  static constexpr int S_M = 0, S_S = TILE, S_XL = 2 * TILE, S_QOH = 3 * TILE, S_QOL = S_QOH + FBOX,
                       S_QLH = S_QOL + FBOX, S_QLL = S_QLH + FBOX;
};

struct K1Bars {
  uint64_t *sfull, *sempty;    // [kK1Ring] item ring
  uint64_t *full, *xready;     // [NS] TMA landed / converters wrote x (kK1Conv arrivals)
  uint64_t *pdone, *sfree;     // [NS] MMA 2 read the stage / storer's TMA store read S
  uint64_t *cfull, *cempty;    // [2] corr accumulator (MMA commit / kK1Conv arrivals)
  uint64_t *qfull, *qempty;    // [2] P partial (MMA commit / 4 arrivals: the h = 0 converters)
  uint64_t *pofull, *poempty;  // [2] P_orth rows (TMA / MMA commit)
  int32_t* ring;
  uint32_t* tmem;
};

template <int R8>
__global__ void __launch_bounds__(kK1Threads, 1)
tc5_k1p_kernel(Tables t, const TcSeg* __restrict__ items, int nitems, int32_t* __restrict__ sched) {
  using G = K1<R8>;
  constexpr int NS = G::NS;
  extern __shared__ __align__(1024) unsigned char k1_raw[];
  unsigned char* base = k1_raw + ((1024u - (s32(k1_raw) & 1023u)) & 1023u);
  const uint32_t sbase = s32(base);
  K1Bars b;
  {
    uint64_t* p = reinterpret_cast<uint64_t*>(base + G::BAR_OFF);
    b.sfull = p; p += kK1Ring;
    b.sempty = p; p += kK1Ring;
    b.full = p; p += NS;
    b.xready = p; p += NS;
    b.pdone = p; p += NS;
    b.sfree = p; p += NS;
    b.cfull = p; p += 2;
    b.cempty = p; p += 2;
    b.qfull = p; p += 2;
    b.qempty = p; p += 2;
    b.pofull = p; p += 2;
    b.poempty = p; p += 2;
    b.ring = reinterpret_cast<int32_t*>(p);
    b.tmem = reinterpret_cast<uint32_t*>(b.ring + kK1Ring);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kK1Ring; ++i) {
      mbar_init(&b.sfull[i], 1);
      mbar_init(&b.sempty[i], kK1SlotReaders);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&b.full[i], 1);
      mbar_init(&b.xready[i], kK1Conv);
      mbar_init(&b.pdone[i], 1);
      mbar_init(&b.sfree[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b.cfull[i], 1);
      mbar_init(&b.cempty[i], kK1Conv);
      mbar_init(&b.qfull[i], 1);
      mbar_init(&b.qempty[i], 4);
      mbar_init(&b.pofull[i], 1);
      mbar_init(&b.poempty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(b.tmem, kK1TmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *b.tmem;
  auto stage_ptr = [&](uint32_t tt) { return base + (tt % NS) * G::STAGE; };

  if (warp == 0) {
    // ---------------- fetcher + TMA producer ----------------
    if (lane == 0) {
      uint32_t f = 0;
      auto fetch = [&]() -> int {
        const int slot = f % kK1Ring;
        mbar_wait(&b.sempty[slot], ((f / kK1Ring) & 1u) ^ 1u);
        int it = atomicAdd(sched, 1);
        if (it >= nitems) it = -1;
        *reinterpret_cast<volatile int32_t*>(b.ring + slot) = it;
        mbar_arrive(&b.sfull[slot]);
        ++f;
        return it;
      };
      const uint64_t pol_stream = policy_evict_first();
      uint64_t pol_keep;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
      uint32_t t_it = 0, b_it = 0;
      bool c_first = true;
      int cur = fetch();
      int nxt = cur >= 0 ? fetch() : -1;
      while (cur >= 0) {
        const TcSeg s = items[cur];
        const LayerDesc& L = t.layers[s.layer];
        if (L.mat) {
          const CUtensorMap* maps = t.tmaps + kTmapsPerLayer * (int64_t)s.layer;
          tmap_acquire(maps + 0);
          tmap_acquire(maps + 1);
          tmap_acquire(maps + 2);
          tmap_acquire(maps + 3);
          tmap_acquire(maps + 13);
          tmap_acquire(maps + 14);
          tmap_acquire(maps + 15);
          tmap_acquire(maps + 16);
          const int pb = b_it % G::NPO;
          mbar_wait(&b.poempty[pb], ((b_it / G::NPO) & 1u) ^ 1u);
          unsigned char* po = base + G::PO_OFF + pb * 2 * G::PO;
          mbar_arrive_tx(&b.pofull[pb], 2u * G::PO);
          tma_load_2d(po, maps + 15, 0, (int)s.row0, &b.pofull[pb], pol_keep);
          tma_load_2d(po + G::PO, maps + 16, 0, (int)s.row0, &b.pofull[pb], pol_keep);
          ++b_it;
          // L2 prefetch of the M / S tiles t.tc5_pf tiles ahead (this block's
          // later tiles, then the next item's first ones)
          const int64_t ntile = (L.m + kK1N - 1) / kK1N;
          const TcSeg sn = items[nxt >= 0 ? nxt : cur];
          const LayerDesc& Ln = t.layers[sn.layer];
          const CUtensorMap* mapsn = t.tmaps + kTmapsPerLayer * (int64_t)sn.layer;
          const bool pf_next = nxt >= 0 && Ln.mat;
          if (pf_next) {
            tmap_acquire(mapsn + 0);
            tmap_acquire(mapsn + 1);
          }
          auto prefetch = [&](int64_t j) {  // tile j of this block (j >= ntile: of the next one)
            if (j < ntile) {
              tma_prefetch_2d(maps + 0, (int)(j * kK1N), (int)s.row0);
              tma_prefetch_2d(maps + 1, (int)(j * kK1N), (int)s.row0);
            } else if (pf_next && (j - ntile) * kK1N < Ln.m) {
              tma_prefetch_2d(mapsn + 0, (int)((j - ntile) * kK1N), (int)sn.row0);
              tma_prefetch_2d(mapsn + 1, (int)((j - ntile) * kK1N), (int)sn.row0);
            }
          };
          const int kPF = t.tc5_pf;
          if (c_first) {  // the CTA's first block: warm the first kPF tiles too
            for (int64_t j = 0; j < kPF; ++j) prefetch(j);
            c_first = false;
          }
          for (int64_t c0 = 0; c0 < L.m; c0 += kK1N, ++t_it) {
            if (kPF > 0) prefetch(c0 / kK1N + kPF);
            const int st = t_it % NS;
            const uint32_t ph = (t_it / NS) & 1u;
            mbar_wait(&b.pdone[st], ph ^ 1u);
            mbar_wait(&b.sfree[st], ph ^ 1u);
            unsigned char* sp = stage_ptr(t_it);
            mbar_arrive_tx(&b.full[st], (uint32_t)(2 * G::TILE + 4 * G::FBOX));
            tma_load_2d(sp + G::S_M, maps + 0, (int)c0, (int)s.row0, &b.full[st], pol_stream);
            tma_load_2d(sp + G::S_S, maps + 1, (int)c0, (int)s.row0, &b.full[st], pol_stream);
            tma_load_2d(sp + G::S_QOH, maps + 2, (int)c0, 0, &b.full[st], pol_keep);
            tma_load_2d(sp + G::S_QOL, maps + 3, (int)c0, 0, &b.full[st], pol_keep);
            tma_load_2d(sp + G::S_QLH, maps + 13, (int)c0, 0, &b.full[st], pol_keep);
            tma_load_2d(sp + G::S_QLL, maps + 14, (int)c0, 0, &b.full[st], pol_keep);
          }
        }
        cur = nxt;
        nxt = cur >= 0 ? fetch() : -1;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t IDC = umma_idesc_tf32(kK1M, kK1N, 0, 1);  // P_orth K-major, Q_loc MN-major
      constexpr uint32_t IDP = umma_idesc_tf32(kK1M, G::PN, 0, 0);  // x K-major, Q_orth K-major
      uint32_t t_it = 0, b_it = 0;
      for (uint32_t c = 0;; ++c) {
        const int cur = ring_read(b.sfull, b.ring, kK1Ring, c);
        if (cur < 0) break;
        const TcSeg s = items[cur];
        const LayerDesc& L = t.layers[s.layer];
        if (L.mat) {
          const uint32_t ntiles = (uint32_t)((L.m + kK1N - 1) / kK1N);
          const int pb = b_it % G::NPO;
          mbar_wait(&b.pofull[pb], (b_it / G::NPO) & 1u);
          const uint32_t poh = sbase + G::PO_OFF + pb * 2 * G::PO, pol = poh + G::PO;
          auto corr = [&](uint32_t tt) {
            const int st = tt % NS, ca = tt & 1;
            mbar_wait(&b.full[st], (tt / NS) & 1u);
            mbar_wait(&b.cempty[ca], ((tt >> 1) & 1u) ^ 1u);
            tc_fence_after();
            const uint32_t sp = sbase + (tt % NS) * G::STAGE;
            const uint32_t d = tbase + (uint32_t)(ca * kK1N);
#pragma unroll
            for (int kg = 0; kg < G::KG; ++kg) {
              const uint64_t ah = umma_sdesc(poh + 32 * kg, 16, 32 * R8, G::PO_LAYOUT);
              const uint64_t al = umma_sdesc(pol + 32 * kg, 16, 32 * R8, G::PO_LAYOUT);
              const uint64_t bh = umma_sdesc(sp + G::S_QLH + 1024 * kg, R8 * 128, 512, kLayoutSw128Atom32);
              const uint64_t bl = umma_sdesc(sp + G::S_QLL + 1024 * kg, R8 * 128, 512, kLayoutSw128Atom32);
              umma_tf32(d, al, bh, IDC, kg > 0 ? 1u : 0u);
              umma_tf32(d, ah, bl, IDC, 1u);
              umma_tf32(d, ah, bh, IDC, 1u);
            }
            umma_commit(&b.cfull[ca]);
          };
          corr(t_it);
          for (uint32_t j = 0; j < ntiles; ++j) {
            const uint32_t tt = t_it + j;
            if (j + 1 < ntiles) corr(tt + 1);
            else umma_commit(&b.poempty[pb]);  // every corr of the block issued: P_orth buffer free when done
            const int st = tt % NS, qa = tt & 1;
            mbar_wait(&b.xready[st], (tt / NS) & 1u);
            mbar_wait(&b.qempty[qa], ((tt >> 1) & 1u) ^ 1u);
            tc_fence_after();
            const uint32_t sp = sbase + (tt % NS) * G::STAGE;
            const uint32_t d = tbase + 64u + (uint32_t)(qa * G::PN);
#pragma unroll
            for (int kk = 0; kk < kK1N / 8; ++kk) {
              const uint64_t ah = umma_sdesc(sp + G::S_M + 32 * kk, 16, 1024, kLayoutSw128);   // x_hi
              const uint64_t al = umma_sdesc(sp + G::S_XL + 32 * kk, 16, 1024, kLayoutSw128);  // x_lo
              const uint64_t bh = umma_sdesc(sp + G::S_QOH + 32 * kk, 16, 1024, kLayoutSw128);
              const uint64_t bl = umma_sdesc(sp + G::S_QOL + 32 * kk, 16, 1024, kLayoutSw128);
              umma_tf32(d, al, bh, IDP, kk > 0 ? 1u : 0u);
              umma_tf32(d, ah, bl, IDP, 1u);
              umma_tf32(d, ah, bh, IDP, 1u);
            }
            umma_commit(&b.qfull[qa]);
            umma_commit(&b.pdone[st]);
          }
          t_it += ntiles;
          ++b_it;
        }
        mbar_arrive(&b.sempty[c % kK1Ring]);
      }
    }
  } else if (warp < kK1WarpStore) {
    // ---------------- converters: x = M + S - corr; P_loc accumulation ----------------
    // two warps per TMEM lane quarter split the tile's 32 columns; the h = 0
    // warp of a quarter also accumulates its rows' P_loc
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    const int i = 32 * q + lane;  // row within the block (= TMEM lane)
    uint32_t t_it = 0;
    for (uint32_t c = 0;; ++c) {
      const int cur = ring_read(b.sfull, b.ring, kK1Ring, c);
      if (cur < 0) break;
      const TcSeg s = items[cur];
      const LayerDesc& L = t.layers[s.layer];
      if (L.mat) {
        const uint32_t ntiles = (uint32_t)((L.m + kK1N - 1) / kK1N);
        float acc[R8];
#pragma unroll
        for (int k = 0; k < R8; ++k) acc[k] = 0.f;
        auto add_partial = [&](uint32_t tt) {
          const int qa = tt & 1;
          mbar_wait(&b.qfull[qa], (tt >> 1) & 1u);
          tc_fence_after();
          uint32_t pv[R8];
          tmem_ld<R8>(tbase + ((uint32_t)(32 * q) << 16) + 64u + (uint32_t)(qa * G::PN), pv);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&b.qempty[qa]);
#pragma unroll
          for (int k = 0; k < R8; ++k) acc[k] += __uint_as_float(pv[k]);
        };
        const int sw = i & 7;
        for (uint32_t j = 0; j < ntiles; ++j) {
          const uint32_t tt = t_it + j;
          const int st = tt % NS, ca = tt & 1;
          mbar_wait(&b.full[st], (tt / NS) & 1u);
          mbar_wait(&b.cfull[ca], (tt >> 1) & 1u);
          tc_fence_after();
          uint32_t cv[16];
          tmem_ld_x16(tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(ca * kK1N + 16 * h), cv);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&b.cempty[ca]);
          unsigned char* sp = stage_ptr(tt);
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int ch = 4 * h + cc;
            const int off = i * 128 + ((ch ^ sw) << 4);
            const float4 mv = *reinterpret_cast<const float4*>(sp + G::S_M + off);
            const float4 sv = *reinterpret_cast<const float4*>(sp + G::S_S + off);
            float4 x;
            x.x = mv.x + sv.x - __uint_as_float(cv[4 * cc + 0]);
            x.y = mv.y + sv.y - __uint_as_float(cv[4 * cc + 1]);
            x.z = mv.z + sv.z - __uint_as_float(cv[4 * cc + 2]);
            x.w = mv.w + sv.w - __uint_as_float(cv[4 * cc + 3]);
            *reinterpret_cast<float4*>(sp + G::S_S + off) = x;
            uint4 h, l;
            split_tf32(x.x, h.x, l.x);
            split_tf32(x.y, h.y, l.y);
            split_tf32(x.z, h.z, l.z);
            split_tf32(x.w, h.w, l.w);
            *reinterpret_cast<uint4*>(sp + G::S_M + off) = h;
            *reinterpret_cast<uint4*>(sp + G::S_XL + off) = l;
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&b.xready[st]);
          if (h == 0 && j > 0) add_partial(tt - 1);
        }
        if (h == 0) add_partial(t_it + ntiles - 1);
        const int64_t row = s.row0 + i;
        if (h == 0 && row < s.row1) {
          const int64_t n = L.n;
          float* Pw = t.pbuf + L.p_off;       // P slot, k-major [r][n]
          float* Pl = t.plsplit + L.ps_off;   // P_loc split [2][n][R8]
#pragma unroll
          for (int k = 0; k < R8; ++k) {
            if (k < L.r) Pw[(int64_t)k * n + row] = acc[k];
            uint32_t h, l;
            split_tf32(acc[k], h, l);
            Pl[row * R8 + k] = __uint_as_float(h);
            Pl[(n + row) * R8 + k] = __uint_as_float(l);
          }
        }
        t_it += ntiles;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&b.sempty[c % kK1Ring]);
    }
  } else {
    // ---------------- storer: S tiles back to global (TMA) + 1-D tensors ----------------
    uint32_t t_it = 0;
    int pend = -1;  // stage whose store is issued but not yet released
    for (uint32_t c = 0;; ++c) {
      const int cur = ring_read(b.sfull, b.ring, kK1Ring, c);
      if (cur < 0) break;
      const TcSeg s = items[cur];
      const LayerDesc& L = t.layers[s.layer];
      if (!L.mat) {  // pack into the P-buffer slot
        const float* grad = t.grads[s.layer];
        float* slot = t.pbuf + L.p_off;
        for (int64_t e = s.row0 + lane; e < s.row1; e += 32 * 8) {
          float v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = (e + 32 * u < s.row1) ? grad[e + 32 * u] : 0.f;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (e + 32 * u < s.row1) slot[e + 32 * u] = v[u];
        }
      } else if (lane == 0) {
        // one bulk group per tile; a stage's S tile is released once its
        // store has been READ (one group behind, so stores overlap)
        const CUtensorMap* smap = t.tmaps + kTmapsPerLayer * (int64_t)s.layer + 1;
        tmap_acquire(smap);
        for (int64_t c0 = 0; c0 < L.m; c0 += kK1N, ++t_it) {
          const int st = t_it % NS;
          mbar_wait(&b.xready[st], (t_it / NS) & 1u);
          tma_store_2d(smap, stage_ptr(t_it) + G::S_S, (int)c0, (int)s.row0);
          bulk_commit();
          if (pend >= 0) {
            bulk_wait_read<1>();
            mbar_arrive(&b.sfree[pend]);
          }
          pend = st;
        }
      }
      if (L.mat) t_it = __shfl_sync(0xffffffffu, t_it, 0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&b.sempty[c % kK1Ring]);
    }
    if (lane == 0) {
      bulk_wait_all();
      if (pend >= 0) mbar_arrive(&b.sfree[pend]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, kK1TmemCols);
  }
  sched_rearm(sched);
}

}  // namespace

size_t tc5_k1p_smem_bytes(int r8) {
  switch (r8) {
    case 8: return K1<8>::SMEM;
    case 16: return K1<16>::SMEM;
    case 32: return K1<32>::SMEM;
    default: return 0;
  }
}

cudaError_t launch_tc5_k1p(int r8, const Tables& t, const TcSeg* items, int nitems, int32_t* sched, int ncta,
                           cudaStream_t st) {
  if (ncta <= 0 || nitems <= 0) return cudaSuccess;
  const size_t smem = tc5_k1p_smem_bytes(r8);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern));
    if (e != cudaSuccess) return e;
    return launch_kernel(kern, dim3(ncta), dim3(kK1Threads), smem, st, false, t, items, nitems, sched);
  };
  switch (r8) {
    case 8: return go(tc5_k1p_kernel<8>);
    case 16: return go(tc5_k1p_kernel<16>);
    case 32: return go(tc5_k1p_kernel<32>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace acp
