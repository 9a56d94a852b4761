// Tensor-core K1 kernels with the double-deferred residual.
//
// Alg. 2 P:221-222 (P-step) and P:226-227 (Q-step) with the residual of each
// step left implicit: after a step the error is E = S - A B^T, where S is the
// step's input sum M' (written back into the E region) and (A, B) are the
// step's local factor and the reused (orthogonalised) one. The next step
// forms M' = M + E_prev = M + S - A B^T on the fly, writes it back as its own
// S, and projects it:
//
//   mode 0, P-step:  x = M + S - P_orth Q_loc^T;  S <- x;  P_loc = x Q_orth
//                    (P slot <- P_loc for the all-reduce; P_loc split kept)
//   mode 1, Q-step:  x = M + S - P_loc Q_orth^T;  S <- x;  Q_loc = x^T P_orth
//                    (per-segment partials; col_reduce_kernel sums them)
//
// so each K1 streams 12 B per element (read M, S; write S) and nothing has to
// hold a whole row: the P-step's row sums accumulate across column panels.
// Both rank-r products run on the tensor cores (mma.sync m16n8k8 TF32) in
// 3xTF32 form, x = hi + lo, so the result keeps fp32-class accuracy; the
// factors arrive pre-split (hi, lo) from the kernels that produce them.
//
// CTA = 8 consumer warps + 1 producer warp. The producer streams tiles of M
// and S (plus the tile's factor panels) with 16-byte cp.async into padded
// shared-memory rows (conflict-free fragment reads), completing on the
// stage's mbarrier (cp.async.mbarrier.arrive.noinc); consumers release
// stages through a second mbarrier. Vectors are packed into the parity's
// buffer by the consumer threads.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "k_common.cuh"
#include "k_nvls.cuh"

namespace acp {
namespace {

constexpr int kTcNW = 8;  // consumer warps

// ---- P-step geometry: tile = 128 rows (one 16-row block per warp) x 32
// columns, loaded as 2-D TMA boxes (rows of 128 B, SWIZZLE_128B: the 16-byte
// chunk c of row i sits at chunk c ^ (i & 7)). Each 8-column MMA block j uses
// chunks j and j + 4 (columns 4j..4j+3, 16+4j..16+4j+3), which makes every
// fragment read of the tile and of the factor boxes bank-conflict free.
constexpr int kPTR = 128, kPBC = 32;
constexpr int kPNB = 2;   // boxes per P-step tile (tile = 128 rows x 64 columns: 256 B per row)
constexpr int kPBOX = kPTR * kPBC;
__host__ __device__ constexpr int p_stage_floats(int r8) { return kPNB * (2 * kPBOX + 4 * r8 * kPBC); }

struct TcShared {
  float* ring;
  uint64_t* full;
  uint64_t* empty;
  int stages;
  int stage_floats;
};

__device__ __forceinline__ uint32_t lds_u32(const float* p) { return __float_as_uint(*p); }
// float offset of (row, 16-byte chunk) in a 128B-swizzled box of 32-float rows
__device__ __forceinline__ int swz(int row, int chunk) { return row * 32 + ((chunk ^ (row & 7)) << 2); }

__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void group_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Stage release with S written back by TMA: thread 0 of the consumers
// releases a stage only after the store that reads it has read it; the
// previous tile's stage is released one tile late so the store overlaps.
struct StageRelease {
  int pending = -1;
  __device__ __forceinline__ void after_store(const TcShared& sh, int stage) {
    bulk_commit();
    bulk_wait_read<1>();
    if (pending >= 0) mbar_arrive(&sh.empty[pending]);
    pending = stage;
  }
  __device__ __forceinline__ void immediate(const TcShared& sh, int stage) {
    if (pending >= 0) {
      bulk_wait_read<0>();
      mbar_arrive(&sh.empty[pending]);
      pending = -1;
    }
    mbar_arrive(&sh.empty[stage]);
  }
  __device__ __forceinline__ void finish() { bulk_wait_all(); }
};

// Two adjacent 8-column MMA blocks (jp, jp + 1) of C fragments -> 16-byte
// stores that fill whole 32-byte sectors: lanes t and t ^ 1 trade one pair so
// each lane holds 4 consecutive columns of a row (block jp for even t,
// block jp + 1 for odd t). ca / cb: this lane's own pair columns in the blocks.
__device__ __forceinline__ void store_pair(float* Ra, float* Rb, int64_t ca, int64_t cb, bool odd,
                                           const float (&a)[4], const float (&b)[4]) {
  const float s0 = odd ? a[0] : b[0], s1 = odd ? a[1] : b[1];
  const float s2 = odd ? a[2] : b[2], s3 = odd ? a[3] : b[3];
  const float r0 = __shfl_xor_sync(0xffffffffu, s0, 1), r1 = __shfl_xor_sync(0xffffffffu, s1, 1);
  const float r2 = __shfl_xor_sync(0xffffffffu, s2, 1), r3 = __shfl_xor_sync(0xffffffffu, s3, 1);
  const int64_t c = odd ? cb - 2 : ca;
  const float4 va = odd ? make_float4(r0, r1, b[0], b[1]) : make_float4(a[0], a[1], r0, r1);
  const float4 vb = odd ? make_float4(r2, r3, b[2], b[3]) : make_float4(a[2], a[3], r2, r3);
  __stcs(reinterpret_cast<float4*>(Ra + c), va);
  __stcs(reinterpret_cast<float4*>(Rb + c), vb);
}
// masked fallback: each lane stores its own pairs (rows / columns checked)
__device__ __forceinline__ void store_own(float* Ra, float* Rb, int64_t col, int64_t m, bool oka, bool okb,
                                          const float (&x)[4]) {
  const bool ca0 = col < m, ca1 = col + 1 < m;
  if (oka && ca0) Ra[col] = x[0];
  if (oka && ca1) Ra[col + 1] = x[1];
  if (okb && ca0) Rb[col] = x[2];
  if (okb && ca1) Rb[col + 1] = x[3];
}

template <int R8>
__device__ void tcp_producer(const Tables& t, const TcSeg* segs, int sb, int se, const TcShared& sh) {
  const int lane = threadIdx.x & 31;
  const uint64_t pol = policy_evict_first();
  uint64_t pol_keep;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
  int stage = 0;
  uint32_t phase = 0;
  constexpr uint32_t kTx = (uint32_t)(kPNB * (2 * kPBOX + 4 * R8 * kPBC)) * 4u;
  for (int si = sb; si < se; ++si) {
    const TcSeg s = segs[si];
    const LayerDesc& L = t.layers[s.layer];
    if (!L.mat) continue;
    const int64_t m = L.m;
    const float* grad = t.grads[s.layer];
    const float* S = t.E + L.e_off;
    const bool v16 = (m % 4 == 0) && ((reinterpret_cast<uintptr_t>(grad) & 15u) == 0);
    const CUtensorMap* maps = t.tmaps + kTmapsPerLayer * (int64_t)s.layer;  // M, S, Q_orth hi/lo, Q_loc hi/lo
    if (v16 && lane < 6) tmap_acquire(maps + lane);
    const float* fq[4] = {t.qsplit + L.qs_off, t.qsplit + L.qs_off + (int64_t)R8 * m,
                          t.qlsplit + L.qs_off, t.qlsplit + L.qs_off + (int64_t)R8 * m};
    for (int64_t r0 = s.row0; r0 < s.row1; r0 += kPTR) {
      const int nr = (int)((s.row1 - r0) < kPTR ? (s.row1 - r0) : kPTR);
      for (int64_t c0 = 0; c0 < m; c0 += kPNB * kPBC) {
        if (lane == 0) mbar_wait(&sh.empty[stage], phase ^ 1u);
        __syncwarp();
        // stage: [M box b][S box b][factor a, box b] (a: Q_orth hi, lo, Q_loc hi, lo)
        float* dM = sh.ring + (size_t)stage * sh.stage_floats;
        float* dS = dM + kPNB * kPBOX;
        float* dF = dS + kPNB * kPBOX;
        if (v16) {
          // boxes: rows beyond n / columns beyond m are zero-filled by the TMA
          if (lane == 0) {
            mbar_arrive_tx(&sh.full[stage], kTx);
#pragma unroll
            for (int b = 0; b < kPNB; ++b) {
              const int cb = (int)c0 + kPBC * b;
              tma_load_2d(dM + b * kPBOX, maps + 0, cb, (int)r0, &sh.full[stage], pol);
              tma_load_2d(dS + b * kPBOX, maps + 1, cb, (int)r0, &sh.full[stage], pol);
#pragma unroll
              for (int a = 0; a < 4; ++a)
                tma_load_2d(dF + (a * kPNB + b) * R8 * kPBC, maps + 2 + a, cb, 0, &sh.full[stage], pol_keep);
            }
          }
        } else {
          // unaligned layer: 4-byte async copies into the same swizzled layout
          if (lane == 0) mbar_arrive(&sh.full[stage]);
          for (int it = lane; it < kPTR * kPNB * kPBC; it += 32) {
            const int i = it / (kPNB * kPBC), j = it - i * (kPNB * kPBC);
            const bool ok = i < nr && c0 + j < m;
            const int64_t off = ok ? (r0 + i) * m + c0 + j : 0;
            const int d = (j >> 5) * kPBOX + swz(i, (j & 31) >> 2) + (j & 3);
            cp_async4(dM + d, grad + off, ok ? 4u : 0u);
            cp_async4(dS + d, S + off, ok ? 4u : 0u);
          }
          for (int it = lane; it < 4 * R8 * kPNB * kPBC; it += 32) {
            const int a = it / (R8 * kPNB * kPBC), rem = it - a * (R8 * kPNB * kPBC);
            const int k = rem / (kPNB * kPBC), j = rem - k * (kPNB * kPBC);
            const bool ok = c0 + j < m;
            cp_async4(dF + (a * kPNB + (j >> 5)) * R8 * kPBC + swz(k, (j & 31) >> 2) + (j & 3),
                      fq[a] + (ok ? k * m + c0 + j : 0), ok ? 4u : 0u);
          }
        }
        cp_async_arrive(&sh.full[stage]);
        if (++stage == sh.stages) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  }
}

template <int R8>
__device__ void tcp_consumer(const Tables& t, const TcSeg* segs, int sb, int se, const TcShared& sh) {
  constexpr int KB = R8 / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int rw = 16 * warp + g;  // this lane's first tile row (second: rw + 8, same swizzle)
  // loop-invariant fragment offsets (floats) inside a stage's boxes, per
  // 8-column block j: X / Q_orth pairs at chunk cj, correction column at cg
  int offX[4], offQ[4], offL0[4], offL1[4], colj[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int cj = tq < 2 ? j : j + 4, oc = 2 * (tq & 1);
    const int cg = g < 4 ? j : j + 4, og = g & 3;
    offX[j] = swz(rw, cj) + oc;
    offQ[j] = swz(g, cj) + oc;               // + 256 * nb (rows 8nb + g)
    offL0[j] = swz(tq, cg) + og;             // + 256 * kb (rows 8kb + tq)
    offL1[j] = swz(tq + 4, cg) + og;         // rows 8kb + tq + 4
    colj[j] = 4 * cj + oc;
  }
  int stage = 0;
  uint32_t phase = 0;
  for (int si = sb; si < se; ++si) {
    if (!t.layers[segs[si].layer].mat) {  // vectors: pack into the P-buffer slots
      si = vector_run(t, segs, si, se, warp, kTcNW, [&](const TcSeg& s, const LayerDesc& L, int first, int stride) {
             const float* grad = t.grads[s.layer];
             float* slot = t.pbuf + L.p_off;
             for (int64_t i = s.row0 + first; i < s.row1; i += stride) slot[i] = grad[i];
           }) - 1;
      continue;
    }
    const TcSeg s = segs[si];
    const LayerDesc& L = t.layers[s.layer];
    float* grad = t.grads[s.layer];
    const int64_t m = L.m, n = L.n;
    const int r = L.r;
    float* S = t.E + L.e_off;
    // S: 16-byte stores of whole 32-byte sectors (lane pairs trade a column
    // pair); a shared-memory + TMA store variant needs a CTA barrier per tile
    // and measured slower here (1.10 vs 0.83 ms, BERT-L r = 8)
    const bool v4 = (m % 4 == 0) && ((reinterpret_cast<uintptr_t>(grad) & 15u) == 0);
    const float* Ps = t.psplit + L.ps_off;   // P_orth [2][n][R8]
    float* Pl = t.plsplit + L.ps_off;        // P_loc  [2][n][R8]
    float* Pw = t.pbuf + L.p_off;            // P slot, k-major [r][n]
    for (int64_t r0 = s.row0; r0 < s.row1; r0 += kPTR) {
      const int64_t ra = r0 + rw, rb = ra + 8;
      const bool oka = ra < s.row1, okb = rb < s.row1;
      // A fragments of P_orth (rows ra, rb; ranks 8kb + tq, + 4), hi and lo;
      // rows past the segment are zero, so their x (zero-filled tiles) is 0
      uint32_t ah[KB][4], al[KB][4];
#pragma unroll
      for (int kb = 0; kb < KB; ++kb) {
        const int k0 = 8 * kb + tq;
        ah[kb][0] = oka ? __float_as_uint(Ps[ra * R8 + k0]) : 0u;
        ah[kb][1] = okb ? __float_as_uint(Ps[rb * R8 + k0]) : 0u;
        ah[kb][2] = oka ? __float_as_uint(Ps[ra * R8 + k0 + 4]) : 0u;
        ah[kb][3] = okb ? __float_as_uint(Ps[rb * R8 + k0 + 4]) : 0u;
        al[kb][0] = oka ? __float_as_uint(Ps[(n + ra) * R8 + k0]) : 0u;
        al[kb][1] = okb ? __float_as_uint(Ps[(n + rb) * R8 + k0]) : 0u;
        al[kb][2] = oka ? __float_as_uint(Ps[(n + ra) * R8 + k0 + 4]) : 0u;
        al[kb][3] = okb ? __float_as_uint(Ps[(n + rb) * R8 + k0 + 4]) : 0u;
      }
      float acc[KB][4];
#pragma unroll
      for (int kb = 0; kb < KB; ++kb) acc[kb][0] = acc[kb][1] = acc[kb][2] = acc[kb][3] = 0.f;
      const bool rows_full = r0 + kPTR <= s.row1;
      float* Sa = S + ra * m;
      float* Sb = S + rb * m;
      for (int64_t c00 = 0; c00 < m; c00 += kPNB * kPBC) {
        mbar_wait(&sh.full[stage], phase);
        const float* sM0 = sh.ring + (size_t)stage * sh.stage_floats;
        const float* sS0 = sM0 + kPNB * kPBOX;
        const float* fF0 = sS0 + kPNB * kPBOX;
        const bool full = rows_full && (c00 + kPNB * kPBC <= m) && v4;
        // the tensor core accumulates with truncation: keep each MMA chain
        // short (one panel) and sum the panels in fp32 round-to-nearest
        float pa[KB][4];
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) pa[kb][0] = pa[kb][1] = pa[kb][2] = pa[kb][3] = 0.f;
#pragma unroll
        for (int bx = 0; bx < kPNB; ++bx) {
        const int64_t c0 = c00 + kPBC * bx;
        const float* sM = sM0 + bx * kPBOX;
        const float* sS = sS0 + bx * kPBOX;
        const float* fQh = fF0 + (0 * kPNB + bx) * R8 * kPBC;
        const float* fQl = fF0 + (1 * kPNB + bx) * R8 * kPBC;
        const float* fLh = fF0 + (2 * kPNB + bx) * R8 * kPBC;
        const float* fLl = fF0 + (3 * kPNB + bx) * R8 * kPBC;
#pragma unroll
        for (int jp = 0; jp < kPBC / 8; jp += 2) {
          float x[2][4];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int j = jp + u;
            // correction C = P_orth Q_loc^T (16 rows x 8 columns)
            float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
              const int o0 = offL0[j] + 256 * kb, o1 = offL1[j] + 256 * kb;
              mma3(c, ah[kb], al[kb], lds_u32(fLh + o0), lds_u32(fLh + o1), lds_u32(fLl + o0),
                   lds_u32(fLl + o1));
            }
            const float2 m0 = *reinterpret_cast<const float2*>(sM + offX[j]);
            const float2 m1 = *reinterpret_cast<const float2*>(sM + offX[j] + 256);
            const float2 s0 = *reinterpret_cast<const float2*>(sS + offX[j]);
            const float2 s1 = *reinterpret_cast<const float2*>(sS + offX[j] + 256);
            x[u][0] = m0.x + s0.x - c[0];
            x[u][1] = m0.y + s0.y - c[1];
            x[u][2] = m1.x + s1.x - c[2];
            x[u][3] = m1.y + s1.y - c[3];
          }
          if (full) {
            store_pair(Sa, Sb, c0 + colj[jp], c0 + colj[jp + 1], tq & 1, x[0], x[1]);
          } else {
            store_own(Sa, Sb, c0 + colj[jp], m, oka, okb, x[0]);
            store_own(Sa, Sb, c0 + colj[jp + 1], m, oka, okb, x[1]);
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int j = jp + u;
            // projection P += x Q_orth; A's k index t <-> column n = 2t, t + 4 <-> 2t + 1
            uint32_t xh[4], xl[4];
            split_tf32(x[u][0], xh[0], xl[0]);
            split_tf32(x[u][2], xh[1], xl[1]);
            split_tf32(x[u][1], xh[2], xl[2]);
            split_tf32(x[u][3], xh[3], xl[3]);
#pragma unroll
            for (int nb = 0; nb < KB; ++nb) {
              const int o = offQ[j] + 256 * nb;
              const float2 bh = *reinterpret_cast<const float2*>(fQh + o);
              const float2 bl = *reinterpret_cast<const float2*>(fQl + o);
              mma3(pa[nb], xh, xl, __float_as_uint(bh.x), __float_as_uint(bh.y),
                   __float_as_uint(bl.x), __float_as_uint(bl.y));
            }
          }
        }
        }
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
          acc[kb][0] += pa[kb][0];
          acc[kb][1] += pa[kb][1];
          acc[kb][2] += pa[kb][2];
          acc[kb][3] += pa[kb][3];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.empty[stage]);
        if (++stage == sh.stages) {
          stage = 0;
          phase ^= 1u;
        }
      }
      // P_loc rows -> P slot (k-major, all-reduce payload) + split copy
#pragma unroll
      for (int nb = 0; nb < KB; ++nb) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int k = 8 * nb + 2 * tq + (h & 1);
          const int64_t row = (h < 2) ? ra : rb;
          const bool ok = (h < 2) ? oka : okb;
          if (ok && k < r) {
            const float v = acc[nb][h];
            Pw[(int64_t)k * n + row] = v;
            uint32_t hi, lo;
            split_tf32(v, hi, lo);
            Pl[row * R8 + k] = __uint_as_float(hi);
            Pl[(n + row) * R8 + k] = __uint_as_float(lo);
          }
        }
      }
    }
  }
}

// ---- Q-step: tiles of tr rows x pc columns, staged as pc/32 boxes of
// tr x 32 floats (SWIZZLE_128B); warps own 16-column blocks (cbw each) and
// walk the tile's 8-row k-steps. Scalar reads (row 2t / 2t+1, column g / g+8)
// hit 32 distinct banks under the swizzle. Row factors (P_loc, P_orth hi/lo)
// arrive by cp.async into rows of R8 + 4 floats.
constexpr int kQRS_PAD = 4;

__host__ __device__ constexpr int q_nbox(int pc) { return (pc + 31) / 32; }
__host__ __device__ constexpr int q_stage_floats(int tr, int pc, int r8) {
  return (2 * q_nbox(pc) * tr * 32 + 4 * tr * (r8 + kQRS_PAD) + 255) / 256 * 256;
}

template <int R8>
__device__ void tcq_producer(const Tables& t, const TcSeg* segs, int sb, int se, const TcShared& sh) {
  constexpr int RS = R8 + kQRS_PAD;
  const int lane = threadIdx.x & 31;
  const uint64_t pol = policy_evict_first();
  int stage = 0;
  uint32_t phase = 0;
  for (int si = sb; si < se; ++si) {
    const TcSeg s = segs[si];
    const LayerDesc& L = t.layers[s.layer];
    if (!L.mat) continue;
    const int64_t m = L.m, n = L.n;
    const TcMap mp = L.tq;
    const float* grad = t.grads[s.layer];
    const float* S = t.E + L.e_off;
    const int64_t c0 = (int64_t)s.panel * mp.pc;
    const int cols = (int)((m - c0) < mp.pc ? (m - c0) : mp.pc);
    const int nbox = q_nbox(mp.pc);
    const int tr = mp.tr;
    const bool v16 = (m % 4 == 0) && ((reinterpret_cast<uintptr_t>(grad) & 15u) == 0);
    const CUtensorMap* maps = t.tmaps + kTmapsPerLayer * (int64_t)s.layer + 6;  // M, S with tr-row boxes
    if (v16 && lane < 2) tmap_acquire(maps + lane);
    const float* fr[4] = {t.plsplit + L.ps_off, t.plsplit + L.ps_off + n * R8,
                          t.psplit + L.ps_off, t.psplit + L.ps_off + n * R8};
    for (int64_t r0 = s.row0; r0 < s.row1; r0 += tr) {
      const int nr = (int)((s.row1 - r0) < tr ? (s.row1 - r0) : tr);
      if (lane == 0) mbar_wait(&sh.empty[stage], phase ^ 1u);
      __syncwarp();
      float* dM = sh.ring + (size_t)stage * sh.stage_floats;
      float* dS = dM + nbox * tr * 32;
      float* dF = dS + nbox * tr * 32;
      if (v16) {
        if (lane == 0) {
          mbar_arrive_tx(&sh.full[stage], 2u * (uint32_t)(nbox * tr * 32 * 4));
          for (int b = 0; b < nbox; ++b) {
            tma_load_2d(dM + b * tr * 32, maps + 0, (int)(c0 + 32 * b), (int)r0, &sh.full[stage], pol);
            tma_load_2d(dS + b * tr * 32, maps + 1, (int)(c0 + 32 * b), (int)r0, &sh.full[stage], pol);
          }
        }
      } else {
        if (lane == 0) mbar_arrive(&sh.full[stage]);
        for (int it = lane; it < tr * nbox * 32; it += 32) {
          const int i = it / (nbox * 32), col = it - i * (nbox * 32);
          const bool ok = i < nr && col < cols;
          const int64_t off = ok ? (r0 + i) * m + c0 + col : 0;
          const int w = col & 31;
          const int d = (col >> 5) * tr * 32 + swz(i, w >> 2) + (w & 3);
          cp_async4(dM + d, grad + off, ok ? 4u : 0u);
          cp_async4(dS + d, S + off, ok ? 4u : 0u);
        }
      }
      // row factors [row][R8] (P_loc hi, lo, P_orth hi, lo): 16-byte chunks
      // (R8 / 4 per row: shifts and masks only, no runtime division)
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const float* src = fr[a] + r0 * R8;
        float* dst = dF + a * tr * RS;
        for (int it = lane; it < tr * (R8 / 4); it += 32) {
          const int i = it / (R8 / 4), j = it % (R8 / 4);
          const bool ok = i < nr;
          cp_async16(dst + i * RS + 4 * j, ok ? src + i * R8 + 4 * j : src, ok ? 16u : 0u);
        }
      }
      cp_async_arrive(&sh.full[stage]);
      if (++stage == sh.stages) {
        stage = 0;
        phase ^= 1u;
      }
    }
  }
}

template <int R8, int CBW>
__device__ void tcq_consumer(const Tables& t, const TcSeg* segs, int sb, int se, const TcShared& sh) {
  constexpr int KB = R8 / 8;
  constexpr int RS = R8 + kQRS_PAD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  StageRelease rel;
  for (int si = sb; si < se; ++si) {
    if (!t.layers[segs[si].layer].mat) {  // vectors: pack into the Q-buffer slots
      si = vector_run(t, segs, si, se, warp, kTcNW, [&](const TcSeg& s, const LayerDesc& L, int first, int stride) {
             const float* grad = t.grads[s.layer];
             float* slot = t.qbuf + L.q_off;
             for (int64_t i = s.row0 + first; i < s.row1; i += stride) slot[i] = grad[i];
           }) - 1;
      continue;
    }
    const TcSeg s = segs[si];
    const LayerDesc& L = t.layers[s.layer];
    const int64_t m = L.m;
    const int r = L.r;
    const TcMap mp = L.tq;
    float* S = t.E + L.e_off;
    const int64_t c0 = (int64_t)s.panel * mp.pc;
    const int cols = (int)((m - c0) < mp.pc ? (m - c0) : mp.pc);
    const int nbox = q_nbox(mp.pc);
    const int tr = mp.tr;
    const int cg = warp % mp.wc, rg = warp / mp.wc;
    const int ksteps = tr / 8;
    const float* Qh = t.qsplit + L.qs_off;   // Q_orth [2][R8][m]
    const float* Ql = Qh + (int64_t)R8 * m;
    // S is written back through shared memory + TMA store (map 7) when rows
    // are 16-byte aligned; otherwise each lane stores its own elements
    const bool tst = (m % 4 == 0);
    const CUtensorMap* smap = t.tmaps + kTmapsPerLayer * (int64_t)s.layer + 7;
    // this warp's column blocks (16 columns each) inside the panel
    uint32_t ah[CBW][KB][4], al[CBW][KB][4];
    float acc[CBW][KB][4];
    int offa[CBW], offb[CBW];  // x at (row 2t, column g) and (row 2t, column g + 8); rows 2t+1: + 32 / xor
    int offa1[CBW], offb1[CBW];
    bool blk[CBW];
#pragma unroll
    for (int j = 0; j < CBW; ++j) {
      const int cl = (cg * CBW + j) * 16;
      blk[j] = cl < mp.pc;  // uniform per warp
      const int64_t ca = c0 + cl + g, cb2 = ca + 8;
      const bool oka = cl + g < cols, okb = cl + g + 8 < cols;
#pragma unroll
      for (int kb = 0; kb < KB; ++kb) {
        const int64_t k0 = 8 * kb + tq;
        ah[j][kb][0] = oka ? __float_as_uint(Qh[k0 * m + ca]) : 0u;
        ah[j][kb][1] = okb ? __float_as_uint(Qh[k0 * m + cb2]) : 0u;
        ah[j][kb][2] = oka ? __float_as_uint(Qh[(k0 + 4) * m + ca]) : 0u;
        ah[j][kb][3] = okb ? __float_as_uint(Qh[(k0 + 4) * m + cb2]) : 0u;
        al[j][kb][0] = oka ? __float_as_uint(Ql[k0 * m + ca]) : 0u;
        al[j][kb][1] = okb ? __float_as_uint(Ql[k0 * m + cb2]) : 0u;
        al[j][kb][2] = oka ? __float_as_uint(Ql[(k0 + 4) * m + ca]) : 0u;
        al[j][kb][3] = okb ? __float_as_uint(Ql[(k0 + 4) * m + cb2]) : 0u;
        acc[j][kb][0] = acc[j][kb][1] = acc[j][kb][2] = acc[j][kb][3] = 0.f;
      }
      const int box = (cl >> 5) * tr * 32, w = (cl & 31) + g;
      offa[j] = box + swz(2 * tq, w >> 2) + (w & 3);
      offb[j] = box + swz(2 * tq, (w + 8) >> 2) + (w & 3);
      offa1[j] = box + swz(2 * tq + 1, w >> 2) + (w & 3);
      offb1[j] = box + swz(2 * tq + 1, (w + 8) >> 2) + (w & 3);
    }
    // the S tile goes back per 32-column box: its writers (the wr row-group
    // warps of the one or two column groups covering it) meet at named
    // barrier 2 + box and the first of them stores it, so no warp waits on
    // the whole CTA each tile. A CTA-wide barrier first: the ids / counts of
    // this segment must not meet a slower warp of the previous one.
    const int cpb = 2 / CBW;                      // column groups per box
    const int mybox = (cg * CBW * 16) >> 5;
    const bool boxed = tst && mybox < nbox;
    const bool storer = boxed && rg == 0 && (cg % cpb) == 0;
    const int bwriters = 32 * mp.wr * cpb;
    consumers_sync();
    for (int64_t r0 = s.row0; r0 < s.row1; r0 += tr) {
      mbar_wait(&sh.full[stage], phase);
      const float* sM = sh.ring + (size_t)stage * sh.stage_floats;
      float* sS = sh.ring + (size_t)stage * sh.stage_floats + nbox * tr * 32;
      const float* fLh = sS + nbox * tr * 32;   // P_loc hi [tr][RS]
      const float* fLl = fLh + tr * RS;
      const float* fPh = fLl + tr * RS;   // P_orth hi
      const float* fPl = fPh + tr * RS;
      float ta[CBW][KB][4];  // this tile's sums (short MMA chains, see the P-step)
#pragma unroll
      for (int j = 0; j < CBW; ++j)
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) ta[j][kb][0] = ta[j][kb][1] = ta[j][kb][2] = ta[j][kb][3] = 0.f;
      // per-tile pointers: every shared load / store below is [pointer + constant]
      const int ks0 = rg;  // this warp's first k-step (k-steps ks0, ks0 + wr, ...)
      const float* pL = fLh + (8 * ks0 + g) * RS + tq;        // P_loc rows 8ks+g, ranks 8kb+t (+4)
      const float* pLl = fLl + (8 * ks0 + g) * RS + tq;
      const float* pP = fPh + (8 * ks0 + 2 * tq) * RS + g;    // P_orth rows 8ks+2t (+1), ranks 8kb+g
      const float* pPl = fPl + (8 * ks0 + 2 * tq) * RS + g;
      const float* xM[CBW][4];
      float* xS[CBW][4];
#pragma unroll
      for (int j = 0; j < CBW; ++j) {
        const int o[4] = {offa[j], offa1[j], offb[j], offb1[j]};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          xM[j][e] = sM + o[e] + 256 * ks0;
          xS[j][e] = sS + o[e] + 256 * ks0;
        }
      }
      auto kstep = [&](const int kk, const int ks) {  // kk: k-step index relative to ks0 (unrolled)
        const int fo = 8 * RS * kk;  // kk: rows 8 kk below the warp's first k-step
        const int xo = 256 * kk;
        // B fragments: P_loc (k = rank, n = row) and P_orth (k = row, n = rank)
        uint32_t lbh[KB][2], lbl[KB][2], pbh[KB][2], pbl[KB][2];
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
          lbh[kb][0] = lds_u32(pL + fo + 8 * kb);
          lbh[kb][1] = lds_u32(pL + fo + 8 * kb + 4);
          lbl[kb][0] = lds_u32(pLl + fo + 8 * kb);
          lbl[kb][1] = lds_u32(pLl + fo + 8 * kb + 4);
          pbh[kb][0] = lds_u32(pP + fo + 8 * kb);
          pbh[kb][1] = lds_u32(pP + fo + RS + 8 * kb);
          pbl[kb][0] = lds_u32(pPl + fo + 8 * kb);
          pbl[kb][1] = lds_u32(pPl + fo + RS + 8 * kb);
        }
#pragma unroll
        for (int j = 0; j < CBW; ++j) {
          if (!blk[j]) continue;
          // correction C^T = Q_orth P_loc^T (16 columns x 8 rows)
          float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int kb = 0; kb < KB; ++kb)
            mma3(c, ah[j][kb], al[j][kb], lbh[kb][0], lbh[kb][1], lbl[kb][0], lbl[kb][1]);
          // c0 (col g, row 2t), c1 (col g, row 2t+1), c2 (col g+8, row 2t), c3 (col g+8, row 2t+1)
          float x[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) x[e] = xM[j][e][xo] + xS[j][e][xo] - c[e];
          if (tst) {  // back into the S tile; the tile is stored by TMA below
#pragma unroll
            for (int e = 0; e < 4; ++e) xS[j][e][xo] = x[e];
          } else {
            const int rowa = 8 * ks + 2 * tq;
            float* Sa = S + (r0 + rowa) * m + c0;
            float* Sb = Sa + m;
            const int ca = (cg * CBW + j) * 16 + g, cb2 = ca + 8;
            const bool va = r0 + rowa < s.row1, vb = r0 + rowa + 1 < s.row1;
            if (ca < cols) {
              if (va) __stcs(Sa + ca, x[0]);
              if (vb) __stcs(Sb + ca, x[1]);
            }
            if (cb2 < cols) {
              if (va) __stcs(Sa + cb2, x[2]);
              if (vb) __stcs(Sb + cb2, x[3]);
            }
          }
          // projection Q += x^T P_orth: A = x^T (columns x rows), k t <-> row 2t
          uint32_t xh[4], xl[4];
          split_tf32(x[0], xh[0], xl[0]);
          split_tf32(x[2], xh[1], xl[1]);
          split_tf32(x[1], xh[2], xl[2]);
          split_tf32(x[3], xh[3], xl[3]);
#pragma unroll
          for (int nb = 0; nb < KB; ++nb)
            mma3(ta[j][nb], xh, xl, pbh[nb][0], pbh[nb][1], pbl[nb][0], pbl[nb][1]);
        }
      };
      if constexpr (R8 >= 32) {  // 32-row tiles (tc_q_map): up to 4 k-steps per warp
        if (ks0 < ksteps) kstep(0, ks0);
#pragma unroll 1
        for (int ks = ks0 + mp.wr; ks < ksteps; ks += mp.wr) kstep(ks - ks0, ks);
      } else {  // 16-row tiles: a second k-step only with wr = 1
        if (ks0 < ksteps) kstep(0, ks0);
        if (ks0 + mp.wr < ksteps) kstep(1, ks0 + mp.wr);
      }
#pragma unroll
      for (int j = 0; j < CBW; ++j)
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
          acc[j][kb][0] += ta[j][kb][0];
          acc[j][kb][1] += ta[j][kb][1];
          acc[j][kb][2] += ta[j][kb][2];
          acc[j][kb][3] += ta[j][kb][3];
        }
      if (boxed) {
        fence_async_smem();
        group_bar(2 + mybox, bwriters);
      }
      __syncwarp();
      if (lane == 0) {
        if (storer) {
          tma_store_2d(smap, sS + mybox * tr * 32, (int)(c0 + 32 * mybox), (int)r0);
          rel.after_store(sh, stage);
        } else {
          rel.immediate(sh, stage);
        }
      }
      if (++stage == sh.stages) {
        stage = 0;
        phase ^= 1u;
      }
    }
    // partial slot of row group rg: k-major [r][pc]
    const int64_t stride = ((int64_t)r * mp.pc + 3) / 4 * 4;
    float* part = t.colpart + s.part_off + rg * stride;
#pragma unroll
    for (int j = 0; j < CBW; ++j) {
      const int cl = (cg * CBW + j) * 16;
      if (cl >= cols) break;
#pragma unroll
      for (int nb = 0; nb < KB; ++nb) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int k = 8 * nb + 2 * tq + (h & 1);
          const int col = cl + g + ((h & 2) ? 8 : 0);
          if (k < r && col < cols) part[(int64_t)k * mp.pc + col] = acc[j][nb][h];
        }
      }
    }
  }
  if (lane == 0) rel.finish();
}

// ---- decode (K3 on the tensor cores): grad = scale * A B^T, tile = 128 rows
// (one 16-row block per warp) x 32 columns. B (the m-side factor) streams in
// as 128B-swizzled boxes of R8 x 32 floats: MODE 2 (P-step) reads Q_orth's
// split copy (maps 2, 3), MODE 3 (Q-step) the all-reduced Q slot (map 8),
// split on use. A: P-step the all-reduced P slot (split once per row block),
// Q-step P_orth's split copy. Write-only: 4 B per element.
constexpr int kDNB = 4;  // boxes per decode tile (128 rows x 128 columns)
__host__ __device__ constexpr int d_stage_floats(int r8) { return 2 * kDNB * r8 * kPBC; }

template <int MODE, int R8>
__device__ void tcd_producer(const Tables& t, const TcSeg* segs, int sb, int se, const TcShared& sh) {
  const int lane = threadIdx.x & 31;
  uint64_t pol_keep;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
  int stage = 0;
  uint32_t phase = 0;
  for (int si = sb; si < se; ++si) {
    const TcSeg s = segs[si];
    const LayerDesc& L = t.layers[s.layer];
    if (!L.mat) continue;
    const int64_t m = L.m;
    const CUtensorMap* maps = t.tmaps + kTmapsPerLayer * (int64_t)s.layer;
    const bool v16 = (m % 4 == 0);
    if (v16 && lane < 9) tmap_acquire(maps + lane);
    const float* src0 = MODE == 2 ? t.qsplit + L.qs_off : t.qbuf + L.q_off;
    const float* src1 = MODE == 2 ? t.qsplit + L.qs_off + (int64_t)R8 * m : nullptr;
    const int rows_b = MODE == 2 ? R8 : L.r;  // rows present in the source array
    for (int64_t r0 = s.row0; r0 < s.row1; r0 += kPTR) {
      for (int64_t c0 = 0; c0 < m; c0 += kDNB * kPBC) {
        if (lane == 0) mbar_wait(&sh.empty[stage], phase ^ 1u);
        __syncwarp();
        float* dB = sh.ring + (size_t)stage * sh.stage_floats;  // [array][box] of R8 x 32
        if (v16) {
          if (lane == 0) {
            if constexpr (MODE == 2) {
              mbar_arrive_tx(&sh.full[stage], 2u * kDNB * R8 * kPBC * 4u);
              for (int b = 0; b < kDNB; ++b) {
                tma_load_2d(dB + b * R8 * kPBC, maps + 2, (int)c0 + kPBC * b, 0, &sh.full[stage], pol_keep);
                tma_load_2d(dB + (kDNB + b) * R8 * kPBC, maps + 3, (int)c0 + kPBC * b, 0, &sh.full[stage],
                            pol_keep);
              }
            } else {
              mbar_arrive_tx(&sh.full[stage], (uint32_t)kDNB * R8 * kPBC * 4u);
              for (int b = 0; b < kDNB; ++b)
                tma_load_2d(dB + b * R8 * kPBC, maps + 8, (int)c0 + kPBC * b, 0, &sh.full[stage], pol_keep);
            }
          }
        } else {
          if (lane == 0) mbar_arrive(&sh.full[stage]);
          const int arrays = MODE == 2 ? 2 : 1;
          for (int it = lane; it < arrays * R8 * kDNB * kPBC; it += 32) {
            const int a = it / (R8 * kDNB * kPBC), rem = it - a * (R8 * kDNB * kPBC);
            const int k = rem / (kDNB * kPBC), j = rem - k * (kDNB * kPBC);
            const bool ok = k < rows_b && c0 + j < m;
            const float* src = a == 0 ? src0 : src1;
            cp_async4(dB + (a * kDNB + (j >> 5)) * R8 * kPBC + swz(k, (j & 31) >> 2) + (j & 3),
                      src + (ok ? k * m + c0 + j : 0), ok ? 4u : 0u);
          }
        }
        cp_async_arrive(&sh.full[stage]);
        if (++stage == sh.stages) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  }
}

template <int MODE, int R8>
__device__ void tcd_consumer(const Tables& t, const TcSeg* segs, int sb, int se, const TcShared& sh,
                             float scale) {
  constexpr int KB = R8 / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int rw = 16 * warp + g;
  int offL0[4], offL1[4], colj[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int cj = tq < 2 ? j : j + 4, oc = 2 * (tq & 1);
    const int cg = g < 4 ? j : j + 4, og = g & 3;
    offL0[j] = swz(tq, cg) + og;      // + 256 * kb (rows 8kb + tq)
    offL1[j] = swz(tq + 4, cg) + og;  // rows 8kb + tq + 4
    colj[j] = 4 * cj + oc;
  }
  int stage = 0;
  uint32_t phase = 0;
  for (int si = sb; si < se; ++si) {
    if (!t.layers[segs[si].layer].mat) {  // vectors: unpack from the parity's buffer
      si = vector_run(t, segs, si, se, warp, kTcNW, [&](const TcSeg& s, const LayerDesc& L, int first, int stride) {
             float* grad = t.grads[s.layer];
             const float* slot = (MODE == 2 ? t.pbuf + L.p_off : t.qbuf + L.q_off);
             for (int64_t i = s.row0 + first; i < s.row1; i += stride) grad[i] = slot[i] * scale;
           }) - 1;
      continue;
    }
    const TcSeg s = segs[si];
    const LayerDesc& L = t.layers[s.layer];
    float* grad = t.grads[s.layer];
    const int64_t m = L.m, n = L.n;
    const int r = L.r;
    const bool v4 = (m % 4 == 0) && ((reinterpret_cast<uintptr_t>(grad) & 15u) == 0);
    for (int64_t r0 = s.row0; r0 < s.row1; r0 += kPTR) {
      const int64_t ra = r0 + rw, rb = ra + 8;
      const bool oka = ra < s.row1, okb = rb < s.row1;
      uint32_t ah[KB][4], al[KB][4];
#pragma unroll
      for (int kb = 0; kb < KB; ++kb) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int k = 8 * kb + tq + ((h & 2) ? 4 : 0);
          const int64_t row = (h & 1) ? rb : ra;
          const bool ok = ((h & 1) ? okb : oka) && k < r;
          if constexpr (MODE == 2) {  // all-reduced P slot, k-major fp32: split here
            const float v = ok ? t.pbuf[L.p_off + (int64_t)k * n + row] * scale : 0.f;
            split_tf32(v, ah[kb][h], al[kb][h]);
          } else {                    // P_orth split copy [2][n][R8]
            const float* Ps = t.psplit + L.ps_off;
            ah[kb][h] = ok ? __float_as_uint(Ps[row * R8 + k] ) : 0u;
            al[kb][h] = ok ? __float_as_uint(Ps[(n + row) * R8 + k]) : 0u;
          }
        }
      }
      float* Ga = grad + ra * m;
      float* Gb = grad + rb * m;
      const bool rows_full = r0 + kPTR <= s.row1;
      for (int64_t c00 = 0; c00 < m; c00 += kDNB * kPBC) {
        mbar_wait(&sh.full[stage], phase);
        const float* fB0 = sh.ring + (size_t)stage * sh.stage_floats;
        const bool full = rows_full && (c00 + kDNB * kPBC <= m) && v4;
#pragma unroll 1
        for (int bx = 0; bx < kDNB; ++bx) {  // not unrolled: 2 CTAs / SM cap registers at 96
        const int64_t c0 = c00 + kPBC * bx;
        const float* fBh = fB0 + bx * R8 * kPBC;
        const float* fBl = fB0 + (kDNB + bx) * R8 * kPBC;
        if constexpr (R8 <= 16) {
        // JB 8-column blocks per batch: all their shared loads first, then the
        // MMAs, then the global stores (loads of a later batch cannot move
        // above stores the compiler cannot prove disjoint; batching gives the
        // MMA chains independent neighbours)
        constexpr int JB = R8 <= 8 ? 4 : 2;  // r = 32: streamed pairs (registers)
#pragma unroll
        for (int j0 = 0; j0 < kPBC / 8; j0 += JB) {
        uint32_t bfr[JB][KB][4];
#pragma unroll
        for (int u = 0; u < JB; ++u) {
#pragma unroll
          for (int kb = 0; kb < KB; ++kb) {
            const int o0 = offL0[j0 + u] + 256 * kb, o1 = offL1[j0 + u] + 256 * kb;
            if constexpr (MODE == 2) {
              bfr[u][kb][0] = lds_u32(fBh + o0);
              bfr[u][kb][1] = lds_u32(fBh + o1);
              bfr[u][kb][2] = lds_u32(fBl + o0);
              bfr[u][kb][3] = lds_u32(fBl + o1);
            } else {
              split_tf32(fBh[o0], bfr[u][kb][0], bfr[u][kb][2]);
              split_tf32(fBh[o1], bfr[u][kb][1], bfr[u][kb][3]);
            }
          }
        }
        float cc[JB][4];
#pragma unroll
        for (int u = 0; u < JB; ++u) {
          cc[u][0] = cc[u][1] = cc[u][2] = cc[u][3] = 0.f;
#pragma unroll
          for (int kb = 0; kb < KB; ++kb)
            mma3(cc[u], ah[kb], al[kb], bfr[u][kb][0], bfr[u][kb][1], bfr[u][kb][2], bfr[u][kb][3]);
          if constexpr (MODE == 3) {
#pragma unroll
            for (int h = 0; h < 4; ++h) cc[u][h] *= scale;
          }
        }
#pragma unroll
        for (int u = 0; u < JB; u += 2) {
          const int jp = j0 + u;
          if (full) {
            store_pair(Ga, Gb, c0 + colj[jp], c0 + colj[jp + 1], tq & 1, cc[u], cc[u + 1]);
          } else {
            store_own(Ga, Gb, c0 + colj[jp], m, oka, okb, cc[u]);
            store_own(Ga, Gb, c0 + colj[jp + 1], m, oka, okb, cc[u + 1]);
          }
        }
        }
        } else {
#pragma unroll
        for (int jp = 0; jp < kPBC / 8; jp += 2) {
        float cc[2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int j = jp + u;
          float (&c)[4] = cc[u];
          c[0] = c[1] = c[2] = c[3] = 0.f;
#pragma unroll
          for (int kb = 0; kb < KB; ++kb) {
            const int o0 = offL0[j] + 256 * kb, o1 = offL1[j] + 256 * kb;
            uint32_t bh0, bh1, bl0, bl1;
            if constexpr (MODE == 2) {
              bh0 = lds_u32(fBh + o0);
              bh1 = lds_u32(fBh + o1);
              bl0 = lds_u32(fBl + o0);
              bl1 = lds_u32(fBl + o1);
            } else {
              split_tf32(fBh[o0], bh0, bl0);
              split_tf32(fBh[o1], bh1, bl1);
            }
            mma3(c, ah[kb], al[kb], bh0, bh1, bl0, bl1);
          }
          if constexpr (MODE == 3) {
#pragma unroll
            for (int h = 0; h < 4; ++h) c[h] *= scale;
          }
        }
        if (full) {
          store_pair(Ga, Gb, c0 + colj[jp], c0 + colj[jp + 1], tq & 1, cc[0], cc[1]);
        } else {
          store_own(Ga, Gb, c0 + colj[jp], m, oka, okb, cc[0]);
          store_own(Ga, Gb, c0 + colj[jp + 1], m, oka, okb, cc[1]);
        }
        }
        }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.empty[stage]);
        if (++stage == sh.stages) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  }
}

template <int MODE, int R8>
__global__ void __launch_bounds__(kTcNW * 32 + 32, MODE >= 2 ? 2 : 1)
tc_kernel(Tables t, const TcSeg* __restrict__ segs, const int32_t* __restrict__ cta_begin,
          int stages, int stage_floats, float scale) {
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];  // SWIZZLE_128B boxes
  TcShared sh;
  sh.stages = stages;
  sh.stage_floats = stage_floats;
  // 1024-byte aligned ring (the launch reserves the slack)
  sh.ring = reinterpret_cast<float*>(tc_smem_raw + ((1024u - (s32(tc_smem_raw) & 1023u)) & 1023u));
  sh.full = reinterpret_cast<uint64_t*>(sh.ring + (size_t)stages * stage_floats);
  sh.empty = sh.full + stages;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&sh.full[i], 33);      // lane 0's expect-tx arrive + one noinc arrive per lane
      // one arrival per consumer warp (Q-step K1: a box's storer after its store read it)
      mbar_init(&sh.empty[i], kTcNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int sb = cta_begin[blockIdx.x], se = cta_begin[blockIdx.x + 1];
  prefetch_segs(t, segs, sb, se);
  if constexpr (MODE >= 2) {  // NVLS (NEXT-3): sum the fused buffer over the ranks first
    if (t.nvls_fused) nvls_fused_reduce(t, MODE == 2 ? 0 : 1);
  }
  const bool producer = (threadIdx.x >> 5) == kTcNW;
  if constexpr (MODE == 0) {
    if (producer) tcp_producer<R8>(t, segs, sb, se, sh);
    else tcp_consumer<R8>(t, segs, sb, se, sh);
  } else if constexpr (MODE == 1) {
    if (producer) tcq_producer<R8>(t, segs, sb, se, sh);
    else tcq_consumer<R8, (R8 <= 16 ? 2 : 1)>(t, segs, sb, se, sh);
  } else {
    if (producer) tcd_producer<MODE, R8>(t, segs, sb, se, sh);
    else tcd_consumer<MODE, R8>(t, segs, sb, se, sh, scale);
  }
}

// TC state -> E (eager, rare): dst = S - A B^T with A [2][n][R8], B [2][R8][m]
__global__ void tc_materialize_kernel(Tables t, LayerDesc L, int which, float* dst) {
  const int64_t n = L.n, m = L.m;
  const int r = L.r, R8 = t.r8;
  const float* S = t.E + L.e_off;
  const float* A = (which == 1 ? t.psplit : t.plsplit) + L.ps_off;
  const float* B = (which == 1 ? t.qlsplit : t.qsplit) + L.qs_off;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n * m;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / m, j = idx - i * m;
    float x = S[idx];
    for (int k = 0; k < r; ++k) {
      const float a = A[i * R8 + k] + A[(n + i) * R8 + k];
      const float b = B[(int64_t)k * m + j] + B[((int64_t)R8 + k) * m + j];
      x = fmaf(-a, b, x);
    }
    dst[idx] = x;
  }
}

}  // namespace

int tc_p_stage_floats(int r8) { return p_stage_floats(r8); }

int tc_q_map(int64_t m, int r8, TcMap* out) {
  const int cbw = r8 <= 16 ? 2 : 1;
  const int64_t maxpc = (int64_t)16 * cbw * kTcNW;
  const int64_t np = (m + maxpc - 1) / maxpc;
  int64_t pc = (m + np - 1) / np;
  pc = (pc + 31) / 32 * 32;  // whole 32-column boxes: the S store never touches another panel
  const int ncb = (int)(pc / 16);
  const int need = (ncb + cbw - 1) / cbw;
  int wc = 1;
  while (wc < need && wc < kTcNW) wc <<= 1;
  const int wr = kTcNW / wc;
  // >= 2 k-steps per tile; 4 at r = 32 (narrow panels: longer tiles amortise
  // the per-tile handshakes; r = 8 / 16 prefer the deeper ring of 16-row tiles)
  const int ksmin = r8 >= 32 ? 4 : 2;
  const int tr = 8 * (wr > ksmin ? wr : ksmin);
  out->pc = (int32_t)pc;
  out->np = (int16_t)np;
  out->wc = (int16_t)wc;
  out->wr = (int16_t)wr;
  out->tr = (int16_t)tr;
  out->cbw = (int16_t)cbw;
  out->pad_ = 0;
  return q_stage_floats(tr, (int)pc, r8);
}

size_t tc_smem_bytes(int stages, int stage_floats) {
  return (size_t)stages * stage_floats * 4 + (size_t)stages * 16 + 1024;
}

// Host: 2-D fp32 tensor map (inner dim `cols`, `rows` rows, row pitch `cols`
// floats) with a box of 32 columns x box_rows rows, SWIZZLE_128B, zero OOB fill.
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool tc_encode_map(CUtensorMap* out, const float* base, int64_t cols, int64_t rows, int box_rows, bool atom32,
                   int box_cols) {
  std::memset(out, 0, sizeof(CUtensorMap));
  auto enc = tmap_encoder();
  if (!enc || !base || cols % 4 != 0 || (reinterpret_cast<uintptr_t>(base) & 15u) != 0) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  // swizzle span = the box row: 128 B (32 floats), or 64 / 32 B for narrow boxes
  const CUtensorMapSwizzle sw = atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                       : (box_cols == 8 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                        : (box_cols == 16 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                                          : CU_TENSOR_MAP_SWIZZLE_128B));
  const cuuint32_t estr[2] = {1, 1};
  return enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
int tc_p_box_rows() { return kPTR; }

cudaError_t launch_tc(int mode, int r8, const Tables& t, const TcSeg* segs, const int32_t* cb, int ncta,
                      int stages, int stage_floats, float scale, cudaStream_t st) {
  if (ncta <= 0) return cudaSuccess;
  const size_t smem = tc_smem_bytes(stages, stage_floats);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern));
    if (e != cudaSuccess) return e;
    // the NVLS-fused decode barriers its whole grid (k_nvls.cuh): cooperative
    return launch_kernel(kern, dim3(ncta), dim3(kTcNW * 32 + 32), smem, st, mode >= 2 && t.nvls_fused != 0,
                         t, segs, cb, stages, stage_floats, scale);
  };
  switch (mode * 100 + r8) {
    case 8: return go(tc_kernel<0, 8>);
    case 16: return go(tc_kernel<0, 16>);
    case 32: return go(tc_kernel<0, 32>);
    case 108: return go(tc_kernel<1, 8>);
    case 116: return go(tc_kernel<1, 16>);
    case 132: return go(tc_kernel<1, 32>);
    case 208: return go(tc_kernel<2, 8>);
    case 216: return go(tc_kernel<2, 16>);
    case 232: return go(tc_kernel<2, 32>);
    case 308: return go(tc_kernel<3, 8>);
    case 316: return go(tc_kernel<3, 16>);
    case 332: return go(tc_kernel<3, 32>);
    default: return cudaErrorInvalidValue;
  }
}

int tc_d_stage_floats(int r8) { return d_stage_floats(r8); }

cudaError_t launch_tc_materialize(const Tables& t, const LayerDesc& L, int which, float* dst,
                                  cudaStream_t s) {
  if (!L.mat) return cudaSuccess;
  const int64_t total = L.n * L.m;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  tc_materialize_kernel<<<grid, 256, 0, s>>>(t, L, which, dst ? dst : t.E + L.e_off);
  return cudaGetLastError();
}

}  // namespace acp
