// K2 -- orthogonalisation of the reused factors (Alg. 2 P:220 / P:225,
// "Orthogonalize" = reduced-QR Q factor), batched over every layer.
//
// Algorithm: CholeskyQR2 with float64 Gram / Cholesky:
//   phase 0: G1 = A^T A            (partial Gram per 256-row segment, fp64)
//            last segment of the layer: G1 = R1^T R1 (Cholesky), W1 = R1^-1
//   phase 1: A1 = A W1  (columns flagged degenerate replaced by the seeded
//            Gaussian column), G2 = A1^T A1, last segment: W2 = R2^-1
//   phase 2: Q = A1 W2
// Q equals the reduced-QR factor with R_kk > 0 that the oracle's MGS2 computes
// (same column space and orientation; DESIGN.md derives the degenerate case).
// Unlike a per-layer Gram-Schmidt, every phase is a grid-wide data-parallel
// sweep, so a 30522 x 32 factor is spread over 120 CTAs instead of serialising
// 2r dependent reductions on one SM. The Gram partials are summed in a fixed
// order (deterministic: every rank computes bit-identical factors).
#include <algorithm>

#include "k_common.cuh"

namespace acp {
namespace {

constexpr double kDegTol2 = 1e-12;      // (1e-6)^2, reading C6

template <int RT, int SEG>
constexpr size_t orth_smem() {
  constexpr int kLd = SEG + 1;
  const size_t seg = (size_t)2 * RT * kLd * 4 + (size_t)3 * RT * RT * 8 + kThreads * 8 + 16;
  // orth_local: [r][len] floats + Gs / Rm / Wm + per-warp pair sums + mask
  const size_t loc = RT > 8 ? 0
                            : (size_t)4 * ((kOrthLocalFloats + 3) & ~3) + (size_t)3 * RT * RT * 8 +
                                  (size_t)(kThreads / 32) * (RT * (RT + 1) / 2) * 8 + 32;
  return seg > loc ? seg : loc;
}

// Layer `s.layer`'s phase `phase` may start once lflag[layer] >= ready_epoch
// (set by the layer's last segment of the previous phase).
__device__ __forceinline__ long long orth_epoch(int64_t step, int phase) { return step * 4 + phase; }

// Cholesky G = R^T R (R upper) and W = R^-1 of one layer's r x r Gram by one
// warp, with lane l holding column l in registers (RT >= 16; the smem-based
// left-looking version below serialises ~r^2 dependent shared-memory round
// trips, ~20 us at r = 32). Right-looking: at step k the pivot comes from
// lane k by a shuffle, every lane forms its entry of row k of R, and the
// trailing columns are updated with row k broadcast lane by lane. Reading C6
// as in the smem version: a column whose Schur pivot is <= 1e-12 of its
// squared norm (or whose norm is 0) is dropped (row and column of R zero,
// R_kk = 1, W_kk = 0); a non-finite diagonal raises the sticky flag and is
// not repaired. W = R^-1 column by column in registers (lane l:
// back substitution, R rows read from shared memory).
// The factorisation and inverse (one warp); W goes to Wout (global or shared
// memory), mydg = column l dropped, nonfinite = a non-finite diagonal seen.
template <int RT>
__device__ __forceinline__ void chol_regs_core(double* Gs, double* Rm, double* Wout, int r, bool& mydg,
                                               bool& nonfinite) {
  const int l = threadIdx.x & 31;
  double a[RT];  // column l of the (Schur-updated) Gram
#pragma unroll
  for (int i = 0; i < RT; ++i) a[i] = (i < r && l < r) ? Gs[i * r + l] : 0.0;
  double myrinv = 1.0;  // 1 / R_ll (lane l)
#pragma unroll
  for (int k = 0; k < RT; ++k) {
    if (k >= r) break;
    const double dkk = __shfl_sync(0xffffffffu, a[k], k);  // Schur pivot G'[k][k]
    const double gkk = Gs[k * r + k];                      // squared norm of column k
    const bool fin = isfinite(gkk);
    nonfinite |= !fin;
    const bool dg = fin && (!(gkk > 0.0) || !(dkk > kDegTol2 * gkk));
    // reciprocal square root + products: no sqrt and division in the chain
    const double rinv = dg ? 1.0 : rsqrt(dkk);
    const double rkk = dg ? 1.0 : dkk * rinv;
    double rkl = 0.0;  // R[k][l]
    if (l == k) {
      rkl = rkk;
      mydg = dg;
      myrinv = rinv;
    } else if (l > k && l < r) {
      rkl = dg ? 0.0 : a[k] * rinv;
    }
    if (l >= k && l < r) Rm[k * r + l] = rkl;
    if (dg && l < k) Rm[l * r + k] = 0.0;  // a dropped column has no entries above R_kk
#pragma unroll
    for (int i = k + 1; i < RT; ++i) {
      const double rki = __shfl_sync(0xffffffffu, rkl, i);
      if (l > k) a[i] = fma(-rki, rkl, a[i]);
    }
  }
  __syncwarp();
  // the Gram's diagonal is not read again: it holds 1 / R_ii for the
  // back substitution (independent loads instead of divisions in the chain)
  if (l < r) Gs[l * r + l] = myrinv;
  __syncwarp();
  // W = R^-1, column l: w[i] = (delta_il - sum_{i<j<=l} R[i][j] w[j]) / R[i][i]
  double w[RT];
#pragma unroll
  for (int i = RT - 1; i >= 0; --i) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int j = i + 1; j < RT; ++j) {
      if (j <= l && j < r) {
        if ((j - i) & 1) s0 = fma(Rm[i * r + j], w[j], s0);
        else s1 = fma(Rm[i * r + j], w[j], s1);
      }
    }
    w[i] = 0.0;
    if (i < r && i <= l && l < r) {
      const double riinv = Gs[i * r + i];
      // a dropped column l: W_ll = 0 (its output column is replaced by the
      // seeded one); its entries above are 0 either way, since R_il = 0
      w[i] = (i == l) ? (mydg ? 0.0 : riinv) : -(s0 + s1) * riinv;
    }
  }
  if (l < r) {
#pragma unroll
    for (int i = 0; i < RT; ++i)
      if (i < r) Wout[i * r + l] = (i <= l) ? w[i] : 0.0;
  }
}

template <int RT>
__device__ __noinline__ void chol_inv_regs(const Tables& t, const LayerDesc& L, double* Gs, double* Rm,
                                           double* Wout, int r, int phase, int64_t step) {
  const int l = threadIdx.x & 31;
  bool mydg = false, nonfinite = false;
  chol_regs_core<RT>(Gs, Rm, Wout, r, mydg, nonfinite);
  __threadfence();  // every lane's W columns visible before lane 0 publishes (see orth_item)
  __syncwarp();
  const uint32_t dmask = __ballot_sync(0xffffffffu, mydg && l < r);
  const bool anynf = __any_sync(0xffffffffu, nonfinite);
  if (l == 0) {
    if (anynf) atomicOr(t.nonfinite, 1);
    if (phase == 0) t.degmask[L.deg_idx] = dmask;
    t.orthcnt[L.deg_idx] = 0;  // re-arm
    __threadfence();
    // publish: the layer's next phase may start
    *reinterpret_cast<volatile long long*>(t.orthflag + L.deg_idx) = orth_epoch(step, phase + 1);
  }
}

// Cholesky G = R^T R (R upper) and W = R^-1 of one layer's r x r Gram (r <=
// 32) by one warp, lane l owning column l (left-looking; shared memory). A
// degenerate column (residual <= 1e-6 of its norm) is dropped (C6): its row
// and column of R are zero, R_kk = 1, and W_kk = 0 (its output column is
// replaced by the seeded Gaussian one). A non-finite column is NOT repaired
// (non-finite input is an error): it propagates NaN and is
// reported through `nonfinite`. Out: Rm, Wm (r x r, row-major, W upper
// triangular with zeros below), dmask (bit k: column k dropped).
__device__ __forceinline__ void chol_small(double* Gs, double* Rm, double* Wm, int r,
                                           uint32_t& dmask, bool& nonfinite) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < r; ++k) {
    const double gkk = Gs[k * r + k];
    double d = gkk;
    for (int j = 0; j < k; ++j) {
      const double rjk = Rm[j * r + k];
      d = fma(-rjk, rjk, d);
    }
    const bool fin = isfinite(gkk);
    nonfinite |= !fin;
    const bool dg = fin && (!(gkk > 0.0) || !(d > kDegTol2 * gkk));
    // 1 / R_kk by one reciprocal square root, then products: the column
    // step's dependent chain no longer holds a sqrt AND a division (the
    // one-warp Cholesky is most of a small K2 item's latency)
    const double rinv = dg ? 1.0 : rsqrt(d);
    const double rkk = dg ? 1.0 : d * rinv;
    if (dg) dmask |= 1u << k;
    if (lane < r) {
      if (dg) {
        if (lane < k) Rm[lane * r + k] = 0.0;
        else if (lane > k) Rm[k * r + lane] = 0.0;
      } else if (lane > k) {
        double v = Gs[k * r + lane];
        for (int j = 0; j < k; ++j) v = fma(-Rm[j * r + k], Rm[j * r + lane], v);
        Rm[k * r + lane] = v * rinv;
      }
      if (lane == k) Rm[k * r + k] = rkk;
    }
    __syncwarp();
    // G_kk is not read again (later steps read rows k' > k off the
    // diagonal): keep 1 / R_kk there for the back substitution
    if (lane == k) Gs[k * r + k] = rinv;
  }
  __syncwarp();
  if (lane < r) {
    const int l = lane;  // back substitution for column l of W
    for (int i = l; i >= 0; --i) {
      double v = (i == l) ? 1.0 : 0.0;
      for (int j = i + 1; j <= l; ++j) v = fma(-Rm[i * r + j], Wm[j * r + l], v);
      Wm[i * r + l] = v * Gs[i * r + i];
    }
    if ((dmask >> l) & 1u) Wm[l * r + l] = 0.0;
    for (int i = l + 1; i < r; ++i) Wm[i * r + l] = 0.0;
  }
  __syncwarp();
}

// The seeded Gaussian entry that replaces column l of a factor whose
// column l was dropped (reading C6); out of line (rare path, large body).
__device__ __noinline__ double degenerate_value(uint64_t seed, int layer, int64_t step, int l, int64_t row) {
  return (double)gaussian_at(column_key(seed, kTagDegenerate, (uint64_t)layer, (uint64_t)step, (uint64_t)l),
                             (uint64_t)row);
}

// One (phase, segment) work item of K2. Returns after the item; the layer's
// last segment of phases 0 / 1 also computes W1 / W2 and publishes the
// layer's next phase through lflag.
template <int RT, int SEG>
__device__ void orth_item(const Tables& t, int side, const OrthSeg& s, int phase, uint64_t seed,
                          int64_t step, unsigned char* orth_smem_raw) {
  constexpr int kSeg = SEG;       // rows staged per CTA (one shot)
  constexpr int kLd = kSeg + 1;   // padded smem row (bank spread)
  float* A = reinterpret_cast<float*>(orth_smem_raw);  // [RT][kLd] input rows (fp32)
  float* B = A + RT * kLd;                               // [RT][kLd] phase-1 output rows
  double* Wm = reinterpret_cast<double*>(B + RT * kLd);  // [RT*RT]
  double* Gs = Wm + RT * RT;
  double* Rm = Gs + RT * RT;
  double* gred = Rm + RT * RT;                            // [kThreads]
  int* flag = reinterpret_cast<int*>(gred + kThreads);

  const LayerDesc L = t.layers[s.layer];
  const int r = L.r;
  const int64_t len = side == 0 ? L.m : L.n;
  float* F = side == 0 ? t.qbuf + L.q_off : t.pbuf + L.p_off;  // k-major [r][len]
  double* W1 = t.wmat + L.w_off;
  double* W2 = W1 + r * r;
  const int tid = threadIdx.x;
  const int nr = (int)(s.row1 - s.row0);
  if (phase > 0) {  // wait for the layer's previous phase (W1 / W2 published)
    if (tid == 0) {
      volatile long long* f = t.orthflag + L.deg_idx;
      const long long want = orth_epoch(step, phase);
      const uint64_t t0 = globaltimer_ns();
      while (*f < want) {
        __nanosleep(64);
        if (globaltimer_ns() - t0 > kSpinLimitNs) __trap();  // broken epoch: fail loudly
      }
      __threadfence();
    }
    __syncthreads();
  }

  // stage the segment's rows (coalesced along rows, k-major source). F, W and
  // degmask are rewritten inside this launch by other SMs (phase 1 writes F in
  // place), so every load of them bypasses L1 (__ldcg): a line this SM cached
  // in an earlier phase would otherwise be read back stale.
  for (int idx = tid; idx < r * kSeg; idx += kThreads) {
    const int k = idx / kSeg, i = idx - k * kSeg;
    A[k * kLd + i] = i < nr ? __ldcg(F + (int64_t)k * len + s.row0 + i) : 0.f;
  }
  uint32_t deg = 0;
  if (phase > 0) {
    const double* Wsrc = phase == 1 ? W1 : W2;
    for (int i = tid; i < r * r; i += kThreads) Wm[i] = __ldcg(Wsrc + i);
    if (phase == 1) deg = __ldcg(t.degmask + L.deg_idx);
  }
  __syncthreads();
  const float* G = A;  // rows the Gram is taken of
  if (RT >= 16 && phase > 0) {
    // r >= 16: thread per row, the row's r values in registers (one fp32 ->
    // fp64 conversion each) and W zero-padded to RT x RT in shared memory
    // (compile-time offsets, broadcast reads), fully unrolled so the r
    // independent output chains interleave. The element-per-thread loop
    // below re-reads and re-converts a_k for every output column and runs
    // each output's dependent chain back to back: r = 32 items of 20-35 us.
    double* Wp = Gs;  // Gs is free until this item's Gram (last segment)
    for (int idx = tid; idx < RT * RT; idx += kThreads) {
      const int k = idx / RT, l = idx - k * RT;
      Wp[idx] = (k < r && l < r) ? Wm[k * r + l] : 0.0;
    }
    __syncthreads();
    for (int i = tid; i < kSeg; i += kThreads) {
      double a[RT];
#pragma unroll
      for (int k = 0; k < RT; ++k) a[k] = (k < r && i < nr) ? (double)A[k * kLd + i] : 0.0;
      const int64_t row = s.row0 + i;
#pragma unroll
      for (int l0 = 0; l0 < RT; l0 += 4) {
        float vf[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int l = l0 + u;
          double v = 0.0;
#pragma unroll
          for (int k = 0; k <= l; ++k) v = fma(a[k], Wp[k * RT + l], v);
          if ((deg >> l) & 1u) v = degenerate_value(seed, s.layer, step, l, row);
          vf[u] = (i < nr && l < r) ? (float)v : 0.f;
          B[l * kLd + i] = vf[u];
          if (i < nr && l < r) F[(int64_t)l * len + row] = vf[u];
        }
        if (phase == 2 && t.r8 > 0 && i < nr) {
          // TC path split copies (Q side k-major [2][R8][m], P side row-major
          // [2][n][R8]: four consecutive columns -> one 16-byte store each)
          const int64_t R8 = t.r8;
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) split_tf32(vf[u], hi[u], lo[u]);
          if (side == 0) {
            float* d = t.qsplit + L.qs_off;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (l0 + u < r) {
                d[(l0 + u) * len + row] = __uint_as_float(hi[u]);
                d[(R8 + l0 + u) * len + row] = __uint_as_float(lo[u]);
              }
            }
          } else if (l0 < r) {
            float* d = t.psplit + L.ps_off;
            // columns l0 .. l0 + 3 < R8 (R8 is a multiple of 8); beyond r the
            // split of 0 is 0, as the slot's padding expects
            *reinterpret_cast<float4*>(d + row * R8 + l0) =
                make_float4(__uint_as_float(hi[0]), __uint_as_float(hi[1]), __uint_as_float(hi[2]),
                            __uint_as_float(hi[3]));
            *reinterpret_cast<float4*>(d + (len + row) * R8 + l0) =
                make_float4(__uint_as_float(lo[0]), __uint_as_float(lo[1]), __uint_as_float(lo[2]),
                            __uint_as_float(lo[3]));
          }
        }
      }
    }
    if (phase == 2) {
      __syncthreads();  // smem reuse by the CTA's next item
      return;
    }
    __syncthreads();
    G = B;
  } else if (phase > 0) {
    // apply W (upper triangular): out_l = sum_{k<=l} a_k W_kl; a column
    // flagged degenerate becomes the seeded Gaussian column (reading C6)
    for (int idx = tid; idx < r * kSeg; idx += kThreads) {
      const int l = idx / kSeg, i = idx - l * kSeg;
      float vf = 0.f;
      if (i < nr) {
        double v = 0.0;
        if ((deg >> l) & 1u) {
          v = (double)gaussian_at(column_key(seed, kTagDegenerate, (uint64_t)s.layer,
                                             (uint64_t)step, (uint64_t)l),
                                  (uint64_t)(s.row0 + i));
        } else {
          for (int k = 0; k <= l; ++k) v = fma((double)A[k * kLd + i], Wm[k * r + l], v);
        }
        vf = (float)v;
        F[(int64_t)l * len + s.row0 + i] = vf;
        if (phase == 2 && t.r8 > 0) {
          // TC path: 3xTF32 split copies (Q side k-major [2][R8][m], P side
          // row-major [2][n][R8]) for the tensor-core K1 kernels
          uint32_t hi, lo;
          split_tf32(vf, hi, lo);
          const int64_t row = s.row0 + i, R8 = t.r8;
          if (side == 0) {
            float* d = t.qsplit + L.qs_off;
            d[l * len + row] = __uint_as_float(hi);
            d[(R8 + l) * len + row] = __uint_as_float(lo);
          } else {
            float* d = t.psplit + L.ps_off;
            d[row * R8 + l] = __uint_as_float(hi);
            d[(len + row) * R8 + l] = __uint_as_float(lo);
          }
        }
      }
      B[l * kLd + i] = vf;
    }
    if (phase == 2) {
      __syncthreads();  // smem reuse by the CTA's next item
      return;
    }
    __syncthreads();
    G = B;
  }

  // partial Gram of this segment (fp64): pair pi <-> (k, l), l <= k, with
  // S row splits per pair
  const int NP = r * (r + 1) / 2;
  const int S = NP <= kThreads ? kThreads / NP : 1;
  const int sp = NP <= kThreads ? tid % S : 0;
  double* part = t.gram + s.gram_off;
  if constexpr (RT >= 16) {
    // 4 x 4 register blocks over the full RT x RT Gram (RT = 32: 64 blocks
    // x 4 row splits; RT = 16: 16 blocks x 16 splits; splits summed by
    // shuffles): 8 shared loads + 8 fp32 -> fp64 conversions per 16 DFMA.
    // (2 x 2 blocks took one conversion per DFMA; the F2F rate bound the
    // r = 32 Gram.) Lanes of a warp read 8 consecutive column blocks at 4
    // consecutive rows: conflict-free with the padded row stride.
    constexpr int BS = 4, BPR = RT / BS, NB = BPR * BPR, SB = kThreads / NB;
    static_assert(NB * SB == kThreads && (SB & (SB - 1)) == 0 && SB <= 32, "Gram block split");
    const int bk = (tid / SB) / BPR, bl = (tid / SB) % BPR, ss = tid % SB;
    const int k0 = BS * bk, l0 = BS * bl;
    const float* gk[BS];
    const float* gl[BS];
#pragma unroll
    for (int u = 0; u < BS; ++u) {
      gk[u] = G + (k0 + u < r ? k0 + u : 0) * kLd;
      gl[u] = G + (l0 + u < r ? l0 + u : 0) * kLd;
    }
    double c[BS][BS];
#pragma unroll
    for (int u = 0; u < BS; ++u)
#pragma unroll
      for (int v = 0; v < BS; ++v) c[u][v] = 0.0;
    for (int i = ss; i < nr; i += SB) {
      double a[BS], b[BS];
#pragma unroll
      for (int u = 0; u < BS; ++u) {
        a[u] = gk[u][i];
        b[u] = gl[u][i];
      }
#pragma unroll
      for (int u = 0; u < BS; ++u)
#pragma unroll
        for (int v = 0; v < BS; ++v) c[u][v] = fma(a[u], b[v], c[u][v]);
    }
#pragma unroll
    for (int off = SB / 2; off > 0; off >>= 1)
#pragma unroll
      for (int u = 0; u < BS; ++u)
#pragma unroll
        for (int v = 0; v < BS; ++v) c[u][v] += __shfl_down_sync(0xffffffffu, c[u][v], off, SB);
    if (ss == 0) {
#pragma unroll
      for (int u = 0; u < BS; ++u)
#pragma unroll
        for (int v = 0; v < BS; ++v)
          if (k0 + u < r && l0 + v < r) part[(k0 + u) * r + l0 + v] = c[u][v];
    }
  } else if (NP <= kThreads) {
    const int pi = tid / S;
    double a = 0.0;
    int k = 0, l = 0;
    if (pi < NP) {
      while ((k + 1) * (k + 2) / 2 <= pi) ++k;
      l = pi - k * (k + 1) / 2;
      for (int i = sp; i < nr; i += S) a = fma((double)G[k * kLd + i], (double)G[l * kLd + i], a);
    }
    gred[tid] = a;
    __syncthreads();
    if (sp == 0 && pi < NP) {
      double g = 0.0;
      for (int j = 0; j < S; ++j) g += gred[tid + j];
      part[k * r + l] = g;
      part[l * r + k] = g;
    }
  } else {
    for (int pi = tid; pi < NP; pi += kThreads) {
      int k = 0;
      while ((k + 1) * (k + 2) / 2 <= pi) ++k;
      const int l = pi - k * (k + 1) / 2;
      double a = 0.0;
      for (int i = 0; i < nr; ++i) a = fma((double)G[k * kLd + i], (double)G[l * kLd + i], a);
      part[k * r + l] = a;
      part[l * r + k] = a;
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int old = atomicAdd(t.orthcnt + L.deg_idx, 1);
    *flag = (old == s.nseg - 1);
  }
  __syncthreads();
  const int last = *flag;
  __syncthreads();  // *flag is rewritten by the CTA's next item
  if (!last) return;
  __threadfence();

  // last segment of the layer: sum the partials in segment order
  const double* gbase = t.gram + (s.gram_off - (int64_t)s.seg * r * r);
  for (int idx = tid; idx < r * r; idx += kThreads) {
    double g = 0.0;
    for (int j = 0; j < s.nseg; ++j) g += __ldcg(gbase + (int64_t)j * r * r + idx);
    Gs[idx] = g;
    Rm[idx] = 0.0;
  }
  __syncthreads();
  if constexpr (RT >= 16) {
    if (tid < 32) chol_inv_regs<RT>(t, L, Gs, Rm, phase == 0 ? W1 : W2, r, phase, step);
  } else if (tid < 32) {
    const int lane = tid;
    uint32_t dmask = 0;
    bool nonfinite = false;
    chol_small(Gs, Rm, Wm, r, dmask, nonfinite);
    double* Wout = phase == 0 ? W1 : W2;
    if (lane < r) {
      const int l = lane;
      for (int i = 0; i < r; ++i) Wout[i * r + l] = Wm[i * r + l];
    }
    // every lane's W columns must be visible GPU-wide before lane 0 publishes
    // the flag the next phase's items (other SMs) wait on: without this, lane
    // 0 could publish while lanes 1..r-1 had not stored (or made visible)
    // their columns, and a phase-1/2 item read a stale column of W (left by
    // the previous K2 launch) -- a rare ~2e-4 full-size parity failure
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      if (nonfinite) atomicOr(t.nonfinite, 1);
      if (phase == 0) t.degmask[L.deg_idx] = dmask;
      t.orthcnt[L.deg_idx] = 0;  // re-arm
      __threadfence();
      // publish: the layer's next phase may start
      *reinterpret_cast<volatile long long*>(t.orthflag + L.deg_idx) = orth_epoch(step, phase + 1);
    }
  }
  __syncthreads();
}

// K2 of one whole small factor (r * len <= kOrthLocalFloats, r <= 8) in one
// CTA: the same three CholeskyQR2 steps as orth_item, with __syncthreads
// between them instead of the cross-CTA epoch flags and partial Grams (a
// ResNet layer's three phases otherwise cost three queue rounds and two
// flag hand-offs for a few microseconds of arithmetic). Same arithmetic per
// element: fp64 Gram of the fp32 rows, fp64 apply rounded to fp32, the
// degenerate-column rule (C6) on the first Cholesky only.
template <int RT>
__device__ void orth_local(const Tables& t, int side, const OrthSeg& s, uint64_t seed, int64_t step,
                           unsigned char* smem_raw) {
  constexpr int NP = RT * (RT + 1) / 2;
  constexpr int NWP = kThreads / 32;
  const LayerDesc L = t.layers[s.layer];
  const int r = L.r;
  const int len = (int)(side == 0 ? L.m : L.n);
  float* F = side == 0 ? t.qbuf + L.q_off : t.pbuf + L.p_off;  // k-major [r][len]
  float* A = reinterpret_cast<float*>(smem_raw);                 // [r][len]
  double* Gs = reinterpret_cast<double*>(smem_raw + 4 * ((kOrthLocalFloats + 3) & ~3));
  double* Rm = Gs + RT * RT;
  double* Wm = Rm + RT * RT;
  double* red = Wm + RT * RT;                                    // [NWP][NP]
  uint32_t* dsh = reinterpret_cast<uint32_t*>(red + NWP * NP);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total = r * len;
  // stage the factor (contiguous k-major [r][len]) with ONE bulk copy: an
  // item of 4608 x 4 spent ~15k cycles in 18 rounds of dependent 4-byte
  // loads. The size is rounded up to 16 bytes (the arena slots are 16-byte
  // aligned and padded, so the tail stays inside the arena).
  {
    uint64_t* bar = reinterpret_cast<uint64_t*>(dsh + 2);
    const uint32_t bytes = (uint32_t)(((total + 3) & ~3) * 4);
    if (tid == 0) {
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      fence_async_smem();  // generic-proxy writes to A by the previous item
      mbar_arrive_tx(bar, bytes);
      bulk_g2s(A, F, bytes, bar, policy_evict_first());
    }
    __syncthreads();
    mbar_wait(bar, 0);
  }
  bool nonfinite = false;
  uint32_t deg = 0;
  for (int pass = 0; pass < 2; ++pass) {
    // Gram of the current rows (fp64): rows strided over the threads, all
    // pairs (k <= l) per thread, then a fixed-order warp / CTA reduction
    double g[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) g[p] = 0.0;
    for (int i = tid; i < len; i += kThreads) {
      double a[RT];
#pragma unroll
      for (int k = 0; k < RT; ++k) a[k] = k < r ? (double)A[k * len + i] : 0.0;
#pragma unroll
      for (int k = 0, p = 0; k < RT; ++k)
#pragma unroll
        for (int l = 0; l <= k; ++l, ++p) g[p] = fma(a[k], a[l], g[p]);
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) g[p] += __shfl_xor_sync(0xffffffffu, g[p], off);
    }
    if (lane == 0) {
#pragma unroll
      for (int p = 0; p < NP; ++p) red[warp * NP + p] = g[p];
    }
    __syncthreads();
    for (int p = tid; p < NP; p += kThreads) {
      int k = 0;
      while ((k + 1) * (k + 2) / 2 <= p) ++k;
      const int l = p - k * (k + 1) / 2;
      double v = 0.0;
      for (int w = 0; w < NWP; ++w) v += red[w * NP + p];
      if (k < r && l < r) {
        Gs[k * r + l] = v;
        Gs[l * r + k] = v;
      }
    }
    for (int i = tid; i < r * r; i += kThreads) Rm[i] = 0.0;
    __syncthreads();
    if (warp == 0) {
      uint32_t dmask = 0;
      if constexpr (RT <= 4) {
        // register right-looking Cholesky (shuffles, no shared-memory chains):
        // ResNet-50 K2 26.4 -> 23.9 us, BERT-L r=4 42 -> 39; at RT = 8 its
        // registers (190) halve the kernel's occupancy and it is slower
        bool mydg = false;
        chol_regs_core<RT>(Gs, Rm, Wm, r, mydg, nonfinite);
        dmask = __ballot_sync(0xffffffffu, mydg && lane < r);
        __syncwarp();
      } else {
        chol_small(Gs, Rm, Wm, r, dmask, nonfinite);
      }
      if (lane == 0 && pass == 0) *dsh = dmask;
    }
    __syncthreads();
    if (pass == 0) deg = *dsh;
    // apply W (upper triangular), thread per row: out_l = sum_{k<=l} a_k W_kl;
    // after the first Cholesky a dropped column becomes the seeded Gaussian
    // column (reading C6); the second apply's output is the factor
    for (int i = tid; i < len; i += kThreads) {
      double a[RT];
#pragma unroll
      for (int k = 0; k < RT; ++k) a[k] = k < r ? (double)A[k * len + i] : 0.0;
#pragma unroll
      for (int l = 0; l < RT; ++l) {
        if (l >= r) break;
        double v = 0.0;
        if (pass == 0 && ((deg >> l) & 1u)) {
          v = (double)gaussian_at(column_key(seed, kTagDegenerate, (uint64_t)s.layer, (uint64_t)step,
                                             (uint64_t)l),
                                  (uint64_t)i);
        } else {
#pragma unroll
          for (int k = 0; k <= l; ++k) v = fma(a[k], Wm[k * r + l], v);
        }
        const float vf = (float)v;
        if (pass == 0) {
          A[l * len + i] = vf;  // this thread's row only: read above, in place
        } else {
          F[(int64_t)l * len + i] = vf;
          if (t.r8 > 0) {  // TC path split copies (as orth_item's phase 2)
            uint32_t hi, lo;
            split_tf32(vf, hi, lo);
            const int64_t row = i, R8 = t.r8;
            if (side == 0) {
              float* d = t.qsplit + L.qs_off;
              d[l * len + row] = __uint_as_float(hi);
              d[(R8 + l) * len + row] = __uint_as_float(lo);
            } else {
              float* d = t.psplit + L.ps_off;
              d[row * R8 + l] = __uint_as_float(hi);
              d[(len + row) * R8 + l] = __uint_as_float(lo);
            }
          }
        }
      }
    }
    __syncthreads();
  }
  if (warp == 0) {
    if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(t.nonfinite, 1);
  }
}

// K2 as one persistent launch: CTAs take (phase, segment) items from a queue
// ordered by phase (all phase-0 items first), so an item only ever waits on
// items dequeued before it (no deadlock) and a layer's phases follow each
// other without a grid-wide barrier or a kernel boundary. The last CTA to
// exit re-arms the queue and advances the step counter (every CTA read it).
template <int RT, int SEG>
__global__ void __launch_bounds__(kThreads) orth_kernel(Tables t, int side,
                                                        const OrthSeg* __restrict__ segs, int nseg,
                                                        uint64_t seed) {
  extern __shared__ __align__(16) unsigned char orth_smem_raw[];
  __shared__ int item_sh;
  const int64_t step = *t.step;
  const int total = 3 * nseg;
  int* work = t.orthwork;  // [0] next item, [1] exited CTAs
  for (;;) {
    if (threadIdx.x == 0) item_sh = atomicAdd(work, 1);
    __syncthreads();
    const int it = item_sh;
    __syncthreads();
    if (it >= total) break;
    const int phase = it / nseg;
    const OrthSeg& sg = segs[it - phase * nseg];
    if (sg.local) {  // whole small factor in this CTA (phase-0 pass only)
      if constexpr (RT <= 8) {
        if (phase == 0) orth_local<RT>(t, side, sg, seed, step, orth_smem_raw);
      }
      continue;
    }
    orth_item<RT, SEG>(t, side, sg, phase, seed, step, orth_smem_raw);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(work + 1, 1) == (int)gridDim.x - 1) {
      work[0] = 0;
      work[1] = 0;
      *t.step = step + 1;
      __threadfence();
    }
  }
}

__global__ void fill_kernel(Tables t, int side, uint64_t seed, int tag, int64_t step) {
  if (step < 0) step = *t.step;
  const int layer = blockIdx.y;
  const LayerDesc L = t.layers[layer];
  if (!L.mat) return;
  const int64_t len = side == 1 ? L.n : L.m;
  float* F = side == 1 ? t.pbuf + L.p_off : t.qbuf + L.q_off;
  const int64_t total = (int64_t)L.r * len;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx / len, i = idx - k * len;
    F[idx] = gaussian_at(column_key(seed, (uint64_t)tag, (uint64_t)layer, (uint64_t)step,
                                    (uint64_t)k), (uint64_t)i);
  }
}

// deferred state -> E: dst = S - P Q_loc^T for one matrix layer
__global__ void materialize_kernel(Tables t, int layer, float* dst) {
  const LayerDesc L = t.layers[layer];
  const int64_t n = L.n, m = L.m;
  const int r = L.r;
  const float* S = t.E + L.e_off;
  const float* P = t.pbuf + L.p_off;
  const float* Ql = t.qloc + L.ql_off;
  if (!dst) dst = t.E + L.e_off;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n * m;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / m, j = idx - i * m;
    float x = S[idx];
    for (int k = 0; k < r; ++k) x = fmaf(-P[k * n + i], Ql[k * m + j], x);
    dst[idx] = x;
  }
}

__global__ void finite_scan_kernel(const float* __restrict__ buf, int64_t n, int32_t* flag) {
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(buf[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 2);
}

__global__ void transpose_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                 int64_t rows, int r, int to_kmajor) {
  const int64_t total = rows * r;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / r, k = idx - i * r;  // row-major index (i, k)
    if (to_kmajor) dst[k * rows + i] = src[idx];
    else dst[idx] = src[k * rows + i];
  }
}

}  // namespace

cudaError_t launch_orth(int rt, int seg_rows, const Tables& t, int side, const OrthSeg* segs, int nseg,
                        uint64_t seed, int64_t step, cudaStream_t s, int* launches, int busy_items) {
  if (nseg <= 0) return cudaSuccess;
  if (seg_rows != kOrthRowsPerSeg && (seg_rows != kOrthRowsPerSegLarge || rt > 4))
    return cudaErrorInvalidValue;
  (void)step;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  auto go = [&](auto kern, size_t smem) -> cudaError_t {
    cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern));
    if (e != cudaSuccess) return e;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
    // every CTA must be resident (items wait on each other): at most one wave;
    // and no more CTAs than items that do work (whole-factor items leave
    // two skip entries each in the phase-ordered queue)
    const int items = busy_items > 0 ? std::min(busy_items, 3 * nseg) : 3 * nseg;
    const int grid = std::max(1, std::min(items, nsm * std::max(1, occ)));
    kern<<<grid, kThreads, smem, s>>>(t, side, segs, nseg, seed);
    return cudaGetLastError();
  };
  cudaError_t e;
  switch (rt) {
    case 1:
      e = seg_rows == kOrthRowsPerSegLarge
              ? go(orth_kernel<1, kOrthRowsPerSegLarge>, orth_smem<1, kOrthRowsPerSegLarge>())
              : go(orth_kernel<1, kOrthRowsPerSeg>, orth_smem<1, kOrthRowsPerSeg>());
      break;
    case 2:
      e = seg_rows == kOrthRowsPerSegLarge
              ? go(orth_kernel<2, kOrthRowsPerSegLarge>, orth_smem<2, kOrthRowsPerSegLarge>())
              : go(orth_kernel<2, kOrthRowsPerSeg>, orth_smem<2, kOrthRowsPerSeg>());
      break;
    case 4:
      e = seg_rows == kOrthRowsPerSegLarge
              ? go(orth_kernel<4, kOrthRowsPerSegLarge>, orth_smem<4, kOrthRowsPerSegLarge>())
              : go(orth_kernel<4, kOrthRowsPerSeg>, orth_smem<4, kOrthRowsPerSeg>());
      break;
    case 8: e = go(orth_kernel<8, kOrthRowsPerSeg>, orth_smem<8, kOrthRowsPerSeg>()); break;
    case 16: e = go(orth_kernel<16, kOrthRowsPerSeg>, orth_smem<16, kOrthRowsPerSeg>()); break;
    case 32: e = go(orth_kernel<32, kOrthRowsPerSeg>, orth_smem<32, kOrthRowsPerSeg>()); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  if (launches) ++*launches;
  return cudaSuccess;
}

cudaError_t launch_fill(const Tables& t, const LayerDesc* host_layers, int num_tensors, int side,
                        uint64_t seed, int tag, int64_t step, cudaStream_t s, int* launches) {
  int64_t maxel = 0;
  for (int i = 0; i < num_tensors; ++i) {
    const LayerDesc& L = host_layers[i];
    if (!L.mat) continue;
    const int64_t el = (int64_t)L.r * (side == 1 ? L.n : L.m);
    if (el > maxel) maxel = el;
  }
  if (maxel == 0) return cudaSuccess;
  int64_t bx = (maxel + kThreads - 1) / kThreads;
  if (bx > 1024) bx = 1024;
  dim3 grid((unsigned)bx, (unsigned)num_tensors);
  fill_kernel<<<grid, kThreads, 0, s>>>(t, side, seed, tag, step);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_materialize(const Tables& t, const LayerDesc& L, int layer, float* dst,
                               cudaStream_t s) {
  const int64_t total = L.n * L.m;
  if (!L.mat || total == 0) return cudaSuccess;
  int64_t blocks = (total + kThreads - 1) / kThreads;
  if (blocks > 8192) blocks = 8192;
  materialize_kernel<<<(unsigned)blocks, kThreads, 0, s>>>(t, layer, dst);
  return cudaGetLastError();
}

cudaError_t launch_finite_scan(const float* buf, int64_t n, int32_t* flag, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + kThreads - 1) / kThreads;
  if (blocks > 1184) blocks = 1184;
  finite_scan_kernel<<<(unsigned)blocks, kThreads, 0, s>>>(buf, n, flag);
  return cudaGetLastError();
}

cudaError_t launch_transpose(const float* src, float* dst, int64_t rows, int r, int to_kmajor,
                             cudaStream_t s) {
  const int64_t total = rows * r;
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + kThreads - 1) / kThreads;
  if (blocks > 4096) blocks = 4096;
  transpose_kernel<<<(unsigned)blocks, kThreads, 0, s>>>(src, dst, rows, r, to_kmajor);
  return cudaGetLastError();
}

}  // namespace acp
