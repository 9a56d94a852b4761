// K2 -- orthogonalisation of the reused factors (Alg. 2 P:220 / P:225,
// "Orthogonalize" = reduced-QR Q factor), batched over every layer.
//
// Algorithm: CholeskyQR2 with float64 Gram / Cholesky:
//   phase 0: G1 = A^T A            (partial Gram per 1024-row segment, fp64)
//            last segment of the layer: G1 = R1^T R1 (Cholesky), W1 = R1^-1
//   phase 1: A1 = A W1  (columns flagged degenerate replaced by the seeded
//            Gaussian column), G2 = A1^T A1, last segment: W2 = R2^-1
//   phase 2: Q = A1 W2
// Q equals the reduced-QR factor with R_kk > 0 that the oracle's MGS2 computes
// (same column space and orientation; DESIGN.md derives the degenerate case).
// Unlike a per-layer Gram-Schmidt, every phase is a grid-wide data-parallel
// sweep, so a 30522 x 32 factor is spread over 30 CTAs instead of serialising
// 2r dependent reductions on one SM. The Gram partials are summed in a fixed
// order (deterministic: every rank computes bit-identical factors).
#include "k_common.cuh"

namespace acp {
namespace {

constexpr int kCH = 32;              // factor rows staged per round
constexpr double kDegTol2 = 1e-12;   // (1e-6)^2, reading C6

template <int RT>
__global__ void __launch_bounds__(kThreads) orth_kernel(Tables t, int side,
                                                        const OrthSeg* __restrict__ segs,
                                                        int phase, uint64_t seed, int64_t step) {
  __shared__ double A[RT][kCH + 1];
  __shared__ double B[RT][kCH + 1];
  __shared__ double Wm[RT * RT];
  __shared__ double Gs[RT * RT];
  __shared__ double Rm[RT * RT];
  __shared__ double gred[kThreads];
  __shared__ int flag;

  const OrthSeg s = segs[blockIdx.x];
  const LayerDesc L = t.layers[s.layer];
  const int r = L.r;
  const int64_t len = side == 0 ? L.m : L.n;
  float* F = side == 0 ? t.qbuf + L.q_off : t.pbuf + L.p_off;  // k-major [r][len]
  double* W1 = t.wmat + L.w_off;
  double* W2 = W1 + r * r;
  const int tid = threadIdx.x;

  uint32_t deg = 0;
  if (phase > 0) {
    const double* Wsrc = phase == 1 ? W1 : W2;
    for (int i = tid; i < r * r; i += kThreads) Wm[i] = Wsrc[i];
    if (phase == 1) deg = t.degmask[L.deg_idx];
  }

  // Gram pair assignment: pair pi <-> (k, l), l <= k; S row splits per pair
  const int NP = r * (r + 1) / 2;
  const int S = NP <= kThreads ? kThreads / NP : 1;
  int pk[3], pl[3], npairs = 0;
  const int sp = NP <= kThreads ? tid % S : 0;
  for (int j = 0; j < 3; ++j) {
    const int pi = NP <= kThreads ? (j == 0 ? tid / S : NP) : tid + j * kThreads;
    if (pi < NP) {
      int k = 0;
      while ((k + 1) * (k + 2) / 2 <= pi) ++k;
      pk[npairs] = k;
      pl[npairs] = pi - k * (k + 1) / 2;
      ++npairs;
    }
  }
  double acc[3] = {0.0, 0.0, 0.0};

  for (int64_t ch0 = s.row0; ch0 < s.row1; ch0 += kCH) {
    const int nr = (int)((s.row1 - ch0) < kCH ? (s.row1 - ch0) : kCH);
    __syncthreads();
    for (int idx = tid; idx < r * kCH; idx += kThreads) {
      const int k = idx / kCH, i = idx - k * kCH;
      A[k][i] = i < nr ? (double)F[(int64_t)k * len + ch0 + i] : 0.0;
    }
    __syncthreads();
    if (phase > 0) {
      for (int idx = tid; idx < r * kCH; idx += kThreads) {
        const int l = idx / kCH, i = idx - l * kCH;
        double v = 0.0;
        if (i < nr) {
          if ((deg >> l) & 1u) {
            v = (double)gaussian_at(column_key(seed, kTagDegenerate, (uint64_t)s.layer,
                                               (uint64_t)step, (uint64_t)l),
                                    (uint64_t)(ch0 + i));
          } else {
            for (int k = 0; k <= l; ++k) v = fma(A[k][i], Wm[k * r + l], v);
          }
          const float vf = (float)v;
          F[(int64_t)l * len + ch0 + i] = vf;
          v = (double)vf;
        }
        B[l][i] = v;
      }
      __syncthreads();
    }
    if (phase < 2) {
      for (int j = 0; j < npairs; ++j) {
        const int k = pk[j], l = pl[j];
        double a = acc[j];
        if (phase == 0) {
          for (int i = sp; i < nr; i += S) a = fma(A[k][i], A[l][i], a);
        } else {
          for (int i = sp; i < nr; i += S) a = fma(B[k][i], B[l][i], a);
        }
        acc[j] = a;
      }
    }
  }
  if (phase == 2) return;

  // partial Gram of this segment (full symmetric r x r)
  double* part = t.gram + s.gram_off;
  if (NP <= kThreads) {
    gred[tid] = acc[0];
    __syncthreads();
    if (sp == 0 && npairs > 0) {
      double g = 0.0;
      for (int j = 0; j < S; ++j) g += gred[tid + j];
      part[pk[0] * r + pl[0]] = g;
      part[pl[0] * r + pk[0]] = g;
    }
  } else {
    for (int j = 0; j < npairs; ++j) {
      part[pk[j] * r + pl[j]] = acc[j];
      part[pl[j] * r + pk[j]] = acc[j];
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int old = atomicAdd(t.orthcnt + L.deg_idx, 1);
    flag = (old == s.nseg - 1);
  }
  __syncthreads();
  if (!flag) return;
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
  if (tid < 32) {
    const int lane = tid;
    uint32_t dmask = 0;
    // left-looking Cholesky G = R^T R (R upper), lane l owns column l;
    // a degenerate column (residual <= 1e-6 of its norm) is dropped (C6)
    for (int k = 0; k < r; ++k) {
      const double gkk = Gs[k * r + k];
      double d = gkk;
      for (int j = 0; j < k; ++j) {
        const double rjk = Rm[j * r + k];
        d = fma(-rjk, rjk, d);
      }
      const bool dg = !(gkk > 0.0) || !(d > kDegTol2 * gkk);
      const double rkk = dg ? 1.0 : sqrt(d);
      if (dg) dmask |= 1u << k;
      if (lane < r) {
        if (dg) {
          if (lane < k) Rm[lane * r + k] = 0.0;
          else if (lane > k) Rm[k * r + lane] = 0.0;
        } else if (lane > k) {
          double v = Gs[k * r + lane];
          for (int j = 0; j < k; ++j) v = fma(-Rm[j * r + k], Rm[j * r + lane], v);
          Rm[k * r + lane] = v / rkk;
        }
        if (lane == k) Rm[k * r + k] = rkk;
      }
      __syncwarp();
    }
    // W = R^-1 (upper triangular), lane l solves column l; W_kk = 0 for a
    // dropped column (its output column is replaced by a seeded one)
    double* Wout = phase == 0 ? W1 : W2;
    if (lane < r) {
      const int l = lane;
      for (int i = l; i >= 0; --i) {
        double v = (i == l) ? 1.0 : 0.0;
        for (int j = i + 1; j <= l; ++j) v = fma(-Rm[i * r + j], Wm[j * r + l], v);
        Wm[i * r + l] = v / Rm[i * r + i];
      }
      for (int i = 0; i < r; ++i) {
        double w = i <= l ? Wm[i * r + l] : 0.0;
        if (((dmask >> l) & 1u) && i == l) w = 0.0;
        Wout[i * r + l] = w;
      }
    }
    if (lane == 0) {
      if (phase == 0) t.degmask[L.deg_idx] = dmask;
      t.orthcnt[L.deg_idx] = 0;  // re-arm
    }
  }
}

__global__ void fill_kernel(Tables t, int side, uint64_t seed, int tag, int64_t step) {
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

cudaError_t launch_orth(int rt, const Tables& t, int side, const OrthSeg* segs, int nseg,
                        uint64_t seed, int64_t step, cudaStream_t s, int* launches) {
  if (nseg <= 0) return cudaSuccess;
  for (int phase = 0; phase < 3; ++phase) {
    switch (rt) {
      case 1: orth_kernel<1><<<nseg, kThreads, 0, s>>>(t, side, segs, phase, seed, step); break;
      case 2: orth_kernel<2><<<nseg, kThreads, 0, s>>>(t, side, segs, phase, seed, step); break;
      case 4: orth_kernel<4><<<nseg, kThreads, 0, s>>>(t, side, segs, phase, seed, step); break;
      case 8: orth_kernel<8><<<nseg, kThreads, 0, s>>>(t, side, segs, phase, seed, step); break;
      case 16: orth_kernel<16><<<nseg, kThreads, 0, s>>>(t, side, segs, phase, seed, step); break;
      case 32: orth_kernel<32><<<nseg, kThreads, 0, s>>>(t, side, segs, phase, seed, step); break;
      default: return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (launches) ++*launches;
  }
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
