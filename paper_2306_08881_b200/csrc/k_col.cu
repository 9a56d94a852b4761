// Column kernel: K1 of the Q-step (Alg. 2):  Q_loc = M'^T P, a
// reduction over the n rows of M' = M + E for every column.
//
// A CTA owns a panel of up to 256*W contiguous columns (thread c owns W
// adjacent columns, so a warp's loads are 32*W*4 contiguous bytes) and a
// contiguous row range; the orthonormal P rows of that range are staged in
// shared memory (a broadcast operand: every thread of the panel reads the same
// P row). Each thread accumulates W x r partial sums in registers; when a
// panel is narrower than 256 chunks, the CTA splits into row subgroups whose
// partials are summed in shared memory. Each segment writes one partial slot;
// the last segment of a (layer, panel) to finish (device-scope counter) sums
// the panel's partial slots in a FIXED order into the Q-buffer slot and the
// local-Q copy, so the result is deterministic and bit-identical run to run.
// Reads M and E once (8 B / element); E is rewritten by the Q-step decode
// (k_row.cu mode 2) once Q_loc is complete (H1 "simple variant").
// Vectors are packed into the Q-buffer in the same launch.
#include "k_common.cuh"

namespace acp {
namespace {

constexpr int kCH = 64;   // rows of P staged per round

template <int W>
__device__ __forceinline__ void load_w(const float* p, bool vec, float (&x)[W]) {
  if constexpr (W == 4) {
    if (vec) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(p));
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
      return;
    }
  } else if constexpr (W == 2) {
    if (vec) {
      const float2 v = __ldcs(reinterpret_cast<const float2*>(p));
      x[0] = v.x; x[1] = v.y;
      return;
    }
  }
#pragma unroll
  for (int q = 0; q < W; ++q) x[q] = __ldcs(p + q);
}

template <int RT, int W>
__device__ void col_matrix(const Tables& t, const LayerDesc& L, const ColSeg& s,
                           const float* __restrict__ grad, int ef, float* Ps, float* red,
                           int* flag) {
  const int64_t n = L.n, m = L.m;
  const int r = L.r;
  const int pw = L.pw;
  const int64_t c0 = (int64_t)s.panel * pw;
  const int pcols = (int)((m - c0) < pw ? (m - c0) : pw);
  const int PC = (pcols + W - 1) / W;          // chunks in this panel
  int T = 1;
  while (T < PC) T <<= 1;                       // threads per row subgroup
  const int SG = kThreads / T;                  // row subgroups
  const int sgi = threadIdx.x / T, cl = threadIdx.x - sgi * T;
  const bool active = cl < PC;
  const int64_t col = c0 + (int64_t)cl * W;
  const bool vec = ((reinterpret_cast<uintptr_t>(grad) & (4u * W - 1)) == 0);
  const float* __restrict__ Po = t.pbuf + L.p_off;
  const float* __restrict__ E = t.E + L.e_off;

  float acc[W][RT];
#pragma unroll
  for (int q = 0; q < W; ++q)
#pragma unroll
    for (int k = 0; k < RT; ++k) acc[q][k] = 0.f;

  for (int64_t ch0 = s.row0; ch0 < s.row1; ch0 += kCH) {
    const int nr = (int)((s.row1 - ch0) < kCH ? (s.row1 - ch0) : kCH);
    __syncthreads();  // previous round's readers are done with Ps
    for (int idx = threadIdx.x; idx < RT * kCH; idx += kThreads) {
      const int k = idx / kCH, i = idx - k * kCH;
      Ps[i * RT + k] = (k < r && i < nr) ? __ldg(Po + k * n + ch0 + i) : 0.f;
    }
    __syncthreads();
    if (active) {
      int i = sgi;
      // 4 rows per trip: issue all loads, then the FMAs
      for (; i + 3 * SG < nr; i += 4 * SG) {
        float x[4][W];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t row = ch0 + i + u * SG;
          load_w<W>(grad + row * m + col, vec, x[u]);
          if (ef) {
            float e[W];
            load_w<W>(E + row * m + col, true, e);
#pragma unroll
            for (int q = 0; q < W; ++q) x[u][q] += e[q];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float* prow = Ps + (i + u * SG) * RT;
#pragma unroll
          for (int k = 0; k < RT; ++k) {
            const float pk = prow[k];
#pragma unroll
            for (int q = 0; q < W; ++q) acc[q][k] = fmaf(x[u][q], pk, acc[q][k]);
          }
        }
      }
      for (; i < nr; i += SG) {
        const int64_t row = ch0 + i;
        float x[W];
        load_w<W>(grad + row * m + col, vec, x);
        if (ef) {
          float e[W];
          load_w<W>(E + row * m + col, true, e);
#pragma unroll
          for (int q = 0; q < W; ++q) x[q] += e[q];
        }
        const float* prow = Ps + i * RT;
#pragma unroll
        for (int k = 0; k < RT; ++k) {
          const float pk = prow[k];
#pragma unroll
          for (int q = 0; q < W; ++q) acc[q][k] = fmaf(x[q], pk, acc[q][k]);
        }
      }
    }
  }

  // combine row subgroups (fixed order)
  if (SG > 1) {
    __syncthreads();
    if (sgi > 0) {
#pragma unroll
      for (int q = 0; q < W; ++q)
#pragma unroll
        for (int k = 0; k < RT; ++k) red[(threadIdx.x) * (W * RT) + q * RT + k] = acc[q][k];
    }
    __syncthreads();
    if (sgi == 0) {
      for (int g = 1; g < SG; ++g) {
        const float* src = red + (g * T + cl) * (W * RT);
#pragma unroll
        for (int q = 0; q < W; ++q)
#pragma unroll
          for (int k = 0; k < RT; ++k) acc[q][k] += src[q * RT + k];
      }
    }
  }
  // partial slot, k-major [r][pw]
  if (sgi == 0 && active) {
    float* part = t.colpart + s.part_off;
#pragma unroll
    for (int k = 0; k < RT; ++k) {
      if (k < r) {
#pragma unroll
        for (int q = 0; q < W; ++q)
          if (cl * W + q < pcols) part[(int64_t)k * pw + cl * W + q] = acc[q][k];
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int old = atomicAdd(t.colcnt + s.counter, 1);
    *flag = (old == s.pcount - 1);
  }
  __syncthreads();
  if (*flag) {
    __threadfence();
    // the panel's partial slots are contiguous; this segment's is number pidx
    const int64_t slot = (int64_t)r * pw;
    const int64_t first = s.part_off - (int64_t)s.pidx * slot;
    float* Qs = t.qbuf + L.q_off;
    float* Ql = t.qloc + L.ql_off;
    for (int idx = threadIdx.x; idx < r * pcols; idx += kThreads) {
      const int k = idx / pcols, j = idx - k * pcols;
      float sum = 0.f;
      for (int p = 0; p < s.pcount; ++p) sum += __ldcg(t.colpart + first + p * slot + (int64_t)k * pw + j);
      Qs[(int64_t)k * m + c0 + j] = sum;
      Ql[(int64_t)k * m + c0 + j] = sum;
    }
    if (threadIdx.x == 0) t.colcnt[s.counter] = 0;  // re-arm for the next launch
  }
}

template <int RT>
__global__ void __launch_bounds__(kThreads) col_kernel(Tables t, const ColSeg* __restrict__ segs,
                                                       const int32_t* __restrict__ cta_begin,
                                                       int ef) {
  __shared__ __align__(16) float Ps[kCH * RT];
  __shared__ __align__(16) float red[kThreads * 32];
  __shared__ int flag;
  const int sb = cta_begin[blockIdx.x], se = cta_begin[blockIdx.x + 1];
  prefetch_segs(t, segs, sb, se);
  for (int si = sb; si < se; ++si) {
    const ColSeg s = segs[si];
    const LayerDesc L = t.layers[s.layer];
    const float* grad = t.grads[s.layer];
    if (!L.mat) {
      float* slot = t.qbuf + L.q_off;
      for (int64_t i = s.row0 + threadIdx.x; i < s.row1; i += kThreads) slot[i] = grad[i];
      continue;
    }
    if constexpr (RT <= 8) {
      if (L.W == 4) { col_matrix<RT, 4>(t, L, s, grad, ef, Ps, red, &flag); continue; }
    }
    if constexpr (RT <= 16) {
      if (L.W == 2) { col_matrix<RT, 2>(t, L, s, grad, ef, Ps, red, &flag); continue; }
    }
    col_matrix<RT, 1>(t, L, s, grad, ef, Ps, red, &flag);
  }
}

}  // namespace

cudaError_t launch_col(int rt, const Tables& t, const ColSeg* segs, const int32_t* cta_begin,
                       int ncta, int ef, cudaStream_t s) {
  if (ncta <= 0) return cudaSuccess;
  dim3 grid(ncta), block(kThreads);
  switch (rt) {
    case 1: col_kernel<1><<<grid, block, 0, s>>>(t, segs, cta_begin, ef); break;
    case 2: col_kernel<2><<<grid, block, 0, s>>>(t, segs, cta_begin, ef); break;
    case 4: col_kernel<4><<<grid, block, 0, s>>>(t, segs, cta_begin, ef); break;
    case 8: col_kernel<8><<<grid, block, 0, s>>>(t, segs, cta_begin, ef); break;
    case 16: col_kernel<16><<<grid, block, 0, s>>>(t, segs, cta_begin, ef); break;
    case 32: col_kernel<32><<<grid, block, 0, s>>>(t, segs, cta_begin, ef); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace acp
