// Row kernels: every row of M' = M + E is independent given the reused,
// orthonormal factor, so one pass over the row suffices.
//
//   mode 0  K1, P-step (Alg. 2):  P_loc[i,:] = M'[i,:] Q,
//           E[i,:] = M'[i,:] - P_loc[i,:] Q^T   -- the row stays in registers
//           between the projection and the residual, so M and E are read once
//           and E written once (12 B / element); P_loc goes to the P-buffer slot.
//           ef = 3: projection only (Power-SGD's first projection, Alg. 1
//           P:180-181, whose residual is formed after the second one): 8 B.
//   mode 1  K3, P-step decode:  grad[i,:] = scale * P_agg[i,:] Q^T
//           (write-only stream, 4 B / element).
//   mode 2  K3, Q-step residual + decode:
//           E[i,:] = M'[i,:] - P[i,:] Q_loc^T,  grad[i,:] = scale * P[i,:] Q_agg^T
//           (reads M and E, writes E and grad: 16 B / element).
//
// Vectors (1-D params) ride in the same launch: mode 0 packs them into the
// P-buffer, modes 1/2 unpack (x scale) from the P-/Q-buffer.
//
// Work decomposition: each CTA (256 threads) walks a host-built, contiguous,
// byte-balanced range of segments (layer, rows). A matrix row is owned by a
// group of G threads (G | 256); thread l of the group owns float4 column
// chunks c = l + v*G, v < V, so a warp's loads are 512 contiguous bytes
// (128-bit coalesced). The factor Q (k-major, r rows of m floats) is read
// through L1 (__ldg) and reused by every row of the layer the CTA processes;
// M and E use streaming (.cs) accesses so they do not evict it.
#include "k_common.cuh"
#include "k_nvls.cuh"

namespace acp {
namespace {

constexpr int kRedSlots = 64;  // max R*RT values reduced per group

__host__ __device__ constexpr int rows_k1p(int V, int RT) {
  return (8 / V) < (64 / RT) ? ((8 / V) > 0 ? 8 / V : 1) : ((64 / RT) > 0 ? 64 / RT : 1);
}
__host__ __device__ constexpr int rows_k3p(int RT) { return (64 / RT) < 8 ? (64 / RT) : 8; }
__host__ __device__ constexpr int rows_k3q(int RT) {
  return (64 / RT) < 4 ? ((64 / RT) > 0 ? 64 / RT : 1) : 4;
}

// Sum N per-thread values over a row group of G threads; every thread of the
// group ends with the group sums. Fixed order => deterministic.
template <int N>
__device__ __forceinline__ void group_sum(float (&a)[N], int G, float* red, int& phase) {
  if (G <= 32) {
    for (int off = G >> 1; off > 0; off >>= 1) {
#pragma unroll
      for (int i = 0; i < N; ++i) a[i] += __shfl_xor_sync(0xffffffffu, a[i], off);
    }
    return;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] += __shfl_xor_sync(0xffffffffu, a[i], off);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* buf = red + (phase & 1) * (8 * kRedSlots);
  ++phase;
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (lane == (i & 31)) buf[warp * kRedSlots + i] = a[i];
  __syncthreads();
  const int nw = G >> 5;
  const int w0 = (warp / nw) * nw;
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      float4 s = *reinterpret_cast<const float4*>(buf + w0 * kRedSlots + i);
      for (int w = 1; w < nw; ++w) s = f4add(s, *reinterpret_cast<const float4*>(buf + (w0 + w) * kRedSlots + i));
      a[i] = s.x; a[i + 1] = s.y; a[i + 2] = s.z; a[i + 3] = s.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      float s = buf[w0 * kRedSlots + i];
      for (int w = 1; w < nw; ++w) s += buf[(w0 + w) * kRedSlots + i];
      a[i] = s;
    }
  }
}

// ---- mode 0, fast path ----------------------------------------------------
template <int RT, int V>
__device__ void k1p_fast(const Tables& t, const LayerDesc& L, const float* __restrict__ grad,
                         int64_t row0, int64_t row1, int ef, float* red, int& phase) {
  constexpr int R = rows_k1p(V, RT);
  const int G = L.G;
  const int NG = kThreads / G;
  const int g = threadIdx.x / G, l = threadIdx.x - g * G;
  const int64_t m = L.m, n = L.n;
  const int m4 = (int)(m >> 2);
  const int r = L.r;
  const float* __restrict__ Qo = t.qbuf + L.q_off;
  float* __restrict__ E = t.E + L.e_off;
  float* __restrict__ Ps = t.pbuf + L.p_off;
  const int64_t per_iter = (int64_t)NG * R;
  const int64_t niter = (row1 - row0 + per_iter - 1) / per_iter;
  for (int64_t it = 0; it < niter; ++it) {
    const int64_t base = row0 + (it * NG + g) * R;
    float4 x[R][V];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int64_t row = base + rr;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int c = l + v * G;
        x[rr][v] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < row1 && c < m4) {
          x[rr][v] = ld_cs4(grad + row * m + 4 * c);
          if (ef) x[rr][v] = f4add(x[rr][v], ld_cs4(E + row * m + 4 * c));
        }
      }
    }
    float acc[R * RT];
#pragma unroll
    for (int i = 0; i < R * RT; ++i) acc[i] = 0.f;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c = l + v * G;
      if (c < m4) {
#pragma unroll
        for (int k = 0; k < RT; ++k) {
          if (k < r) {
            const float4 q = ld_f4(Qo + k * m + 4 * c);
#pragma unroll
            for (int rr = 0; rr < R; ++rr) acc[rr * RT + k] += f4dot(x[rr][v], q);
          }
        }
      }
    }
    group_sum<R * RT>(acc, G, red, phase);
    if (ef == 1) {  // ef == 3: Power-SGD projection only (E is updated after Q)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int c = l + v * G;
        if (c < m4) {
#pragma unroll
          for (int k = 0; k < RT; ++k) {
            if (k < r) {
              const float4 q = ld_f4(Qo + k * m + 4 * c);
#pragma unroll
              for (int rr = 0; rr < R; ++rr) f4fma(x[rr][v], -acc[rr * RT + k], q);
            }
          }
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const int64_t row = base + rr;
            if (row < row1) st_cs4(E + row * m + 4 * c, x[rr][v]);
          }
        }
      }
    }
    if (l == 0) {
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const int64_t row = base + rr;
        if (row < row1) {
#pragma unroll
          for (int k = 0; k < RT; ++k)
            if (k < r) Ps[k * n + row] = acc[rr * RT + k];
        }
      }
    }
  }
}

// Factor loads of the decodes. FUSED (NVLS prologue, k_nvls.cuh): the
// all-reduced slot was rewritten inside this launch by the multicast store,
// so it is read through L2 (ld.global.cg), never the non-coherent L1 path.
template <bool CG>
__device__ __forceinline__ float ld_fac(const float* p) { return CG ? __ldcg(p) : __ldg(p); }
template <bool CG>
__device__ __forceinline__ float4 ld_fac4(const float* p) {
  return CG ? __ldcg(reinterpret_cast<const float4*>(p)) : ld_f4(p);
}

// ---- mode 1 (and 3), fast path ----------------------------------------------
// MODE 1: P-step decode (the P slot is the all-reduced one); MODE 3: Q-step
// decode of the deferred path (the Q slot is the all-reduced one).
template <int RT, int MODE, bool FUSED>
__device__ void k3p_fast(const Tables& t, const LayerDesc& L, float* __restrict__ grad,
                         int64_t row0, int64_t row1, float scale) {
  constexpr bool kCgP = FUSED && MODE == 1, kCgQ = FUSED && MODE == 3;
  constexpr int R = rows_k3p(RT);
  const int G = L.G, V = L.V;
  const int NG = kThreads / G;
  const int g = threadIdx.x / G, l = threadIdx.x - g * G;
  const int64_t m = L.m, n = L.n;
  const int m4 = (int)(m >> 2);
  const int r = L.r;
  const float* __restrict__ Qo = t.qbuf + L.q_off;
  const float* __restrict__ Pa = t.pbuf + L.p_off;
  const int64_t per_iter = (int64_t)NG * R;
  const int64_t niter = (row1 - row0 + per_iter - 1) / per_iter;
  for (int64_t it = 0; it < niter; ++it) {
    const int64_t base = row0 + (it * NG + g) * R;
    float p[R][RT];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int64_t row = base + rr;
#pragma unroll
      for (int k = 0; k < RT; ++k)
        p[rr][k] = (k < r && row < row1) ? ld_fac<kCgP>(Pa + k * n + row) * scale : 0.f;
    }
    for (int v = 0; v < V; ++v) {
      const int c = l + v * G;
      if (c >= m4) break;
      float4 o[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) o[rr] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < RT; ++k) {
        if (k < r) {
          const float4 q = ld_fac4<kCgQ>(Qo + k * m + 4 * c);
#pragma unroll
          for (int rr = 0; rr < R; ++rr) f4fma(o[rr], p[rr][k], q);
        }
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const int64_t row = base + rr;
        if (row < row1) st_cs4(grad + row * m + 4 * c, o[rr]);
      }
    }
  }
}

// ---- mode 2, fast path ----------------------------------------------------
template <int RT, bool FUSED>
__device__ void k3q_fast(const Tables& t, const LayerDesc& L, float* __restrict__ grad,
                         int64_t row0, int64_t row1, float scale, int ef) {
  constexpr int R = rows_k3q(RT);
  const int G = L.G, V = L.V;
  const int NG = kThreads / G;
  const int g = threadIdx.x / G, l = threadIdx.x - g * G;
  const int64_t m = L.m, n = L.n;
  const int m4 = (int)(m >> 2);
  const int r = L.r;
  const float* __restrict__ Po = t.pbuf + L.p_off;   // orthonormal P (k-major)
  const float* __restrict__ Ql = t.qloc + L.ql_off;  // local Q (pre all-reduce)
  const float* __restrict__ Qa = t.qbuf + L.q_off;   // aggregated Q
  float* __restrict__ E = t.E + L.e_off;
  const int64_t per_iter = (int64_t)NG * R;
  const int64_t niter = (row1 - row0 + per_iter - 1) / per_iter;
  for (int64_t it = 0; it < niter; ++it) {
    const int64_t base = row0 + (it * NG + g) * R;
    float p[R][RT];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int64_t row = base + rr;
#pragma unroll
      for (int k = 0; k < RT; ++k)
        p[rr][k] = (k < r && row < row1) ? __ldg(Po + k * n + row) : 0.f;
    }
    for (int v = 0; v < V; ++v) {
      const int c = l + v * G;
      if (c >= m4) break;
      float4 e[R], o[R];
      if (ef) {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int64_t row = base + rr;
          e[rr] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row < row1) e[rr] = f4add(ld_cs4(grad + row * m + 4 * c), ld_cs4(E + row * m + 4 * c));
        }
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) o[rr] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < RT; ++k) {
        if (k < r) {
          const float4 qa = ld_fac4<FUSED>(Qa + k * m + 4 * c);
#pragma unroll
          for (int rr = 0; rr < R; ++rr) f4fma(o[rr], p[rr][k], qa);
          if (ef) {
            const float4 ql = ld_f4(Ql + k * m + 4 * c);
#pragma unroll
            for (int rr = 0; rr < R; ++rr) f4fma(e[rr], -p[rr][k], ql);
          }
        }
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const int64_t row = base + rr;
        if (row < row1) {
          if (ef) st_cs4(E + row * m + 4 * c, e[rr]);
          st_cs4(grad + row * m + 4 * c, f4scale(o[rr], scale));
        }
      }
    }
  }
}

// ---- generic path (any m, any alignment): one row at a time per CTA -------
template <int RT>
__device__ __forceinline__ void block_sum(float (&a)[RT], float* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < RT; ++k) a[k] += __shfl_xor_sync(0xffffffffu, a[k], off);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < RT; ++k)
    if (lane == (k & 31)) red[warp * 32 + k] = a[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < RT; ++k) {
    float s = red[k];
    for (int w = 1; w < kThreads / 32; ++w) s += red[w * 32 + k];
    a[k] = s;
  }
  __syncthreads();
}

template <int MODE, int RT, bool CG>
__device__ void row_generic(const Tables& t, const LayerDesc& L, float* __restrict__ grad,
                            int64_t row0, int64_t row1, float scale, int ef, float* red) {
  // one warp per row (lanes stride the columns, shuffle row sums): layers with
  // many short rows (or m % 4 != 0) run without CTA barriers
  (void)red;
  const int64_t m = L.m, n = L.n;
  const int r = L.r;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* __restrict__ Qs = t.qbuf + L.q_off;
  const float* __restrict__ Ql = t.qloc + L.ql_off;
  float* __restrict__ Ps = t.pbuf + L.p_off;
  float* __restrict__ E = t.E + L.e_off;
  for (int64_t row = row0 + warp; row < row1; row += kThreads / 32) {
    float* __restrict__ g = grad + row * m;
    float* __restrict__ e = E + row * m;
    if (MODE == 0) {
      float acc[RT];
#pragma unroll
      for (int k = 0; k < RT; ++k) acc[k] = 0.f;
      for (int64_t j = lane; j < m; j += 32) {
        const float x = g[j] + (ef ? e[j] : 0.f);
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) acc[k] = fmaf(x, __ldg(Qs + k * m + j), acc[k]);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int k = 0; k < RT; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
      if (ef == 1) {  // ef == 3: projection only (Power-SGD)
        for (int64_t j = lane; j < m; j += 32) {
          float x = g[j] + e[j];
#pragma unroll
          for (int k = 0; k < RT; ++k)
            if (k < r) x = fmaf(-acc[k], __ldg(Qs + k * m + j), x);
          e[j] = x;
        }
      }
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) Ps[k * n + row] = acc[k];
      }
    } else {
      float p[RT];
#pragma unroll
      for (int k = 0; k < RT; ++k) p[k] = (k < r) ? ld_fac<CG>(Ps + k * n + row) : 0.f;
      for (int64_t j = lane; j < m; j += 32) {
        float o = 0.f;
        if (MODE == 1) {
#pragma unroll
          for (int k = 0; k < RT; ++k)
            if (k < r) o = fmaf(p[k], ld_fac<CG>(Qs + k * m + j), o);
        } else {
          float x = ef ? g[j] + e[j] : 0.f;
#pragma unroll
          for (int k = 0; k < RT; ++k) {
            if (k < r) {
              o = fmaf(p[k], ld_fac<CG>(Qs + k * m + j), o);
              if (ef) x = fmaf(-p[k], ld_fac<CG>(Ql + k * m + j), x);
            }
          }
          if (ef) e[j] = x;
        }
        g[j] = o * scale;
      }
    }
  }
}

template <int MODE, int RT>
__global__ void __launch_bounds__(kThreads) row_kernel(Tables t, const RowSeg* __restrict__ segs,
                                                       const int32_t* __restrict__ cta_begin,
                                                       float scale, int ef) {
  __shared__ __align__(16) float red[2 * 8 * kRedSlots];
  __shared__ __align__(16) float red_gen[8 * 32];
  int phase = 0;
  // NVLS (NEXT-3): sum this parity's fused buffer over the ranks first
  if (MODE != 0 && t.nvls_fused) nvls_fused_reduce(t, MODE == 1 ? 0 : 1);
  // the P-step decode runs after the P-step projection consumed a deferred
  // Q-step residual (k_stream.cu): E is materialised again
  if (MODE == 1 && blockIdx.x == 0 && threadIdx.x == 0) *t.deferred = 0;
  const int sb = cta_begin[blockIdx.x], se = cta_begin[blockIdx.x + 1];
  prefetch_segs(t, segs, sb, se);
  for (int s = sb; s < se; ++s) {
    if (!t.layers[segs[s].layer].mat) {
      // vectors: pack (mode 0) into the P-buffer / unpack (modes 1, 2, 3)
      s = vector_run(t, segs, s, se, threadIdx.x >> 5, kThreads / 32,
                     [&](const RowSeg& sg, const LayerDesc& L, int first, int stride) {
                       float* grad = t.grads[sg.layer];
                       float* slot = (MODE >= 2 ? t.qbuf + L.q_off : t.pbuf + L.p_off);
                       for (int64_t i = sg.row0 + first; i < sg.row1; i += stride) {
                         if (MODE == 0) slot[i] = grad[i];
                         else grad[i] = (t.nvls_fused ? __ldcg(slot + i) : slot[i]) * scale;
                       }
                     }) - 1;
      continue;
    }
    const RowSeg sg = segs[s];
    const LayerDesc L = t.layers[sg.layer];
    float* grad = t.grads[sg.layer];
    const bool fast = L.G > 0 && ((reinterpret_cast<uintptr_t>(grad) & 15u) == 0);
    if (!fast) {
      if (MODE != 0 && t.nvls_fused)
        row_generic<MODE == 3 ? 1 : MODE, RT, true>(t, L, grad, sg.row0, sg.row1, scale, ef, red_gen);
      else
        row_generic<MODE == 3 ? 1 : MODE, RT, false>(t, L, grad, sg.row0, sg.row1, scale, ef, red_gen);
      continue;
    }
    if constexpr (MODE == 0) {
      switch (L.V) {
        case 1: k1p_fast<RT, 1>(t, L, grad, sg.row0, sg.row1, ef, red, phase); break;
        case 2: k1p_fast<RT, 2>(t, L, grad, sg.row0, sg.row1, ef, red, phase); break;
        case 3: k1p_fast<RT, 3>(t, L, grad, sg.row0, sg.row1, ef, red, phase); break;
        case 4: k1p_fast<RT, 4>(t, L, grad, sg.row0, sg.row1, ef, red, phase); break;
        case 5: k1p_fast<RT, 5>(t, L, grad, sg.row0, sg.row1, ef, red, phase); break;
        case 6: k1p_fast<RT, 6>(t, L, grad, sg.row0, sg.row1, ef, red, phase); break;
        case 7: k1p_fast<RT, 7>(t, L, grad, sg.row0, sg.row1, ef, red, phase); break;
        default: k1p_fast<RT, 8>(t, L, grad, sg.row0, sg.row1, ef, red, phase); break;
      }
    } else if constexpr (MODE == 1 || MODE == 3) {
      if (t.nvls_fused) k3p_fast<RT, MODE, true>(t, L, grad, sg.row0, sg.row1, scale);
      else k3p_fast<RT, MODE, false>(t, L, grad, sg.row0, sg.row1, scale);
    } else {
      if (t.nvls_fused) k3q_fast<RT, true>(t, L, grad, sg.row0, sg.row1, scale, ef);
      else k3q_fast<RT, false>(t, L, grad, sg.row0, sg.row1, scale, ef);
    }
  }
}

template <int MODE>
cudaError_t launch_row_mode(int rt, const Tables& t, const RowSeg* segs, const int32_t* cb,
                            int ncta, float scale, int ef, cudaStream_t s) {
  dim3 grid(ncta), block(kThreads);
  // the NVLS-fused decode barriers its whole grid (k_nvls.cuh): cooperative
  const bool coop = MODE != 0 && t.nvls_fused;
  switch (rt) {
    case 1: return launch_kernel(row_kernel<MODE, 1>, grid, block, 0, s, coop, t, segs, cb, scale, ef);
    case 2: return launch_kernel(row_kernel<MODE, 2>, grid, block, 0, s, coop, t, segs, cb, scale, ef);
    case 4: return launch_kernel(row_kernel<MODE, 4>, grid, block, 0, s, coop, t, segs, cb, scale, ef);
    case 8: return launch_kernel(row_kernel<MODE, 8>, grid, block, 0, s, coop, t, segs, cb, scale, ef);
    case 16: return launch_kernel(row_kernel<MODE, 16>, grid, block, 0, s, coop, t, segs, cb, scale, ef);
    case 32: return launch_kernel(row_kernel<MODE, 32>, grid, block, 0, s, coop, t, segs, cb, scale, ef);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

int row_kernel_ctas_per_sm(int mode, int rt) {
  int n = 1;
  auto occ = [&](auto kern) { cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, 0); };
#define ACP_OCC(M)                                      \
  switch (rt) {                                        \
    case 1: occ(row_kernel<M, 1>); break;              \
    case 2: occ(row_kernel<M, 2>); break;              \
    case 4: occ(row_kernel<M, 4>); break;              \
    case 8: occ(row_kernel<M, 8>); break;              \
    case 16: occ(row_kernel<M, 16>); break;            \
    default: occ(row_kernel<M, 32>); break;            \
  }
  if (mode == 1) { ACP_OCC(1) }
  else if (mode == 2) { ACP_OCC(2) }
  else if (mode == 3) { ACP_OCC(3) }
  else { ACP_OCC(0) }
#undef ACP_OCC
  return n;
}

int row_rows_per_iter(int mode, int V, int rt) {
  if (mode == 0) return rows_k1p(V, rt);
  if (mode == 1 || mode == 3) return rows_k3p(rt);
  return rows_k3q(rt);
}

cudaError_t launch_row(int mode, int rt, const Tables& t, const RowSeg* segs,
                       const int32_t* cta_begin, int ncta, float scale, int ef,
                       cudaStream_t stream) {
  if (ncta <= 0) return cudaSuccess;
  switch (mode) {
    case 0: return launch_row_mode<0>(rt, t, segs, cta_begin, ncta, scale, ef, stream);
    case 1: return launch_row_mode<1>(rt, t, segs, cta_begin, ncta, scale, ef, stream);
    case 2: return launch_row_mode<2>(rt, t, segs, cta_begin, ncta, scale, ef, stream);
    case 3: return launch_row_mode<3>(rt, t, segs, cta_begin, ncta, scale, ef, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace acp
