// TMA-pipelined streaming kernels for the three passes that read M and E:
//
//   mode 0  K1, P-step (Alg. 2): P_loc = M'Q, E = M' - P_loc Q^T
//   mode 2  K3, Q-step:     E = M' - P Q_loc^T, grad = P Q_agg^T / p
//   mode 3  K1, Q-step:            Q_loc = M'^T P  (column reduction)
//
// with M' = M + E. One producer warp streams contiguous row tiles of M and E
// (row-major, so a tile of TR rows is ONE cp.async.bulk of TR*m*4 bytes per
// tensor -> SASS UBLKCP) into an S-stage shared-memory ring guarded by
// mbarriers (full: TMA complete_tx; empty: one arrive per consumer warp).
// Eight consumer warps read the tile from shared memory (128-bit, conflict
// free), keep the layer's orthonormal r-column factor(s) in REGISTERS for the
// whole segment (thread l owns float4 column chunks c = l + v*G, v < V), and
// write E / grad back with streaming 128-bit stores. A consumer warp releases
// its stage as soon as it has pulled the tile into registers, so the producer
// keeps ~S*2*16 KB of loads in flight per SM independent of compute.
//
// Layers that cannot take the bulk path (m % 4 != 0, m > 5120, gradient not
// 16-byte aligned, too many factor registers) run a generic consumer-only
// path in the same launch; vectors (1-D params) are packed/unpacked here too.
#include "k_common.cuh"

namespace acp {
namespace {

constexpr int kCons = 256;                  // consumer threads (all of the CTA)
constexpr int kConsWarps = kCons / 32;
constexpr int kStreamThreads = kCons;       // thread 0 doubles as the TMA producer
constexpr int kRedSlots = 64;

__device__ __forceinline__ uint32_t s32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(s32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(done)
      : "r"(s32(b)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(s32(dst)),
      "l"(src), "r"(bytes), "r"(s32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void cons_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory");
}
__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

struct Shared {
  float* sM;
  float* sE;
  uint64_t* full;
  uint64_t* empty;
  float* red;    // [2][8][kRedSlots]
  int* flag;
  int stage_floats;
  int stages;
};

// Tile sequence of one CTA: q-th bulk tile uses stage q % S, use (q / S).
// Consumers keep `q`; thread 0 additionally runs the producer cursor and
// keeps up to S tiles in flight ahead of the consumers (no dedicated producer
// warp, so the 8 compute warps keep the full 255-register budget).
struct Pipe {
  int64_t q = 0;          // next tile to consume
  // producer state (thread 0)
  int64_t issued = 0;     // tiles issued so far
  int psi = 0;            // producer segment cursor
  int64_t pr0 = -1;       // producer row cursor within segment psi
};

template <int MODE>
__device__ __forceinline__ bool prod_peek(const Tables& t, const StreamSeg* segs, int se, Pipe& pp,
                                          const float** src_m, const float** src_e, uint32_t* bytes,
                                          int64_t* next_r0) {
  constexpr uint32_t kBit = MODE == 0 ? 1u : (MODE == 2 ? 2u : 4u);
  while (pp.psi < se) {
    const StreamSeg& s = segs[pp.psi];
    const LayerDesc& L = t.layers[s.layer];
    const float* grad = t.grads[s.layer];
    const bool fast = L.mat && (L.fast & kBit) && ((reinterpret_cast<uintptr_t>(grad) & 15u) == 0);
    if (pp.pr0 < 0) pp.pr0 = s.row0;
    if (!fast || pp.pr0 >= s.row1) {
      ++pp.psi;
      pp.pr0 = -1;
      continue;
    }
    const int TR = MODE == 3 ? L.trc : L.tr;
    const int64_t nr = (s.row1 - pp.pr0) < TR ? (s.row1 - pp.pr0) : TR;
    *src_m = grad + pp.pr0 * L.m;
    *src_e = t.E + L.e_off + pp.pr0 * L.m;
    *bytes = (uint32_t)(nr * L.m * 4);
    *next_r0 = pp.pr0 + TR;
    return true;
  }
  return false;
}

// Called by thread 0 before consuming tile pp.q: makes sure tile q has been
// issued (blocking on its stage if needed) and opportunistically issues the
// following tiles whose stages are already free.
template <int MODE>
__device__ void prod_pump(const Tables& t, const StreamSeg* segs, int se, Pipe& pp,
                          const Shared& sh, uint64_t pol) {
  while (pp.issued < pp.q + sh.stages) {
    const int stage = (int)(pp.issued % sh.stages);
    const float *sm_src, *se_src;
    uint32_t bytes;
    int64_t nr0;
    if (!prod_peek<MODE>(t, segs, se, pp, &sm_src, &se_src, &bytes, &nr0)) break;
    if (pp.issued >= sh.stages) {
      const uint32_t par = (uint32_t)(((pp.issued / sh.stages) - 1) & 1);
      if (pp.issued == pp.q) mbar_wait(&sh.empty[stage], par);
      else if (!mbar_test(&sh.empty[stage], par)) break;
    }
    mbar_arrive_tx(&sh.full[stage], 2 * bytes);
    bulk_g2s(sh.sM + (size_t)stage * sh.stage_floats, sm_src, bytes, &sh.full[stage], pol);
    bulk_g2s(sh.sE + (size_t)stage * sh.stage_floats, se_src, bytes, &sh.full[stage], pol);
    pp.pr0 = nr0;
    ++pp.issued;
  }
}

// Group sum over G threads (G | 256); every thread of the group gets the sums.
template <int N>
__device__ __forceinline__ void group_sum(float (&a)[N], int G, float* red, int& rph) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    if (off < G) {
#pragma unroll
      for (int i = 0; i < N; ++i) a[i] += __shfl_xor_sync(0xffffffffu, a[i], off);
    }
  }
  if (G <= 32) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* buf = red + (rph & 1) * (kConsWarps * kRedSlots);
  ++rph;
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (lane == (i & 31)) buf[warp * kRedSlots + i] = a[i];
  cons_sync();
  const int nw = G >> 5;
  const int w0 = (warp / nw) * nw;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    float s = buf[w0 * kRedSlots + i];
    for (int w = 1; w < nw; ++w) s += buf[(w0 + w) * kRedSlots + i];
    a[i] = s;
  }
}

template <int RT>
__device__ __forceinline__ void block_sum_cons(float (&a)[RT], float* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < RT; ++k) a[k] += __shfl_xor_sync(0xffffffffu, a[k], off);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  cons_sync();
#pragma unroll
  for (int k = 0; k < RT; ++k)
    if (lane == (k & 31)) red[warp * 32 + k] = a[k];
  cons_sync();
#pragma unroll
  for (int k = 0; k < RT; ++k) {
    float s = red[k];
    for (int w = 1; w < kConsWarps; ++w) s += red[w * 32 + k];
    a[k] = s;
  }
}

__host__ __device__ constexpr bool v_ok(int mode, int V, int RT) {
  return mode == 0 ? V * RT <= 24 : (mode == 2 ? 2 * V * RT <= 40 : V * RT <= 24);
}

// ---------------------------------------------------------------------------
// fast (bulk-pipelined) segment, consumer side
// ---------------------------------------------------------------------------
template <int MODE, int RT, int V>
__device__ void seg_fast(const Tables& t, const LayerDesc& L, const StreamSeg& s,
                         float* __restrict__ grad, float scale, const Shared& sh, Pipe& pp,
                         int& rph, const StreamSeg* segs, int se, uint64_t pol) {
  const int G = MODE == 3 ? L.gc : L.G;
  const int TR = MODE == 3 ? L.trc : L.tr;
  const int NG = kCons / G;
  const int RR = TR / NG;
  const int g = threadIdx.x / G, l = threadIdx.x - g * G;
  const int lane = threadIdx.x & 31;
  const int64_t m = L.m, n = L.n;
  const int m4 = (int)(m >> 2);
  const int r = L.r;
  float* __restrict__ E = t.E + L.e_off;

  // factor(s) in registers for the whole segment
  float4 qa[V][RT];   // mode 0: Q (orthonormal); mode 2: Q_agg
  float4 qb[MODE == 2 ? V : 1][MODE == 2 ? RT : 1];  // mode 2: Q_loc
  float4 acc3[MODE == 3 ? V : 1][MODE == 3 ? RT : 1];
  if constexpr (MODE == 0 || MODE == 2) {
    const float* Qf = t.qbuf + L.q_off;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c = l + v * G;
#pragma unroll
      for (int k = 0; k < RT; ++k) {
        qa[v][k] = (c < m4 && k < r) ? ld_f4(Qf + k * m + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
        if constexpr (MODE == 2)
          qb[v][k] = (c < m4 && k < r) ? ld_f4(t.qloc + L.ql_off + k * m + 4 * c)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int k = 0; k < RT; ++k) acc3[v][k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const float* __restrict__ Pf = t.pbuf + L.p_off;  // k-major [r][n]
  float* __restrict__ Pw = t.pbuf + L.p_off;

  for (int64_t r0 = s.row0; r0 < s.row1; r0 += TR) {
    const int nr = (int)((s.row1 - r0) < TR ? (s.row1 - r0) : TR);
    if (threadIdx.x == 0) prod_pump<MODE>(t, segs, se, pp, sh, pol);
    const int stage = (int)(pp.q % sh.stages);
    mbar_wait(&sh.full[stage], (uint32_t)((pp.q / sh.stages) & 1));
    const float* tM = sh.sM + (size_t)stage * sh.stage_floats;
    const float* tE = sh.sE + (size_t)stage * sh.stage_floats;
    for (int j = 0; j < RR; ++j) {
      const int li = g + NG * j;
      const bool valid = li < nr;
      const int64_t row = r0 + li;
      float pk[RT];
      if constexpr (MODE != 0) {
#pragma unroll
        for (int k = 0; k < RT; ++k) pk[k] = (valid && k < r) ? __ldg(Pf + k * n + row) : 0.f;
      }
      float4 x[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int c = l + v * G;
        x[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid && c < m4) x[v] = f4add(lds4(tM + li * m + 4 * c), lds4(tE + li * m + 4 * c));
      }
      if (j == RR - 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.empty[stage]);
      }
      if constexpr (MODE == 0) {
        float acc[RT];
#pragma unroll
        for (int k = 0; k < RT; ++k) {
          float a = 0.f;
#pragma unroll
          for (int v = 0; v < V; ++v) a += f4dot(x[v], qa[v][k]);
          acc[k] = a;
        }
        group_sum<RT>(acc, G, sh.red, rph);
        if (valid) {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const int c = l + v * G;
            if (c < m4) {
              float4 e = x[v];
#pragma unroll
              for (int k = 0; k < RT; ++k) f4fma(e, -acc[k], qa[v][k]);
              st_cs4(E + row * m + 4 * c, e);
            }
          }
          if (l == 0) {
#pragma unroll
            for (int k = 0; k < RT; ++k)
              if (k < r) Pw[k * n + row] = acc[k];
          }
        }
      } else if constexpr (MODE == 2) {
        if (valid) {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const int c = l + v * G;
            if (c < m4) {
              float4 e = x[v], o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int k = 0; k < RT; ++k) {
                f4fma(e, -pk[k], qb[v][k]);
                f4fma(o, pk[k], qa[v][k]);
              }
              st_cs4(E + row * m + 4 * c, e);
              st_cs4(grad + row * m + 4 * c, f4scale(o, scale));
            }
          }
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int k = 0; k < RT; ++k) {
            acc3[v][k].x = fmaf(x[v].x, pk[k], acc3[v][k].x);
            acc3[v][k].y = fmaf(x[v].y, pk[k], acc3[v][k].y);
            acc3[v][k].z = fmaf(x[v].z, pk[k], acc3[v][k].z);
            acc3[v][k].w = fmaf(x[v].w, pk[k], acc3[v][k].w);
          }
      }
    }
    ++pp.q;
  }
  if constexpr (MODE == 3) {
    // partial slot g of this segment: k-major [r][m]
    float* part = t.colpart + s.part_off + (int64_t)g * r * m;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c = l + v * G;
      if (c < m4) {
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) *reinterpret_cast<float4*>(part + k * m + 4 * c) = acc3[v][k];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// generic segment (any m / alignment), consumer threads only
// ---------------------------------------------------------------------------
template <int MODE, int RT>
__device__ void seg_generic(const Tables& t, const LayerDesc& L, const StreamSeg& s,
                            float* __restrict__ grad, float scale, float* red) {
  const int64_t m = L.m, n = L.n;
  const int r = L.r;
  const float* __restrict__ Qs = t.qbuf + L.q_off;
  const float* __restrict__ Ql = t.qloc + L.ql_off;
  float* __restrict__ Ps = t.pbuf + L.p_off;
  float* __restrict__ E = t.E + L.e_off;
  if constexpr (MODE == 3) {
    float* part = t.colpart + s.part_off;
    for (int64_t c0 = 0; c0 < m; c0 += kCons) {
      const int64_t c = c0 + threadIdx.x;
      float acc[RT];
#pragma unroll
      for (int k = 0; k < RT; ++k) acc[k] = 0.f;
      if (c < m) {
        for (int64_t row = s.row0; row < s.row1; ++row) {
          const float x = grad[row * m + c] + E[row * m + c];
#pragma unroll
          for (int k = 0; k < RT; ++k)
            if (k < r) acc[k] = fmaf(x, __ldg(Ps + k * n + row), acc[k]);
        }
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) part[k * m + c] = acc[k];
        for (int gsl = 1; gsl < s.nslot; ++gsl)
          for (int k = 0; k < r; ++k) part[(int64_t)gsl * r * m + k * m + c] = 0.f;
      }
    }
    return;
  }
  for (int64_t row = s.row0; row < s.row1; ++row) {
    float* __restrict__ gr = grad + row * m;
    float* __restrict__ er = E + row * m;
    if constexpr (MODE == 0) {
      float acc[RT];
#pragma unroll
      for (int k = 0; k < RT; ++k) acc[k] = 0.f;
      for (int64_t j = threadIdx.x; j < m; j += kCons) {
        const float x = gr[j] + er[j];
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) acc[k] = fmaf(x, __ldg(Qs + k * m + j), acc[k]);
      }
      block_sum_cons<RT>(acc, red);
      for (int64_t j = threadIdx.x; j < m; j += kCons) {
        float x = gr[j] + er[j];
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) x = fmaf(-acc[k], __ldg(Qs + k * m + j), x);
        er[j] = x;
      }
      if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) Ps[k * n + row] = acc[k];
      }
    } else {
      float p[RT];
#pragma unroll
      for (int k = 0; k < RT; ++k) p[k] = (k < r) ? __ldg(Ps + k * n + row) : 0.f;
      for (int64_t j = threadIdx.x; j < m; j += kCons) {
        float x = gr[j] + er[j], o = 0.f;
#pragma unroll
        for (int k = 0; k < RT; ++k) {
          if (k < r) {
            o = fmaf(p[k], __ldg(Qs + k * m + j), o);
            x = fmaf(-p[k], __ldg(Ql + k * m + j), x);
          }
        }
        er[j] = x;
        gr[j] = o * scale;
      }
    }
  }
}

// last segment of a layer to finish (mode 3): sum the layer's partial slots in
// slot order into the Q-buffer slot and the local-Q copy
__device__ void col_finish(const Tables& t, const LayerDesc& L, const StreamSeg& s, int* flag) {
  __threadfence();
  cons_sync();
  if (threadIdx.x == 0) {
    const int old = atomicAdd(t.colcnt + s.layer, s.nslot);
    *flag = (old + s.nslot == s.pcount);
  }
  cons_sync();
  if (!*flag) return;
  __threadfence();
  const int64_t m = L.m;
  const int r = L.r;
  const int64_t slot = (int64_t)r * m;
  const float* first = t.colpart + s.part_off - (int64_t)s.pidx * slot;
  float* Qs = t.qbuf + L.q_off;
  float* Ql = t.qloc + L.ql_off;
  const int64_t total = slot;
  if ((m & 3) == 0) {
    for (int64_t i = 4 * threadIdx.x; i < total; i += 4 * kCons) {
      float4 acc = __ldcg(reinterpret_cast<const float4*>(first + i));
      for (int p = 1; p < s.pcount; ++p)
        acc = f4add(acc, __ldcg(reinterpret_cast<const float4*>(first + p * slot + i)));
      *reinterpret_cast<float4*>(Qs + i) = acc;
      *reinterpret_cast<float4*>(Ql + i) = acc;
    }
  } else {
    for (int64_t i = threadIdx.x; i < total; i += kCons) {
      float acc = __ldcg(first + i);
      for (int p = 1; p < s.pcount; ++p) acc += __ldcg(first + p * slot + i);
      Qs[i] = acc;
      Ql[i] = acc;
    }
  }
  if (threadIdx.x == 0) t.colcnt[s.layer] = 0;  // re-arm
}

template <int MODE, int RT>
__global__ void __launch_bounds__(kStreamThreads, 1)
    stream_kernel(Tables t, const StreamSeg* __restrict__ segs, const int32_t* __restrict__ cta_begin,
                  float scale, int stages, int stage_floats) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Shared sh;
  sh.stages = stages;
  sh.stage_floats = stage_floats;
  sh.sM = reinterpret_cast<float*>(smem_raw);
  sh.sE = sh.sM + (size_t)stages * stage_floats;
  sh.full = reinterpret_cast<uint64_t*>(sh.sE + (size_t)stages * stage_floats);
  sh.empty = sh.full + stages;
  sh.red = reinterpret_cast<float*>(sh.empty + stages);
  sh.flag = reinterpret_cast<int*>(sh.red + 2 * kConsWarps * kRedSlots);
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&sh.full[i], 1);
      mbar_init(&sh.empty[i], kConsWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int sb = cta_begin[blockIdx.x], se = cta_begin[blockIdx.x + 1];
  constexpr uint32_t kBit = MODE == 0 ? 1u : (MODE == 2 ? 2u : 4u);

  const uint64_t pol = policy_evict_first();
  // ---------------- consumers ----------------
  Pipe pp;
  pp.psi = sb;
  int rph = 0;
  for (int si = sb; si < se; ++si) {
    const StreamSeg s = segs[si];
    const LayerDesc L = t.layers[s.layer];
    float* grad = t.grads[s.layer];
    if (!L.mat) {
      if (MODE == 0) {
        float* slot = t.pbuf + L.p_off;
        for (int64_t i = s.row0 + threadIdx.x; i < s.row1; i += kCons) slot[i] = grad[i];
      } else if (MODE == 3) {
        float* slot = t.qbuf + L.q_off;
        for (int64_t i = s.row0 + threadIdx.x; i < s.row1; i += kCons) slot[i] = grad[i];
      } else {
        const float* slot = t.qbuf + L.q_off;
        for (int64_t i = s.row0 + threadIdx.x; i < s.row1; i += kCons) grad[i] = slot[i] * scale;
      }
      continue;
    }
    const bool fast = (L.fast & kBit) && ((reinterpret_cast<uintptr_t>(grad) & 15u) == 0);
    if (!fast) {
      seg_generic<MODE, RT>(t, L, s, grad, scale, sh.red);
    } else {
      const int V = MODE == 3 ? L.vc : L.V;
      switch (V) {
#define ACP_CASE(VV)                                                       \
  case VV:                                                                 \
    if constexpr (v_ok(MODE, VV, RT)) seg_fast<MODE, RT, VV>(t, L, s, grad, scale, sh, pp, rph, segs, se, pol); \
    break;
        ACP_CASE(1)
        ACP_CASE(2)
        ACP_CASE(3)
        ACP_CASE(4)
        ACP_CASE(5)
#undef ACP_CASE
        default: break;
      }
    }
    if constexpr (MODE == 3) col_finish(t, L, s, sh.flag);
  }
}

template <int MODE>
cudaError_t launch_mode(int rt, const Tables& t, const StreamSeg* segs, const int32_t* cb, int ncta,
                        float scale, int stages, int stage_floats, cudaStream_t st) {
  const size_t smem = (size_t)2 * stages * stage_floats * 4 + 2 * stages * 8 +
                      2 * kConsWarps * kRedSlots * 4 + 16;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<ncta, kStreamThreads, smem, st>>>(t, segs, cb, scale, stages, stage_floats);
    return cudaGetLastError();
  };
  switch (rt) {
    case 1: return go(stream_kernel<MODE, 1>);
    case 2: return go(stream_kernel<MODE, 2>);
    case 4: return go(stream_kernel<MODE, 4>);
    case 8: return go(stream_kernel<MODE, 8>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool stream_v_ok(int mode, int V, int rt) { return V >= 1 && V <= 5 && v_ok(mode, V, rt); }

size_t stream_smem_bytes(int stages, int stage_floats) {
  return (size_t)2 * stages * stage_floats * 4 + 2 * stages * 8 + 2 * kConsWarps * kRedSlots * 4 + 16;
}

cudaError_t launch_stream(int mode, int rt, const Tables& t, const StreamSeg* segs,
                          const int32_t* cta_begin, int ncta, float scale, int stages,
                          int stage_floats, cudaStream_t s) {
  if (ncta <= 0) return cudaSuccess;
  switch (mode) {
    case 0: return launch_mode<0>(rt, t, segs, cta_begin, ncta, scale, stages, stage_floats, s);
    case 2: return launch_mode<2>(rt, t, segs, cta_begin, ncta, scale, stages, stage_floats, s);
    case 3: return launch_mode<3>(rt, t, segs, cta_begin, ncta, scale, stages, stage_floats, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace acp
