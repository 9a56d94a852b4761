// TMA-pipelined streaming kernels for the three passes that read M and E:
//
//   mode 0  K1, P-step (Alg. 2): P_loc = M'Q, E = M' - P_loc Q^T
//   mode 2  K3, Q-step:     E = M' - P Q_loc^T, grad = P Q_agg^T / p
//   mode 3  K1, Q-step:            Q_loc = M'^T P  (column reduction)
//
// with M' = M + E. Thread 0 of the CTA doubles as the producer: it streams
// contiguous row tiles of M and E (row-major, so a tile of tr rows is ONE
// cp.async.bulk of tr*m*4 bytes per tensor, SASS UBLKCP) into an S-stage
// shared-memory ring guarded by mbarriers (full: TMA complete_tx; empty: one
// arrive per warp), keeping up to S tiles in flight. All NW warps compute:
// each pulls its slice of the tile from shared memory into registers
// (128-bit, conflict-free), releases the stage at once, and then works from
// registers, with the layer's r-column factor(s) also held in registers for
// the whole segment. Outputs (E, grad) leave with streaming 128-bit stores.
// A row is covered either by a sub-warp lane group (small m) or by gw whole
// warps (large m; row sums combined through shared memory behind a named
// barrier of the row group), so each lane holds at most a few float4 chunks
// and the code stays branch-free (StreamMap in acp_internal.h).
//
// Layers that cannot take the bulk path (m % 4 != 0, m too large for the
// register budget, gradient not 16-byte aligned) run a generic path in the
// same launch; vectors (1-D params) are packed/unpacked here too.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "k_common.cuh"

namespace acp {
namespace {

// NW consumer warps + 1 producer warp per CTA, CPS CTAs per SM (9 warps ->
// at most 3 per SM sub-partition -> 168 registers per thread), TT = tile
// target (floats per tensor per stage).
template <int MODE>
struct Cfg;
// K1 P-step: factor in registers (nc*RT float4)
// (NW here is the r = 8 count; r <= 4 runs 12 consumer warps: nw_of)
template <> struct Cfg<0> { static constexpr int NW = 8, CPS = 1, TT = 8192; };
// K3 Q-step: two factors in registers (2*nc*RT float4), no barriers
template <> struct Cfg<2> { static constexpr int NW = 8, CPS = 1, TT = 4096; };
// K1 Q-step: accumulators nc*RT float4 in registers
template <> struct Cfg<3> { static constexpr int NW = 8, CPS = 1, TT = 8192; };

// Consumer warps per CTA. K1-P at r <= 4: 12 warps (13 with the producer ->
// at most 4 per SM sub-partition -> 128 registers, nc <= 3): measured 0.87 ms
// vs 0.96 ms with 8 warps x 168 registers on BERT-L (latency-bound loop).
__host__ __device__ constexpr int nw_of(int mode, int RT) {
  return (mode == 0 && RT <= 4) ? 12 : 8;
}

__host__ __device__ constexpr int nc_max(int mode, int RT) {
  return mode == 0 ? (RT <= 4 ? 3 : (RT == 8 ? 4 : 0))
                   : (mode == 2 ? (RT <= 4 ? 3 : (RT == 8 ? 1 : 0)) : (RT <= 4 ? 4 : (RT == 8 ? 2 : 0)));
}

template <int NT>
__device__ __forceinline__ void cta_sync1() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}
__device__ __forceinline__ void group_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 zero4() { return make_float4(0.f, 0.f, 0.f, 0.f); }

struct Shared {
  float* sM;
  float* sE;
  uint64_t* full;
  uint64_t* empty;
  float* red;    // [2][16 warps][8] row-group partial sums
  float* gred;   // generic path block reduction [16][32]
  float4* cred;  // column mode: cross-row-slot combine [NW*32]
  float* sQl;    // K1-P deferred: local Q factor of the segment's layer [RT][m]
  float* sP;     // per stage: the tile's P rows [tr][RT] (staged by the producer warp)
  int ptile;     // floats per stage in sP
  int* flag;
  int stage_floats;
  int stages;
};

// Consumer position in the tile ring (stage, phase parity).
struct Pipe {
  int stage = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void advance(int stages) {
    if (++stage == stages) {
      stage = 0;
      phase ^= 1u;
    }
  }
};

template <int MODE>
struct ModeIdx { static constexpr int v = MODE == 0 ? 0 : (MODE == 2 ? 1 : 2); };

template <int MODE>
__device__ __forceinline__ bool is_fast(const LayerDesc& L, const float* grad) {
  return L.mat && L.sm[ModeIdx<MODE>::v].tr > 0 && ((reinterpret_cast<uintptr_t>(grad) & 15u) == 0);
}

// Producer warp (lane 0): walk the CTA's segments and issue every bulk tile
// as soon as its ring stage is released by all consumer warps.
template <int MODE>
__device__ void producer(const Tables& t, const StreamSeg* segs, int sb, int se, const Shared& sh,
                         int stage_p) {
  // lane 0 drives the ring (waits + bulk copies); when the consumers need the
  // tile's rows of the P factor (stage_p), the whole warp gathers them into
  // the stage's sP slot ([row][RT], zero-padded) before lane 0 arms the stage
  const int lane = threadIdx.x & 31;
  const uint64_t pol = policy_evict_first();
  int stage = 0;
  uint32_t phase = 0;
  for (int si = sb; si < se; ++si) {
    const StreamSeg s = segs[si];
    const LayerDesc& L = t.layers[s.layer];
    const float* grad = t.grads[s.layer];
    if (!is_fast<MODE>(L, grad)) continue;
    const StreamMap mp = L.sm[ModeIdx<MODE>::v];
    const int64_t m = L.m, n = L.n;
    const int r = L.r;
    const int tr = mp.tr;
    const int64_t c0 = (int64_t)s.panel * mp.pcols;
    const int64_t cols = (m - c0) < mp.pcols ? (m - c0) : mp.pcols;
    const float* pm = grad + s.row0 * m + c0;
    const float* pe = t.E + L.e_off + s.row0 * m + c0;
    const float* Pf = t.pbuf + L.p_off;
    const int RTp = sh.ptile > 0 ? sh.ptile / tr : 0;  // row stride in sP (>= r)
    // L2 prefetch of the tiles t.stream_pf ahead of the ring (whole-row
    // tiles): more HBM reads in flight than the shared-memory stages hold
    const int pf = (cols == m) ? t.stream_pf : 0;
    auto prefetch_tile = [&](int64_t rp) {
      if (rp < s.row1) {
        const uint32_t pb = (uint32_t)(((s.row1 - rp) < tr ? (s.row1 - rp) : tr) * m * 4);
        bulk_prefetch_l2(grad + rp * m, pb);
        bulk_prefetch_l2(t.E + L.e_off + rp * m, pb);
      }
    };
    if (pf > 0 && lane == 0)
      for (int j = 1; j <= pf; ++j) prefetch_tile(s.row0 + (int64_t)j * tr);
    for (int64_t r0 = s.row0; r0 < s.row1; r0 += tr) {
      const int64_t nr = (s.row1 - r0) < tr ? (s.row1 - r0) : tr;
      if (pf > 0 && lane == 0 && r0 > s.row0) prefetch_tile(r0 + (int64_t)pf * tr);
      if (lane == 0) mbar_wait(&sh.empty[stage], phase ^ 1u);
      __syncwarp();
      if (lane == 0) {
        float* dM = sh.sM + (size_t)stage * sh.stage_floats;
        float* dE = sh.sE + (size_t)stage * sh.stage_floats;
        if (cols == m) {  // whole rows: one contiguous copy per tensor
          const uint32_t bytes = (uint32_t)(nr * m * 4);
          mbar_arrive_tx(&sh.full[stage], 2 * bytes);
          bulk_g2s(dM, pm, bytes, &sh.full[stage], pol);
          bulk_g2s(dE, pe, bytes, &sh.full[stage], pol);
        } else {          // panel: one copy per row, smem row stride pcols
          const uint32_t rb = (uint32_t)(cols * 4);
          mbar_arrive_tx(&sh.full[stage], (uint32_t)(2 * nr) * rb);
          for (int64_t i = 0; i < nr; ++i) {
            bulk_g2s(dM + i * mp.pcols, pm + i * m, rb, &sh.full[stage], pol);
            bulk_g2s(dE + i * mp.pcols, pe + i * m, rb, &sh.full[stage], pol);
          }
        }
      }
      if (stage_p) {
        // the tile's P rows, gathered with async 4-byte copies (zero-filled
        // beyond r / nr); each lane's arrive fires when its copies landed, so
        // the producer never waits on these loads
        float* dP = sh.sP + (size_t)stage * sh.ptile;
        for (int idx = lane; idx < tr * RTp; idx += 32) {
          const int i = idx / RTp, k = idx - i * RTp;
          const bool ok = i < nr && k < r;
          cp_async4(dP + idx, ok ? Pf + (int64_t)k * n + r0 + i : Pf, ok ? 4u : 0u);
        }
        cp_async_arrive(&sh.full[stage]);
      }
      pm += nr * m;
      pe += nr * m;
      if (++stage == sh.stages) {
        stage = 0;
        phase ^= 1u;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K1 P-step, bulk-pipelined, lean consumer loop (~14 thread-instructions per
// element at r = 4): invalid chunks / rows read a valid (clamped) shared
// address and contribute 0 through zero factor registers or are simply not
// stored, so the loop has no data-dependent selects; dot products accumulate
// straight into the row sums with FMAs; whole-warp rows use an unconditional
// 5-level butterfly; rows spread over gw warps are combined by RT lanes
// after one named barrier and broadcast with RT shuffles.
// ---------------------------------------------------------------------------
template <int RT, int NC>
__device__ void seg_k1p(const Tables& t, const LayerDesc& L, const StreamSeg& s,
                        const Shared& sh, Pipe& pp, int& rph, int defer, int projonly) {
  constexpr int NW = nw_of(0, RT);
  const StreamMap mp = L.sm[0];
  const int lg = mp.lg, gw = mp.gw, rs = mp.rs, TR = mp.tr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = warp % gw, wrow = warp / gw;
  const int lgi = lane / lg, li = lane - lgi * lg;
  const int rowslot = wrow * (32 / lg) + lgi;
  const int NRS = (NW / gw) * (32 / lg);
  const int m = (int)L.m;
  const int n = (int)L.n;
  const int r = L.r;
  const int m4 = m >> 2;
  const int cbase = sub * lg * NC + li;
  int coff[NC];
  bool cval[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c = cbase + lg * i;
    cval[i] = c < m4;
    coff[i] = 4 * (cval[i] ? c : 0);
  }
  float4 qa[NC][RT];
  {
    const float* Qf = t.qbuf + L.q_off;
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
      for (int k = 0; k < RT; ++k) qa[i][k] = (cval[i] && k < r) ? ld_f4(Qf + k * m + coff[i]) : zero4();
  }
  float* __restrict__ E = t.E + L.e_off;
  float* __restrict__ Pw = t.pbuf + L.p_off;
  const bool pwriter = (sub == 0) && (li == 0);
  if (defer) {
    // deferred Q-step residual: stage this layer's local Q (k-major) in
    // shared memory; E_prev = S - P_o Q_loc^T is formed on the fly per row
    const float* Ql = t.qloc + L.ql_off;
    cta_sync1<NW * 32>();  // previous segment's readers are done
    for (int idx = threadIdx.x; idx < RT * m4; idx += NW * 32) {
      const int k = idx / m4, c = idx - k * m4;
      *reinterpret_cast<float4*>(sh.sQl + k * m + 4 * c) = k < r ? ld_f4(Ql + k * m + 4 * c) : zero4();
    }
    cta_sync1<NW * 32>();
  }
  // x = M + S - sum_k po[k] Q_loc[k] (po = 0 when E is materialised)
  auto corrected = [&](const float* tM, const float* tE, int toff, int i, const float (&po)[RT]) {
    float4 xi = f4add(lds4(tM + toff + coff[i]), lds4(tE + toff + coff[i]));
    if (defer) {
#pragma unroll
      for (int k = 0; k < RT; ++k) f4fma(xi, -po[k], lds4(sh.sQl + k * m + coff[i]));
    }
    return xi;
  };
  for (int64_t r0 = s.row0; r0 < s.row1; r0 += TR) {
    const int nr = (int)((s.row1 - r0) < TR ? (s.row1 - r0) : TR);
    const int stage = pp.stage;
    mbar_wait(&sh.full[stage], pp.phase);
    const float* tM = sh.sM + (size_t)stage * sh.stage_floats;
    const float* tE = sh.sE + (size_t)stage * sh.stage_floats;
    for (int j = 0; j < rs; ++j) {
      const int tri = rowslot + NRS * j;
      const bool rval = tri < nr;
      const int toff = (rval ? tri : 0) * m;
      // RT >= 8: x is re-read from shared memory for the residual (registers
      // go to the factor); the stage is then released after the residual
      constexpr bool kReload = RT >= 8;
      float po[RT];  // P_o row staged by the producer (zero beyond r)
      {
        const float* ps = sh.sP + (size_t)stage * sh.ptile + (rval ? tri : 0) * (sh.ptile / TR);
#pragma unroll
        for (int k = 0; k < RT; ++k) po[k] = defer ? ps[k] : 0.f;
      }
      float4 x[kReload ? 1 : NC];
      float acc[RT];
#pragma unroll
      for (int k = 0; k < RT; ++k) acc[k] = 0.f;
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const float4 xi = corrected(tM, tE, toff, i, po);
        if constexpr (!kReload) x[i] = xi;
#pragma unroll
        for (int k = 0; k < RT; ++k) {
          acc[k] = fmaf(xi.x, qa[i][k].x, acc[k]);
          acc[k] = fmaf(xi.y, qa[i][k].y, acc[k]);
          acc[k] = fmaf(xi.z, qa[i][k].z, acc[k]);
          acc[k] = fmaf(xi.w, qa[i][k].w, acc[k]);
        }
      }
      if (!kReload && j == rs - 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.empty[stage]);
      }
      if (lg == 32) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
          for (int k = 0; k < RT; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
      } else {
        for (int off = lg >> 1; off > 0; off >>= 1)
#pragma unroll
          for (int k = 0; k < RT; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
      }
      if (gw > 1) {
        float* buf = sh.red + (rph & 1) * (16 * 8);
        ++rph;
        float mine = acc[0];
#pragma unroll
        for (int k = 1; k < RT; ++k)
          if (lane == k) mine = acc[k];
        if (lane < RT) buf[warp * 8 + lane] = mine;
        cta_sync1<NW * 32>();
        float tot = 0.f;
        if (lane < RT) {
          const float* gb = buf + (wrow * gw) * 8 + lane;
          for (int w = 0; w < gw; ++w) tot += gb[w * 8];
        }
#pragma unroll
        for (int k = 0; k < RT; ++k) acc[k] = __shfl_sync(0xffffffffu, tot, k);
      }
      const int64_t row = r0 + tri;
      if (!projonly) {
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          float4 e;
          if constexpr (kReload) e = corrected(tM, tE, toff, i, po);
          else e = x[i];
#pragma unroll
          for (int k = 0; k < RT; ++k) f4fma(e, -acc[k], qa[i][k]);
          if (rval && cval[i]) st_cs4(E + row * m + coff[i], e);
        }
      }
      if (kReload && j == rs - 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.empty[stage]);
      }
      if (rval && pwriter) {
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) Pw[(int64_t)k * n + row] = acc[k];
      }
    }
    pp.advance(sh.stages);
  }
}

// ---------------------------------------------------------------------------
// fast (bulk-pipelined) segment
// ---------------------------------------------------------------------------
template <int MODE, int RT, int NC>
__device__ void seg_fast(const Tables& t, const LayerDesc& L, const StreamSeg& s,
                         float* __restrict__ grad, float scale, const Shared& sh, Pipe& pp,
                         int& rph, int defer) {
  constexpr int NW = nw_of(MODE, RT);
  const StreamMap mp = L.sm[ModeIdx<MODE>::v];
  const int lg = mp.lg, gw = mp.gw, rs = mp.rs, TR = mp.tr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = warp % gw, wrow = warp / gw;
  const int lgi = lane / lg, li = lane - lgi * lg;
  const int rowslot = wrow * (32 / lg) + lgi;
  const int NRS = (NW / gw) * (32 / lg);
  const int m = (int)L.m;
  const int n = (int)L.n;
  const int r = L.r;
  const int pc = mp.pcols;                         // smem row stride (floats)
  const int c0 = s.panel * pc;                     // first column of the panel
  const int m4 = ((m - c0) < pc ? (m - c0) : pc) >> 2;  // chunks in this panel
  const int cbase = sub * lg * NC + li;
  int coff[NC];
  bool cval[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c = cbase + lg * i;
    cval[i] = c < m4;
    coff[i] = 4 * (cval[i] ? c : 0);
  }
  float* __restrict__ E = t.E + L.e_off + c0;      // panel origin (global)
  grad += c0;

  // factor(s) in registers for the whole segment (k >= r and invalid chunks: 0)
  float4 qa[MODE == 3 ? 1 : NC][MODE == 3 ? 1 : RT];
  float4 qb[MODE == 2 ? NC : 1][MODE == 2 ? RT : 1];
  float4 acc3[MODE == 3 ? NC : 1][MODE == 3 ? RT : 1];
  if constexpr (MODE != 3) {
    const float* Qf = t.qbuf + L.q_off + c0;
    const float* Ql = t.qloc + L.ql_off + c0;
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
      for (int k = 0; k < RT; ++k) {
        const bool ok = cval[i] && k < r;
        qa[i][k] = ok ? ld_f4(Qf + k * m + coff[i]) : zero4();
        if constexpr (MODE == 2) qb[i][k] = ok ? ld_f4(Ql + k * m + coff[i]) : zero4();
      }
  } else {
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
      for (int k = 0; k < RT; ++k) acc3[i][k] = zero4();
  }

  for (int64_t r0 = s.row0; r0 < s.row1; r0 += TR) {
    const int nr = (int)((s.row1 - r0) < TR ? (s.row1 - r0) : TR);
    const int stage = pp.stage;
    mbar_wait(&sh.full[stage], pp.phase);
    const float* tM = sh.sM + (size_t)stage * sh.stage_floats;
    const float* tE = sh.sE + (size_t)stage * sh.stage_floats;
    for (int j = 0; j < rs; ++j) {
      const int tri = rowslot + NRS * j;  // row within the tile
      const bool rval = tri < nr;
      const int64_t row = r0 + (rval ? tri : 0);
      const int toff = (rval ? tri : 0) * pc;
      float4 x[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const float4 a = lds4(tM + toff + coff[i]);
        const float4 b = lds4(tE + toff + coff[i]);
        x[i] = (rval && cval[i]) ? f4add(a, b) : zero4();
      }
      // P row staged by the producer (zero beyond r): read BEFORE the stage
      // is released -- the producer regathers the stage's P rows for a later
      // tile as soon as every warp has arrived (reading it after the arrive
      // was a rare cross-warp race: one warp's rows projected on the next
      // tile's P rows, ~5e-4 on a Q factor panel)
      float pk[RT];
      if constexpr (MODE != 0) {
        const float* ps = sh.sP + (size_t)stage * sh.ptile + (rval ? tri : 0) * (sh.ptile / TR);
#pragma unroll
        for (int k = 0; k < RT; ++k) pk[k] = ps[k];
      }
      if (j == rs - 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.empty[stage]);
      }
      if constexpr (MODE == 0) {
        float acc[RT];
#pragma unroll
        for (int k = 0; k < RT; ++k) {
          float a = 0.f;
#pragma unroll
          for (int i = 0; i < NC; ++i) a += f4dot(x[i], qa[i][k]);
          acc[k] = a;
        }
        // sum over the lg lanes of the row group (butterfly: all lanes get it)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          if (off < lg) {
#pragma unroll
            for (int k = 0; k < RT; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
          }
        }
        // ... and over the gw warps of the row group (shared memory). The
        // barrier spans the whole CTA: named barriers with per-group thread
        // counts could alias across consecutive segments with different gw.
        if (gw > 1) {
          float* buf = sh.red + (rph & 1) * (16 * 8);  // [2][16 warps][8]
          if (lane < RT) {
            float v = acc[0];
#pragma unroll
            for (int k = 1; k < RT; ++k)
              if (lane == k) v = acc[k];
            buf[warp * 8 + lane] = v;
          }
          cta_sync1<NW * 32>();  // uniform across the CTA (every warp has the same rows)
          const float* gb = buf + (wrow * gw) * 8;
#pragma unroll
          for (int k = 0; k < RT; ++k) acc[k] = 0.f;
          for (int w = 0; w < gw; ++w) {
            if constexpr (RT >= 4) {
#pragma unroll
              for (int k = 0; k < RT; k += 4) {
                const float4 v = lds4(gb + w * 8 + k);
                acc[k] += v.x;
                acc[k + 1] += v.y;
                acc[k + 2] += v.z;
                acc[k + 3] += v.w;
              }
            } else {
#pragma unroll
              for (int k = 0; k < RT; ++k) acc[k] += gb[w * 8 + k];
            }
          }
        }
        ++rph;
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          float4 e = x[i];
#pragma unroll
          for (int k = 0; k < RT; ++k) f4fma(e, -acc[k], qa[i][k]);
          if (rval && cval[i]) st_cs4(E + row * m + coff[i], e);
        }
        if (rval && sub == 0 && li == 0) {
#pragma unroll
          for (int k = 0; k < RT; ++k)
            if (k < r) t.pbuf[L.p_off + (int64_t)k * n + row] = acc[k];
        }
      } else {
        if constexpr (MODE == 2) {
#pragma unroll
          for (int i = 0; i < NC; ++i) {
            float4 e = x[i], o = zero4();
#pragma unroll
            for (int k = 0; k < RT; ++k) {
              f4fma(e, -pk[k], qb[i][k]);
              f4fma(o, pk[k], qa[i][k]);
            }
            if (rval && cval[i]) {
              st_cs4(E + row * m + coff[i], e);
              st_cs4(grad + row * m + coff[i], f4scale(o, scale));
            }
          }
        } else {
          if (defer) {  // deferred Q-step residual: keep S = M' in E
            const int64_t rowg = r0 + tri;
#pragma unroll
            for (int i = 0; i < NC; ++i)
              if (rval && cval[i]) st_cs4(E + rowg * m + coff[i], x[i]);
          }
#pragma unroll
          for (int i = 0; i < NC; ++i)
#pragma unroll
            for (int k = 0; k < RT; ++k) {
              acc3[i][k].x = fmaf(x[i].x, pk[k], acc3[i][k].x);
              acc3[i][k].y = fmaf(x[i].y, pk[k], acc3[i][k].y);
              acc3[i][k].z = fmaf(x[i].z, pk[k], acc3[i][k].z);
              acc3[i][k].w = fmaf(x[i].w, pk[k], acc3[i][k].w);
            }
        }
      }
    }
    pp.advance(sh.stages);
  }
  if constexpr (MODE == 3) {
    // combine the row slots of the CTA (fixed order) and write ONE partial
    // slot for this segment: k-major [r][pc], stride round4(r * pc)
    float* part = t.colpart + s.part_off;
    const int rpw = 32 / lg;  // row slots per warp
#pragma unroll
    for (int i = 0; i < NC; ++i) {
#pragma unroll
      for (int k = 0; k < RT; ++k) {
        cta_sync1<NW * 32>();
        sh.cred[threadIdx.x] = acc3[i][k];
        cta_sync1<NW * 32>();
        if (rowslot == 0 && cval[i] && k < r) {
          float4 sum = acc3[i][k];
          for (int j = 1; j < NRS; ++j) {
            const int w = (j / rpw) * gw + sub, ln = (j % rpw) * lg + li;
            sum = f4add(sum, sh.cred[w * 32 + ln]);
          }
          *reinterpret_cast<float4*>(part + (int64_t)k * pc + coff[i]) = sum;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// generic segment (any m / alignment)
// ---------------------------------------------------------------------------
template <int NT, int RT>
__device__ __forceinline__ void block_sum(float (&a)[RT], float* red) {
  constexpr int NWp = NT / 32;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < RT; ++k) a[k] += __shfl_xor_sync(0xffffffffu, a[k], off);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  cta_sync1<NT>();
#pragma unroll
  for (int k = 0; k < RT; ++k)
    if (lane == (k & 31)) red[warp * 32 + k] = a[k];
  cta_sync1<NT>();
#pragma unroll
  for (int k = 0; k < RT; ++k) {
    float s = red[k];
    for (int w = 1; w < NWp; ++w) s += red[w * 32 + k];
    a[k] = s;
  }
}

template <int MODE, int RT>
__device__ void seg_generic(const Tables& t, const LayerDesc& L, const StreamSeg& s,
                            float* __restrict__ grad, float scale, float* red, int defer) {
  // Generic path (m % 4 != 0, very wide m, or an unaligned gradient): plain
  // coalesced scalar accesses. Rows are spread over the warps (one warp per
  // row, lanes stride the columns, warp-shuffle row sums) so a layer with many
  // short rows does not serialise on CTA barriers; the column reduction
  // (mode 3) gives each thread a column and unrolls its row loop.
  constexpr int NWc = nw_of(MODE, RT);
  constexpr int NT = NWc * 32;
  (void)red;
  const int64_t m = L.m, n = L.n;
  const int r = L.r;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* __restrict__ Qs = t.qbuf + L.q_off;
  const float* __restrict__ Ql = t.qloc + L.ql_off;
  float* __restrict__ Ps = t.pbuf + L.p_off;
  float* __restrict__ E = t.E + L.e_off;
  // column range of this segment's panel (modes 2, 3; generic layers have one)
  const StreamMap mp = L.sm[ModeIdx<MODE>::v];
  const int64_t pc = (MODE != 0 && mp.tr > 0) ? mp.pcols : m;
  const int64_t c0 = (int64_t)s.panel * pc;
  const int64_t c1 = (c0 + pc) < m ? (c0 + pc) : m;
  if constexpr (MODE == 3) {
    float* part = t.colpart + s.part_off;
    for (int64_t cb = c0; cb < c1; cb += NT) {
      const int64_t c = cb + threadIdx.x;
      if (c < c1) {
        float acc[RT];
#pragma unroll
        for (int k = 0; k < RT; ++k) acc[k] = 0.f;
        int64_t row = s.row0;
        for (; row + 4 <= s.row1; row += 4) {
          float x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) x[u] = grad[(row + u) * m + c] + E[(row + u) * m + c];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (defer) E[(row + u) * m + c] = x[u];  // deferred residual: keep S = M'
#pragma unroll
            for (int k = 0; k < RT; ++k)
              if (k < r) acc[k] = fmaf(x[u], __ldg(Ps + k * n + row + u), acc[k]);
          }
        }
        for (; row < s.row1; ++row) {
          const float x = grad[row * m + c] + E[row * m + c];
          if (defer) E[row * m + c] = x;
#pragma unroll
          for (int k = 0; k < RT; ++k)
            if (k < r) acc[k] = fmaf(x, __ldg(Ps + k * n + row), acc[k]);
        }
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) part[k * pc + (c - c0)] = acc[k];
      }
    }
    return;
  }
  const int projonly = (MODE == 0) && (defer & 2);  // Power-SGD: no residual here
  defer &= 1;
  for (int64_t row = s.row0 + warp; row < s.row1; row += NWc) {
    float* __restrict__ gr = grad + row * m;
    float* __restrict__ er = E + row * m;
    if constexpr (MODE == 0) {
      float po[RT];  // deferred: E_prev = S - P_o Q_loc^T (P slot still holds P_o)
#pragma unroll
      for (int k = 0; k < RT; ++k) po[k] = (defer && k < r) ? Ps[k * n + row] : 0.f;
      float acc[RT];
#pragma unroll
      for (int k = 0; k < RT; ++k) acc[k] = 0.f;
      for (int64_t j = lane; j < m; j += 32) {
        float x = gr[j] + er[j];
        if (defer) {
#pragma unroll
          for (int k = 0; k < RT; ++k)
            if (k < r) x = fmaf(-po[k], __ldg(Ql + k * m + j), x);
        }
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) acc[k] = fmaf(x, __ldg(Qs + k * m + j), acc[k]);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int k = 0; k < RT; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
      for (int64_t j = lane; j < m && !projonly; j += 32) {
        float x = gr[j] + er[j];
        if (defer) {
#pragma unroll
          for (int k = 0; k < RT; ++k)
            if (k < r) x = fmaf(-po[k], __ldg(Ql + k * m + j), x);
        }
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) x = fmaf(-acc[k], __ldg(Qs + k * m + j), x);
        er[j] = x;
      }
      __syncwarp();  // every lane has read P_o of this row
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < RT; ++k)
          if (k < r) Ps[k * n + row] = acc[k];
      }
    } else {
      float p[RT];
#pragma unroll
      for (int k = 0; k < RT; ++k) p[k] = (k < r) ? __ldg(Ps + k * n + row) : 0.f;
      for (int64_t j = c0 + lane; j < c1; j += 32) {
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

template <int MODE, int RT>
__global__ void __launch_bounds__(nw_of(MODE, RT) * 32 + 32, Cfg<MODE>::CPS)
    stream_kernel(Tables t, const StreamSeg* __restrict__ segs, const int32_t* __restrict__ cta_begin,
                  float scale, int stages, int stage_floats, int factor_floats, int defer,
                  int ptile) {
  constexpr int NT = nw_of(MODE, RT) * 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Shared sh;
  sh.stages = stages;
  sh.stage_floats = stage_floats;
  sh.sM = reinterpret_cast<float*>(smem_raw);
  sh.sE = sh.sM + (size_t)stages * stage_floats;
  sh.full = reinterpret_cast<uint64_t*>(sh.sE + (size_t)stages * stage_floats);
  sh.empty = sh.full + stages;
  sh.red = reinterpret_cast<float*>(sh.empty + stages);
  sh.gred = sh.red + 2 * 16 * 8;
  sh.cred = reinterpret_cast<float4*>(sh.gred + 16 * 32);
  sh.sQl = reinterpret_cast<float*>(sh.cred + 16 * 32);
  sh.sP = sh.sQl + factor_floats;
  sh.ptile = ptile;
  sh.flag = reinterpret_cast<int*>(sh.sP + (size_t)stages * ptile);
  // the producer warp stages P rows (32 cp.async arrivals per tile) for the
  // Q-step kernels and, when the residual is deferred, for the P-step one
  const int stage_p = (ptile > 0) && (MODE != 0 || ((defer & 1) && *t.deferred));
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&sh.full[i], stage_p ? 33 : 1);
      mbar_init(&sh.empty[i], nw_of(MODE, RT));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int sb = cta_begin[blockIdx.x], se = cta_begin[blockIdx.x + 1];
  prefetch_segs(t, segs, sb, se);
  // deferred Q-step residual: K1 Q-step raises the flag (nothing in that
  // launch reads it); K1 P-step reads it (cleared later by the P decode)
  // defer bit 1 (mode 0): projection only, no residual (Power-SGD, whose
  // residual is formed after the second projection)
  const int projonly = (MODE == 0) && (defer & 2);
  defer &= 1;
  int dflag = 0;
  if (MODE == 3 && defer && blockIdx.x == 0 && threadIdx.x == 0) *t.deferred = 1;
  if (MODE == 0 && defer) dflag = *t.deferred;
  if ((threadIdx.x >> 5) == nw_of(MODE, RT)) {  // producer warp
    producer<MODE>(t, segs, sb, se, sh, stage_p);
    return;
  }
  Pipe pp;
  int rph = 0;
  for (int si = sb; si < se; ++si) {
    if (!t.layers[segs[si].layer].mat) {
      si = vector_run(t, segs, si, se, threadIdx.x >> 5, NT / 32,
                      [&](const StreamSeg& s, const LayerDesc& L, int first, int stride) {
                        float* grad = t.grads[s.layer];
                        if (MODE == 0 || MODE == 3) {
                          float* slot = (MODE == 0 ? t.pbuf + L.p_off : t.qbuf + L.q_off);
                          for (int64_t i = s.row0 + first; i < s.row1; i += stride) slot[i] = grad[i];
                        } else {
                          const float* slot = t.qbuf + L.q_off;
                          for (int64_t i = s.row0 + first; i < s.row1; i += stride) grad[i] = slot[i] * scale;
                        }
                      }) - 1;
      continue;
    }
    const StreamSeg s = segs[si];
    const LayerDesc& L = t.layers[s.layer];
    float* grad = t.grads[s.layer];
    if (!is_fast<MODE>(L, grad)) {
      seg_generic<MODE, RT>(t, L, s, grad, scale, sh.gred, MODE == 0 ? (dflag | (projonly << 1)) : defer);
    } else {
      switch (L.sm[ModeIdx<MODE>::v].nc) {
#define ACP_CASE(NCV)                                                            \
  case NCV:                                                                      \
    if constexpr (NCV <= nc_max(MODE, RT)) {                                     \
      if constexpr (MODE == 0) seg_k1p<RT, NCV>(t, L, s, sh, pp, rph, dflag, projonly); \
      else seg_fast<MODE, RT, NCV>(t, L, s, grad, scale, sh, pp, rph, defer);   \
    }                                                                            \
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
  }
}

// ---------------------------------------------------------------------------
// K1 P-step at r <= 4, two rows per pass (k1p_kernel, the default for the
// ACP P-step at r <= 4; ACP_K1P_OLD=1 selects stream_kernel<0> / seg_k1p).
// Same tiles, ring and thread-to-column map as seg_k1p, with the per-row
// overhead that made seg_k1p issue-bound (ncu: ~480 warp instructions per
// row slot, 40 per element, of which 12 are the arithmetic) taken out:
//  * the producer role is folded into consumer warp 0, which fills the ring
//    at each tile start (two bulk copies per tile, from addresses cached
//    per segment): 12 warps = 3 per SM sub-partition -> 168 registers
//    instead of the 128 a 13th warp leaves, which pays for two rows in
//    flight per warp;
//  * the P_o rows of the deferred correction are not gathered into the
//    ring by the producer (32 lanes of 4-byte cp.async per tile: with the
//    1-row tiles of ResNet's wide layers that made warp 0 the bottleneck,
//    every other warp waiting at the pass barrier -- 0.149 vs 0.101 ms)
//    but loaded by the consumers from the P slot one pass ahead;
//  * the 2*RT row sums of the two rows are reduced by a transposing
//    butterfly (each level halves the values a lane carries: 2*RT - 1 +
//    5 - log2(2*RT) shuffles instead of 5 * 2*RT), rows spread over gw warps
//    take one named barrier per two rows, and the cross-warp sum is spread
//    over the lanes that share a value;
//  * the staged Q_loc columns of the deferred correction are loaded once
//    for both rows, and the deferred / not-deferred loops are separate
//    instantiations.
// Measured (B200, A/B against ACP_K1P_OLD=1, same box): BERT-L r=4 K1-P'
// 0.836 -> 0.689 ms (4.04 GB: 5.87 TB/s), ResNet-50 0.1015 -> 0.0825,
// ResNet-152 0.218 -> 0.177. A variant with 8 consumer warps + a producer
// warp (168 registers, up to 4 chunks per lane) spilled at r = 4 and left
// ResNet's m = 4608 layers without a map (generic path): 0.75 ms.
// ---------------------------------------------------------------------------
constexpr int kK1pWarps = 12;

// Ring producer state (warp 0; identical in its 32 lanes). The current
// segment's addresses are cached here when the producer reaches it, so a
// tile costs warp 0 no dependent descriptor loads (a 1-row tile of a
// ResNet layer is only ~700 cycles of work for the CTA, and every warp
// waits for warp 0 at the tile's pass barrier).
struct Prod {
  int si;            // segment of the next tile (a fast segment with rows left, or se)
  int stage;
  uint32_t phase;
  int issued;        // tiles issued so far
  int64_t r0, row1;  // next tile's first row, segment end
  const float* gm;   // M row r0
  const float* ge;   // E row r0
  uint32_t rowb;     // bytes per row
  int tr;
};

__device__ __forceinline__ void prod_seek(const Tables& t, const StreamSeg* segs, int se, Prod& pr) {
  for (; pr.si < se; ++pr.si) {
    const StreamSeg s = segs[pr.si];
    const LayerDesc& L = t.layers[s.layer];
    const float* grad = t.grads[s.layer];
    if (!is_fast<0>(L, grad) || s.row0 >= s.row1) continue;
    pr.r0 = s.row0;
    pr.row1 = s.row1;
    pr.gm = grad + s.row0 * L.m;
    pr.ge = t.E + L.e_off + s.row0 * L.m;
    pr.rowb = (uint32_t)(L.m * 4);
    pr.tr = L.sm[0].tr;
    return;
  }
}

// Issue the next tile into pr.stage (its stage is known to be free): one
// bulk copy per tensor (whole rows) by lane 0. (The P_o rows of the
// deferred correction are not staged: the consumers load them from the P
// slot one pass ahead.)
__device__ __forceinline__ void prod_issue(const Tables& t, const StreamSeg* segs, int se,
                                           const Shared& sh, Prod& pr, uint64_t pol) {
  const int lane = threadIdx.x & 31;
  const int tr = pr.tr;
  const int64_t nr = (pr.row1 - pr.r0) < tr ? (pr.row1 - pr.r0) : tr;
  if (lane == 0) {
    uint64_t* full = &sh.full[pr.stage];
    const uint32_t bytes = (uint32_t)nr * pr.rowb;
    mbar_arrive_tx(full, 2 * bytes);
    bulk_g2s(sh.sM + (size_t)pr.stage * sh.stage_floats, pr.gm, bytes, full, pol);
    bulk_g2s(sh.sE + (size_t)pr.stage * sh.stage_floats, pr.ge, bytes, full, pol);
  }
  ++pr.issued;
  if (++pr.stage == sh.stages) {
    pr.stage = 0;
    pr.phase ^= 1u;
  }
  pr.r0 += tr;
  const int64_t adv = (int64_t)tr * (pr.rowb >> 2);
  pr.gm += adv;
  pr.ge += adv;
  if (pr.r0 >= pr.row1) {
    ++pr.si;
    prod_seek(t, segs, se, pr);
  }
}

// Warp 0 issues tiles while fewer than `upto` are issued; called at each
// tile start with upto = tile + stages, i.e. it fills the ring. The last of
// those tiles reuses the stage of the previous tile, so this waits until
// every warp has released that one (in layers whose rows span several warps
// the pass barrier has already ensured it). Issuing only what is free at
// that moment collapses the lookahead to one tile whenever the warps drift
// apart, and extra early refill attempts (right after the last pass's
// cross-warp barrier) delay warp 0 at the next barrier: both measured
// slower.
__device__ __forceinline__ void produce(const Tables& t, const StreamSeg* segs, int se, const Shared& sh,
                                        Prod& pr, int upto, bool block, uint64_t pol) {
  const int lane = threadIdx.x & 31;
  while (pr.si < se && pr.issued < upto) {
    uint32_t ok = 1;
    if (lane == 0) {
      if (block) mbar_wait(&sh.empty[pr.stage], pr.phase ^ 1u);
      else ok = mbar_test(&sh.empty[pr.stage], pr.phase ^ 1u) ? 1u : 0u;
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    if (!ok) break;
    prod_issue(t, segs, se, sh, pr, pol);
  }
}

template <int RT, int NC, bool DEFER>
__device__ void seg_k1p2(const Tables& t, const StreamSeg* segs, int se, const LayerDesc& L,
                         const StreamSeg& s, const Shared& sh, Pipe& pp, Prod& pr, int& consumed,
                         int& rph, uint64_t pol) {
  constexpr int NW = kK1pWarps;
  const StreamMap mp = L.sm[0];
  const int lg = mp.lg, gw = mp.gw, rs = mp.rs, TR = mp.tr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = warp % gw, wrow = warp / gw;
  const int lgi = lane / lg, li = lane - lgi * lg;
  const int rowslot = wrow * (32 / lg) + lgi;
  const int NRS = (NW / gw) * (32 / lg);
  const int m = (int)L.m;
  const int n = (int)L.n;
  const int r = L.r;
  const int m4 = m >> 2;
  const int cbase = sub * lg * NC + li;
  int coff[NC];
  bool cval[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c = cbase + lg * i;
    cval[i] = c < m4;
    coff[i] = 4 * (cval[i] ? c : 0);
  }
  float4 qa[NC][RT];
  {
    const float* Qf = t.qbuf + L.q_off;
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
      for (int k = 0; k < RT; ++k) qa[i][k] = (cval[i] && k < r) ? ld_f4(Qf + k * m + coff[i]) : zero4();
  }
  float* __restrict__ E = t.E + L.e_off;
  float* __restrict__ Pw = t.pbuf + L.p_off;
  if constexpr (DEFER) {
    // stage this layer's local Q (k-major) for E_prev = S - P_o Q_loc^T
    const float* Ql = t.qloc + L.ql_off;
    cta_sync1<NW * 32>();  // previous segment's readers are done
    for (int idx = threadIdx.x; idx < RT * m4; idx += NW * 32) {
      const int k = idx / m4, c = idx - k * m4;
      *reinterpret_cast<float4*>(sh.sQl + k * m + 4 * c) = k < r ? ld_f4(Ql + k * m + 4 * c) : zero4();
    }
    cta_sync1<NW * 32>();
  }
  // P_o rows of the deferred correction, straight from the P slot (which
  // still holds P_o until this kernel overwrites the row with P_loc, after
  // every warp of the row group has read it), loaded one pass ahead so the
  // L2 latency overlaps the previous pass
  float pn[2][RT];
  auto load_po = [&](int64_t r0x, int jx) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t rw = r0x + rowslot + NRS * (jx + h);
      const bool ok = (jx + h < rs) && (rw < s.row1);
#pragma unroll
      for (int k = 0; k < RT; ++k) pn[h][k] = (ok && k < r) ? __ldcg(Pw + (int64_t)k * n + rw) : 0.f;
    }
  };
  if constexpr (DEFER) load_po(s.row0, 0);
  for (int64_t r0 = s.row0; r0 < s.row1; r0 += TR) {
    const int nr = (int)((s.row1 - r0) < TR ? (s.row1 - r0) : TR);
    if (warp == 0) produce(t, segs, se, sh, pr, consumed + sh.stages, true, pol);
    const int stage = pp.stage;
    mbar_wait(&sh.full[stage], pp.phase);
    const float* tM = sh.sM + (size_t)stage * sh.stage_floats;
    const float* tE = sh.sE + (size_t)stage * sh.stage_floats;
    // one pass over ROWS (2, or 1 for an odd tail) rows of the tile
    auto pass = [&](auto rows_c, int j) {
      constexpr int ROWS = decltype(rows_c)::value;
      constexpr int V = ROWS * RT;                       // row sums carried
      constexpr int LOGV = V == 1 ? 0 : (V == 2 ? 1 : (V == 4 ? 2 : 3));
      constexpr int G = 32 >> LOGV;                      // lanes sharing one reduced value
      int tri[ROWS], toff[ROWS];
      bool rv[ROWS];
      int64_t row[ROWS];
#pragma unroll
      for (int h = 0; h < ROWS; ++h) {
        tri[h] = rowslot + NRS * (j + h);
        rv[h] = tri[h] < nr;
        toff[h] = (rv[h] ? tri[h] : 0) * m;
        row[h] = r0 + tri[h];
      }

      float4 x[ROWS][NC];
      float v[V];
#pragma unroll
      for (int q = 0; q < V; ++q) v[q] = 0.f;
#pragma unroll
      for (int i = 0; i < NC; ++i) {
#pragma unroll
        for (int h = 0; h < ROWS; ++h)
          x[h][i] = f4add(lds4(tM + toff[h] + coff[i]), lds4(tE + toff[h] + coff[i]));
        if constexpr (DEFER) {
#pragma unroll
          for (int k = 0; k < RT; ++k) {
            const float4 ql = lds4(sh.sQl + k * m + coff[i]);  // shared by the rows
#pragma unroll
            for (int h = 0; h < ROWS; ++h) f4fma(x[h][i], -pn[h][k], ql);
          }
        }
#pragma unroll
        for (int h = 0; h < ROWS; ++h)
#pragma unroll
          for (int k = 0; k < RT; ++k) {
            float& a = v[h * RT + k];
            a = fmaf(x[h][i].x, qa[i][k].x, a);
            a = fmaf(x[h][i].y, qa[i][k].y, a);
            a = fmaf(x[h][i].z, qa[i][k].z, a);
            a = fmaf(x[h][i].w, qa[i][k].w, a);
          }
      }
      if constexpr (DEFER) {
        // P_o of the next pass (the next row pair of this tile, else the
        // next tile's first), in flight during this pass's reduction
        if (j + 2 < rs) load_po(r0, j + 2);
        else if (r0 + TR < s.row1) load_po(r0 + TR, 0);
      }
      if (j + ROWS >= rs) {  // the tile's last pass: release the stage
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.empty[stage]);
      }
      float tot[V];
      if (lg == 32) {
        // transposing butterfly: at the level with offset 16 >> l a lane
        // hands half of its values to its partner and keeps the other half
        // (lane bit 4 - l picks which), until one value is left; the last
        // 5 - LOGV levels are a plain butterfly on that value
#pragma unroll
        for (int lev = 0; lev < 5; ++lev) {
          const int off = 16 >> lev;
          const int w = lev < LOGV ? (V >> lev) : 1;
          if (w > 1) {
            const bool up = (lane & off) != 0;
            const int hw = w >> 1;
#pragma unroll
            for (int q = 0; q < hw; ++q) {
              const float send = up ? v[q] : v[q + hw];
              const float keep = up ? v[q + hw] : v[q];
              v[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
          } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
          }
        }
        const int qi = LOGV == 0 ? 0 : ((lane >> (5 - LOGV)) & (V - 1));  // this lane's row sum
        if (gw > 1) {
          float* buf = sh.red + (rph & 1) * (16 * 8);
          ++rph;
          if ((lane & (G - 1)) == 0) buf[warp * 8 + qi] = v[0];
          cta_sync1<NW * 32>();
          float sum = 0.f;
          for (int w = lane & (G - 1); w < gw; w += G) sum += buf[(wrow * gw + w) * 8 + qi];
#pragma unroll
          for (int off = 1; off < G; off <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
          v[0] = sum;
        }
        if (sub == 0 && (lane & (G - 1)) == 0) {
          const int h = qi / RT, k = qi - h * RT;
          int64_t rw = row[0];  // row[h] without a local-memory array
          bool ok = rv[0];
#pragma unroll
          for (int hh = 1; hh < ROWS; ++hh)
            if (h == hh) {
              rw = row[hh];
              ok = rv[hh];
            }
          if (k < r && ok) Pw[(int64_t)k * n + rw] = v[0];
        }
#pragma unroll
        for (int q = 0; q < V; ++q) tot[q] = __shfl_sync(0xffffffffu, v[0], q << (5 - LOGV));
      } else {
        for (int off = lg >> 1; off > 0; off >>= 1)
#pragma unroll
          for (int q = 0; q < V; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
#pragma unroll
        for (int q = 0; q < V; ++q) tot[q] = v[q];
        if (li == 0) {
#pragma unroll
          for (int h = 0; h < ROWS; ++h)
#pragma unroll
            for (int k = 0; k < RT; ++k)
              if (k < r && rv[h]) Pw[(int64_t)k * n + row[h]] = tot[h * RT + k];
        }
      }
#pragma unroll
      for (int h = 0; h < ROWS; ++h) {
        float* __restrict__ er = E + row[h] * m;
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          float4 a = x[h][i];
#pragma unroll
          for (int k = 0; k < RT; ++k) f4fma(a, -tot[h * RT + k], qa[i][k]);
          if (rv[h] && cval[i]) st_cs4(er + coff[i], a);
        }
      }
    };
    int j = 0;
    for (; j + 2 <= rs; j += 2) pass(std::integral_constant<int, 2>{}, j);
    if (j < rs) pass(std::integral_constant<int, 1>{}, j);
    pp.advance(sh.stages);
    ++consumed;
  }
}

__device__ __forceinline__ Shared make_shared(unsigned char* smem_raw, int stages, int stage_floats,
                                              int factor_floats, int ptile) {
  Shared sh;
  sh.stages = stages;
  sh.stage_floats = stage_floats;
  sh.sM = reinterpret_cast<float*>(smem_raw);
  sh.sE = sh.sM + (size_t)stages * stage_floats;
  sh.full = reinterpret_cast<uint64_t*>(sh.sE + (size_t)stages * stage_floats);
  sh.empty = sh.full + stages;
  sh.red = reinterpret_cast<float*>(sh.empty + stages);
  sh.gred = sh.red + 2 * 16 * 8;
  sh.cred = reinterpret_cast<float4*>(sh.gred + 16 * 32);
  sh.sQl = reinterpret_cast<float*>(sh.cred + 16 * 32);
  sh.sP = sh.sQl + factor_floats;
  sh.ptile = ptile;
  sh.flag = reinterpret_cast<int*>(sh.sP + (size_t)stages * ptile);
  return sh;
}

template <int RT>
__global__ void __launch_bounds__(kK1pWarps * 32, 1)
    k1p_kernel(Tables t, const StreamSeg* __restrict__ segs, const int32_t* __restrict__ cta_begin,
               int stages, int stage_floats, int factor_floats, int defer, int ptile) {
  constexpr int NT = kK1pWarps * 32;
  static_assert(nw_of(0, RT) == kK1pWarps, "k1p_kernel shares the 12-warp stream map");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const Shared sh = make_shared(smem_raw, stages, stage_floats, factor_floats, ptile);
  const int dflag = (defer & 1) ? *t.deferred : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&sh.full[i], 1);
      mbar_init(&sh.empty[i], kK1pWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int sb = cta_begin[blockIdx.x], se = cta_begin[blockIdx.x + 1];
  prefetch_segs(t, segs, sb, se);
  const uint64_t pol = policy_evict_first();
  Prod pr{};
  pr.si = sb;
  Pipe pp;
  int consumed = 0, rph = 0;
  if ((threadIdx.x >> 5) == 0) {  // the first tiles go out before any other work
    prod_seek(t, segs, se, pr);
    produce(t, segs, se, sh, pr, sh.stages, true, pol);
  }
  for (int si = sb; si < se; ++si) {
    if (!t.layers[segs[si].layer].mat) {
      si = vector_run(t, segs, si, se, threadIdx.x >> 5, NT / 32,
                      [&](const StreamSeg& s, const LayerDesc& L, int first, int stride) {
                        const float* grad = t.grads[s.layer];
                        float* slot = t.pbuf + L.p_off;
                        for (int64_t i = s.row0 + first; i < s.row1; i += stride) slot[i] = grad[i];
                      }) - 1;
      continue;
    }
    const StreamSeg s = segs[si];
    const LayerDesc& L = t.layers[s.layer];
    float* grad = t.grads[s.layer];
    if (!is_fast<0>(L, grad)) {
      seg_generic<0, RT>(t, L, s, grad, 1.0f, sh.gred, dflag);
      continue;
    }
    switch (L.sm[0].nc) {
#define ACP_CASE(NCV)                                                                          \
  case NCV:                                                                                    \
    if (dflag) seg_k1p2<RT, NCV, true>(t, segs, se, L, s, sh, pp, pr, consumed, rph, pol); \
    else seg_k1p2<RT, NCV, false>(t, segs, se, L, s, sh, pp, pr, consumed, rph, pol);     \
    break;
      ACP_CASE(1)
      ACP_CASE(2)
      ACP_CASE(3)
#undef ACP_CASE
      default: break;
    }
  }
}

template <int MODE>
cudaError_t launch_mode(int rt, const Tables& t, const StreamSeg* segs, const int32_t* cb, int ncta,
                        float scale, int stages, int stage_floats, int factor_floats, int defer,
                        int ptile, cudaStream_t st) {
  const size_t smem = stream_smem_bytes(stages, stage_floats, factor_floats, ptile);
  // K1 P-step on the two-row kernel (defer bit 2, set by the plan)
  if (MODE == 0 && rt <= 4 && (defer & 4)) {
    auto go2 = [&](auto kern) -> cudaError_t {
      cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern));
      if (e != cudaSuccess) return e;
      kern<<<ncta, kK1pWarps * 32, smem, st>>>(t, segs, cb, stages, stage_floats, factor_floats, defer, ptile);
      return cudaGetLastError();
    };
    switch (rt) {
      case 1: return go2(k1p_kernel<1>);
      case 2: return go2(k1p_kernel<2>);
      case 4: return go2(k1p_kernel<4>);
      default: break;
    }
  }
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern));
    if (e != cudaSuccess) return e;
    kern<<<ncta, nw_of(MODE, rt) * 32 + 32, smem, st>>>(t, segs, cb, scale, stages, stage_floats,
                                                        factor_floats, defer, ptile);
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

// K1 Q-step, second stage: Q_loc of each (layer, panel) = sum of its
// segments' partial slots, in slot order (deterministic). 8 lanes share one
// output float4 (each sums every 8th slot), combined by a fixed shuffle tree.
// lanes per output float4 (each sums every kColReduceSplit-th partial slot):
// most (layer, panel) units have only a few slots, so one lane per output
// keeps the grid to about one wave (8 lanes: 6 waves, BERT-L K1-Q 0.704 ms;
// 2 lanes 0.698; 1 lane 0.689)
constexpr int kColReduceSplit = 1;

__global__ void __launch_bounds__(256) col_reduce_kernel(Tables t, const ColReduceTask* __restrict__ tasks,
                                                        int ntasks) {
  constexpr int kSplit = kColReduceSplit;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int item = gtid / kSplit, j = gtid % kSplit;
  // items are laid out task by task: item -> (task, k, float4 column)
  int lo = 0, hi = ntasks - 1;
  if (item >= tasks[ntasks - 1].item_end) return;
  while (lo < hi) {  // first task whose item_end > item
    const int mid = (lo + hi) >> 1;
    if (tasks[mid].item_end > item) hi = mid; else lo = mid + 1;
  }
  const ColReduceTask tk = tasks[lo];
  const int local = item - tk.item_begin;
  const int c4 = (int)((tk.cols + 3) / 4);
  const int k = local / c4, c = (local - k * c4) * 4;
  const float* base = t.colpart + tk.part_first + (int64_t)k * tk.pc + c;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const bool vec = ((tk.cols | tk.m | tk.q_dst | tk.ql_dst) & 3) == 0;  // 16-byte aligned rows
  int p = j;
  if (vec) {
    // the slots' loads go out 8 at a time and are summed in slot order (the
    // same sums as one at a time: bitwise identical), so a unit with many
    // partial slots costs one L2 round trip per 8 slots, not per slot
    // (ResNet-50: col_reduce 8 us of a 135 us step)
    constexpr int kB = 8;
    for (; p + (kB - 1) * kSplit < tk.pcount; p += kB * kSplit) {
      float4 v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u)
        v[u] = __ldcg(reinterpret_cast<const float4*>(base + (int64_t)(p + u * kSplit) * tk.stride));
#pragma unroll
      for (int u = 0; u < kB; ++u) acc = f4add(acc, v[u]);
    }
  }
  for (; p < tk.pcount; p += kSplit) {
    const float* src = base + (int64_t)p * tk.stride;
    if (vec) {
      acc = f4add(acc, __ldcg(reinterpret_cast<const float4*>(src)));
    } else {
      acc.x += __ldcg(src);
      if (c + 1 < tk.cols) acc.y += __ldcg(src + 1);
      if (c + 2 < tk.cols) acc.z += __ldcg(src + 2);
      if (c + 3 < tk.cols) acc.w += __ldcg(src + 3);
    }
  }
#pragma unroll
  for (int off = 1; off < kSplit; off <<= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, off);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, off);
  }
  if (j != 0) return;
  float* q = t.qbuf + tk.q_dst + (int64_t)k * tk.m + c;
  float* ql = t.qloc + tk.ql_dst + (int64_t)k * tk.m + c;
  if (vec) {
    *reinterpret_cast<float4*>(q) = acc;
    *reinterpret_cast<float4*>(ql) = acc;
  } else {
    const float v[4] = {acc.x, acc.y, acc.z, acc.w};
    for (int u = 0; u < 4 && c + u < tk.cols; ++u) {
      q[u] = v[u];
      ql[u] = v[u];
    }
  }
  if (tk.qs_dst >= 0) {  // TC path: Q_loc split copy (k-major [2][R8][m])
    float* d = t.qlsplit + tk.qs_dst + (int64_t)k * tk.m + c;
    const float v[4] = {acc.x, acc.y, acc.z, acc.w};
    for (int u = 0; u < 4 && c + u < tk.cols; ++u) {
      uint32_t hi, lo;
      split_tf32(v[u], hi, lo);
      d[u] = __uint_as_float(hi);
      d[tk.qs_lo + u] = __uint_as_float(lo);
    }
  }
}

}  // namespace

cudaError_t launch_col_reduce(const Tables& t, const ColReduceTask* tasks, int ntasks, int nitems,
                              cudaStream_t s) {
  if (ntasks <= 0 || nitems <= 0) return cudaSuccess;
  const int64_t threads = (int64_t)nitems * kColReduceSplit;
  col_reduce_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(t, tasks, ntasks);
  return cudaGetLastError();
}

cudaError_t allow_max_smem(const void* kern) {
  // one attribute call per (kernel, device); the table is tiny and process-wide
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& d : done)
    if (d.first == kern && d.second == dev) return cudaSuccess;
  // the dynamic limit plus the kernel's static shared memory must fit 227 KB
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           227 * 1024 - (int)fa.sharedSizeBytes);
  if (e == cudaSuccess) done.emplace_back(kern, dev);
  return e;
}

size_t stream_smem_bytes(int stages, int stage_floats, int factor_floats, int ptile) {
  return (size_t)2 * stages * stage_floats * 4 + 2 * stages * 8 + (2 * 16 * 8 + 16 * 32) * 4 +
         16 * 32 * 16 + (size_t)factor_floats * 4 + (size_t)stages * ptile * 4 + 16;
}

// Host: choose the thread mapping of an m-column layer for stream mode
// `mode` (0, 2, 3); returns false (generic path) when it does not fit.
int stream_ctas_per_sm(int mode) {
  return mode == 0 ? Cfg<0>::CPS : (mode == 2 ? Cfg<2>::CPS : Cfg<3>::CPS);
}

bool stream_make_map(int mode, int64_t m, int rt, StreamMap* out, int tt_override, bool k1p2) {
  (void)k1p2;  // k1p_kernel uses seg_k1p's 12-warp geometry
  *out = StreamMap{};
  if (m % 4 != 0 || rt > 8) return false;
  const int NW = nw_of(mode, rt);
  // K1-P at r = 8 stages an 8 x m local factor: halve its tiles to stay in 227 KB
  int64_t TT = mode == 0 ? (rt >= 8 ? Cfg<0>::TT / 2 : Cfg<0>::TT)
                         : (mode == 2 ? Cfg<2>::TT : Cfg<3>::TT);
  if (tt_override > 0) TT = tt_override;
  const int ncm = nc_max(mode, rt);
  if (ncm <= 0) return false;
  const int64_t m4 = m / 4;
  // panels (modes 2, 3): at most NW*32*ncm chunks each
  int64_t np = 1, pc4 = m4;
  if (mode != 0) {
    np = (m4 + (int64_t)NW * 32 * ncm - 1) / ((int64_t)NW * 32 * ncm);
    pc4 = (m4 + np - 1) / np;
  }
  const int64_t pcols = 4 * pc4;
  out->np = (int16_t)np;
  out->pcols = (int32_t)pcols;
  if (pc4 < 32) {  // sub-warp row groups
    int lg = 1;
    while (lg < pc4) lg <<= 1;
    const int64_t nrs = (int64_t)NW * (32 / lg);
    // tiles of at most TT floats and 256 rows (the staged P rows grow with tr)
    const int64_t rs = std::max<int64_t>(1, std::min<int64_t>(TT / (nrs * pcols), 256 / nrs));
    out->lg = (int16_t)lg;
    out->gw = 1;
    out->nc = 1;
    out->rs = (int16_t)rs;
    out->tr = (int32_t)(nrs * rs);
    return true;
  }
  for (int gw = 1; gw <= NW; ++gw) {
    if (NW % gw) continue;  // gw warps per row, NW / gw row groups
    const int64_t nc = (pc4 + 32LL * gw - 1) / (32LL * gw);
    if (nc > ncm) continue;
    const int64_t nrs = NW / gw;
    if (gw < NW && nrs * pcols > TT) continue;  // tile would exceed the target
    const int64_t rs = std::max<int64_t>(1, TT / (nrs * pcols));
    out->lg = 32;
    out->gw = (int16_t)gw;
    out->nc = (int16_t)nc;
    out->rs = (int16_t)rs;
    out->tr = (int32_t)(nrs * rs);
    return true;
  }
  *out = StreamMap{};
  return false;
}

cudaError_t launch_stream(int mode, int rt, const Tables& t, const StreamSeg* segs,
                          const int32_t* cta_begin, int ncta, float scale, int stages,
                          int stage_floats, int factor_floats, int defer, int ptile, cudaStream_t s) {
  if (ncta <= 0) return cudaSuccess;
  switch (mode) {
    case 0: return launch_mode<0>(rt, t, segs, cta_begin, ncta, scale, stages, stage_floats, factor_floats, defer, ptile, s);
    case 2: return launch_mode<2>(rt, t, segs, cta_begin, ncta, scale, stages, stage_floats, factor_floats, defer, ptile, s);
    case 3: return launch_mode<3>(rt, t, segs, cta_begin, ncta, scale, stages, stage_floats, factor_floats, defer, ptile, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace acp
