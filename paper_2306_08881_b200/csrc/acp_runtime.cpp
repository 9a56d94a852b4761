// Host runtime behind include/acp.h: plan (shape policy, ranks, fused-buffer
// layout, buckets, byte-balanced work lists), fused-buffer scheduler
// (per-bucket projection -> NCCL all-reduce on a comm stream -> decode), and
// the C ABI. See DESIGN.md for the layout and the readings it implements.
#include "acp.h"
#include "acp_internal.h"

#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace acp {
int row_rows_per_iter(int mode, int V, int rt);
}

using namespace acp;

namespace {

thread_local std::string g_err;

acp_status fail(acp_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

inline int64_t round4(int64_t x) { return (x + 3) / 4 * 4; }
inline size_t align256(size_t x) { return (x + 255) / 256 * 256; }

constexpr int kMaxRank = 32;

struct Launch {
  int kind = 0;          // 0 register row kernel, 1 register col kernel, 2 TMA stream kernel,
                         // 3 tensor-core K1 (k_tc.cu; mode 0 P-step, 1 Q-step)
  int mode = 0;          // row: 0/1/2; stream: 0/2/3
  int64_t seg_off = 0;   // first segment (row, col or stream array)
  int64_t cb_off = 0;    // first entry of cta_begin
  int ncta = 0;
  int stages = 0, stage_floats = 0, factor_floats = 0, defer = 0, ptile = 0;
  int64_t red_off = 0;   // K1 Q-step: first ColReduceTask of this launch
  int nred = 0, nitems = 0;
  double bytes = 0;      // algorithmic bytes moved by this launch
};

struct Unit {
  int layer;
  int panel;             // col kernel panel (-1 otherwise)
  int64_t count;         // rows (matrix) or elements (vector)
  double cost;           // bytes per row / element
  int64_t align;         // preferred split granularity
};

struct Plan {
  int T = 0, RT = 1, nsm = 148, nmat = 0;
  bool ef = true;
  bool defer = false;   // deferred Q-step residual (stream kernels)
  bool psgd = false;    // ACP_POWERSGD: the Power-SGD baseline (NEXT-1)
  bool tc = false;      // tensor-core K1 + double-deferred residual
  bool k1p2 = false;    // SIMT K1-P' on the two-row kernel (k_stream.cu k1p_kernel); ACP_K1P_OLD=1: seg_k1p
  bool bucketed = false;  // multi-rank scheduler (world_size > 1 or ACP_BUCKETED)
  bool tc5 = false;       // TC path decodes on tcgen05 / TMEM (k_tc5.cu); ACP_NO_TC5=1: mma.sync
  int R8 = 0;           // TC path: rank padded to a multiple of 8
  int64_t qs_elems = 0, ps_elems = 0;  // TC path: split-factor array sizes (floats)
  std::vector<TcSeg> tcsegs;
  std::vector<LayerDesc> L;
  int64_t N = 0, e_elems = 0, arena[2] = {0, 0}, ql_elems = 0, wmat_elems = 0;
  std::vector<std::vector<int>> buckets[2];
  std::vector<int64_t> boff[2], bcnt[2];
  std::vector<int> bucket_of[2];
  std::vector<int64_t> payload[2];
  std::vector<RowSeg> rowsegs;
  std::vector<ColSeg> colsegs;
  std::vector<StreamSeg> streamsegs;
  std::vector<ColReduceTask> redtasks;
  std::vector<OrthSeg> orthsegs[2];
  std::vector<int32_t> ctab;
  Launch k1_all[2], k3_all[2];
  // tcgen05 K1 P-step (k_tc5k1.cu): items of the TMA-able layers (+ vectors),
  // and a mma.sync launch for the matrices with m % 4 != 0; used when every
  // such layer's gradient is 16-byte aligned (acp_ctx::tc5k1_ok), else k1_all
  bool tc5k1 = false;
  Launch k1_t5, k1_t5rest;
  // SIMT K1-P' split by layer width (ACP_K1P_SPLIT): the wide layers' staged
  // local factor no longer sets the ring depth of the narrow ones
  Launch k1_wide;
  Launch k3_fused[2];  // decodes planned as one resident wave (NVLS-fused prologue)
  // world_size > 1: compute groups = runs of consecutive buckets whose
  // projection / decode run as one launch; each bucket is still its own
  // all-reduce (the paper's fusion rule), issued as an NCCL group per compute
  // group as soon as the group's projection has finished.
  std::vector<Launch> k1_g[2], k3_g[2];
  std::vector<Launch> k1_b[2];  // WFBP API: one projection launch per bucket
  std::vector<std::pair<int, int>> groups[2];  // [first bucket, last bucket]
  double orth_bytes[2] = {0, 0};
  int orth_seg[2] = {kOrthRowsPerSeg, kOrthRowsPerSeg};  // K2 rows per work item, per side
  int64_t colpart_elems = 0, colcnt_n = 1, gram_elems = 1;
  // workspace byte offsets
  size_t off_E = 0, off_P = 0, off_Q = 0, off_QL = 0, off_colpart = 0, off_colcnt = 0,
         off_gram = 0, off_wmat = 0, off_orthcnt = 0, off_degmask = 0, off_layers = 0,
         off_orthflag = 0, off_orthwork = 0,
         off_grads = 0, off_rowsegs = 0, off_colsegs = 0, off_streamsegs = 0, off_orth[2] = {0, 0},
         off_ctab = 0, off_step = 0, off_red = 0, off_defer = 0,
         off_qsplit = 0, off_qlsplit = 0, off_psplit = 0, off_plsplit = 0, off_tcsegs = 0,
         off_tmaps = 0, off_nvargs = 0, off_fsync = 0, off_nvepoch = 0, off_nonfinite = 0, off_tc5sched = 0,
         total = 0;
};

// Split `units` into `grid` contiguous, cost-balanced CTA ranges of segments.
// Fixed cost of one segment (factor loads into registers / shared memory,
// the ring's first tile), in byte equivalents, per launch kind: without it
// CTAs that get many small layers (ResNet) finish last. Measured on 1x B200
// (profiles/r01_v8_balance.md): 96 KB for the SIMT kernels, 160 KB for the
// tensor-core K1, 0 for the tensor-core decodes. For the SIMT stream and row
// kernels the cost grows to 1% of a CTA's share (at most 256 KB) on big
// models: round 2, two-row K1-P', sweep of the fixed cost -- BERT-L r=4 best
// at 256 KB (0.947 vs 0.959 ms at 96), ResNet-50 / 152 best at 96 (0.136 /
// 0.258 vs 0.141 / 0.273 at 256); 1% of the share is ~270 KB for BERT-L and
// ~20 KB for ResNet-50. ACP_SEG_COST_KB overrides (fixed, every kind).
enum SegKind { kSegStream = 0, kSegRow = 1, kSegCol = 2, kSegTcK1 = 3, kSegTcDec = 4 };
double seg_cost_bytes(SegKind k) {
  if (const char* e = std::getenv("ACP_SEG_COST_KB")) return std::atof(e) * 1024.0;
  static const double kb[5] = {96, 96, 96, 160, 0};
  return kb[k] * 1024.0;
}
bool seg_cost_adapts(SegKind k) {
  return !std::getenv("ACP_SEG_COST_KB") && (k == kSegStream || k == kSegRow);
}

template <class Emit>
int split_units(const std::vector<Unit>& units, int nsm, double min_share, int max_grid,
                std::vector<int32_t>& ctab, double seg_cost, Emit emit, bool adapt = false) {
  double total = 0;
  for (const Unit& u : units) total += u.cost * (double)u.count + seg_cost;
  if (total <= 0) {
    ctab.push_back(0);
    return 0;
  }
  int grid = (int)std::ceil(total / min_share);
  grid = std::max(1, std::min(grid, max_grid));
  // whole waves: a multiple of the SM count (max_grid is one), so every SM
  // gets the same number of equal shares
  if (grid > nsm && nsm > 0) grid = std::min(max_grid, (grid + nsm - 1) / nsm * nsm);
  if (adapt) {
    const double sc = std::min(256.0 * 1024.0, total / grid / 100.0);
    if (sc > seg_cost) {
      total += (sc - seg_cost) * (double)units.size();
      seg_cost = sc;
    }
  }
  const double share = (total + seg_cost * grid) / grid;  // + one split segment per CTA
  const size_t cb0 = ctab.size();
  int nseg = 0;
  ctab.push_back(0);
  int cta = 0;
  double done = 0;
  for (const Unit& u : units) {
    int64_t pos = 0;
    while (pos < u.count) {
      const double budget = share * (cta + 1) - done - seg_cost;
      int64_t take = (int64_t)std::ceil(std::max(0.0, budget) / u.cost);
      take = (take + u.align - 1) / u.align * u.align;
      // segment boundaries stay on multiples of align (TC tiles must not
      // straddle two segments): never less than one aligned chunk
      if (take < u.align) take = u.align;
      take = std::min(take, u.count - pos);
      emit(u, pos, pos + take);
      ++nseg;
      done += u.cost * (double)take + seg_cost;
      pos += take;
      if (done >= share * (cta + 1) - 1e-6 * share && cta < grid - 1) {
        ++cta;
        ctab.push_back(nseg);
      }
    }
  }
  while ((int)(ctab.size() - cb0) < grid + 1) ctab.push_back(nseg);
  return grid;
}

// plan_only: host-only plan (acp_plan_create): no CUDA calls, 148 SMs assumed.
acp_status build_plan(const acp_config* cfg, Plan& P, bool plan_only = false) {
  if (!cfg) return fail(ACP_E_INVAL, "config is NULL");
  if (cfg->abi_version != ACP_ABI_VERSION) return fail(ACP_E_INVAL, "abi_version mismatch");
  if (cfg->num_tensors < 1) return fail(ACP_E_INVAL, "num_tensors must be >= 1");
  if (!cfg->rows || !cfg->cols) return fail(ACP_E_INVAL, "rows/cols are NULL");
  if (cfg->rank < 1) return fail(ACP_E_INVAL, "rank must be >= 1");
  if (cfg->rank > kMaxRank) return fail(ACP_E_INVAL, "rank > 32 is not supported");
  if (cfg->world_size < 1) return fail(ACP_E_INVAL, "world_size must be >= 1");
  int nsm = 148;
  if (!plan_only) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev)
      return fail(ACP_E_INVAL, "invalid CUDA device");
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cfg->device) != cudaSuccess)
      return fail(ACP_E_CUDA, "cannot query SM count");
  }
  P.nsm = nsm;
  P.bucketed = cfg->world_size > 1 || (cfg->flags & ACP_BUCKETED) != 0;
  P.T = cfg->num_tensors;
  P.ef = !(cfg->flags & ACP_NO_EF);
  P.psgd = (cfg->flags & ACP_POWERSGD) != 0;
  if (P.psgd && (cfg->flags & (ACP_NO_EF | ACP_NO_REUSE)))
    return fail(ACP_E_INVAL, "ACP_POWERSGD cannot be combined with ACP_NO_EF / ACP_NO_REUSE");
  P.L.assign(P.T, LayerDesc{});
  int rmax = 1;
  for (int i = 0; i < P.T; ++i) {
    LayerDesc& L = P.L[i];
    const int64_t n = cfg->rows[i], m = cfg->cols[i];
    if (n < 1 || m < 0) return fail(ACP_E_INVAL, "tensor " + std::to_string(i) + ": bad shape");
    L.n = n;
    L.m = m;
    L.mat = m > 0 ? 1 : 0;
    L.r = L.mat ? (int)std::min<int64_t>(cfg->rank, std::min(n, m)) : 0;
    L.deg_idx = i;
    rmax = std::max(rmax, L.r);
    P.N += L.mat ? n * m : n;
    if (L.mat) ++P.nmat;
  }
  while (P.RT < rmax) P.RT <<= 1;
  // tensor-core K1 with the double-deferred residual for r >= 8 (the SIMT
  // stream kernels are faster at r <= 4); ACP_TC=1 / ACP_NO_TC=1 override
  const char* tc_env = std::getenv("ACP_TC");
  P.tc = P.ef && !P.psgd && P.RT <= 32 && !std::getenv("ACP_NO_TC") &&
         (P.RT >= 8 || (tc_env && std::atoi(tc_env) != 0));
  P.R8 = P.tc ? std::max(8, (P.RT + 7) / 8 * 8) : 0;
  {
    const char* e = std::getenv("ACP_K1P_OLD");
    P.k1p2 = P.ef && !P.psgd && P.RT <= 4 && !(e && std::atoi(e) != 0);
  }
  P.tc5 = P.tc && !std::getenv("ACP_NO_TC5");
  // tcgen05 K1 P-step: faster than the mma.sync kernel at r = 32 (BERT-L
  // proj_p 1.22 -> 1.09 ms), slower at r = 16 (0.93 -> 0.99) and r = 8
  // (BERT-Base 0.28 -> 0.31): default at R8 = 32; ACP_TC5K1=1 / 0 forces it
  const char* k1env = std::getenv("ACP_TC5K1");
  P.tc5k1 = P.tc5 && !std::getenv("ACP_NO_TC5K1") && (k1env ? std::atoi(k1env) != 0 : P.R8 >= 32);
  int tc_q_stage = 0;
  // offsets
  int64_t e = 0, ql = 0, w = 0, so[2] = {0, 0}, qs = 0, ps = 0;
  for (int p = 0; p < 2; ++p) P.payload[p].resize(P.T);
  for (int i = 0; i < P.T; ++i) {
    LayerDesc& L = P.L[i];
    P.payload[0][i] = L.mat ? L.n * L.r : L.n;
    P.payload[1][i] = L.mat ? L.m * L.r : L.n;
    L.p_off = so[0];
    L.q_off = so[1];
    so[0] += round4(P.payload[0][i]);
    so[1] += round4(P.payload[1][i]);
    if (L.mat) {
      L.e_off = e;
      e += round4(L.n * L.m);
      L.ql_off = ql;
      ql += round4(L.m * L.r);
      L.w_off = w;
      w += 2LL * L.r * L.r;
      // row kernel thread-group shape
      L.G = 0;
      L.V = 0;
      if (L.m % 4 == 0 && L.m / 4 <= (int64_t)kThreads * kMaxV) {
        const int64_t m4 = L.m / 4;
        double best = 1e30;
        for (int G = kThreads; G >= 1; G >>= 1) {
          const int64_t V = (m4 + G - 1) / G;
          if (V > kMaxV) continue;
          const double score = (double)(G * V - m4) / (double)(G * V) + 0.02 * std::abs((double)V - 4.0);
          if (score < best) {
            best = score;
            L.G = G;
            L.V = (int)V;
          }
        }
      }
      L.qs_off = -1;
      L.ps_off = -1;
      if (P.tc) {
        L.qs_off = qs;
        qs += round4(2LL * P.R8 * L.m);
        L.ps_off = ps;
        ps += round4(2LL * P.R8 * L.n);
        tc_q_stage = std::max(tc_q_stage, tc_q_map(L.m, P.R8, &L.tq));
      }
      L.W = (L.m % 4 == 0 && P.RT <= 8) ? 4 : ((L.m % 2 == 0 && P.RT <= 16) ? 2 : 1);
      L.pw = kThreads * L.W;
      // TMA stream kernels: thread mapping per mode (tr == 0: generic path)
      if (P.ef) {
        // A/B knobs (measured, off by default): half-size K1-P' tiles for the
        // wide layers (ACP_K1P_WIDE_TT), splitting K1-P' by width
        // (ACP_K1P_SPLIT) and a larger ring budget (ACP_STREAM_BUDGET_KB)
        // give the narrow layers 3 ring stages, but the step is not faster
        // (BERT-L r=4 1.031-1.044 vs 1.027 ms): K1-P' is issue/latency-bound,
        // not ring-depth-bound (scripts/micro/read_pattern.cu streams this
        // traffic at 100% of the copy peak with 3 x 64 KB stages)
        static const int wide_m = std::getenv("ACP_K1P_WIDE") ? std::atoi(std::getenv("ACP_K1P_WIDE")) : 4096;
        static const int wide_tt = std::getenv("ACP_K1P_WIDE_TT") ? std::atoi(std::getenv("ACP_K1P_WIDE_TT")) : 0;
        stream_make_map(0, L.m, P.RT, &L.sm[0], (wide_m > 0 && L.m >= wide_m && P.RT <= 4) ? wide_tt : 0,
                        P.k1p2);
        // K1-P stages the layer's local Q (RT x m) next to two ring stages
        const StreamMap& m0 = L.sm[0];
        if (m0.tr > 0 && 4 * ((int64_t)P.RT * L.m + 4LL * m0.tr * m0.pcols + 2LL * m0.tr * P.RT) +
                                 24 * 1024 > 227 * 1024)
          L.sm[0] = StreamMap{};  // generic path
        stream_make_map(2, L.m, P.RT, &L.sm[1]);
        stream_make_map(3, L.m, P.RT, &L.sm[2]);
      }
    } else {
      L.e_off = -1;
      L.ql_off = -1;
      L.w_off = -1;
      L.qs_off = -1;
      L.ps_off = -1;
    }
  }
  P.qs_elems = qs;
  P.ps_elems = ps;
  P.e_elems = e;
  P.ql_elems = ql;
  P.wmat_elems = std::max<int64_t>(w, 1);
  P.arena[0] = so[0];
  P.arena[1] = so[1];
  // buckets per parity (greedy, seal when >= cap)
  for (int p = 0; p < 2; ++p) {
    int64_t F = 0;
    for (int i = 0; i < P.T; ++i) F += P.payload[p][i];
    const double rate = (double)F / (double)P.N;
    int64_t cap = cfg->default_bucket_bytes;
    if (cap > 0) cap = std::max<int64_t>(1024, (int64_t)std::ceil((double)cap * rate));
    P.bucket_of[p].assign(P.T, 0);
    std::vector<int> cur;
    int64_t tot = 0;
    for (int i = 0; i < P.T; ++i) {
      cur.push_back(i);
      tot += 4 * P.payload[p][i];
      if (cap >= 0 && tot >= cap) {
        P.buckets[p].push_back(cur);
        cur.clear();
        tot = 0;
      }
    }
    if (!cur.empty()) P.buckets[p].push_back(cur);
    for (size_t b = 0; b < P.buckets[p].size(); ++b) {
      const int first = P.buckets[p][b].front(), last = P.buckets[p][b].back();
      const int64_t off = p == 0 ? P.L[first].p_off : P.L[first].q_off;
      const int64_t end = (p == 0 ? P.L[last].p_off : P.L[last].q_off) + round4(P.payload[p][last]);
      P.boff[p].push_back(off);
      P.bcnt[p].push_back(end - off);
      for (int i : P.buckets[p][b]) P.bucket_of[p][i] = (int)b;
    }
  }

  // ---- work lists ----
  const int max_grid = nsm * 8;
  const double min_share = 256.0 * 1024;
  const bool ef = P.ef;
  auto row_launch = [&](int mode, const std::vector<int>& tensors, bool one_wave = false) {
    std::vector<Unit> units;
    double bytes = 0;
    for (int i : tensors) {
      const LayerDesc& L = P.L[i];
      if (!L.mat) {
        units.push_back({i, -1, L.n, 8.0, 1024});
        bytes += 8.0 * L.n;
        continue;
      }
      const double bpe = mode == 0 ? (ef ? (P.psgd ? 8.0 : 12.0) : 4.0)
                                   : ((mode == 1 || mode == 3) ? 4.0 : (ef ? 16.0 : 8.0));
      int64_t align = 1;
      if (L.G > 0) align = (int64_t)(kThreads / L.G) * row_rows_per_iter(mode, L.V, P.RT);
      // balance by expected time, not bytes: the generic path is several
      // times slower per byte (it set the tail of ResNet-50's conv1)
      units.push_back({i, -1, L.n, bpe * (double)L.m * (L.G > 0 ? 1.0 : 6.0), align});
      // algorithmic bytes: M/E stream + factor traffic (each factor touched once)
      bytes += bpe * (double)L.n * (double)L.m;
      if (mode == 0) bytes += 4.0 * L.r * (double)(L.m + L.n);
      if (mode == 1 || mode == 3) bytes += 4.0 * L.r * (double)(L.m + L.n);
      if (mode == 2) bytes += 4.0 * L.r * (double)(2 * L.m + L.n);
    }
    Launch ln;
    ln.kind = 0;
    ln.mode = mode;
    ln.seg_off = (int64_t)P.rowsegs.size();
    ln.cb_off = (int64_t)P.ctab.size();
    // fused NVLS decodes: one resident wave, so the prologue can barrier the grid
    const int grid_cap = (one_wave && (mode == 1 || mode == 2 || mode == 3))
                             ? std::min(max_grid, nsm * std::max(1, row_kernel_ctas_per_sm(mode, P.RT)))
                             : max_grid;
    ln.ncta = split_units(units, nsm, min_share, grid_cap, P.ctab, seg_cost_bytes(kSegRow), [&](const Unit& u, int64_t a, int64_t b) {
      RowSeg s{};
      s.layer = u.layer;
      s.row0 = a;
      s.row1 = b;
      P.rowsegs.push_back(s);
    }, seg_cost_adapts(kSegRow));
    // cta_begin entries are relative to the launch's first segment
    ln.bytes = bytes;
    return ln;
  };
  auto col_launch = [&](const std::vector<int>& tensors) {
    std::vector<Unit> units;
    double bytes = 0;
    int counters = 0;
    for (int i : tensors) {
      const LayerDesc& L = P.L[i];
      if (!L.mat) {
        units.push_back({i, -1, L.n, 8.0, 1024});
        bytes += 8.0 * L.n;
        continue;
      }
      const int64_t npan = (L.m + L.pw - 1) / L.pw;
      for (int64_t pn = 0; pn < npan; ++pn) {
        const int64_t pcols = std::min<int64_t>(L.pw, L.m - pn * L.pw);
        units.push_back({i, (int)pn, L.n, (ef ? 8.0 : 4.0) * (double)pcols, 16});
      }
      bytes += (ef ? 8.0 : 4.0) * (double)L.n * (double)L.m + 4.0 * L.r * (double)(L.n + 2 * L.m);
    }
    Launch ln;
    ln.kind = 1;
    ln.seg_off = (int64_t)P.colsegs.size();
    ln.cb_off = (int64_t)P.ctab.size();
    int64_t part = 0;
    int prev_layer = -1, prev_panel = -1;
    size_t panel_first = 0;
    auto close_panel = [&]() {
      if (prev_layer < 0) return;
      const int cnt = (int)(P.colsegs.size() - panel_first);
      for (size_t k = panel_first; k < P.colsegs.size(); ++k) P.colsegs[k].pcount = cnt;
    };
    ln.ncta = split_units(units, nsm, min_share, max_grid, P.ctab, seg_cost_bytes(kSegCol), [&](const Unit& u, int64_t a, int64_t b) {
      ColSeg s{};
      s.layer = u.layer;
      s.panel = u.panel;
      s.row0 = a;
      s.row1 = b;
      if (u.panel >= 0) {
        if (u.layer != prev_layer || u.panel != prev_panel) {
          close_panel();
          prev_layer = u.layer;
          prev_panel = u.panel;
          panel_first = P.colsegs.size();
          ++counters;
        }
        s.counter = counters - 1;
        s.pidx = (int)(P.colsegs.size() - panel_first);
        s.part_off = part;
        part += (int64_t)P.L[u.layer].r * P.L[u.layer].pw;
      } else {
        close_panel();
        prev_layer = -1;
        prev_panel = -1;
        s.counter = -1;
      }
      P.colsegs.push_back(s);
    });
    close_panel();
    P.colpart_elems = std::max(P.colpart_elems, part);
    P.colcnt_n = std::max<int64_t>(P.colcnt_n, counters);
    ln.bytes = bytes;
    return ln;
  };
  // TMA stream launch (mode 0: K1 P-step, 2: K3 Q-step, 3: K1 Q-step).
  // stream_waves > 1 over-decomposes the grid so the hardware CTA scheduler
  // balances layers whose per-byte cost differs (dynamic load balance).
  int stream_waves = 1;
  if (const char* env = std::getenv("ACP_STREAM_WAVES")) stream_waves = std::max(1, std::atoi(env));
  bool smem_overflow = false;
  auto stream_launch = [&](int mode, const std::vector<int>& tensors) {
    const int mi = mode == 0 ? 0 : (mode == 2 ? 1 : 2);
    std::vector<Unit> units;
    double bytes = 0;
    int64_t stage_floats = 32, factor_floats = 0, max_tr = 0;
    for (int i : tensors) {
      const LayerDesc& L = P.L[i];
      if (!L.mat) {
        units.push_back({i, -1, L.n, 8.0, 1024});
        bytes += 8.0 * L.n;
        continue;
      }
      const double bpe = mode == 0 ? (P.psgd ? 8.0 : 12.0)
                                   : (mode == 2 ? 16.0 : (P.defer ? 12.0 : 8.0));
      const StreamMap& mp = L.sm[mi];
      const bool fast = mp.tr > 0;
      const int64_t tr = fast ? mp.tr : 1;
      const int64_t pc = fast ? mp.pcols : L.m;
      const int np = fast ? mp.np : 1;
      if (fast) stage_floats = std::max<int64_t>(stage_floats, tr * pc);
      if (fast) max_tr = std::max<int64_t>(max_tr, tr);
      if (fast && mode == 0 && P.defer)  // staged Q_loc [RT][m]
        factor_floats = std::max<int64_t>(factor_floats, (int64_t)P.RT * L.m);
      for (int pn = 0; pn < np; ++pn) {
        const int64_t cols = std::min<int64_t>(pc, L.m - (int64_t)pn * pc);
        // time-weighted cost (generic path ~8x, sub-warp rows ~2x per byte)
        static const double w_sub = std::getenv("ACP_W_SUBWARP") ? std::atof(std::getenv("ACP_W_SUBWARP")) : 2.0;
        static const double w_gen = std::getenv("ACP_W_GENERIC") ? std::atof(std::getenv("ACP_W_GENERIC")) : 8.0;
        const double mult = fast ? (mp.lg < 32 ? w_sub : 1.0) : w_gen;
        units.push_back({i, pn, L.n, bpe * (double)cols * mult, tr});
      }
      bytes += bpe * (double)L.n * (double)L.m;
      if (mode == 0) bytes += 4.0 * L.r * (double)(L.m + L.n);
      if (mode == 2) bytes += 4.0 * L.r * (double)(2 * L.m + L.n);
      if (mode == 3) bytes += 4.0 * L.r * (double)(L.n + 2 * L.m);
    }
    Launch ln;
    ln.kind = 2;
    ln.mode = mode;
    ln.seg_off = (int64_t)P.streamsegs.size();
    ln.cb_off = (int64_t)P.ctab.size();
    stage_floats = (stage_floats + 31) / 32 * 32;
    const int cps = stream_ctas_per_sm(mode);
    // P rows per stage (modes 2, 3 always; mode 0 when deferred): [tr][RT]
    const bool need_p = mode != 0 || (P.defer && !P.k1p2);  // k1p_kernel reads P_o from the slot
    // row stride RT in sP; the kernel derives it as ptile / tr per layer, so
    // size per-layer slots as tr_layer * RT and reserve max_tr * RT per stage
    ln.ptile = need_p ? (int)(max_tr * P.RT) : 0;
    static const int budget_kb = std::getenv("ACP_STREAM_BUDGET_KB") ? std::atoi(std::getenv("ACP_STREAM_BUDGET_KB")) : 200;
    const int64_t budget = (cps == 1 ? budget_kb : 96) * 1024 - 4 * factor_floats;
    int stages = (int)std::min<int64_t>(8, budget / (2 * 4 * stage_floats + 4 * ln.ptile));
    ln.stages = std::max(2, stages);
    ln.stage_floats = (int)stage_floats;
    ln.factor_floats = (int)factor_floats;
    if (stream_smem_bytes(ln.stages, ln.stage_floats, ln.factor_floats, ln.ptile) > 227 * 1024)
      smem_overflow = true;
    ln.defer = (P.defer && (mode == 0 || mode == 3)) ? 1 : 0;
    if (P.psgd && mode == 0) ln.defer = 2;  // projection only (no residual write)
    if (P.k1p2 && mode == 0) ln.defer |= 4;  // two-row kernel (its own stream map)
    int64_t part = 0;
    int prev_layer = -1, prev_panel = -1;
    ln.red_off = (int64_t)P.redtasks.size();
    ln.ncta = split_units(units, nsm, min_share, nsm * cps * stream_waves, P.ctab, seg_cost_bytes(kSegStream), [&](const Unit& u, int64_t a, int64_t b) {
      StreamSeg s{};
      s.layer = u.layer;
      s.row0 = a;
      s.row1 = b;
      s.panel = u.panel < 0 ? 0 : u.panel;
      const LayerDesc& L = P.L[u.layer];
      if (mode == 3 && L.mat) {
        const StreamMap& mp = L.sm[2];
        const int64_t pc = mp.tr > 0 ? mp.pcols : L.m;
        const int64_t stride = round4((int64_t)L.r * pc);
        if (u.layer != prev_layer || u.panel != prev_panel) {
          // new (layer, panel) output unit: its partial slots are contiguous
          prev_layer = u.layer;
          prev_panel = u.panel;
          ColReduceTask tk{};
          const int64_t c0 = (int64_t)s.panel * pc;
          tk.part_first = part;
          tk.stride = stride;
          tk.pc = pc;
          tk.cols = std::min<int64_t>(pc, L.m - c0);
          tk.m = L.m;
          tk.q_dst = L.q_off + c0;
          tk.ql_dst = L.ql_off + c0;
          tk.qs_dst = -1;
          tk.pcount = 0;
          tk.item_begin = ln.nitems;
          ln.nitems += (int)(L.r * ((tk.cols + 3) / 4));
          tk.item_end = ln.nitems;
          P.redtasks.push_back(tk);
          ++ln.nred;
        }
        s.nslot = 1;
        s.part_off = part;
        s.pidx = P.redtasks.back().pcount++;
        part += stride;
      }
      P.streamsegs.push_back(s);
    }, seg_cost_adapts(kSegStream));
    if (mode == 3) P.colpart_elems = std::max(P.colpart_elems, part);
    ln.bytes = bytes;
    return ln;
  };
  const bool use_stream = P.ef && P.RT <= 8;
  // the deferred Q-step residual needs the stream kernels' layouts; the
  // environment switch keeps the 24-B/element Q-step for comparison
  P.defer = use_stream && !P.psgd && !P.tc && !std::getenv("ACP_NO_DEFER");
  // Power-SGD: the SIMT stream kernels at r <= 8, the register row / column
  // kernels above (projection-only row kernel, column kernel, row decode
  // with the residual): 32 B / element either way
  if (P.psgd && !P.ef) return fail(ACP_E_INVAL, "ACP_POWERSGD needs error feedback");
  // tensor-core K1 launch (mode 0 P-step, 1 Q-step) over `tensors`
  auto tc_launch = [&](int mode, const std::vector<int>& tensors) {
    if (mode >= 2 && P.tc5) {
      // tcgen05 decode (k_tc5.cu): a flat list of work items fetched
      // dynamically by one persistent CTA per SM -- 128-row blocks of every
      // matrix, largest layers (most tiles per block) first, then chunks of
      // the 1-D tensors
      Launch ln;
      ln.kind = 3;
      ln.mode = mode;
      ln.seg_off = (int64_t)P.tcsegs.size();
      std::vector<int> order(tensors);
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        const LayerDesc &A = P.L[a], &B = P.L[b];
        if (A.mat != B.mat) return A.mat > B.mat;
        return A.m > B.m;
      });
      for (int i : order) {
        const LayerDesc& L = P.L[i];
        const int64_t step = L.mat ? 128 : 32768;
        for (int64_t r0 = 0; r0 < L.n; r0 += step) {
          TcSeg sg{};
          sg.layer = i;
          sg.row0 = r0;
          sg.row1 = std::min<int64_t>(L.n, r0 + step);
          P.tcsegs.push_back(sg);
        }
        ln.bytes += L.mat ? 4.0 * (double)L.n * (double)L.m + 4.0 * L.r * (double)(L.n + L.m) : 8.0 * L.n;
      }
      ln.nitems = (int)((int64_t)P.tcsegs.size() - ln.seg_off);
      ln.ncta = std::min(nsm, std::max(1, ln.nitems));
      if (tc5_smem_bytes(P.R8) > 227 * 1024) smem_overflow = true;
      return ln;
    }
    std::vector<Unit> units;
    double bytes = 0;
    for (int i : tensors) {
      const LayerDesc& L = P.L[i];
      if (!L.mat) {
        units.push_back({i, -1, L.n, 8.0, 1024});
        bytes += 8.0 * L.n;
        continue;
      }
      if (mode >= 2) {  // decode: grad written (+ the two factors once)
        bytes += 4.0 * (double)L.n * (double)L.m + 4.0 * L.r * (double)(L.n + L.m);
        units.push_back({i, -1, L.n, 4.0 * (double)L.m * (L.m % 4 ? 6.0 : 1.0), 128});
        continue;
      }
      // algorithmic bytes: M, S read, S written + the factors once
      bytes += 12.0 * (double)L.n * (double)L.m + 4.0 * L.r * (2.0 * L.n + 2.0 * L.m);
      if (mode == 0) {
        units.push_back({i, -1, L.n, 12.0 * (double)L.m * (L.m % 4 ? 6.0 : 1.0), 128});
      } else {
        for (int pn = 0; pn < L.tq.np; ++pn) {
          const int64_t cols = std::min<int64_t>(L.tq.pc, L.m - (int64_t)pn * L.tq.pc);
          units.push_back({i, pn, L.n, 12.0 * (double)cols * (L.m % 4 ? 6.0 : 1.0), L.tq.tr});
        }
      }
    }
    Launch ln;
    ln.kind = 3;
    ln.mode = mode;
    ln.seg_off = (int64_t)P.tcsegs.size();
    ln.cb_off = (int64_t)P.ctab.size();
    ln.stage_floats = std::max(4, mode == 0 ? tc_p_stage_floats(P.R8)
                                            : (mode == 1 ? tc_q_stage : tc_d_stage_floats(P.R8)));
    // mma.sync decodes run two CTAs per SM (more warps to hide the MMA
    // chains); the tcgen05 decodes one persistent CTA per SM
    const int tc_cps = (mode >= 2 && !P.tc5) ? 2 : 1;
    ln.stages = (int)std::max<int64_t>(2, std::min<int64_t>(mode >= 2 ? 8 : 6,
                                                            (200 * 1024 / tc_cps) / (4LL * ln.stage_floats)));
    if (tc_smem_bytes(ln.stages, ln.stage_floats) > 227 * 1024) smem_overflow = true;
    int64_t part = 0;
    int prev_layer = -1, prev_panel = -1;
    ln.red_off = (int64_t)P.redtasks.size();
    ln.ncta = split_units(units, nsm, min_share, nsm * tc_cps, P.ctab,
                          seg_cost_bytes(mode >= 2 ? kSegTcDec : kSegTcK1), [&](const Unit& u, int64_t a, int64_t b) {
      TcSeg sg{};
      sg.layer = u.layer;
      sg.row0 = a;
      sg.row1 = b;

      sg.panel = u.panel < 0 ? 0 : u.panel;
      const LayerDesc& L = P.L[u.layer];
      if (mode == 1 && L.mat) {
        const int64_t pc = L.tq.pc;
        const int64_t stride = round4((int64_t)L.r * pc);
        if (u.layer != prev_layer || u.panel != prev_panel) {
          prev_layer = u.layer;
          prev_panel = u.panel;
          ColReduceTask tk{};
          const int64_t c0 = (int64_t)sg.panel * pc;
          tk.part_first = part;
          tk.stride = stride;
          tk.pc = pc;
          tk.cols = std::min<int64_t>(pc, L.m - c0);
          tk.m = L.m;
          tk.q_dst = L.q_off + c0;
          tk.ql_dst = L.ql_off + c0;
          tk.qs_dst = L.qs_off + c0;
          tk.qs_lo = (int64_t)P.R8 * L.m;
          tk.pcount = 0;
          tk.item_begin = ln.nitems;
          ln.nitems += (int)(L.r * ((tk.cols + 3) / 4));
          tk.item_end = ln.nitems;
          P.redtasks.push_back(tk);
          ++ln.nred;
        }
        sg.nslot = L.tq.wr;
        sg.part_off = part;
        part += (int64_t)L.tq.wr * stride;
        P.redtasks.back().pcount += L.tq.wr;
      }
      P.tcsegs.push_back(sg);
    });
    if (mode == 1) P.colpart_elems = std::max(P.colpart_elems, part);
    ln.bytes = bytes;
    return ln;
  };
  auto k1_launch = [&](int parity, const std::vector<int>& ts) {
    if (P.tc) return tc_launch(parity, ts);
    if (use_stream) return stream_launch(parity == 0 ? 0 : 3, ts);
    return parity == 0 ? row_launch(0, ts) : col_launch(ts);
  };
  auto k3_launch = [&](int parity, const std::vector<int>& ts) {
    if (P.psgd && parity == 0) return Launch{};  // Power-SGD decodes once, after Q
    if (P.tc) return tc_launch(parity == 0 ? 2 : 3, ts);  // write-only decodes
    if (parity == 1 && P.defer) return row_launch(3, ts);  // decode only
    if (parity == 1 && use_stream) return stream_launch(2, ts);
    return row_launch(parity == 0 ? 1 : 2, ts);
  };
  std::vector<int> all(P.T);
  for (int i = 0; i < P.T; ++i) all[i] = i;
  for (int p = 0; p < 2; ++p) {
    P.k1_all[p] = k1_launch(p, all);
    static const bool split = std::getenv("ACP_K1P_SPLIT") ? std::atoi(std::getenv("ACP_K1P_SPLIT")) != 0 : false;
    if (p == 0 && split && use_stream && P.defer) {
      static const int wide_m = std::getenv("ACP_K1P_WIDE") ? std::atoi(std::getenv("ACP_K1P_WIDE")) : 4096;
      std::vector<int> narrow, wide;
      for (int i : all) (P.L[i].mat && P.L[i].m >= wide_m ? wide : narrow).push_back(i);
      if (!wide.empty() && !narrow.empty()) {
        P.k1_all[0] = k1_launch(0, narrow);
        P.k1_wide = k1_launch(0, wide);
      }
    }
    if (p == 0 && P.tc5k1) {
      // tcgen05 P-step: 128-row blocks of every matrix with m % 4 == 0
      // (largest rows first), then vector chunks; the rest via mma.sync
      std::vector<int> rest, mats;
      for (int i : all)
        if (P.L[i].mat && P.L[i].m % 4 != 0) rest.push_back(i);
        else mats.push_back(i);
      std::stable_sort(mats.begin(), mats.end(), [&](int a, int b) {
        const LayerDesc &A = P.L[a], &B = P.L[b];
        if (A.mat != B.mat) return A.mat > B.mat;
        return A.m > B.m;
      });
      Launch ln;
      ln.kind = 5;
      ln.mode = 0;
      ln.seg_off = (int64_t)P.tcsegs.size();
      for (int i : mats) {
        const LayerDesc& L = P.L[i];
        const int64_t step = L.mat ? 128 : 32768;
        for (int64_t r0 = 0; r0 < L.n; r0 += step) {
          TcSeg sg{};
          sg.layer = i;
          sg.row0 = r0;
          sg.row1 = std::min<int64_t>(L.n, r0 + step);
          P.tcsegs.push_back(sg);
        }
        ln.bytes += L.mat ? 12.0 * (double)L.n * (double)L.m + 4.0 * L.r * (2.0 * L.n + 2.0 * L.m) : 8.0 * L.n;
      }
      ln.nitems = (int)((int64_t)P.tcsegs.size() - ln.seg_off);
      ln.ncta = std::min(nsm, std::max(1, ln.nitems));
      if (tc5_k1p_smem_bytes(P.R8) > 227 * 1024) smem_overflow = true;
      P.k1_t5 = ln;
      if (!rest.empty()) P.k1_t5rest = k1_launch(0, rest);
    }
    P.k3_all[p] = k3_launch(p, all);
  }
  if (cfg->world_size > 1) {  // decode variants for the NVLS-fused prologue
    for (int p = 0; p < 2; ++p) {
      if (P.tc) P.k3_fused[p] = P.k3_all[p];  // TC decodes are one wave already
      else if (P.defer || !P.ef) P.k3_fused[p] = row_launch(p == 0 ? 1 : (P.defer ? 3 : 2), all, true);
    }
  }
  if (P.bucketed) {
    // measured on 2xB200 after the load-balance work: 1 group 0.197 / 1.114 ms
    // (ResNet-50 / BERT-L r=4), 2 groups 0.200 / 1.124, 4 groups 0.265 / 1.187
    int ngroups = 1;
    if (const char* env = std::getenv("ACP_COMPUTE_GROUPS")) ngroups = std::max(1, std::atoi(env));
    for (int p = 0; p < 2; ++p) {
      // balance groups by gradient elements, cutting only at bucket boundaries
      const int nb = (int)P.buckets[p].size();
      std::vector<double> w(nb, 0.0);
      double tot = 0;
      for (int b = 0; b < nb; ++b) {
        for (int i : P.buckets[p][b]) w[b] += P.L[i].mat ? (double)P.L[i].n * P.L[i].m : (double)P.L[i].n;
        tot += w[b];
      }
      const int ng = std::min(ngroups, nb);
      double acc = 0;
      int first = 0, made = 0;
      for (int b = 0; b < nb; ++b) {
        acc += w[b];
        const bool last = b == nb - 1;
        if (last || (acc >= tot * (made + 1) / ng && made < ng - 1)) {
          P.groups[p].push_back({first, b});
          std::vector<int> ts;
          for (int bb = first; bb <= b; ++bb)
            ts.insert(ts.end(), P.buckets[p][bb].begin(), P.buckets[p][bb].end());
          P.k1_g[p].push_back(k1_launch(p, ts));
          P.k3_g[p].push_back(k3_launch(p, ts));
          first = b + 1;
          ++made;
        }
      }
    }
  }
  // per-bucket projections for the WFBP API (acp_bucket_ready)
  for (int p = 0; p < 2; ++p)
    for (const auto& bk : P.buckets[p]) P.k1_b[p].push_back(k1_launch(p, bk));
  P.colcnt_n = std::max<int64_t>(P.colcnt_n, P.T);
  if (smem_overflow) return fail(ACP_E_INVAL, "internal: stream kernel shared memory exceeds 227 KB");
  // K2 segments per side (0: Q factors, length m; 1: P factors, length n)
  // Item size: 1024 rows at rank <= 2 when every SM still gets >= one item
  // per phase (fewer queue rounds on the chain: BERT-L r = 1 K2 36.6 -> 28.1
  // us, r = 2 38.8 -> 33.0), else 256 (r = 4 was neutral on BERT-L and slower
  // on ResNet-152, 33.4 -> 42.2 us; K2). ACP_ORTH_SEG=256|1024
  // forces it at rank <= 4.
  const int nsm_plan = P.nsm;
  const char* seg_env = std::getenv("ACP_ORTH_SEG");
  for (int side = 0; side < 2; ++side) {
    int64_t items_large = 0;
    for (int i = 0; i < P.T; ++i)
      if (P.L[i].mat)
        items_large += ((side == 0 ? P.L[i].m : P.L[i].n) + kOrthRowsPerSegLarge - 1) / kOrthRowsPerSegLarge;
    bool large = P.RT <= 2 && items_large >= nsm_plan;
    if (seg_env && P.RT <= 4) large = std::atoi(seg_env) == kOrthRowsPerSegLarge;
    P.orth_seg[side] = large ? kOrthRowsPerSegLarge : kOrthRowsPerSeg;
  }
  // Small factors (r <= 8, r * len <= kOrthLocalFloats) run whole in one CTA
  // (orth_local: no cross-CTA phases); they follow the segmented layers'
  // items in the queue, largest first. ACP_ORTH_LOCAL=0 disables it.
  const char* loc_env = std::getenv("ACP_ORTH_LOCAL");  // 0: off; else the r * len threshold
  const int64_t loc_max = loc_env ? std::min<int64_t>(std::atoll(loc_env), kOrthLocalFloats) : kOrthLocalFloats;
  const bool orth_local = P.RT <= 8 && loc_max > 0;
  for (int side = 0; side < 2; ++side) {
    int64_t g = 0;
    double bytes = 0;
    const int64_t segr = P.orth_seg[side];
    std::vector<std::pair<int64_t, int>> locals;
    for (int i = 0; i < P.T; ++i) {
      const LayerDesc& L = P.L[i];
      if (!L.mat) continue;
      const int64_t len = side == 0 ? L.m : L.n;
      bytes += 4.0 * L.r * (double)len * 5.0;  // read, read+write, read+write
      if (orth_local && (int64_t)L.r * len <= loc_max) {
        locals.emplace_back(-len, i);
        continue;
      }
      const int nseg = (int)((len + segr - 1) / segr);
      for (int j = 0; j < nseg; ++j) {
        OrthSeg s{};
        s.layer = i;
        s.seg = j;
        s.row0 = (int64_t)j * segr;
        s.row1 = std::min<int64_t>(len, s.row0 + segr);
        s.gram_off = g;
        s.nseg = nseg;
        g += (int64_t)L.r * L.r;
        P.orthsegs[side].push_back(s);
      }
    }
    std::stable_sort(locals.begin(), locals.end());
    for (const auto& lc : locals) {
      OrthSeg s{};
      s.layer = lc.second;
      s.row0 = 0;
      s.row1 = -lc.first;
      s.nseg = 1;
      s.local = 1;
      P.orthsegs[side].push_back(s);
    }
    P.gram_elems = std::max<int64_t>(P.gram_elems, g);
    P.orth_bytes[side] = bytes;
  }
  // workspace layout
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align256(o + std::max<size_t>(bytes, 1));
    return at;
  };
  P.off_E = take(4 * (size_t)P.e_elems);
  P.off_P = take(4 * (size_t)P.arena[0]);
  P.off_Q = take(4 * (size_t)P.arena[1]);
  P.off_QL = take(4 * (size_t)P.ql_elems);
  P.off_colpart = take(4 * (size_t)std::max<int64_t>(P.colpart_elems, 1));
  P.off_colcnt = take(4 * (size_t)P.colcnt_n);
  P.off_gram = take(8 * (size_t)P.gram_elems);
  P.off_wmat = take(8 * (size_t)P.wmat_elems);
  P.off_orthcnt = take(4 * (size_t)P.T);
  P.off_orthflag = take(8 * (size_t)P.T);
  P.off_orthwork = take(8);
  P.off_degmask = take(4 * (size_t)P.T);
  P.off_layers = take(sizeof(LayerDesc) * P.L.size());
  P.off_grads = take(8 * (size_t)P.T);
  P.off_rowsegs = take(sizeof(RowSeg) * P.rowsegs.size());
  P.off_colsegs = take(sizeof(ColSeg) * P.colsegs.size());
  P.off_streamsegs = take(sizeof(StreamSeg) * P.streamsegs.size());
  P.off_orth[0] = take(sizeof(OrthSeg) * P.orthsegs[0].size());
  P.off_orth[1] = take(sizeof(OrthSeg) * P.orthsegs[1].size());
  P.off_ctab = take(4 * P.ctab.size());
  P.off_qsplit = take(4 * (size_t)P.qs_elems);
  P.off_qlsplit = take(4 * (size_t)P.qs_elems);
  P.off_psplit = take(4 * (size_t)P.ps_elems);
  P.off_plsplit = take(4 * (size_t)P.ps_elems);
  P.off_tcsegs = take(sizeof(TcSeg) * P.tcsegs.size());
  P.off_tmaps = take(P.tc ? sizeof(CUtensorMap) * kTmapsPerLayer * (size_t)P.T : 0);
  P.off_nvargs = take(sizeof(NvlsArgs));
  P.off_fsync = take(2 * sizeof(FusedSync));
  P.off_nvepoch = take(4 * (size_t)kNvlsMaxCtas);
  P.off_nonfinite = take(4);
  // tcgen05 kernels' dynamic item counters [next item, exited CTAs]: decode P,
  // decode Q, K1 P-step, K1 Q-step
  P.off_tc5sched = take(4 * 8);
  P.off_step = take(8);
  P.off_defer = take(8);
  P.off_red = take(sizeof(ColReduceTask) * P.redtasks.size());
  P.total = o;
  return ACP_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  double bytes;
};

}  // namespace

struct acp_ctx {
  acp_config cfg{};
  Plan P;
  char* ws = nullptr;
  Tables tab{};
  cudaStream_t comm_stream = nullptr;
  std::vector<cudaEvent_t> ev_k1, ev_ar;
  std::vector<float*> grads_cache;
  int64_t step_count = 0;
  bool e_deferred = false;  // host mirror of *tab.deferred
  int tc_state = 0;         // TC path: 0 E = S, 1 E = S - P_orth Q_loc^T, 2 E = S - P_loc Q_orth^T
  // WFBP API state: -1 idle, else the open step's parity; per-bucket flags
  int wf_parity = -1;
  std::vector<char> wf_done;
  std::vector<cudaEvent_t> wf_ev;  // per bucket: all-reduce finished (comm stream)
  // NVLS all-reduce (acp_attach_symmetric)
  bool nvls = false;
  NvlsArgs nv{};
  float* mc_base = nullptr;
  int64_t sym_q_off = 0;           // floats: Q buffer inside the symmetric region
  uint32_t* nvls_epoch = nullptr;  // device (workspace), kNvlsMaxCtas counters
  bool nvls_fusable = false;       // acp_step: all-reduce inside the decode prologue
  bool tc5k1_ok = false;           // tcgen05 K1 usable: every TMA-able layer's gradient 16-B aligned
  std::vector<CUtensorMap> tmaps;  // TC path: host copy of the per-layer TMA maps
  int64_t launches = 0;
  bool plan_only = false;  // acp_plan_create: host plan, no device state
  int next_ar = 0;         // WFBP API: next bucket whose all-reduce may be issued
  bool poisoned = false;
  bool profile = false;
  std::vector<ProfRec> prof;
  size_t prof_used = 0;
  ncclComm_t comm = nullptr;
  // CUDA graphs: one captured step per parity (kernels read the gradient
  // table and the step counter from device memory, so the graph is reusable)
  bool use_graphs = true;
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  int64_t graph_kernels[2] = {0, 0};
};

namespace {

acp_status cuda_fail(acp_ctx* c, cudaError_t e, const char* what) {
  if (c) c->poisoned = true;
  return fail(ACP_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(ctx, call, what)                          \
  do {                                               \
    cudaError_t e_ = (call);                         \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, what); \
  } while (0)

ProfRec* prof_begin(acp_ctx* c, int cls, double bytes, cudaStream_t s) {
  if (!c->profile) return nullptr;
  if (c->prof_used == c->prof.size()) {
    ProfRec r{};
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    c->prof.push_back(r);
  }
  ProfRec* r = &c->prof[c->prof_used++];
  r->cls = cls;
  r->bytes = bytes;
  cudaEventRecord(r->a, s);
  return r;
}
void prof_end(ProfRec* r, cudaStream_t s) {
  if (r) cudaEventRecord(r->b, s);
}

const RowSeg* dev_rowsegs(acp_ctx* c, const Launch& ln) {
  return reinterpret_cast<const RowSeg*>(c->ws + c->P.off_rowsegs) + ln.seg_off;
}
const ColSeg* dev_colsegs(acp_ctx* c, const Launch& ln) {
  return reinterpret_cast<const ColSeg*>(c->ws + c->P.off_colsegs) + ln.seg_off;
}
const StreamSeg* dev_streamsegs(acp_ctx* c, const Launch& ln) {
  return reinterpret_cast<const StreamSeg*>(c->ws + c->P.off_streamsegs) + ln.seg_off;
}
const TcSeg* dev_tcsegs(acp_ctx* c, const Launch& ln) {
  return reinterpret_cast<const TcSeg*>(c->ws + c->P.off_tcsegs) + ln.seg_off;
}
const int32_t* dev_ctab(acp_ctx* c, const Launch& ln) {
  return reinterpret_cast<const int32_t*>(c->ws + c->P.off_ctab) + ln.cb_off;
}

float decode_scale(acp_ctx* c) {
  return (c->cfg.flags & ACP_SUM) ? 1.0f : 1.0f / (float)c->cfg.world_size;
}

acp_status run_k1(acp_ctx* c, int parity, const Launch& ln, cudaStream_t s) {
  if (ln.ncta <= 0) return ACP_OK;
  const int ef = c->P.ef ? 1 : 0;
  ProfRec* r = prof_begin(c, parity == 0 ? ACP_K_PROJ_P : ACP_K_PROJ_Q, ln.bytes, s);
  cudaError_t e;
  if (ln.kind == 5) {
    e = launch_tc5_k1p(c->P.R8, c->tab, dev_tcsegs(c, ln), ln.nitems,
                       reinterpret_cast<int32_t*>(c->ws + c->P.off_tc5sched) + 4, ln.ncta, s);
  } else if (ln.kind == 3) {
    e = launch_tc(ln.mode, c->P.R8, c->tab, dev_tcsegs(c, ln), dev_ctab(c, ln), ln.ncta, ln.stages,
                  ln.stage_floats, 1.0f, s);
    if (e == cudaSuccess && ln.mode == 1 && ln.nred > 0) {
      e = launch_col_reduce(c->tab,
                            reinterpret_cast<const ColReduceTask*>(c->ws + c->P.off_red) + ln.red_off,
                            ln.nred, ln.nitems, s);
      ++c->launches;
    }
  } else if (ln.kind == 2) {
    e = launch_stream(ln.mode, c->P.RT, c->tab, dev_streamsegs(c, ln), dev_ctab(c, ln), ln.ncta,
                      1.0f, ln.stages, ln.stage_floats, ln.factor_floats, ln.defer, ln.ptile, s);
    if (e == cudaSuccess && ln.mode == 3 && ln.nred > 0) {
      e = launch_col_reduce(c->tab,
                            reinterpret_cast<const ColReduceTask*>(c->ws + c->P.off_red) + ln.red_off,
                            ln.nred, ln.nitems, s);
      ++c->launches;
    }
  }
  else if (parity == 0)  // Power-SGD at r > 8: projection only (ef = 3)
    e = launch_row(0, c->P.RT, c->tab, dev_rowsegs(c, ln), dev_ctab(c, ln), ln.ncta, 1.0f,
                   (ef && c->P.psgd) ? 3 : ef, s);
  else
    e = launch_col(c->P.RT, c->tab, dev_colsegs(c, ln), dev_ctab(c, ln), ln.ncta, ef, s);
  prof_end(r, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "projection kernel launch");
  ++c->launches;
  return ACP_OK;
}

// K1 over every tensor: the tcgen05 P-step when planned and usable, else k1_all
acp_status run_k1_all(acp_ctx* c, int parity, cudaStream_t s) {
  const Plan& P = c->P;
  if (parity == 0 && P.tc5k1 && c->tc5k1_ok) {
    acp_status st = run_k1(c, 0, P.k1_t5rest, s);
    if (st != ACP_OK) return st;
    return run_k1(c, 0, P.k1_t5, s);
  }
  acp_status st = run_k1(c, parity, P.k1_all[parity], s);
  if (st == ACP_OK && parity == 0 && P.k1_wide.ncta > 0) st = run_k1(c, 0, P.k1_wide, s);
  return st;
}

acp_status run_k3(acp_ctx* c, int parity, const Launch& ln, cudaStream_t s, bool fused = false) {
  if (ln.ncta <= 0) return ACP_OK;
  const int ef = c->P.ef ? 1 : 0;
  Tables tt = c->tab;
  tt.nvls_fused = fused ? 1 : 0;  // this decode first sums its buffer over the ranks (NVLS)
  ProfRec* r = prof_begin(c, parity == 0 ? ACP_K_DECODE_P : ACP_K_DECODE_Q, ln.bytes, s);
  cudaError_t e =
      (ln.kind == 3 && c->P.tc5)
          ? launch_tc5_decode(ln.mode, c->P.R8, tt, dev_tcsegs(c, ln), ln.nitems,
                              reinterpret_cast<int32_t*>(c->ws + c->P.off_tc5sched) + 2 * (ln.mode - 2), ln.ncta,
                              decode_scale(c), s)
      : ln.kind == 3
          ? launch_tc(ln.mode, c->P.R8, tt, dev_tcsegs(c, ln), dev_ctab(c, ln), ln.ncta, ln.stages,
                      ln.stage_floats, decode_scale(c), s)
      : ln.kind == 2
          ? launch_stream(ln.mode, c->P.RT, tt, dev_streamsegs(c, ln), dev_ctab(c, ln), ln.ncta,
                          decode_scale(c), ln.stages, ln.stage_floats, ln.factor_floats, ln.defer,
                          ln.ptile, s)
          : launch_row(ln.mode, c->P.RT, tt, dev_rowsegs(c, ln), dev_ctab(c, ln),
                       ln.ncta, decode_scale(c), ef, s);
  prof_end(r, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "decode kernel launch");
  ++c->launches;
  return ACP_OK;
}

acp_status run_orth(acp_ctx* c, int parity, cudaStream_t s) {
  const int side = parity == 0 ? 0 : 1;  // P-step orthogonalises Q, Q-step P
  int nl = 0;
  if (c->cfg.flags & ACP_NO_REUSE) {
    cudaError_t e = launch_fill(c->tab, c->P.L.data(), c->P.T, side, c->cfg.seed, 3, -1, s, &nl);
    if (e != cudaSuccess) return cuda_fail(c, e, "fill kernel launch");
  }
  const auto& segs = c->P.orthsegs[side];
  ProfRec* r = prof_begin(c, ACP_K_ORTH, c->P.orth_bytes[side], s);
  int busy = 0;
  for (const OrthSeg& sg : segs) busy += sg.local ? 1 : 3;
  cudaError_t e = launch_orth(c->P.RT, c->P.orth_seg[side], c->tab, side,
                              reinterpret_cast<const OrthSeg*>(c->ws + c->P.off_orth[side]),
                              (int)segs.size(), c->cfg.seed, -1, s, &nl, busy);
  prof_end(r, s);
  c->launches += nl;
  if (e != cudaSuccess) return cuda_fail(c, e, "orthogonalisation kernel launch");
  return ACP_OK;
}

acp_status set_grads(acp_ctx* c, float* const* grads, cudaStream_t s) {
  if (!grads) return fail(ACP_E_INVAL, "grads is NULL");
  bool same = true;
  for (int i = 0; i < c->P.T; ++i) {
    if (!grads[i]) return fail(ACP_E_INVAL, "grads[" + std::to_string(i) + "] is NULL");
    if (grads[i] != c->grads_cache[i]) same = false;
  }
  if (same) return ACP_OK;
  for (int i = 0; i < c->P.T; ++i) c->grads_cache[i] = grads[i];
  // pageable source: staged before return, so the cache can change afterwards
  CK(c, cudaMemcpyAsync(c->ws + c->P.off_grads, c->grads_cache.data(), 8 * (size_t)c->P.T,
                        cudaMemcpyHostToDevice, s), "gradient table upload");
  if (c->P.tc) {
    // TC P-step: TMA maps of the gradients (M) next to the fixed ones (S, factors)
    const Plan& P = c->P;
    c->tmaps.resize(kTmapsPerLayer * (size_t)P.T);
    for (int i = 0; i < P.T; ++i) {
      const LayerDesc& L = P.L[i];
      CUtensorMap* mp = c->tmaps.data() + kTmapsPerLayer * (size_t)i;
      if (!L.mat) {
        std::memset(mp, 0, kTmapsPerLayer * sizeof(CUtensorMap));
        continue;
      }
      const int br = tc_p_box_rows();
      tc_encode_map(mp + 0, c->grads_cache[i], L.m, L.n, br);
      tc_encode_map(mp + 1, c->tab.E + L.e_off, L.m, L.n, br);
      tc_encode_map(mp + 2, c->tab.qsplit + L.qs_off, L.m, P.R8, P.R8);
      tc_encode_map(mp + 3, c->tab.qsplit + L.qs_off + (int64_t)P.R8 * L.m, L.m, P.R8, P.R8);
      tc_encode_map(mp + 4, c->tab.qlsplit + L.qs_off, L.m, P.R8, P.R8);
      tc_encode_map(mp + 5, c->tab.qlsplit + L.qs_off + (int64_t)P.R8 * L.m, L.m, P.R8, P.R8);
      tc_encode_map(mp + 6, c->grads_cache[i], L.m, L.n, L.tq.tr);
      tc_encode_map(mp + 7, c->tab.E + L.e_off, L.m, L.n, L.tq.tr);
      tc_encode_map(mp + 8, c->tab.qbuf + L.q_off, L.m, L.r, P.R8);
      tc_encode_map(mp + 10, c->tab.qsplit + L.qs_off, L.m, P.R8, P.R8, true);
      tc_encode_map(mp + 11, c->tab.qsplit + L.qs_off + (int64_t)P.R8 * L.m, L.m, P.R8, P.R8, true);
      tc_encode_map(mp + 12, c->tab.qbuf + L.q_off, L.m, L.r, P.R8, true);
      tc_encode_map(mp + 13, c->tab.qlsplit + L.qs_off, L.m, P.R8, P.R8, true);
      tc_encode_map(mp + 14, c->tab.qlsplit + L.qs_off + (int64_t)P.R8 * L.m, L.m, P.R8, P.R8, true);
      tc_encode_map(mp + 15, c->tab.psplit + L.ps_off, P.R8, L.n, 128, false, P.R8);
      tc_encode_map(mp + 16, c->tab.psplit + L.ps_off + (int64_t)P.R8 * L.n, P.R8, L.n, 128, false, P.R8);
    }
    CK(c, cudaMemcpyAsync(c->ws + P.off_tmaps, c->tmaps.data(), sizeof(CUtensorMap) * c->tmaps.size(),
                          cudaMemcpyHostToDevice, s), "tensor map upload");
    // the tcgen05 K1 streams M through TMA: usable only with 16-byte-aligned
    // gradients; a change of that decision invalidates the captured graphs
    bool ok = P.tc5k1;
    for (int i = 0; ok && i < P.T; ++i)
      if (P.L[i].mat && P.L[i].m % 4 == 0 && (reinterpret_cast<uintptr_t>(c->grads_cache[i]) & 15u) != 0) ok = false;
    if (ok != c->tc5k1_ok) {
      c->tc5k1_ok = ok;
      for (auto& ge : c->gexec)
        if (ge) {
          cudaGraphExecDestroy(ge);
          ge = nullptr;
        }
    }
  }
  return ACP_OK;
}

acp_status check_ctx(acp_ctx* c) {
  if (!c) return fail(ACP_E_INVAL, "ctx is NULL");
  if (c->plan_only) return fail(ACP_E_STATE, "plan-only context (acp_plan_create): no device state");
  if (c->poisoned) return fail(ACP_E_STATE, "context poisoned by an earlier failure");
  return ACP_OK;
}

// an NCCL failure on another rank (or a transport error) surfaces
// asynchronously; poll it before enqueueing more collectives on the comm.
acp_status poll_nccl(acp_ctx* c) {
  if (!c->comm) return ACP_OK;
  ncclResult_t ar = ncclSuccess;
  const ncclResult_t r = ncclCommGetAsyncError(c->comm, &ar);
  if (r != ncclSuccess) ar = r;
  if (ar != ncclSuccess && ar != ncclInProgress) {
    c->poisoned = true;
    return fail(ACP_E_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar));
  }
  return ACP_OK;
}

}  // namespace

extern "C" {

int32_t acp_abi_version(void) { return ACP_ABI_VERSION; }

const char* acp_last_error(void) { return g_err.c_str(); }

acp_status acp_workspace_bytes(const acp_config* cfg, size_t* out) {
  if (!out) return fail(ACP_E_INVAL, "out is NULL");
  Plan P;
  acp_status st = build_plan(cfg, P);
  if (st != ACP_OK) return st;
  *out = P.total;
  return ACP_OK;
}

acp_status acp_create(const acp_config* cfg, acp_ctx** out) {
  if (!out) return fail(ACP_E_INVAL, "out is NULL");
  *out = nullptr;
  acp_ctx* c = new acp_ctx();
  acp_status st = build_plan(cfg, c->P);
  if (st != ACP_OK) {
    delete c;
    return st;
  }
  if (!cfg->workspace) {
    delete c;
    return fail(ACP_E_INVAL, "workspace is NULL");
  }
  if (cfg->workspace_bytes < c->P.total) {
    delete c;
    return fail(ACP_E_NOMEM, "workspace too small: need " + std::to_string(c->P.total) + " bytes");
  }
  if (cfg->world_size > 1 && !cfg->nccl_comm) {
    // allowed: split API only; acp_step will reject
  }
  c->cfg = *cfg;
  c->cfg.rows = nullptr;
  c->cfg.cols = nullptr;
  c->cfg.q0_host = nullptr;
  c->comm = reinterpret_cast<ncclComm_t>(cfg->nccl_comm);
  c->ws = reinterpret_cast<char*>(cfg->workspace);
  c->grads_cache.assign(c->P.T, nullptr);
  Plan& P = c->P;
  Tables& t = c->tab;
  t.layers = reinterpret_cast<const LayerDesc*>(c->ws + P.off_layers);
  t.grads = reinterpret_cast<float* const*>(c->ws + P.off_grads);
  t.E = reinterpret_cast<float*>(c->ws + P.off_E);
  t.pbuf = reinterpret_cast<float*>(c->ws + P.off_P);
  t.qbuf = reinterpret_cast<float*>(c->ws + P.off_Q);
  t.qloc = reinterpret_cast<float*>(c->ws + P.off_QL);
  t.colpart = reinterpret_cast<float*>(c->ws + P.off_colpart);
  t.colcnt = reinterpret_cast<int32_t*>(c->ws + P.off_colcnt);
  t.gram = reinterpret_cast<double*>(c->ws + P.off_gram);
  t.wmat = reinterpret_cast<double*>(c->ws + P.off_wmat);
  t.orthcnt = reinterpret_cast<int32_t*>(c->ws + P.off_orthcnt);
  t.orthflag = reinterpret_cast<long long*>(c->ws + P.off_orthflag);
  t.orthwork = reinterpret_cast<int32_t*>(c->ws + P.off_orthwork);
  t.degmask = reinterpret_cast<uint32_t*>(c->ws + P.off_degmask);
  t.step = reinterpret_cast<int64_t*>(c->ws + P.off_step);
  t.deferred = reinterpret_cast<int32_t*>(c->ws + P.off_defer);
  t.qsplit = reinterpret_cast<float*>(c->ws + P.off_qsplit);
  t.qlsplit = reinterpret_cast<float*>(c->ws + P.off_qlsplit);
  t.psplit = reinterpret_cast<float*>(c->ws + P.off_psplit);
  t.plsplit = reinterpret_cast<float*>(c->ws + P.off_plsplit);
  t.r8 = P.R8;
  t.tmaps = reinterpret_cast<const CUtensorMap*>(c->ws + P.off_tmaps);
  t.nv = reinterpret_cast<const NvlsArgs*>(c->ws + P.off_nvargs);
  t.fsync = reinterpret_cast<FusedSync*>(c->ws + P.off_fsync);
  t.nvls_fused = 0;
  t.nonfinite = reinterpret_cast<int32_t*>(c->ws + P.off_nonfinite);
  t.stream_pf = std::getenv("ACP_STREAM_PF") ? std::atoi(std::getenv("ACP_STREAM_PF")) : 0;
  // L2 prefetch ahead of the shared-memory rings: measured slower everywhere
  // (BERT-L r=4 / r=8 / r=32, ResNet-50), off by default; A/B switches
  t.tc5_pf = std::getenv("ACP_TC5_PF") ? std::atoi(std::getenv("ACP_TC5_PF")) : 0;
  c->nvls_epoch = reinterpret_cast<uint32_t*>(c->ws + P.off_nvepoch);

  DeviceGuard dg(cfg->device);
  cudaStream_t s = nullptr;
  auto bail = [&](cudaError_t e, const char* what) {
    if (s) cudaStreamDestroy(s);
    delete c;
    return fail(ACP_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  };
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e != cudaSuccess) return bail(e, "stream create");
  if ((e = cudaMemsetAsync(c->ws, 0, P.total, s)) != cudaSuccess) return bail(e, "workspace memset");
  auto up = [&](size_t off, const void* src, size_t bytes) {
    return bytes ? cudaMemcpyAsync(c->ws + off, src, bytes, cudaMemcpyHostToDevice, s) : cudaSuccess;
  };
  if ((e = up(P.off_layers, P.L.data(), sizeof(LayerDesc) * P.L.size())) != cudaSuccess ||
      (e = up(P.off_rowsegs, P.rowsegs.data(), sizeof(RowSeg) * P.rowsegs.size())) != cudaSuccess ||
      (e = up(P.off_colsegs, P.colsegs.data(), sizeof(ColSeg) * P.colsegs.size())) != cudaSuccess ||
      (e = up(P.off_streamsegs, P.streamsegs.data(), sizeof(StreamSeg) * P.streamsegs.size())) != cudaSuccess ||
      (e = up(P.off_tcsegs, P.tcsegs.data(), sizeof(TcSeg) * P.tcsegs.size())) != cudaSuccess ||
      (e = up(P.off_orth[0], P.orthsegs[0].data(), sizeof(OrthSeg) * P.orthsegs[0].size())) != cudaSuccess ||
      (e = up(P.off_orth[1], P.orthsegs[1].data(), sizeof(OrthSeg) * P.orthsegs[1].size())) != cudaSuccess ||
      (e = up(P.off_ctab, P.ctab.data(), 4 * P.ctab.size())) != cudaSuccess ||
      (e = up(P.off_red, P.redtasks.data(), sizeof(ColReduceTask) * P.redtasks.size())) != cudaSuccess)
    return bail(e, "plan upload");
  // Q_0: caller-provided (row-major m x r per matrix) or generated
  std::vector<float> q0;
  if (cfg->q0_host) {
    q0.assign(P.arena[1], 0.f);
    int64_t src = 0;
    for (int i = 0; i < P.T; ++i) {
      const LayerDesc& L = P.L[i];
      if (!L.mat) continue;
      for (int64_t j = 0; j < L.m; ++j)
        for (int k = 0; k < L.r; ++k) q0[L.q_off + (int64_t)k * L.m + j] = cfg->q0_host[src + j * L.r + k];
      src += L.m * L.r;
    }
    if ((e = up(P.off_Q, q0.data(), 4 * q0.size())) != cudaSuccess) return bail(e, "Q0 upload");
  } else {
    int nl = 0;
    if ((e = launch_fill(t, P.L.data(), P.T, 2, cfg->seed, 1, 0, s, &nl)) != cudaSuccess)
      return bail(e, "Q0 generator");
  }
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return bail(e, "create sync");
  cudaStreamDestroy(s);
  s = nullptr;
  if (P.bucketed) {
    if ((e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking)) != cudaSuccess)
      return bail(e, "comm stream");
    const size_t nb = std::max(P.groups[0].size(), P.groups[1].size());
    c->ev_k1.resize(nb);
    c->ev_ar.resize(nb);
    for (size_t b = 0; b < nb; ++b) {
      cudaEventCreateWithFlags(&c->ev_k1[b], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&c->ev_ar[b], cudaEventDisableTiming);
    }
  }
  *out = c;
  g_err.clear();
  return ACP_OK;
}

acp_status acp_plan_create(const acp_config* cfg, acp_ctx** out) {
  if (!out) return fail(ACP_E_INVAL, "out is NULL");
  *out = nullptr;
  acp_ctx* c = new acp_ctx();
  acp_status st = build_plan(cfg, c->P, /*plan_only=*/true);
  if (st != ACP_OK) {
    delete c;
    return st;
  }
  c->cfg = *cfg;
  c->cfg.rows = nullptr;
  c->cfg.cols = nullptr;
  c->cfg.q0_host = nullptr;
  c->cfg.workspace = nullptr;
  c->cfg.nccl_comm = nullptr;
  c->plan_only = true;
  *out = c;
  g_err.clear();
  return ACP_OK;
}

}  // extern "C"

namespace {

// Deferred Q-step residual -> materialised E for every matrix (repeated
// Q-steps, set_state); eager, on stream s.
acp_status materialize_all(acp_ctx* c, cudaStream_t s) {
  if (!c->e_deferred) return ACP_OK;
  for (int i = 0; i < c->P.T; ++i)
    if (c->P.L[i].mat)
      CK(c, launch_materialize(c->tab, c->P.L[i], i, nullptr, s), "materialize E");
  CK(c, cudaMemsetAsync(c->tab.deferred, 0, sizeof(int32_t), s), "clear deferred flag");
  c->e_deferred = false;
  return ACP_OK;
}

// TC path: fold the implicit residual into S (state -> 0) and zero the split
// factor the next K1's correction would pair with it (eager, irregular
// parity sequences and set_state only; the steady state never needs it).
acp_status tc_materialize_all(acp_ctx* c, cudaStream_t s) {
  if (c->tc_state == 0) return ACP_OK;
  for (int i = 0; i < c->P.T; ++i)
    if (c->P.L[i].mat)
      CK(c, launch_tc_materialize(c->tab, c->P.L[i], c->tc_state, nullptr, s), "materialize E");
  CK(c, cudaMemsetAsync(c->tab.qlsplit, 0, 4 * (size_t)c->P.qs_elems, s), "zero Q_loc split");
  CK(c, cudaMemsetAsync(c->tab.plsplit, 0, 4 * (size_t)c->P.ps_elems, s), "zero P_loc split");
  c->tc_state = 0;
  return ACP_OK;
}

// host bookkeeping before/after a K1 of `parity`
acp_status before_k1(acp_ctx* c, int32_t parity, cudaStream_t s) {
  if (c->P.tc) {  // P after P / Q after Q: the steady-state correction does not apply
    if ((parity == 0 && c->tc_state == 2) || (parity == 1 && c->tc_state == 1))
      return tc_materialize_all(c, s);
    return ACP_OK;
  }
  if (parity == 1 && c->e_deferred) return materialize_all(c, s);  // Q after Q
  return ACP_OK;
}
void after_k1(acp_ctx* c, int32_t parity) {
  c->e_deferred = c->P.defer && parity == 1;
  if (c->P.tc) c->tc_state = parity == 0 ? 2 : 1;
}

// All-reduce floats [off, off + cnt) of the parity's fused buffer on the comm
// stream: the NVLS kernel when a symmetric region is attached, else NCCL.
acp_status allreduce_range(acp_ctx* c, int parity, int64_t off, int64_t cnt) {
  float* buf = parity == 0 ? c->tab.pbuf : c->tab.qbuf;
  if (c->nvls) {
    NvlsArgs a = c->nv;
    a.mc = c->mc_base + (parity == 0 ? 0 : c->sym_q_off);
    CK(c, launch_nvls_allreduce(a, off, cnt, c->comm_stream), "NVLS all-reduce");
    ++c->launches;
    return ACP_OK;
  }
  const ncclResult_t nr = ncclAllReduce(buf + off, buf + off, (size_t)cnt, ncclFloat, ncclSum, c->comm,
                                        c->comm_stream);
  if (nr != ncclSuccess) {
    c->poisoned = true;
    return fail(ACP_E_NCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(nr));
  }
  return ACP_OK;
}

// Per compute group: projection K1 of `parity` on s, then the group's buckets
// all-reduced as one NCCL group on the comm stream (event ev_ar[g] marks it).
acp_status project_and_reduce(acp_ctx* c, int32_t parity, cudaStream_t s) {
  acp_status st;
  const Plan& P = c->P;
  float* buf = parity == 0 ? c->tab.pbuf : c->tab.qbuf;
  const size_t ng = P.groups[parity].size();
  for (size_t g = 0; g < ng; ++g) {
    if ((st = run_k1(c, parity, P.k1_g[parity][g], s)) != ACP_OK) return st;
    CK(c, cudaEventRecord(c->ev_k1[g], s), "event record");
    CK(c, cudaStreamWaitEvent(c->comm_stream, c->ev_k1[g], 0), "stream wait");
    const int b0 = P.groups[parity][g].first, b1 = P.groups[parity][g].second;
    double bytes = 0;
    for (int b = b0; b <= b1; ++b) bytes += 4.0 * P.bcnt[parity][b];
    ProfRec* r = prof_begin(c, ACP_K_ALLREDUCE, bytes, c->comm_stream);
    if (c->nvls) {
      // the group's buckets are one contiguous range of the buffer
      const int64_t off = P.boff[parity][b0];
      const int64_t end = P.boff[parity][b1] + P.bcnt[parity][b1];
      if ((st = allreduce_range(c, parity, off, end - off)) != ACP_OK) return st;
    } else {
      ncclResult_t nr = ncclGroupStart();
      for (int b = b0; b <= b1 && nr == ncclSuccess; ++b)
        nr = ncclAllReduce(buf + P.boff[parity][b], buf + P.boff[parity][b],
                           (size_t)P.bcnt[parity][b], ncclFloat, ncclSum, c->comm, c->comm_stream);
      const ncclResult_t ne = ncclGroupEnd();
      if (nr == ncclSuccess) nr = ne;
      if (nr != ncclSuccess) {
        prof_end(r, c->comm_stream);
        c->poisoned = true;
        return fail(ACP_E_NCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(nr));
      }
    }
    prof_end(r, c->comm_stream);
    CK(c, cudaEventRecord(c->ev_ar[g], c->comm_stream), "event record");
  }
  return ACP_OK;
}

// Power-SGD step (ACP_POWERSGD): P = M'Q -> AR(P) -> orth(P) ->
// Q = M'^T P -> AR(Q) -> E = M' - P Q_loc^T, decoded = P Q^T / p.
acp_status enqueue_psgd_step(acp_ctx* c, cudaStream_t s) {
  acp_status st;
  const Plan& P = c->P;
  if (!P.bucketed) {
    if ((st = run_k1(c, 0, P.k1_all[0], s)) != ACP_OK) return st;
    if ((st = run_orth(c, 1, s)) != ACP_OK) return st;
    if ((st = run_k1(c, 1, P.k1_all[1], s)) != ACP_OK) return st;
    return run_k3(c, 1, P.k3_all[1], s);
  }
  if ((st = project_and_reduce(c, 0, s)) != ACP_OK) return st;
  for (size_t g = 0; g < P.groups[0].size(); ++g)
    CK(c, cudaStreamWaitEvent(s, c->ev_ar[g], 0), "stream wait");
  if ((st = run_orth(c, 1, s)) != ACP_OK) return st;  // needs every reduced P
  if ((st = project_and_reduce(c, 1, s)) != ACP_OK) return st;
  for (size_t g = 0; g < P.groups[1].size(); ++g) {
    CK(c, cudaStreamWaitEvent(s, c->ev_ar[g], 0), "stream wait");
    if ((st = run_k3(c, 1, P.k3_g[1][g], s)) != ACP_OK) return st;
  }
  return ACP_OK;
}

// Enqueue one whole step (orthogonalise, per-bucket projection + all-reduce,
// decode) on stream s; used eagerly and for graph capture.
acp_status enqueue_step(acp_ctx* c, int32_t parity, cudaStream_t s) {
  if (c->P.psgd) return enqueue_psgd_step(c, s);
  acp_status st;
  if ((st = run_orth(c, parity, s)) != ACP_OK) return st;
  const Plan& P = c->P;
  if (!P.bucketed) {
    if ((st = run_k1_all(c, parity, s)) != ACP_OK) return st;
    if ((st = run_k3(c, parity, P.k3_all[parity], s)) != ACP_OK) return st;
    return ACP_OK;
  }
  if (c->nvls && c->nvls_fusable) {
    // NEXT-3: one projection launch, then the decode sums the buffer over the
    // ranks in the switch before decoding (no all-reduce launch, no comm stream)
    if ((st = run_k1_all(c, parity, s)) != ACP_OK) return st;
    ProfRec* r = prof_begin(c, ACP_K_ALLREDUCE, 0.0, s);  // marker only: fused into the decode
    prof_end(r, s);
    return run_k3(c, parity, P.k3_fused[parity], s, true);
  }
  if ((st = project_and_reduce(c, parity, s)) != ACP_OK) return st;
  for (size_t g = 0; g < P.groups[parity].size(); ++g) {
    CK(c, cudaStreamWaitEvent(s, c->ev_ar[g], 0), "stream wait");
    if ((st = run_k3(c, parity, P.k3_g[parity][g], s)) != ACP_OK) return st;
  }
  return ACP_OK;
}

// Sticky non-finite flag: bit 0 set by K2 (non-finite factor),
// bit 1 by the fused-buffer scan (scan = true: ACP_CHECK_FINITE after a step).
acp_status check_finite(acp_ctx* c, int parity, cudaStream_t s, bool scan = true) {
  if (scan) {
    const float* buf = parity == 0 ? c->tab.pbuf : c->tab.qbuf;
    CK(c, launch_finite_scan(buf, c->P.arena[parity], c->tab.nonfinite, s), "finite scan");
    ++c->launches;
  }
  int32_t flag = 0;
  CK(c, cudaMemcpyAsync(&flag, c->tab.nonfinite, 4, cudaMemcpyDeviceToHost, s), "flag read");
  CK(c, cudaStreamSynchronize(s), "flag sync");
  if (flag) {
    c->poisoned = true;
    return fail(ACP_E_NONFINITE, std::string("non-finite value ") +
                                     ((flag & 1) ? "in a factor reaching the orthogonaliser" : "") +
                                     ((flag & 3) == 3 ? " and " : "") +
                                     ((flag & 2) ? "in the all-reduced fused buffer" : "") + " (SPEC S:63)");
  }
  return ACP_OK;
}

acp_status capture_step(acp_ctx* c, int32_t parity) {
  if (!c->cap_stream) CK(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking), "capture stream");
  const int64_t l0 = c->launches;
  CK(c, cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal), "begin capture");
  acp_status st = enqueue_step(c, parity, c->cap_stream);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->cap_stream, &g);
  if (st != ACP_OK) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "end capture");
  e = cudaGraphInstantiate(&c->gexec[parity], g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(c, e, "graph instantiate");
  c->graph_kernels[parity] = c->launches - l0;
  c->launches = l0;
  return ACP_OK;
}

}  // namespace

extern "C" {

acp_status acp_step(acp_ctx* c, int32_t parity, float* const* grads, void* stream) {
  acp_status st = check_ctx(c);
  if (st != ACP_OK) return st;
  if (parity != 0 && parity != 1) return fail(ACP_E_INVAL, "parity must be 0 or 1");
  if (c->P.bucketed && !c->comm)
    return fail(ACP_E_INVAL, "world_size > 1 / ACP_BUCKETED needs an NCCL communicator (or use the split API)");
  if (c->wf_parity >= 0) return fail(ACP_E_INVAL, "acp_step: a bucket step is open (acp_step_begin)");
  if ((st = poll_nccl(c)) != ACP_OK) return st;
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((st = set_grads(c, grads, s)) != ACP_OK) return st;
  if (c->P.psgd) parity = 0;  // one Power-SGD step does both projections
  if ((st = before_k1(c, parity, s)) != ACP_OK) return st;
  if (c->use_graphs && !c->profile) {
    if (!c->gexec[parity] && (st = capture_step(c, parity)) != ACP_OK) return st;
    CK(c, cudaGraphLaunch(c->gexec[parity], s), "graph launch");
    c->launches += c->graph_kernels[parity];
  } else if ((st = enqueue_step(c, parity, s)) != ACP_OK) {
    return st;
  }
  after_k1(c, parity);
  ++c->step_count;
  if (c->cfg.flags & ACP_CHECK_FINITE) return check_finite(c, c->P.psgd ? 1 : parity, s);
  return ACP_OK;
}

acp_status acp_step_begin(acp_ctx* c, int32_t parity, float* const* grads, void* stream) {
  acp_status st = check_ctx(c);
  if (st != ACP_OK) return st;
  if (parity != 0 && parity != 1) return fail(ACP_E_INVAL, "parity must be 0 or 1");
  if (c->P.psgd) return fail(ACP_E_INVAL, "the bucket API runs ACP-SGD only (not ACP_POWERSGD)");
  if (c->wf_parity >= 0) return fail(ACP_E_INVAL, "acp_step_begin: a step is already open");
  if (c->P.bucketed && !c->comm)
    return fail(ACP_E_INVAL, "world_size > 1 / ACP_BUCKETED needs an NCCL communicator");
  if ((st = poll_nccl(c)) != ACP_OK) return st;
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((st = set_grads(c, grads, s)) != ACP_OK) return st;
  if ((st = before_k1(c, parity, s)) != ACP_OK) return st;
  if ((st = run_orth(c, parity, s)) != ACP_OK) return st;
  const size_t nb = c->P.buckets[parity].size();
  c->wf_done.assign(nb, 0);
  while (c->wf_ev.size() < 2 * nb) {
    cudaEvent_t ev;
    CK(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event create");
    c->wf_ev.push_back(ev);
  }
  c->wf_parity = parity;
  c->next_ar = 0;
  return ACP_OK;
}

acp_status acp_bucket_ready(acp_ctx* c, int32_t b, void* stream) {
  acp_status st = check_ctx(c);
  if (st != ACP_OK) return st;
  const int parity = c->wf_parity;
  if (parity < 0) return fail(ACP_E_INVAL, "acp_bucket_ready: no open step (acp_step_begin)");
  const Plan& P = c->P;
  if (b < 0 || b >= (int32_t)P.buckets[parity].size()) return fail(ACP_E_INVAL, "bucket index out of range");
  if (c->wf_done[b]) return fail(ACP_E_INVAL, "bucket made ready twice");
  if ((st = poll_nccl(c)) != ACP_OK) return st;
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((st = run_k1(c, parity, P.k1_b[parity][b], s)) != ACP_OK) return st;
  c->wf_done[b] = 1;
  if (P.bucketed) {
    CK(c, cudaEventRecord(c->wf_ev[2 * b], s), "event record");
    // collectives strictly in bucket-index order (identical on every rank,
    // whatever order the hooks fired in): issue every ready prefix bucket
    const int nb = (int)P.buckets[parity].size();
    while (c->next_ar < nb && c->wf_done[c->next_ar]) {
      const int a = c->next_ar;
      CK(c, cudaStreamWaitEvent(c->comm_stream, c->wf_ev[2 * a], 0), "stream wait");
      ProfRec* r = prof_begin(c, ACP_K_ALLREDUCE, 4.0 * P.bcnt[parity][a], c->comm_stream);
      st = allreduce_range(c, parity, P.boff[parity][a], P.bcnt[parity][a]);
      prof_end(r, c->comm_stream);
      if (st != ACP_OK) return st;
      CK(c, cudaEventRecord(c->wf_ev[2 * a + 1], c->comm_stream), "event record");
      ++c->next_ar;
    }
  }
  return ACP_OK;
}

acp_status acp_step_end(acp_ctx* c, void* stream) {
  acp_status st = check_ctx(c);
  if (st != ACP_OK) return st;
  const int parity = c->wf_parity;
  if (parity < 0) return fail(ACP_E_INVAL, "acp_step_end: no open step");
  for (size_t b = 0; b < c->wf_done.size(); ++b)
    if (!c->wf_done[b]) return fail(ACP_E_INVAL, "acp_step_end: bucket " + std::to_string(b) + " not ready");
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (c->P.bucketed)
    for (size_t b = 0; b < c->wf_done.size(); ++b)
      CK(c, cudaStreamWaitEvent(s, c->wf_ev[2 * b + 1], 0), "stream wait");
  if ((st = run_k3(c, parity, c->P.k3_all[parity], s)) != ACP_OK) return st;
  after_k1(c, parity);
  ++c->step_count;
  c->wf_parity = -1;
  return ACP_OK;
}

static int64_t sym_layout(const Plan& P, int64_t* q_off, int64_t* flag_off) {
  const int64_t qo = (P.arena[0] + 63) / 64 * 64;                 // floats, 256-byte aligned
  const int64_t fo = ((qo + P.arena[1]) * 4 + 255) / 256 * 256;   // bytes
  if (q_off) *q_off = qo;
  if (flag_off) *flag_off = fo;
  return fo + (int64_t)kNvlsFlagRows * kNvlsMaxCtas * kNvlsMaxRanks * 4;
}

acp_status acp_symmetric_bytes(acp_ctx* c, int64_t* out) {
  if (!c || !out) return fail(ACP_E_INVAL, "bad arguments");
  *out = sym_layout(c->P, nullptr, nullptr);
  return ACP_OK;
}

acp_status acp_attach_symmetric(acp_ctx* c, void* local, void* multicast, void* const* peers,
                                int32_t rank, int64_t bytes) {
  acp_status st = check_ctx(c);
  if (st != ACP_OK) return st;
  const int world = c->cfg.world_size;
  if (world < 2 || world > kNvlsMaxRanks) return fail(ACP_E_INVAL, "NVLS needs 2 <= world_size <= 8");
  if (!local || !multicast || !peers || rank < 0 || rank >= world)
    return fail(ACP_E_INVAL, "bad symmetric buffer arguments");
  int64_t qo = 0, fo = 0;
  if (bytes < sym_layout(c->P, &qo, &fo)) return fail(ACP_E_INVAL, "symmetric region too small");
  if (c->wf_parity >= 0) return fail(ACP_E_INVAL, "a bucket step is open");
  DeviceGuard dg(c->cfg.device);
  char* base = reinterpret_cast<char*>(local);
  float* np = reinterpret_cast<float*>(base);
  float* nq = np + qo;
  CK(c, cudaDeviceSynchronize(), "attach sync");
  CK(c, cudaMemcpy(np, c->tab.pbuf, 4 * (size_t)c->P.arena[0], cudaMemcpyDeviceToDevice), "move P buffer");
  CK(c, cudaMemcpy(nq, c->tab.qbuf, 4 * (size_t)c->P.arena[1], cudaMemcpyDeviceToDevice), "move Q buffer");
  CK(c, cudaMemset(base + fo, 0, kNvlsFlagRows * kNvlsMaxCtas * kNvlsMaxRanks * 4), "zero flags");
  CK(c, cudaMemset(c->nvls_epoch, 0, 4 * kNvlsMaxCtas), "epoch zero");
  c->tab.pbuf = np;
  c->tab.qbuf = nq;
  c->mc_base = reinterpret_cast<float*>(multicast);
  c->sym_q_off = qo;
  c->nv = NvlsArgs{};
  c->nv.my_flags = reinterpret_cast<uint32_t*>(base + fo);
  for (int p = 0; p < world; ++p)
    c->nv.peer_flags[p] = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(peers[p]) + fo);
  c->nv.epoch = c->nvls_epoch;
  c->nv.rank = rank;
  c->nv.world = world;
  c->nv.mc_buf[0] = c->mc_base;
  c->nv.mc_buf[1] = c->mc_base + qo;
  c->nv.n_buf[0] = (c->P.arena[0] + 3) / 4 * 4;
  c->nv.n_buf[1] = (c->P.arena[1] + 3) / 4 * 4;
  CK(c, cudaMemcpy(c->ws + c->P.off_nvargs, &c->nv, sizeof(NvlsArgs), cudaMemcpyHostToDevice), "NVLS args");
  CK(c, cudaMemset(c->ws + c->P.off_fsync, 0, 2 * sizeof(FusedSync)), "fused sync");
  c->nvls = true;
  // the decode kernels (row / TC) sum the buffer in their prologue; the
  // stream K3-Q (ACP_NO_DEFER) and Power-SGD keep the separate kernel
  c->nvls_fusable = (!c->P.psgd && (c->P.tc || c->P.defer || !c->P.ef)) && !std::getenv("ACP_NVLS_UNFUSED");
  // captured graphs and TMA maps hold the old buffer addresses
  for (int p = 0; p < 2; ++p)
    if (c->gexec[p]) {
      cudaGraphExecDestroy(c->gexec[p]);
      c->gexec[p] = nullptr;
    }
  std::fill(c->grads_cache.begin(), c->grads_cache.end(), nullptr);
  return ACP_OK;
}

acp_status acp_check_finite(acp_ctx* c, void* stream) {
  acp_status st = check_ctx(c);
  if (st != ACP_OK) return st;
  DeviceGuard dg(c->cfg.device);
  return check_finite(c, 0, reinterpret_cast<cudaStream_t>(stream), /*scan=*/false);
}

acp_status acp_set_graphs(acp_ctx* c, int32_t enable) {
  if (!c) return fail(ACP_E_INVAL, "ctx is NULL");
  c->use_graphs = enable != 0;
  return ACP_OK;
}

acp_status acp_compress(acp_ctx* c, int32_t parity, float* const* grads, float** out_buffer,
                        int64_t* out_count, void* stream) {
  acp_status st = check_ctx(c);
  if (st != ACP_OK) return st;
  if (parity != 0 && parity != 1) return fail(ACP_E_INVAL, "parity must be 0 or 1");
  if (!out_buffer || !out_count) return fail(ACP_E_INVAL, "output pointers are NULL");
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((st = set_grads(c, grads, s)) != ACP_OK) return st;
  if ((st = before_k1(c, parity, s)) != ACP_OK) return st;
  // Power-SGD's first projection uses the previous Q as it is
  if (!(c->P.psgd && parity == 0) && (st = run_orth(c, parity, s)) != ACP_OK) return st;
  if ((st = run_k1_all(c, parity, s)) != ACP_OK) return st;
  after_k1(c, parity);
  *out_buffer = parity == 0 ? c->tab.pbuf : c->tab.qbuf;
  *out_count = c->P.arena[parity];
  ++c->step_count;
  return ACP_OK;
}

acp_status acp_decompress(acp_ctx* c, int32_t parity, float* const* grads, void* stream) {
  acp_status st = check_ctx(c);
  if (st != ACP_OK) return st;
  if (parity != 0 && parity != 1) return fail(ACP_E_INVAL, "parity must be 0 or 1");
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((st = set_grads(c, grads, s)) != ACP_OK) return st;
  return run_k3(c, parity, c->P.k3_all[parity], s);
}

acp_status acp_get_state(acp_ctx* c, int32_t i, float* Pm, float* Qm, float* Em, void* stream) {
  acp_status st = check_ctx(c);
  if (st != ACP_OK) return st;
  if (i < 0 || i >= c->P.T || !c->P.L[i].mat) return fail(ACP_E_INVAL, "not a matrix tensor");
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const LayerDesc& L = c->P.L[i];
  if (Pm) CK(c, launch_transpose(c->tab.pbuf + L.p_off, Pm, L.n, L.r, 0, s), "state transpose");
  if (Qm) CK(c, launch_transpose(c->tab.qbuf + L.q_off, Qm, L.m, L.r, 0, s), "state transpose");
  if (Em) {
    if (c->P.tc && c->tc_state != 0)  // E = S - A B^T, formed on the fly (state unchanged)
      CK(c, launch_tc_materialize(c->tab, L, c->tc_state, Em, s), "materialize E");
    else if (c->e_deferred)  // E = S - P Q_loc^T, formed on the fly (state unchanged)
      CK(c, launch_materialize(c->tab, L, i, Em, s), "materialize E");
    else
      CK(c, cudaMemcpyAsync(Em, c->tab.E + L.e_off, 4 * (size_t)(L.n * L.m),
                            cudaMemcpyDeviceToDevice, s), "state copy");
  }
  return ACP_OK;
}

acp_status acp_set_state(acp_ctx* c, int32_t i, const float* Pm, const float* Qm, const float* Em,
                         void* stream) {
  acp_status st = check_ctx(c);
  if (st != ACP_OK) return st;
  if (i < 0 || i >= c->P.T || !c->P.L[i].mat) return fail(ACP_E_INVAL, "not a matrix tensor");
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const LayerDesc& L = c->P.L[i];
  if ((st = materialize_all(c, s)) != ACP_OK) return st;  // other layers keep their E
  if ((st = tc_materialize_all(c, s)) != ACP_OK) return st;
  if (Pm) CK(c, launch_transpose(Pm, c->tab.pbuf + L.p_off, L.n, L.r, 1, s), "state transpose");
  if (Qm) CK(c, launch_transpose(Qm, c->tab.qbuf + L.q_off, L.m, L.r, 1, s), "state transpose");
  if (Em) CK(c, cudaMemcpyAsync(c->tab.E + L.e_off, Em, 4 * (size_t)(L.n * L.m),
                               cudaMemcpyDeviceToDevice, s), "state copy");
  return ACP_OK;
}

acp_status acp_plan_info(acp_ctx* c, int32_t i, int64_t out[6]) {
  if (!c) return fail(ACP_E_INVAL, "ctx is NULL");
  if (i < 0 || i >= c->P.T || !out) return fail(ACP_E_INVAL, "bad tensor index");
  const LayerDesc& L = c->P.L[i];
  out[0] = L.r;
  out[1] = L.p_off;
  out[2] = L.q_off;
  out[3] = L.mat ? L.e_off : -1;
  out[4] = c->P.bucket_of[0][i];
  out[5] = c->P.bucket_of[1][i];
  return ACP_OK;
}

acp_status acp_num_buckets(acp_ctx* c, int32_t parity, int32_t* out) {
  if (!c || !out || (parity != 0 && parity != 1)) return fail(ACP_E_INVAL, "bad arguments");
  *out = (int32_t)c->P.buckets[parity].size();
  return ACP_OK;
}

acp_status acp_bucket_range(acp_ctx* c, int32_t parity, int32_t b, int64_t* off, int64_t* cnt) {
  if (!c || !off || !cnt || (parity != 0 && parity != 1) || b < 0 ||
      b >= (int32_t)c->P.buckets[parity].size())
    return fail(ACP_E_INVAL, "bad arguments");
  *off = c->P.boff[parity][b];
  *cnt = c->P.bcnt[parity][b];
  return ACP_OK;
}

acp_status acp_profile_enable(acp_ctx* c, int32_t enable) {
  if (!c) return fail(ACP_E_INVAL, "ctx is NULL");
  c->profile = enable != 0;
  return ACP_OK;
}

acp_status acp_profile_reset(acp_ctx* c) {
  if (!c) return fail(ACP_E_INVAL, "ctx is NULL");
  c->prof_used = 0;
  return ACP_OK;
}

acp_status acp_profile_read(acp_ctx* c, int32_t cls, double* ms, int64_t* launches, double* bytes) {
  if (!c || !ms || !launches || !bytes || cls < 0 || cls >= ACP_K_NUM)
    return fail(ACP_E_INVAL, "bad arguments");
  DeviceGuard dg(c->cfg.device);
  double tot = 0, by = 0;
  int64_t n = 0;
  for (size_t k = 0; k < c->prof_used; ++k) {
    ProfRec& r = c->prof[k];
    if (r.cls != cls) continue;
    CK(c, cudaEventSynchronize(r.b), "profile event sync");
    float t = 0;
    CK(c, cudaEventElapsedTime(&t, r.a, r.b), "profile elapsed");
    tot += t;
    by += r.bytes;
    ++n;
  }
  *ms = tot;
  *launches = n;
  *bytes = by;
  return ACP_OK;
}

acp_status acp_launch_count(acp_ctx* c, int64_t* out) {
  if (!c || !out) return fail(ACP_E_INVAL, "bad arguments");
  *out = c->launches;
  return ACP_OK;
}

acp_status acp_destroy(acp_ctx* c) {
  if (!c) return ACP_OK;
  if (c->plan_only) {
    delete c;
    return ACP_OK;
  }
  DeviceGuard dg(c->cfg.device);
  for (auto& ge : c->gexec)
    if (ge) cudaGraphExecDestroy(ge);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->comm_stream) {
    cudaStreamSynchronize(c->comm_stream);
    cudaStreamDestroy(c->comm_stream);
  }
  for (auto ev : c->ev_k1) cudaEventDestroy(ev);
  for (auto ev : c->ev_ar) cudaEventDestroy(ev);
  for (auto ev : c->wf_ev) cudaEventDestroy(ev);
  for (auto& r : c->prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  delete c;
  return ACP_OK;
}

acp_status acp_nccl_unique_id(uint8_t out_id[128]) {
  if (!out_id) return fail(ACP_E_INVAL, "out is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(ACP_E_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out_id, &id, 128);
  return ACP_OK;
}

acp_status acp_nccl_comm_create(const uint8_t id_bytes[128], int32_t nranks, int32_t rank,
                                int32_t device, void** out) {
  if (!id_bytes || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(ACP_E_INVAL, "bad arguments");
  DeviceGuard dg(device);
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, 128);
  ncclComm_t comm = nullptr;
  ncclResult_t r = ncclCommInitRank(&comm, nranks, id, rank);
  if (r != ncclSuccess) return fail(ACP_E_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  *out = comm;
  return ACP_OK;
}

acp_status acp_nccl_comm_destroy(void* comm) {
  if (!comm) return ACP_OK;
  ncclResult_t r = ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return fail(ACP_E_NCCL, std::string("ncclCommDestroy: ") + ncclGetErrorString(r));
  return ACP_OK;
}

}  // extern "C"
