// Internal declarations shared by the host runtime (acp_runtime.cpp) and the
// sm_100a kernels. Not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace acp {

constexpr int kThreads = 256;          // every hot kernel runs 256-thread CTAs
constexpr int kMaxV = 8;               // row kernel: float4 chunks per thread per row
constexpr int kOrthRowsPerSeg = 256;   // K2 work unit (factor rows), staged at once
constexpr int kOrthLocalFloats = 18432;  // K2: factors with r * len <= this (r <= 8) run in one CTA
constexpr int kOrthRowsPerSegLarge = 1024;  // K2 unit at rank <= 2 (<= 4 forced) when a phase has
                                           // >= one item per SM (fewer queue rounds)

// Thread mapping of a matrix layer onto a TMA stream kernel CTA (NW warps):
// a row is covered by `gw` warps (lg = 32) or by `lg` lanes of one warp
// (gw = 1, 32/lg rows per warp); lane li of the row group owns float4 column
// chunks c = sub*lg*nc + li + lg*i, i < nc (sub = warp index within the row
// group). A tile holds tr = (NW/gw)*(32/lg)*rs rows (rs rows per row slot,
// processed one after another). tr == 0: the layer takes the generic path.
// Column panels (modes 2, 3 only): the row is split into np panels of pcols
// columns (the last one narrower); each panel is a separate work unit, so the
// per-thread factor registers stay bounded for wide layers.
struct StreamMap {
  int32_t tr;
  int16_t lg, gw, nc, rs;
  int32_t pcols;
  int16_t np, pad_;
};

// Tensor-core K1 Q-step mapping of one layer (k_tc.cu): column panels of pc
// columns (multiple of 16), warps = wc column groups (cbw 16-column blocks
// each) x wr row groups; tiles of tr rows; each segment writes wr partial slots.
struct TcMap {
  int32_t pc;
  int16_t np, wc, wr, tr, cbw, pad_;
};

// Per-tensor descriptor uploaded once (device copy of the plan).
struct LayerDesc {
  int64_t n, m;        // matrix n x m; vector: n = length, m = 0
  int32_t r;           // r_i (0 for vectors)
  int32_t mat;         // 1 matrix, 0 vector
  int64_t e_off;       // float offset into E (matrices)
  int64_t p_off;       // float offset of the slot in the P-buffer
  int64_t q_off;       // float offset of the slot in the Q-buffer
  int64_t ql_off;      // float offset into the local-Q copy (matrices)
  int32_t G;           // row kernel: threads per row (0 = generic path)
  int32_t V;           // row kernel: float4 chunks per thread per row
  int32_t W;           // col kernel: columns per thread (4, 2 or 1)
  int32_t pw;          // col kernel: panel width in columns (= 256 * W)
  int64_t w_off;       // K2: offset (doubles) of this layer's two r x r W matrices
  int32_t deg_idx;     // K2: index into the degenerate-mask / counter arrays
  int32_t pad_;
  StreamMap sm[3];     // stream kernels: [0] K1 P-step, [1] K3 Q-step, [2] K1 Q-step
  int64_t qs_off;      // TC path: offset of the layer's [2][R8][m] Q-side split factors
  int64_t ps_off;      // TC path: offset of the layer's [2][n][R8] P-side split factors
  TcMap tq;            // TC path: K1 Q-step mapping
};

// Tensor-core K1 work unit (k_tc.cu): rows [row0, row1) of matrix `layer`
// (column panel `panel` on Q-steps), or elements of a vector (packed).
// Q-steps: the segment writes nslot partial slots (r x pc floats, k-major,
// stride round4(r * pc)) starting at part_off.
struct TcSeg {
  int32_t layer;
  int32_t panel;
  int64_t row0, row1;
  int64_t part_off;
  int32_t nslot;
  int32_t pad_;
};

// Stream-kernel work unit: rows [row0, row1) of matrix `layer` (or elements of
// a vector). Column mode: the segment writes `nslot` partial slots (r x m
// floats each, k-major) starting at part_off; the layer's `pcount` slots are
// contiguous and slot index of this segment's first one is `pidx`. Slots are
// r x pcols floats (k-major), stride round4(r * pcols).
struct StreamSeg {
  int32_t layer;
  int32_t nslot;
  int64_t row0, row1;
  int64_t part_off;
  int32_t pidx;
  int32_t pcount;
  int32_t panel;     // column panel (modes 2, 3)
  int32_t counter;   // mode 3: completion counter of (layer, panel)
};

// Row-kernel work unit: rows [row0, row1) of matrix `layer`, or elements
// [row0, row1) of vector `layer`.
struct RowSeg {
  int32_t layer;
  int32_t pad_;
  int64_t row0, row1;
};

// Column-kernel (K1 Q-step) work unit: rows [row0, row1) of panel `panel` of
// matrix `layer`; writes its partial slot (r x pw floats at part_off); the
// panel's pcount partial slots are contiguous and the last segment of the
// panel to finish sums them in order into the Q slot (completion counter
// `counter`). Vectors: pack elements [row0, row1).
struct ColSeg {
  int32_t layer;
  int32_t panel;
  int64_t row0, row1;
  int64_t part_off;    // float offset of this segment's partial slot
  int32_t pidx;        // index of this segment's partial among its panel's
  int32_t pcount;      // number of partials of (layer, panel), contiguous
  int32_t counter;     // completion counter of (layer, panel)
  int32_t pad_;
};

// K2 (orthogonalisation) work unit: rows [row0, row1) of factor `layer`
// (the Q factor on P-steps, the P factor on Q-steps).
struct OrthSeg {
  int32_t layer;
  int32_t seg;         // index of this segment among the layer's segments
  int64_t row0, row1;
  int64_t gram_off;    // double offset of this segment's partial Gram (r x r)
  int32_t nseg;        // segments of this layer
  int32_t gram_first;  // segment index of the layer's first partial (gram_off of seg 0)
  int32_t local;       // 1: the whole factor in one CTA (orth_local), nseg = 1
  int32_t pad_;
};

// K1 Q-step second stage: one (layer, panel) output unit. Items
// [item_begin, item_end) of the flattened (k, float4 column) space.
struct ColReduceTask {
  int64_t part_first;   // float offset of the unit's first partial slot
  int64_t stride;       // slot stride (floats)
  int64_t pc;           // slot row length (panel width, floats)
  int64_t cols;         // columns of this panel
  int64_t m;            // layer width (Q slot row length)
  int64_t q_dst, ql_dst;  // float offsets of column c0 of k-row 0 in the Q-buffer / local-Q copy
  int64_t qs_dst;       // TC path: offset of column c0 in the Q_loc split array (-1: none)
  int64_t qs_lo;        // TC path: offset of the lo half (R8 * m)
  int32_t pcount;       // partial slots of the unit
  int32_t item_begin, item_end;
  int32_t pad_;
};

struct NvlsArgs;
struct FusedSync;

struct Tables {
  const LayerDesc* layers;
  float* const* grads;   // device table of gradient pointers
  float* E;
  float* pbuf;
  float* qbuf;
  float* qloc;
  float* colpart;
  int32_t* colcnt;
  double* gram;
  double* wmat;
  int32_t* orthcnt;
  long long* orthflag;   // K2: per layer, epoch of the phase that may start (step * 4 + phase)
  int32_t* orthwork;     // K2 persistent queue: [0] next item, [1] exited CTAs
  uint32_t* degmask;
  int64_t* step;         // device step counter (keys the method's random draws)
  int32_t* deferred;     // 1: E holds S = M' of the last Q-step (E = S - P Q_loc^T
                         //    is applied lazily by the next P-step), 0: E is materialised
  // tensor-core path (double-deferred residual): 3xTF32 split
  // copies (hi, lo) of the factors, ranks padded to r8 with zeros
  float* qsplit;         // Q_orth  [2][R8][m] per layer (written by K2, side 0)
  float* qlsplit;        // Q_loc   [2][R8][m] (written by the Q-step column reduce)
  float* psplit;         // P_orth  [2][n][R8] (written by K2, side 1)
  float* plsplit;        // P_loc   [2][n][R8] (written by the P-step TC kernel)
  int32_t r8;            // padded rank (multiple of 8), 0: TC path off
  const CUtensorMap* tmaps;
  // NVLS all-reduce fused into the decode prologue (acp_attach_symmetric):
  // nvls_fused != 0 -> the decode of parity p first sums buffer p over the
  // ranks in the switch (k_nvls.cuh)
  const NvlsArgs* nv;
  FusedSync* fsync;
  int32_t* nonfinite;  // sticky flag: bit 0 K2 saw a non-finite factor, bit 1 finite scan hit
  int32_t stream_pf;   // stream kernels: tiles prefetched into L2 ahead of the shared ring (0: off)
  int32_t tc5_pf;      // tcgen05 K1: M / S tiles prefetched into L2 ahead
  int32_t nvls_fused;
};
// TC path TMA maps per layer: [M, S, Q_orth hi, lo, Q_loc hi, lo] (P-step
// boxes), [M, S] (Q-step boxes of tq.tr rows), [Q slot] (R8-row boxes),
// [unused], for the tcgen05 decode's column factor (32-byte-atom swizzle)
// [Q_orth hi, lo, Q slot] (10-12), and for the tcgen05 K1 P-step [Q_loc hi,
// lo] (32-byte-atom swizzle, 13-14) and [P_orth hi, lo] (R8 x 128-row boxes,
// swizzle = R8 * 4 bytes, 15-16)
constexpr int kTmapsPerLayer = 17;

// NVLS all-reduce (k_nvls.cu): the fused buffers live in a
// symmetric region bound to a multicast object; flags for the cross-rank
// barriers sit behind the buffers in the same region.
constexpr int kNvlsMaxCtas = 64, kNvlsMaxRanks = 8;
struct NvlsArgs {
  float* mc;                              // multicast address of the buffer being reduced
  uint32_t* my_flags;                     // this rank's flag region
  uint32_t* peer_flags[kNvlsMaxRanks];    // every rank's flag region, as mapped here
  uint32_t* epoch;                        // [kNvlsMaxCtas] per-CTA launch counters (local)
  int32_t rank, world;
  float* mc_buf[2];                       // multicast address of the P / Q buffer
  int64_t n_buf[2];                       // floats of the P / Q buffer (multiple of 4)
};
// Fused all-reduce in the decode prologue: per parity, a grid arrival
// counter, a release word and the launch epoch (monotonic, graph-safe).
struct FusedSync {
  uint32_t gcount, release, epoch, pad_;
};
// flag area: rows 0-1 separate all-reduce kernel, rows 2-5 fused prologue
// (two per parity)
constexpr int kNvlsFlagRows = 6;
// sum over ranks of floats [off, off + cnt) of the buffer behind a.mc (16-byte aligned)
cudaError_t launch_nvls_allreduce(const NvlsArgs& a, int64_t off, int64_t cnt, cudaStream_t s);
// CTAs of a decode row kernel resident per SM (the fused prologue needs the
// whole grid resident)
int row_kernel_ctas_per_sm(int mode, int rt);

// launches (all on `stream`, 256 threads, grid = ncta)
// mode 0: K1 P-step (projection + residual + pack into P-buffer)
// mode 1: K3 P-step decode (+ unpack from P-buffer)
// mode 2: K3 Q-step residual + decode (+ unpack from Q-buffer)
// mode 3: K3 Q-step decode only, deferred residual (+ unpack from Q-buffer)
// (mode 1 also clears *t.deferred: the P-step's K1 has consumed it)
cudaError_t launch_row(int mode, int rt, const Tables& t, const RowSeg* segs,
                       const int32_t* cta_begin, int ncta, float scale, int ef,
                       cudaStream_t stream);
// K1 Q-step: column projection into the Q-buffer + local-Q copy (+ pack)
cudaError_t launch_col(int rt, const Tables& t, const ColSeg* segs, const int32_t* cta_begin,
                       int ncta, int ef, cudaStream_t stream);
// TMA-pipelined streaming kernels (k_stream.cu): mode 0 K1 P-step, mode 2 K3
// Q-step, mode 3 K1 Q-step. rt <= 8, error feedback on.
cudaError_t launch_col_reduce(const Tables& t, const ColReduceTask* tasks, int ntasks, int nitems,
                              cudaStream_t stream);
// Raise the dynamic shared-memory limit of a kernel once per device.
cudaError_t allow_max_smem(const void* kern);
// defer = 1 (deferred Q-step residual): mode 3 also writes
// S = M + E back into E and raises *t.deferred; mode 0 applies
// E_prev = S - P Q_loc^T on the fly when *t.deferred is set (Q_loc staged in
// factor_floats of shared memory).
cudaError_t launch_stream(int mode, int rt, const Tables& t, const StreamSeg* segs,
                          const int32_t* cta_begin, int ncta, float scale, int stages,
                          int stage_floats, int factor_floats, int defer, int ptile,
                          cudaStream_t stream);
// E (or dst) = S - P Q_loc^T for one matrix layer (deferred state -> E)
cudaError_t launch_materialize(const Tables& t, const LayerDesc& L, int layer, float* dst,
                               cudaStream_t stream);
// tt_override > 0: tile target (floats per tensor per stage) instead of the mode's default
bool stream_make_map(int mode, int64_t m, int rt, StreamMap* out, int tt_override = 0, bool k1p2 = false);
// Tensor-core K1 (k_tc.cu). mode 0: P-step (x = M + S - P_orth Q_loc^T,
// S = x, P_loc = x Q_orth -> P slot + P_loc split), mode 1: Q-step
// (x = M + S - P_loc Q_orth^T, S = x, Q partials = x^T P_orth -> colpart).
// mode 2 / 3: decode on the tensor cores, grad = scale * P Q^T (P-step: the
// all-reduced P slot with Q_orth; Q-step: P_orth with the all-reduced Q slot).
cudaError_t launch_tc(int mode, int r8, const Tables& t, const TcSeg* segs, const int32_t* cta_begin,
                      int ncta, int stages, int stage_floats, float scale, cudaStream_t stream);
int tc_d_stage_floats(int r8);
// tcgen05 decodes (k_tc5.cu): mode 2 P-step, mode 3 Q-step; one CTA per SM
// (items: 128-row blocks / vector chunks fetched dynamically through the
// counter pair `sched`, which must start at {0, 0}; the kernel re-arms it)
cudaError_t launch_tc5_decode(int mode, int r8, const Tables& t, const TcSeg* items, int nitems, int32_t* sched,
                              int ncta, float scale, cudaStream_t stream);
size_t tc5_smem_bytes(int r8);
// tcgen05 K1 P-step (k_tc5k1.cu): items = 128-row blocks of layers with
// m % 4 == 0 and 16-byte-aligned gradients, and 1-D tensor chunks
cudaError_t launch_tc5_k1p(int r8, const Tables& t, const TcSeg* items, int nitems, int32_t* sched, int ncta,
                           cudaStream_t stream);
size_t tc5_k1p_smem_bytes(int r8);
size_t tc_smem_bytes(int stages, int stage_floats);
// host: encode a 2-D TMA map (fp32 rows x cols, 32-column boxes of box_rows
// rows, SWIZZLE_128B); false (map zeroed) when the layout does not allow it
bool tc_encode_map(CUtensorMap* out, const float* base, int64_t cols, int64_t rows, int box_rows,
                   bool atom32 = false, int box_cols = 32);
int tc_p_box_rows();
int tc_p_stage_floats(int r8);
// K1 Q-step tile geometry of an m-column layer; returns stage floats
int tc_q_map(int64_t m, int r8, TcMap* out);
// TC state -> E: dst = S - A B^T (which 1: A = P_orth, B = Q_loc; 2: A = P_loc, B = Q_orth)
cudaError_t launch_tc_materialize(const Tables& t, const LayerDesc& L, int which, float* dst,
                                  cudaStream_t stream);
int stream_ctas_per_sm(int mode);
size_t stream_smem_bytes(int stages, int stage_floats, int factor_floats, int ptile);
// K2: CholeskyQR2 of the factors named by segs (side 0: Q factors in the
// Q-buffer, length m; side 1: P factors in the P-buffer, length n).
// busy_items: items that do work (whole-factor items + 3 per segment);
// the grid is capped there (the other queue entries are skips).
cudaError_t launch_orth(int rt, int seg_rows, const Tables& t, int side, const OrthSeg* segs, int nseg,
                        uint64_t seed, int64_t step, cudaStream_t stream, int* launches,
                        int busy_items = 0);
// Fill factor slots with counter-based N(0,1) (tag, step): side as above, or
// side 2 = Q_0 into the Q-buffer. Layers = all matrices. step < 0: use the
// device step counter (*t.step). The orthogonaliser reads *t.step and its
// last phase increments it, so a captured CUDA graph stays valid.
cudaError_t launch_fill(const Tables& t, const LayerDesc* host_layers, int num_tensors, int side,
                        uint64_t seed, int tag, int64_t step, cudaStream_t stream, int* launches);
// ACP_CHECK_FINITE: *flag |= 2 if any of buf[0, n) is not finite
cudaError_t launch_finite_scan(const float* buf, int64_t n, int32_t* flag, cudaStream_t stream);
// k-major slot <-> row-major rows x r (state access)
cudaError_t launch_transpose(const float* src, float* dst, int64_t rows, int r, int to_kmajor,
                             cudaStream_t stream);

}  // namespace acp
