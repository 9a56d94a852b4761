/*
 * acp.h -- C ABI of the B200-native ACP-SGD hot path.
 *
 * ACP-SGD = "alternate compressed Power-SGD" with error feedback,
 * Algorithm 2 of arXiv 2306.08881 ("Evaluation and Optimization of Gradient
 * Compression for Distributed Deep Learning").
 * "P:n" below is PAPER.md line n; "S:n" is SPEC.md line n; "C<k>" is a
 * reading listed in DESIGN.md "Readings".
 *
 * One call of acp_step() runs, for EVERY tensor of a data-parallel worker's
 * gradient set, one iteration of Alg. 2 (parity 0 = the paper's odd t,
 * parity 1 = even t; C1):
 *
 *   parity 0 (P-step)          parity 1 (Q-step)
 *   Q  <- Orthogonalize(Q_{t-1})          P  <- Orthogonalize(P_{t-1})
 *   M' <- M + E_{t-1}                     M' <- M + E_{t-1}
 *   P  <- M' Q            (local)         Q  <- M'^T P          (local)
 *   E  <- M' - P Q^T      (local P, C3)   E  <- M' - P Q^T      (local Q, C3)
 *   P  <- All-Reduce(P)   (sum, C2)       Q  <- All-Reduce(Q)   (sum, C2)
 *   grad <- P Q^T / p         grad <- P Q^T / p
 *
 * 1-D tensors (biases, norms) are not compressed; they are copied into
 * the same fused buffer as the fresh factors and all-reduced with them
 * (P:257 numbers, C8): grad <- All-Reduce(grad) / p.
 *
 * Layout (all float32, little endian):
 *   - gradient of tensor i: caller-owned, row-major n_i x m_i (n = dim0,
 *     m = prod(dims[1:]), "reshaped into matrices", C9), overwritten in
 *     place with the decoded (averaged) gradient;
 *   - fused buffers ("P-buffer" used on parity 0, "Q-buffer" on parity 1):
 *     one slot per tensor in READY order, slot i starting at a multiple of 4
 *     floats (16 B) and padded to a multiple of 4 floats; a matrix slot holds
 *     its fresh factor k-major (column k of P, n_i floats, then column k+1 ...;
 *     resp. of Q, m_i floats each), a vector slot holds the vector;
 *   - buckets (tensor fusion, C10): greedy in ready order, sealed
 *     once their payload (4 * elements, unpadded) reaches
 *     cap = max(1 KiB, ceil(default_bucket_bytes * rate_parity)),
 *     rate_P = (sum n_i r_i + N_v)/N, rate_Q = (sum m_i r_i + N_v)/N; a bucket
 *     is the contiguous float range of its slots (padding included);
 *   - E: one float region per matrix (row-major n_i x m_i) in ready order,
 *     each starting at a multiple of 4 floats.
 *   r_i = min(rank, n_i, m_i) (C7).
 *
 * Ownership: the caller owns the gradients, the workspace (device memory of at
 * least acp_workspace_bytes()), the CUDA stream and the NCCL communicator.
 * Every device buffer the library uses lives in the caller's workspace (or,
 * after acp_attach_symmetric, in the caller's symmetric region); the library
 * itself only creates CUDA streams, events and graph executables. It keeps
 * the gradient pointers of the last call (a host copy and a device table in
 * the workspace) only to skip re-uploading an unchanged table; a captured
 * step graph reads the table, so the pointers passed to a call must stay
 * valid until the work that call enqueued has finished. All device work is
 * enqueued asynchronously on the caller's stream (plus one internal stream
 * for the all-reduces when world_size > 1 or ACP_BUCKETED).
 *
 * Errors: functions return acp_status. ACP_E_INVAL means the arguments were
 * rejected with no side effects; ACP_E_CUDA / ACP_E_NCCL poison the context
 * and every later call on it returns ACP_E_STATE. An asynchronous NCCL error
 * (ncclCommGetAsyncError, polled at the entry of every acp_step /
 * acp_step_begin / acp_bucket_ready) also poisons it with ACP_E_NCCL.
 * acp_last_error() returns a thread-local description of the last non-OK
 * status. Non-finite values: gradients pass through the projections and the
 * all-reduce unchecked (as SPEC S:141 does for collectives); the
 * orthogonaliser, whose input must be finite, does not repair a
 * non-finite factor (NaN propagates to the outputs) but raises a sticky
 * device flag that acp_check_finite() reports as ACP_E_NONFINITE; with
 * ACP_CHECK_FINITE every acp_step also scans its all-reduced fused buffer
 * and checks the flag synchronously (debug mode). All ranks must issue
 * identical parity sequences.
 */
#ifndef ACP_H
#define ACP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACP_ABI_VERSION 1

typedef struct acp_ctx acp_ctx;

typedef enum {
  ACP_OK = 0,
  ACP_E_INVAL = 1,  /* invalid argument or configuration; nothing changed   */
  ACP_E_CUDA = 2,   /* a CUDA call failed; context poisoned                  */
  ACP_E_NCCL = 3,   /* an NCCL call failed; context poisoned                 */
  ACP_E_NOMEM = 4,  /* workspace smaller than acp_workspace_bytes()          */
  ACP_E_STATE = 5,  /* context poisoned by an earlier failure, or a call that
                       a plan-only context (acp_plan_create) cannot serve   */
  ACP_E_NONFINITE = 6 /* a non-finite value reached the orthogonaliser or the
                       all-reduced buffer (acp_check_finite / ACP_CHECK_FINITE);
                       context poisoned                                     */
} acp_status;

/* flags */
enum {
  ACP_NO_EF = 1u,     /* error feedback off: E == 0 (ablation, C12)      */
  ACP_NO_REUSE = 2u,  /* query reuse off: orthogonalise a fresh seeded N(0,1)
                         factor each step instead of the previous aggregated
                         one (ablation, C12)                            */
  ACP_SUM = 4u,       /* decoded gradient = sum over workers (default: / p)   */
  ACP_POWERSGD = 8u,  /* run the Power-SGD baseline instead (Alg. 1;
                         NEXT-1): each step projects twice, P = M'Q -> AR(P) ->
                         orth(P) -> Q = M'^T P -> AR(Q), E = M' - P Q_loc^T,
                         decoded = P Q^T / p. acp_step ignores parity; in the
                         split API acp_compress(0) forms P (no orthogonalisation),
                         acp_compress(1) orthogonalises the reduced P and forms
                         Q, acp_decompress(1) decodes (acp_decompress(0) is a
                         no-op). Needs error feedback; not
                         combinable with ACP_NO_EF / ACP_NO_REUSE            */
  ACP_BUCKETED = 16u, /* run the multi-rank scheduler (compute groups, the comm
                         stream, one NCCL all-reduce per bucket inside an NCCL
                         group, events, graph capture) even at world_size == 1;
                         needs nccl_comm (a 1-rank communicator). Lets one GPU
                         exercise the whole all-reduce path (P:223 / P:228)   */
  ACP_CHECK_FINITE = 32u /* debug: after each acp_step scan the all-reduced fused
                         buffer for non-finite values and synchronise the
                         stream; the step returns ACP_E_NONFINITE on a hit or
                         when the orthogonaliser saw a non-finite factor
                                                                    */
};

typedef struct {
  int32_t abi_version;           /* ACP_ABI_VERSION                                    */
  int32_t num_tensors;           /* >= 1, in READY order (reverse parameter order)     */
  const int64_t* rows;           /* host, num_tensors: n_i = dim0 (vector: its length) */
  const int64_t* cols;           /* host, num_tensors: m_i = prod(dims[1:]) >= 1, or
                                    0 to mark a 1-D (vector) tensor of length rows[i]  */
  int32_t rank;                  /* r >= 1; per tensor r_i = min(r, n_i, m_i)          */
  int32_t world_size;            /* p >= 1 (divisor of the decoded gradient)           */
  void* nccl_comm;               /* ncclComm_t of p ranks, required iff world_size > 1
                                    and acp_step() is used (the split API needs none)  */
  uint64_t seed;                 /* seeds the method's own draws (Q_0 when q0_host is
                                    NULL, rank-deficiency repair, NO_REUSE); identical
                                    on all ranks                                       */
  const float* q0_host;          /* optional host array: for each matrix in ready order
                                    its Q_0 (m_i x r_i, row-major), concatenated; NULL:
                                    Q_0 from the counter-based generator   */
  int64_t default_bucket_bytes;  /* 25 MiB in the paper; 0 = one tensor per
                                    bucket; < 0 = a single bucket                      */
  uint32_t flags;                /* ACP_NO_EF | ACP_NO_REUSE | ACP_SUM                 */
  int32_t device;                /* CUDA device ordinal the context runs on            */
  void* workspace;               /* device memory, >= acp_workspace_bytes()            */
  size_t workspace_bytes;
} acp_config;

/* Bytes of device workspace the configuration needs (E + both fused buffers +
 * scratch). Reads only the shape fields of *cfg. */
acp_status acp_workspace_bytes(const acp_config* cfg, size_t* out_bytes);

/* Build the plan, upload it into the workspace, write Q_0, zero E.
 * Synchronous (returns after the device work is done). */
acp_status acp_create(const acp_config* cfg, acp_ctx** out_ctx);

/* Plan-only context: the host part of acp_create (shape policy, r_i, slot
 * offsets, buckets of both parities, C7-C10) with no device, no
 * workspace and no communicator -- cfg->device, workspace and nccl_comm are
 * ignored and the work split assumes 148 SMs. acp_plan_info,
 * acp_num_buckets, acp_bucket_range and acp_destroy serve it; every other
 * call returns ACP_E_STATE. Used to check on CPU hosts that all ranks derive
 * the same bucket sequence. ACP_E_INVAL on a bad shape config. */
acp_status acp_plan_create(const acp_config* cfg, acp_ctx** out_ctx);

/* Non-finite check: synchronises cuda_stream, then returns
 * ACP_E_NONFINITE (and poisons the context) if the orthogonaliser saw a
 * non-finite factor -- or, with ACP_CHECK_FINITE, a step's all-reduced buffer
 * held a non-finite value -- since the context was created; ACP_OK otherwise. */
acp_status acp_check_finite(acp_ctx* ctx, void* cuda_stream);

/* One ACP-SGD step (see top). grads: host array of num_tensors DEVICE
 * pointers, each to the tensor's fp32 contiguous gradient, overwritten with
 * the decoded mean. parity: 0 = P-step, 1 = Q-step. cuda_stream: a
 * cudaStream_t (NULL = legacy default stream). Asynchronous. */
acp_status acp_step(acp_ctx* ctx, int32_t parity, float* const* grads, void* cuda_stream);

/* Split API (simulated workers / external all-reduce): acp_compress runs the
 * orthogonalisation and the fused projection + pack of ALL tensors and returns
 * the parity's whole fused buffer (device pointer and float count); the caller
 * replaces its contents by the element-wise SUM over workers; acp_decompress
 * then decodes into grads. Both asynchronous on cuda_stream. */
acp_status acp_compress(acp_ctx* ctx, int32_t parity, float* const* grads,
                        float** out_buffer, int64_t* out_count, void* cuda_stream);
acp_status acp_decompress(acp_ctx* ctx, int32_t parity, float* const* grads, void* cuda_stream);

/* Bucket-granular step for wait-free back-propagation (WFBP, P:236, P:262;
 * SURVEY NEXT-2). The same step as acp_step, split so that each bucket's
 * projection and all-reduce start as soon as the bucket's gradients exist:
 *   acp_step_begin(ctx, parity, grads, s)   orthogonalise the reused factors
 *                                           (they do not depend on this step's
 *                                           gradients); grads as in acp_step,
 *                                           the pointers must stay valid until
 *                                           acp_step_end
 *   acp_bucket_ready(ctx, b, s)             bucket b (of this parity, ready
 *                                           order, acp_num_buckets) is complete:
 *                                           project + pack its tensors on s and
 *                                           (world_size > 1) all-reduce its
 *                                           buffer range on the comm stream
 *   acp_step_end(ctx, s)                    wait for every bucket's all-reduce,
 *                                           decode all tensors into grads
 * Every bucket must be made ready exactly once between begin and end, in any
 * order: the projection runs at once, but the all-reduces are issued strictly
 * in bucket-index order (a bucket that becomes ready before a lower-indexed
 * one waits for it), so every rank issues the same collective sequence even
 * when its hooks fire in a different order. Eager launches (no CUDA graph). Errors: ACP_E_INVAL on a bucket
 * index out of range / a bucket made ready twice / calls out of order
 * (context not poisoned); CUDA / NCCL failures poison the context. */
acp_status acp_step_begin(acp_ctx* ctx, int32_t parity, float* const* grads, void* cuda_stream);
acp_status acp_bucket_ready(acp_ctx* ctx, int32_t bucket, void* cuda_stream);
acp_status acp_step_end(acp_ctx* ctx, void* cuda_stream);

/* NVLS all-reduce (world_size > 1, NVSwitch systems with
 * multicast). The caller allocates a symmetric buffer of
 * acp_symmetric_bytes() bytes on every rank (same size, bound to one
 * NVLink-SHARP multicast object, e.g. torch symmetric memory) and passes this
 * rank's unicast address, the multicast address, every rank's unicast
 * address as mapped on this device (peers[world_size], index = rank in the
 * symmetric group) and this rank's index. The context moves its fused P / Q
 * buffers into the region and from then on all-reduces each compute group
 * (acp_step) or bucket (acp_bucket_ready) with its own kernel: in-switch
 * reduction (multimem.ld_reduce) + multicast store, instead of NCCL.
 * Collective: every rank calls it, then the caller barriers before the next
 * step. Synchronous. ACP_E_INVAL: world_size == 1, too small a region,
 * world_size > 8. */
acp_status acp_symmetric_bytes(acp_ctx* ctx, int64_t* out_bytes);
acp_status acp_attach_symmetric(acp_ctx* ctx, void* local, void* multicast, void* const* peers,
                                int32_t rank, int64_t bytes);

/* State of matrix tensor i (tests, checkpoint/resume). Device pointers; any
 * may be NULL to skip. P: n_i x r_i row-major, Q: m_i x r_i row-major,
 * E: n_i x m_i row-major. Asynchronous on cuda_stream. */
acp_status acp_get_state(acp_ctx* ctx, int32_t tensor, float* P, float* Q, float* E,
                         void* cuda_stream);
acp_status acp_set_state(acp_ctx* ctx, int32_t tensor, const float* P, const float* Q,
                         const float* E, void* cuda_stream);

/* Plan of tensor i: out[0] = r_i (0 for vectors), out[1] = slot offset in the
 * P-buffer (floats), out[2] = slot offset in the Q-buffer, out[3] = E offset
 * (-1 for vectors), out[4] = P-bucket index, out[5] = Q-bucket index. */
acp_status acp_plan_info(acp_ctx* ctx, int32_t tensor, int64_t out[6]);

/* Number of buckets of a parity, and bucket b's [offset, count) in floats
 * within that parity's fused buffer. */
acp_status acp_num_buckets(acp_ctx* ctx, int32_t parity, int32_t* out);
acp_status acp_bucket_range(acp_ctx* ctx, int32_t parity, int32_t bucket, int64_t* offset,
                            int64_t* count);

/* Kernel timing for roofline reporting. When enabled, every kernel launch is
 * bracketed by CUDA events on its launching stream. acp_profile_read
 * synchronises the context's streams and returns, for kernel class k
 * (ACP_K_*), the summed event time (ms), the number of launches and the
 * summed ALGORITHMIC bytes moved. Reset clears. */
enum { ACP_K_ORTH = 0, ACP_K_PROJ_P = 1, ACP_K_PROJ_Q = 2, ACP_K_DECODE_P = 3,
       ACP_K_DECODE_Q = 4, ACP_K_ALLREDUCE = 5, ACP_K_NUM = 6 };
acp_status acp_profile_enable(acp_ctx* ctx, int32_t enable);
acp_status acp_profile_reset(acp_ctx* ctx);
acp_status acp_profile_read(acp_ctx* ctx, int32_t kernel_class, double* ms, int64_t* launches,
                            double* algorithmic_bytes);

/* CUDA graphs (default on): the first acp_step of each parity is captured
 * into a graph (kernels + NCCL calls) that later steps replay with a single
 * launch; the gradient pointers are read from a device table refreshed
 * before each launch, so new pointers do not need a new capture. Profiling
 * (acp_profile_enable) always runs eagerly. */
acp_status acp_set_graphs(acp_ctx* ctx, int32_t enable);

/* Number of kernels this context has launched so far (its own kernels, not
 * NCCL's). */
acp_status acp_launch_count(acp_ctx* ctx, int64_t* out);

acp_status acp_destroy(acp_ctx* ctx);

/* thread-local description of the last non-OK status ("" if none) */
const char* acp_last_error(void);
int32_t acp_abi_version(void);

/* NCCL bootstrap helpers (the caller broadcasts the 128-byte id over its own
 * process group, e.g. torch.distributed, then every rank creates the comm). */
acp_status acp_nccl_unique_id(uint8_t out_id[128]);
acp_status acp_nccl_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank,
                                int32_t device, void** out_comm);
acp_status acp_nccl_comm_destroy(void* comm);

#ifdef __cplusplus
}
#endif
#endif /* ACP_H */
