/*
 * gt.h -- C ABI of libgt.so: full-graph multi-head sparse graph attention (forward + backward)
 * on B200 (sm_100a), single- or multi-GPU (1D node-row partition).
 *
 * The operation (PAPER.md, arXiv 2604.16715):
 *   Eq. 2, Eq. 4, Eq. 5, per head t of the [N, h, d] tensors:
 *     s_e   = scale * <q_{i,t}, k_{j,t}>            for each stored entry e = (i, j) of row i of A
 *     U_e   = exp(s_e) / sum_{e' in row i} exp(s_e')                 (edge softmax over row i)
 *     Y_i,t = sum_{e in row i} U_e v_{j,t}                             (SpMM)
 *     LSE_i,t = log sum_{e in row i} exp(s_e)        (natural log; -inf for an empty row, Y = 0)
 *   Backward (Section 2.2: "three SpMM operations and one SDDMM"):
 *     dP_e  = <dY_i,t, v_{j,t}>                      (SDDMM)
 *     D_i,t = sum_e U_e dP_e
 *     dS_e  = scale * U_e (dP_e - D_i,t)            (softmax backward)
 *     dQ_i  = sum_{e in row i} dS_e k_j   (SpMM, A)
 *     dK_j  = sum_{e in column j} dS_e q_i (SpMM, A^T)
 *     dV_j  = sum_{e in column j} U_e dY_i (SpMM, A^T)
 *   "scale" is the factor of Q K^T: 1/sqrt(d) in Eq. 4.  The paper never reconciles d (feature
 *   dim) with the head dim d'; gt_opts.scale = 0 selects 1/sqrt(heads * d), the
 *   paper-literal full feature dim (reading Z2).  Any positive value may be passed.
 *
 * Graph (CSR, "represented in a sparse format such as COO or CSR"): row i lists the keys
 * node i attends to (reading Z3); columns strictly increasing per row, no duplicates (Z6).
 *
 * Multi-GPU (Alg. 1 GP-AG, generalised): rank r owns rows [row_lo, row_hi) of every
 * [N, h, d] tensor.  Remote K||V rows needed by its edges are fetched by an all-gather
 * (GT_ALLGATHER) or by a halo exchange of only the cut-edge columns (GT_HALO) — as copies into a
 * receive table (gt_opts.transport = 0) or loaded by the kernels straight from the owners over
 * NVLink (transport = 1).  The backward either fetches Q||dY||(LSE, D) of in-neighbour rows the
 * same way and each owner computes dK, dV of its own columns ("transposed-owner", reading Z11), or
 * sends fp32 partial dK||dV to the owners (gt_opts.bwd_mode = 1, the paper's reduce-scatter).
 * GT_A2A is the paper's head-parallel GP-A2A (Alg. 2).  GT_AUTO picks the strategy with
 * the cost model of Eq. 6-8 over measured exchange times (Alg. 3, at fixed
 * world).
 *
 * Per-entry state (gt_opts.edge_state, on by default when it fits): the forward keeps each entry's
 * logit and the row pass its (P, dS) (Table 1 keeps Z and U per edge), so the
 * backward does not recompute them.
 *
 * Conventions
 *   - All functions return gt_status; they never abort or throw.  The message of the last
 *     non-OK status of the calling thread is in gt_last_error().
 *   - Argument / configuration / graph errors are detected synchronously and have no side effects.
 *   - Device work is enqueued on the caller's stream; calls return after enqueue.  Asynchronous
 *     CUDA faults surface as GT_ECUDA on a later call.
 *   - Collective calls (gt_plan, gt_attn_fwd, gt_attn_bwd with world > 1) must be made by every
 *     rank in the same order.  A plan is used by one host thread at a time.
 *   - Supported shapes: heads in {1,2,4,8}, heads*d in {64, 128, 256, 512}.
 *     Others return GT_ECONFIG.
 */
#ifndef GT_H_
#define GT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gt_plan_s* gt_plan_t;     /* opaque; owned by the library, released by gt_free */
typedef struct gt_loopback_s* gt_loopback_t; /* opaque in-process multi-rank group (tests) */
typedef struct gt_hostipc_s* gt_hostipc_t;   /* opaque host-bootstrapped CUDA-IPC group (one process per rank) */

typedef enum {
  GT_OK = 0,
  GT_EINVAL = 1,   /* bad argument or shape ("shape error") */
  GT_EGRAPH = 2,   /* CSR invariant violated: row_ptr not monotone, column out of range,
                      columns not strictly increasing */
  GT_ECONFIG = 3,  /* unsupported heads/d/dtype/world combination ("configuration error") */
  GT_ENOMEM = 4,   /* device or host allocation failed */
  GT_ECUDA = 5,    /* CUDA runtime error (possibly from earlier asynchronous work) */
  GT_ENCCL = 6,    /* NCCL error, NCCL unavailable, or collective protocol mismatch */
  GT_ESTATE = 7    /* call out of order (gt_attn_bwd before any gt_attn_fwd on a plan that retains
                      forward state: world > 1, entry-state logits, GP-A2A) */
} gt_status;

typedef enum { GT_F32 = 0, GT_BF16 = 1 } gt_dtype;

typedef enum {
  GT_AUTO = 0,      /* cost-model choice (world > 1); GT_SINGLE when world == 1 */
  GT_SINGLE = 1,    /* world == 1 only */
  GT_ALLGATHER = 2, /* GP-AG: every rank receives every remote K||V row (Alg. 1) */
  GT_HALO = 3,      /* only the rows its cut edges touch (reading of Alg. 3's open set) */
  GT_A2A = 4        /* GP-A2A head parallelism (Alg. 2): all-to-all of Q, K, V by head group,
                       every rank runs all N rows for heads / world heads, all-to-all of Y back.  Needs
                       heads % world == 0 and a supported (heads / world, d) shape; Q, K, V (and LSE)
                       head slices are retained from gt_attn_fwd for gt_attn_bwd. */
} gt_strategy;

typedef enum {
  GT_COMM_NONE = 0,     /* world == 1 */
  GT_COMM_NCCL = 1,     /* comm = ncclComm_t (from gt_nccl_comm_create), one process per GPU */
  GT_COMM_LOOPBACK = 2, /* comm = gt_loopback_t; all ranks are host threads of one process on
                           devices that can address each other (tests on a single GPU) */
  GT_COMM_HOSTIPC = 3   /* comm = gt_hostipc_t (gt_hostipc_create); one process per rank, devices that can
                           map each other's allocations with CUDA IPC (several processes on one GPU, or
                           GPUs of one node); host collectives through caller callbacks (e.g. gloo) */
} gt_comm_kind;

/* Host CSR of the GLOBAL graph, identical on every rank; borrowed for the duration of gt_plan.
 * row_ptr: int64[n + 1], row_ptr[0] = 0, nondecreasing, row_ptr[n] = nnz.
 * col_idx: int32[nnz], each in [0, n), strictly increasing within a row. */
typedef struct {
  const int64_t* row_ptr;
  const int32_t* col_idx;
} gt_csr;

typedef struct {
  int rank;                /* this rank, 0 <= rank < world */
  int comm_kind;           /* gt_comm_kind */
  void* comm;              /* ncclComm_t, gt_loopback_t or gt_hostipc_t, borrowed; NULL iff world == 1 */
  int dtype;               /* gt_dtype of q, k, v, y, dy, dq, dk, dv */
  float scale;             /* multiplier of Q K^T; 0 => 1/sqrt(heads * d) */
  int strategy;            /* gt_strategy */
  int validate;            /* 1 => O(n + nnz) CSR checks in gt_plan (GT_EGRAPH on failure) */
  int partition;           /* 0 => rows+edges balanced (reading Z9), 1 => node-balanced */
  int device;              /* CUDA device ordinal; -1 => the calling thread's current device */
  int heavy_threshold;     /* rows/columns with more entries are split into chunks; 0 => 512 */
  const char* beta_profile;/* optional path of a measured-beta JSON (GT_AUTO): {"allgather": B,
                              "halo": B, "a2a": B}, B = seconds per exchanged row, a number or an
                              object keyed by the GPU count ({"2": .., "8": ..}, as written by
                              paper_2604_16715_b200.agp); given strategies skip the plan-time probe.
                              NULL => probe every candidate.  Unreadable file => GT_EINVAL. */
  int profile;             /* 1 => record CUDA events around every stage (gt_plan_timings) */
  int edge_state;          /* per-entry state of the backward (Table 1 keeps U per edge,
                              P:166): 0 => materialise when it fits in 85 % of free device memory,
                              1 => materialise (GT_ENOMEM if it does not fit), -1 => never
                              (recompute q.k in the row pass, q.k and dY.v in the column pass).
                              Materialised, the forward stores base-2 logits (4 h B per owned-row
                              entry, fp32), the row pass (P, dS) (4 h B per owned-row entry as bf16x2 for bf16
                              plans, 8 h B as fp32 pairs for fp32 plans),
                              and the plan holds a 4 B CSC -> CSR map per owned-column entry. */
  int bwd_mode;            /* world > 1 backward dataflow (reading Z11 of PAPER.md P:113):
                              0 => transposed owner: the owner of column j computes dK_j, dV_j after
                                   receiving q || dY || (LSE, D) of its remote in-neighbour rows;
                              1 => reduce-scatter (paper-faithful): every rank computes fp32 partial
                                   dK || dV of the remote columns its rows touch and sends them to the
                                   owners (all-gather: a reduce-scatter; halo: the reverse halo), which
                                   sum them in a fixed order.  2 D fp32 per exchanged row. */
  int transport;           /* world > 1 transport of remote rows (strategies halo / all-gather):
                              0 => pack + all-to-all-v / all-gather (NCCL or loopback) into a receive
                                   table, on a side stream overlapped with the owned-column entries;
                              1 => fused peer gather: every rank publishes its K || V
                                   rows (forward) and Q || dY rows (backward) in plan buffers shared
                                   with the peers, and shares its (LSE, D) array in place (CUDA IPC
                                   for NCCL ranks, one GPU per process, peer access over NVLink; the
                                   pointer itself for loopback ranks); the forward / row-pass /
                                   column-pass kernels load remote rows directly from the owners,
                                   with device-side barriers instead of copies.  Needs world <= 8
                                   and bwd_mode = 0. */
  int cuda_graphs;         /* 1 => world-1 plans replay their launch sequence as CUDA graphs (the
                              first call of each direction runs eagerly; later calls are captured
                              once per set of tensor pointers, up to 4, and replayed).  Not used on
                              the legacy default stream or with profile = 1.  Small graphs, whose
                              steps are launch-bound, gain most. */
  int kv_fp8;              /* 1 => fp8 K || V storage (reading Z25): gt_attn_fwd
                              quantises k and v per (row, head) to e4m3 with a power-of-two scale 2^e
                              (e the smallest integer with max |x| <= 448 2^e; x8 = RNE(x 2^-e)) into a
                              plan-owned table [k8 | v8 | scales] (2 d h + 8 h B per row instead of
                              4 d h), and the forward and the row pass gather it: the results are the
                              attention of q, dY on the DEQUANTISED K^ = 2^e k8, V^ = 2^e v8 (products
                              in f16 x e4m3 with fp32 accumulation; q and dY enter as f16 after a
                              per-(row, head) power-of-two normalisation).  A backward whose k, v are
                              not the last forward's re-quantises them.  Needs world == 1, a bf16
                              plan, heads * d >= 128 and the materialised entry state (edge_state
                              >= 0 and fitting); else GT_ECONFIG.  0 => K, V gathered as given. */
  int reserve_sms;         /* world > 1: SMs per GPU left free for the communication kernels while the
                              forward's owned-column phase overlaps the K || V exchange; 0 => 16, -1 =>
                              none (tune per interconnect / NCCL channel count) */
  int hot_cols;            /* > 0 => hot-column table (world 1; not with kv_fp8): the K || V rows of the
                              hot_cols columns with the most entries (power-law hubs, e.g. R-MAT) are
                              packed by every gt_attn_fwd into one contiguous plan table that the
                              forward and row-pass kernels read under an L2 access-policy window
                              (persisting), and the plan's CSR entries of those columns point into
                              it.  Sets the device's persisting-L2 limit.  Results are unchanged
                              (the same values are read).  Measured slower on the C3 / C5
                              benchmarks: an option for graphs whose hubs LRU
                              evicts.  0 => off. */
} gt_opts;

typedef struct {
  int world, rank, strategy, dtype, heads, d;
  float scale;
  int64_t n, nnz;                 /* global graph */
  int64_t row_lo, row_hi;         /* owned rows [row_lo, row_hi) */
  int64_t n_local, nnz_local;     /* owned rows, stored entries in owned rows */
  int64_t nnz_in_local;           /* stored entries in owned columns (column pass) */
  int64_t halo_out_rows;          /* remote rows received in the forward exchange */
  int64_t halo_in_rows;           /* remote rows received in the backward exchange */
  int64_t exch_fwd_bytes;         /* bytes this rank receives per gt_attn_fwd */
  int64_t exch_bwd_bytes;         /* bytes this rank receives per gt_attn_bwd */
  int64_t send_fwd_bytes, send_bwd_bytes;
  int64_t device_bytes;           /* device memory held by the plan */
  int64_t heavy_rows, heavy_row_chunks, heavy_cols, heavy_col_chunks;
  int launches_fwd, launches_bwd; /* libgt kernels launched per call */
  double beta_s_per_row[5];       /* measured exchange time per received row, by strategy (s) */
  double predicted_ms[5];         /* cost-model time of fwd+bwd, by strategy (ms) */
  double agp_score[5];            /* Alg. 3 score p * t_comm / (p - 1) per strategy (ms) */
  int agp_feasible[5];            /* Eq. 14 feasibility: score <= t_iter(1) */
  double alpha_s_per_unit;        /* cost-model compute seconds per (edge + row) */
  int edge_state;                 /* 1 if the plan materialises per-entry state (gt_opts.edge_state) */
  int64_t edge_state_bytes;       /* device bytes of that state */
  int bwd_mode;                   /* backward dataflow in use (gt_opts.bwd_mode; 0 when world == 1) */
  int transport;                  /* forward K || V transport in use (gt_opts.transport) */
  int64_t fwd_gen;                /* gt_attn_fwd calls made on this plan */
  int64_t stale_bwds;             /* gt_attn_bwd calls whose (q, k, v, lse) were not those of the last
                                     gt_attn_fwd (they re-fetched / recomputed the forward's state) */
  int kv_fp8;                     /* 1 if K, V are gathered from the plan's fp8 table (gt_opts.kv_fp8) */
  int64_t kv_fp8_bytes;           /* device bytes of that table */
  int64_t hot_cols;               /* columns in the hot-column table (gt_opts.hot_cols) */
  int64_t hot_entries;            /* owned-row entries that read it */
  int bwd_colfirst;               /* 1: a backward of the last forward runs column-first (world 1, stored
                                     logits): (LSE2, D) of every row, the column pass (dP with its own v_j,
                                     dK, dV, dS per entry), then a row pass gathering k_j alone (dQ);
                                     GT_COLFIRST=0 selects the row-first order */
} gt_plan_info;

/* Fills *o with defaults: rank 0, world-1 comm, bf16, scale 0, GT_AUTO, validate 1,
 * partition 0, device -1, heavy_threshold 0, beta_profile NULL. */
void gt_default_opts(gt_opts* o);

/* Builds a plan: validates the CSR, uploads it, builds the transposed pattern A^T (CSC, rows
 * ascending per column), partitions rows, computes halo sets and send lists, bins rows and
 * columns by degree, allocates exchange buffers and, for world > 1 with GT_AUTO, measures the
 * exchanges and chooses a strategy (rank 0 decides; the decision is broadcast).  Collective.
 * heads, d: the [N, heads, d] layout of every feature tensor.  world: number of ranks.
 * On success *out owns device memory until gt_free. */
gt_status gt_plan(const gt_csr* csr, int64_t n, int64_t nnz, int heads, int d, int world, const gt_opts* opts,
                  gt_plan_t* out);

gt_status gt_plan_info_get(gt_plan_t plan, gt_plan_info* out);

/* Copies plan-internal integer tables to host memory for bit-exact tests.
 * what: GT_EXPORT_* below; peer: rank index for the SEND_* tables (ignored otherwise).
 * dst: host buffer of cap elements (int64 for BOUNDS and CSC_PTR, int32 otherwise); *len receives
 * the element count (dst may be NULL to query).  GT_EINVAL if cap < len. */
enum {
  GT_EXPORT_BOUNDS = 0,     /* int64[world + 1] row partition */
  GT_EXPORT_HALO_OUT = 1,   /* int32 global ids of remote rows received in the forward */
  GT_EXPORT_HALO_IN = 2,    /* int32 global ids of remote rows received in the backward */
  GT_EXPORT_SEND_OUT = 3,   /* int32 global ids this rank sends to `peer` in the forward */
  GT_EXPORT_SEND_IN = 4,    /* int32 global ids this rank sends to `peer` in the backward */
  GT_EXPORT_CSC_PTR = 5,    /* int64[n_local + 1] column pointers of the owned columns */
  GT_EXPORT_CSC_IDX = 6,    /* int32[nnz_in_local] global row ids, ascending within a column */
  GT_EXPORT_HEAVY_ROWS = 7, /* int32 local ids of rows split into chunks */
  GT_EXPORT_HEAVY_COLS = 8, /* int32 local ids of columns split into chunks */
  GT_EXPORT_KV8 = 9         /* uint8[n_local * row] the fp8 K || V table of the last quantisation
                               (gt_opts.kv_fp8): per row k8[heads d] | v8[heads d] | 2^ek f32[heads] |
                               2^ev f32[heads], padded to 16 B; len counts bytes.  Synchronises the
                               device.  Empty when kv_fp8 is off. */
};
gt_status gt_plan_export(gt_plan_t plan, int what, int peer, void* dst, int64_t cap, int64_t* len);

/* Forward.  q, k, v: device [n_local, heads, d] of opts.dtype, contiguous, 16-byte aligned,
 * caller-owned.  y: device [n_local, heads, d] (output, same dtype).  lse: device float32
 * [n_local, heads] (output; natural-log normaliser, -inf for empty rows).  stream: cudaStream_t
 * (NULL = legacy default stream).  Retains the exchanged K||V rows until the next gt_attn_fwd.
 * Collective when world > 1. */
gt_status gt_attn_fwd(gt_plan_t plan, const void* q, const void* k, const void* v, void* y, float* lse,
                      void* stream);

/* Backward.  q, k, v, y, lse as passed to / produced by the matching gt_attn_fwd; dy: device
 * [n_local, heads, d] upstream gradient.  dq, dk, dv: device [n_local, heads, d] outputs (same
 * dtype, round-to-nearest-even from fp32 accumulation).  Collective when world > 1.
 * D_i = sum_e U_e dP_e is taken as <dY_i, Y_i> (equal, since sum_e U_e = 1), so the
 * row pass knows it before its first entry; dS_e = U_e (dP_e - D_i).  With bf16 tensors the weights
 * U_e, dS_e of the SpMM products are rounded to bf16 (the products are exact in fp32 and accumulated
 * in fp32), as the PV and dS K products of FlashAttention are (reading Z23).
 * Order (world 1, materialised logits of this forward): column-first - a kernel writes (LSE2, D) of
 * every row, the column pass over A^T computes dP_e = <dY_i, v_j> with its own v_j, U_e from the
 * logit, dS_e, accumulates dK, dV and stores dS_e per entry; the row pass then gathers k_j alone for
 * dQ (bitwise the results of the row-first order; GT_COLFIRST=0 at gt_plan selects row-first, which
 * world > 1, the host-buffer path and backward calls of another forward always use).
 * The plan retains state of the LAST gt_attn_fwd it ran (the received K||V rows when world > 1, the
 * per-entry logits with edge_state, the head slices with GT_A2A), tagged with that forward's
 * (q, k, v, lse) pointers.  gt_attn_bwd uses the state only when its own (q, k, v, lse) are those
 * tensors; otherwise (another forward ran in between, e.g. several layers sharing one plan, or no
 * forward ran at all) it re-fetches the K||V rows / head slices for these k, v and recomputes the
 * logits from q, k — correct for any call order, at the cost of the extra exchange and dot products
 * (gt_plan_info.stale_bwds counts such calls).  With world > 1 every rank must see the same match,
 * which holds when all ranks make the same sequence of calls on live tensors. */
gt_status gt_attn_bwd(gt_plan_t plan, const void* q, const void* k, const void* v, const void* y, const float* lse,
                      const void* dy, void* dq, void* dk, void* dv, void* stream);

/* End-to-end step with HOST buffers (pinned for full speed): copies q, k, v, dy host->device,
 * runs gt_attn_fwd and gt_attn_bwd, copies y, lse, dq, dk, dv device->host, and returns when all of
 * it is done.  The copies run on two plan-owned copy streams ordered by events against `stream`
 * (PCIe is full duplex): k, v, q in, then the forward while dy arrives; y and lse go out during the
 * backward, dq during the column pass, dk and dv last.  Device staging buffers are allocated on
 * first use and owned by the plan.  Any output pointer may be NULL to skip its copy. */
gt_status gt_attn_fwd_bwd_host(gt_plan_t plan, const void* q, const void* k, const void* v, const void* dy,
                               void* y, float* lse, void* dq, void* dk, void* dv, void* stream);

/* Per-stage device time accumulated since the last call (requires opts.profile = 1), in ms, summed
 * over calls, measured with CUDA events on the stream each stage was launched on:
 *   ms[0] forward exchange (pack + transfer)   ms[1] forward kernels (K1 + chunked rows + merge)
 *   ms[2] backward row pass (dQ, D)            ms[3] backward exchange (pack + transfer)
 *   ms[4] backward column pass (dK, dV)
 * calls[i] = number of times stage i ran.  Synchronises the recorded events; resets the sums. */
gt_status gt_plan_timings(gt_plan_t plan, double* ms /* [5] */, int64_t* calls /* [5] */);

/* Synchronises the plan's internal streams and frees everything it owns.  NULL is a no-op. */
void gt_free(gt_plan_t plan);

/* Thread-local message for the last non-OK status returned to this thread. */
const char* gt_last_error(void);

/* ------------------------------------------------------------------ multi-rank plumbing -- */
/* NCCL bootstrap (one process per GPU): rank 0 calls gt_nccl_unique_id, the 128-byte id is
 * broadcast by the caller (e.g. torch.distributed), then every rank calls gt_nccl_comm_create
 * with its CUDA device current.  NCCL is loaded at run time (libnccl.so.2); GT_ENCCL if absent. */
gt_status gt_nccl_unique_id(void* uid128);
gt_status gt_nccl_comm_create(const void* uid128, int world, int rank, void** comm);
void gt_nccl_comm_destroy(void* comm);

/* In-process group of `world` ranks run by `world` host threads (the loopback transport copies
 * device-to-device on the caller's streams).  Used to test the multi-rank path on one GPU. */
gt_status gt_loopback_create(int world, gt_loopback_t* out);
void gt_loopback_destroy(gt_loopback_t g);

/* Host-bootstrapped CUDA-IPC group (GT_COMM_HOSTIPC): one process per rank, device current at
 * creation.  Device data moves as in Alg. 1 - all-to-all-v of packed rows, all-gather -
 * by CUDA IPC: the sender publishes the IPC handle of the allocation holding its rows and an
 * interprocess event recorded after they were written; receivers wait on the event on their stream
 * and copy out of the mapped allocation; senders wait on the receivers' "done" events before reusing
 * their rows.  Host collectives go through coll->allgather(ctx, send, recv, bytes): every rank passes
 * `bytes` bytes, recv[world * bytes] receives them in rank order; host-synchronous; 0 = success
 * (anything else => GT_ENCCL).  gt_hostipc_create is collective; the callback must stay valid until
 * gt_hostipc_destroy, which must follow gt_free of every plan using the group. */
typedef struct {
  void* ctx;
  int (*allgather)(void* ctx, const void* send, void* recv, int64_t bytes);
} gt_host_coll;
gt_status gt_hostipc_create(const gt_host_coll* coll, int world, int rank, gt_hostipc_t* out);
void gt_hostipc_destroy(gt_hostipc_t g);

/* ------------------------------------------------------------- host-only planning helpers -- */
/* Row partition (reading Z9): mode 0 => bounds[r] = min{ i : row_ptr[i] + i >= ceil(r (nnz + n) / p) },
 * mode 1 => node-balanced.  bounds: int64[p + 1].  No device work. */
gt_status gt_partition(int64_t n, const int64_t* row_ptr, int p, int mode, int64_t* bounds);

/* Halo set of the owned range [lo, hi): inward = 0 => remote columns referenced by owned rows;
 * inward = 1 => remote rows with an entry in an owned column.  Ascending int32 global ids.
 * out may be NULL to query *len.  No device work. */
gt_status gt_halo(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t lo, int64_t hi, int inward,
                  int32_t* out, int64_t cap, int64_t* len);

/* Rows the rank owning [lo, hi) sends to the rank owning [peer_lo, peer_hi) (ascending int32 global
 * ids): inward = 0 => forward K||V rows = owned columns referenced by the peer's rows (the peer's
 * halo intersected with [lo, hi)); inward = 1 => backward Q||dY rows = owned rows with an entry
 * in a peer column.  Exactly the lists gt_plan uses.  No device work. */
gt_status gt_send_list(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t lo, int64_t hi,
                       int64_t peer_lo, int64_t peer_hi, int inward, int32_t* out, int64_t cap, int64_t* len);

/* Cost model of Eq. 7 with Eq. 8 (alpha(p) = alpha(1)/p):
 *   t_iter(p) = alpha1 * E / p + beta_c(p) * N.   beta[c * (P + 1) + p] = beta_c(p) in s/node. */
double gt_estimate_iter_time(double alpha1, const double* beta, int n_strategies, int P, int c, int p, double N,
                             double E);

/* Algorithm 3: k = t_iter1 / N; for i = 2..P, each strategy c: b = beta_c(i); keep
 * (i b / (i - 1), c, i) when it is <= k; return the argmin (ties: smaller i, then smaller c).
 * No feasible candidate => *c_out = -1, *s_out = 1 (single GPU, reading Z12).
 * beta layout as in gt_estimate_iter_time.  *score_out = the chosen score (or 0). */
gt_status gt_agp_select(double N, double t_iter1, const double* beta, int n_strategies, int P, int* c_out,
                        int* s_out, double* score_out);

/* Least-squares fit of t = beta * x in log-log space (Fig. 2): returns beta =
 * exp(mean(log t - log x)) over m >= 2 samples; GT_EINVAL on non-positive samples. */
gt_status gt_fit_beta(const double* x, const double* t, int m, double* beta);

/* Library build / capability string (compile flags, architecture). */
const char* gt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GT_H_ */
