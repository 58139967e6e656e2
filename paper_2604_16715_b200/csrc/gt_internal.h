// Internal declarations of libgt.so (not part of the ABI; see include/gt.h).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <array>
#include <functional>
#include <string>
#include <vector>

#include "../../include/gt.h"

namespace gt {

// ------------------------------------------------------------------ errors --
void set_error(const std::string& msg);
gt_status fail(gt_status s, const std::string& msg);

#define GT_CUDA_TRY(expr)                                                                  \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return ::gt::fail(GT_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));     \
  } while (0)

#define GT_TRY(expr)                 \
  do {                               \
    gt_status _s = (expr);           \
    if (_s != GT_OK) return _s;      \
  } while (0)

// ------------------------------------------------------------- device memory --
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  gt_status alloc(size_t n);
  void release();
  template <typename T> T* as() const { return static_cast<T*>(p); }
  ~DevBuf() { release(); }
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// ------------------------------------------------------------------- comm --
// Transport for the two exchanges of a step (forward K||V rows, backward Q||dY||stats rows).
// A "pattern" is an all-to-all-v of fixed-size rows: send_cnt[s] rows to peer s from
// send_buf + send_off[s] rows, recv_cnt[s] rows from peer s into recv_buf + recv_off[s] rows.
struct Comm {
  virtual ~Comm() = default;
  virtual int world() const = 0;
  virtual int rank() const = 0;
  // all-to-all-v of rows of `row_bytes` bytes, enqueued on `stream`.
  virtual gt_status exchange(const void* send_buf, const int64_t* send_off, const int64_t* send_cnt,
                             void* recv_buf, const int64_t* recv_off, const int64_t* recv_cnt,
                             int64_t row_bytes, cudaStream_t stream) = 0;
  // all-gather of `rows` rows per rank (padded blocks): recv_buf is [world, rows, row_bytes].
  virtual gt_status all_gather(const void* send_buf, void* recv_buf, int64_t rows, int64_t row_bytes,
                               cudaStream_t stream) = 0;
  // broadcast of a small host value from rank 0 (host-synchronous).
  virtual gt_status broadcast_host(void* data, int64_t bytes, cudaStream_t stream) = 0;
  // max over ranks of a host double (host-synchronous).
  virtual gt_status max_host(double* v, cudaStream_t stream) = 0;
  virtual gt_status barrier(cudaStream_t stream) = 0;
  // device-side barrier enqueued on `stream`: work after it on any rank's stream starts only once every
  // rank's stream has reached it (no host synchronisation).
  virtual gt_status stream_barrier(cudaStream_t stream) = 0;
  // collective, host-synchronous: peers[s] = an address of rank s's device buffer `local` valid in this
  // process (CUDA IPC for one process per GPU; the pointer itself for in-process ranks).
  virtual gt_status share_pointers(void* local, void** peers, cudaStream_t stream) = 0;
};

Comm* make_nccl_comm(void* nccl_comm, int world, int rank, gt_status* st);
Comm* make_loopback_comm(gt_loopback_t g, int world, int rank, gt_status* st);
Comm* make_hostipc_comm(gt_hostipc_t g, int world, int rank, gt_status* st);

// ------------------------------------------------------------------- plan --
struct ChunkTable {        // rows (or columns) split into chunks of <= chunk edges
  std::vector<int32_t> ids;        // local ids of heavy rows/cols, ascending
  std::vector<int32_t> first;      // first chunk of each heavy id (size ids.size() + 1)
  std::vector<int64_t> chunk_lo;   // [nchunks] entry range start (offset in the CSR/CSC slice)
  std::vector<int64_t> chunk_hi;
  std::vector<int32_t> chunk_owner;// [nchunks] local row/col id
  DevBuf d_ids, d_first, d_lo, d_hi, d_owner;
  int64_t nchunks() const { return (int64_t)chunk_lo.size(); }
};

// Work items of one kernel launch: entry range [beg, end) in the CSR (CSC) slice and the owner
// (>= 0: the row/column, finished in place; < 0: chunk -1 - c of a ChunkTable, merged later).
// Listed in row (column) order so resident warps sweep a narrow window of rows.
struct WorkList {
  std::vector<int64_t> beg, end;
  std::vector<int32_t> own;
  DevBuf d_beg, d_end, d_own, d_counter;
  int64_t n = 0;
  // rows (columns) without entries are not work items (one atomicAdd each would dominate graphs
  // with many of them, e.g. R-MAT's 56 %): a streaming kernel writes their outputs
  std::vector<int32_t> empty;
  DevBuf d_empty;
};

// One segment of a row's entries assigned to a phase (0 or 1) of a split pass.
struct Segment {
  int64_t lo, hi;
  int phase;
};

}  // namespace gt

struct gt_plan_s {
  // identity
  int world = 1, rank = 0, heads = 0, d = 0, dtype = GT_BF16, strategy = GT_SINGLE, device = 0;
  float scale = 0.f;
  int64_t n = 0, nnz = 0;
  int heavy_threshold = 1024;
  std::vector<int64_t> bounds;     // [world + 1]
  int64_t lo = 0, hi = 0, n_local = 0, nnz_local = 0, nnz_in_local = 0;

  // row pass (forward, backward dQ): local CSR over owned rows, columns remapped
  gt::DevBuf d_row_ptr;            // int64[n_local + 1], rebased to 0
  gt::DevBuf d_col;                // int32[nnz_local]: < n_local local row; >= n_local halo slot
  // column pass (dK, dV): CSC of owned columns, rows remapped the same way (halo-in slots)
  gt::DevBuf d_col_ptr;            // int64[n_local + 1], rebased to 0
  gt::DevBuf d_row;                // int32[nnz_in_local]
  std::vector<int64_t> h_col_ptr;  // host copy of d_col_ptr (exports, chunking)

  gt::ChunkTable heavy_rows, heavy_cols;   // rows / columns with more than heavy_threshold entries
  gt::WorkList w_rows, w_cols;              // row pass (and unsplit forward), column pass
  // forward with world > 1: phase A = owned-column entries (runs while K||V rows are exchanged),
  // phase B = remote-column entries; rows touching both are chunks of fwd_chunks, merged at the end
  bool fwd_split = false;
  gt::WorkList w_fwd[2];
  gt::ChunkTable fwd_chunks;
  int stats_stride = 0;                    // floats per row of d_stats: round16(8 heads) / 4
  int64_t n_items_rows = 0, n_items_cols = 0;

  // backward statistics: [n_local, heads, 2] fp32 = (LSE * log2(e), D)
  gt::DevBuf d_stats;
  // heavy-chunk workspaces (fp32)
  gt::DevBuf d_part_fwd;           // [forward chunks, D + 2 heads]
  gt::DevBuf d_part_rowb;          // [row chunks, D]
  gt::DevBuf d_part_colb;          // [col chunks, 2 D]

  // materialised entry state (opts.edge_state; Table 1 stores U per edge): the row
  // pass writes (P, dS) per entry in CSR order, and the column pass gathers them through the
  // CSC -> CSR entry map instead of recomputing q.k and dY.v per entry
  bool es = false;
  bool es_logits = false;          // the forward's logits are part of the state (GT_ES_LOGITS, default 1)
  bool colfirst = true;            // world-1 backward in column-first order (GT_COLFIRST=0: row-first)
  gt::DevBuf d_s2;                 // f32 [nnz_local][heads] base-2 logits of the forward, local CSR order
  gt::DevBuf d_pd;                 // (P, dS) [nnz_local][heads]: bf16x2 (bf16 plans) | f32x2, local CSR order
  gt::DevBuf d_src;                // int32 [nnz_in_local]: local CSR entry of the CSC position, -1 if remote row
  // column pass with world > 1 and es: phase A = local-row entries (stored state, runs while the
  // in-halo stats are exchanged), phase B = remote-row entries (recompute); split columns merged
  bool col_split = false;
  gt::WorkList w_colp[2];
  gt::ChunkTable col_chunks;

  // paper-faithful backward (opts.bwd_mode = 1; "matching Reduce-Scatter", reading
  // Z11): each rank computes fp32 partial dK || dV of the remote columns its rows touch ("halo
  // columns", from the local CSR's remote-column entries grouped by slot), sends them to the owners
  // (the forward pattern reversed: a reduce-scatter for all-gather, a reverse halo for halo), and
  // each owner sums, in a fixed order, its local-row contributions and the received partials.
  bool bwd_reduce = false;
  gt::DevBuf d_hrow, d_hsrc;       // int32 [halo entries]: local row, local CSR entry; grouped by slot
  int64_t n_hent = 0, n_slots = 0;
  gt::WorkList w_hcols;            // one chunk item per <= T-entry piece of a halo column
  gt::ChunkTable hcol_chunks;      // ids = every slot (possibly with no pieces)
  gt::WorkList w_colrs;            // owned columns, owned-row entries; columns with remote in-edges merged
  gt::ChunkTable rs_chunks;
  gt::DevBuf d_part_h;             // f32 [halo pieces][2 D]
  gt::DevBuf d_rs_send;            // f32 [slots][2 D]: summed partials, in slot (= owner-grouped) order
  gt::DevBuf d_part_rs;            // f32 [rs chunks + received rows][2 D] (one index space)
  gt::DevBuf d_mptr, d_midx;       // per merged column: rows of d_part_rs to sum, in a fixed order
  std::vector<int64_t> rs_send_off, rs_send_cnt, rs_recv_off, rs_recv_cnt;
  int64_t rs_recv_rows = 0, rs_row_bytes = 0;

  // multi-rank exchange
  gt::Comm* comm = nullptr;
  bool own_comm = true;
  std::vector<int32_t> halo_out, halo_in;                 // global ids, ascending
  std::vector<std::vector<int32_t>> send_out, send_in;    // [peer] global ids
  std::vector<int64_t> so_off, so_cnt, ro_off, ro_cnt;    // forward pattern (rows)
  std::vector<int64_t> si_off, si_cnt, ri_off, ri_cnt;    // backward pattern (rows)
  int64_t n_max = 0;               // all-gather block rows
  int64_t n_send_out = 0, n_send_in = 0;                  // rows packed per exchange
  int64_t halo_out_rows = 0, halo_in_rows = 0;            // rows of the receive tables
  gt::DevBuf d_send_out_idx, d_send_in_idx;               // int32 local ids to pack
  gt::DevBuf d_send_buf, d_recv_kv;                       // packed rows: forward [k | v], backward [q | dy]
  gt::DevBuf d_recv_qd, d_send_st, d_recv_st;             // backward [q | dy] rows, (LSE2, D) blocks
  int64_t kv_row_bytes = 0;                               // 2 D b: one [k | v] or [q | dy] row
  int64_t st_row_bytes = 0;                               // round16(8 heads): one (LSE2, D) block
  int64_t in_row_bytes = 0;                               // kv + st: bytes per backward-halo row
  cudaEvent_t ev_bwd0 = nullptr, ev_rows = nullptr, ev_side = nullptr, ev_fwd0 = nullptr, ev_halo = nullptr;
  // Which tensors the retained state belongs to (tags = pointers of the caller's tensors):
  //   kv_tag  (k, v):           the K||V rows received / published for the remote columns (world > 1),
  //                             and for GP-A2A the head slices of (q, k, v) (slice_tag)
  //   lg_tag  (q, k, v, lse):   the per-entry logits stored by the forward (edge_state)
  // gt_attn_bwd uses a piece only when its own tensors match that piece's tag; otherwise it re-fetches
  // the rows / slices (and re-tags them) or recomputes the logits (a stale backward).
  const void* kv_tag[2] = {};
  const void* lg_tag[4] = {};
  const void* slice_tag[3] = {};
  bool kv_valid = false, lg_valid = false, slice_valid = false;
  uint64_t fwd_gen = 0;
  int64_t stale_bwds = 0;          // backward calls that could not use the retained state

  // fused peer-gather transport (opts.transport = 1): every rank publishes its K || V
  // rows in d_pub; the forward's remote-column entries and the row pass read remote rows straight from
  // the owners' publish buffers (NVLink peer loads by the attention kernels themselves, overlapped with
  // the math) instead of a pack + exchange + receive copy.  Remote column ids are
  // n_local + (owner << peer_shift) + offset.
  bool peer = false;
  int peer_shift = 0;
  void* peer_base[8] = {};
  gt::DevBuf d_pub;                // [n_local][k | v]
  gt::DevBuf d_iota;               // int32 [n_local] 0, 1, ...
  gt::DevBuf d_pub_qd;             // [n_local][q | dy]: the backward's published rows
  void* peer_qd[8] = {};           // per rank: its d_pub_qd
  void* peer_st[8] = {};           // per rank: its d_stats ((LSE2, D) blocks, written by its row pass)

  // GP-A2A head-parallel strategy (Alg. 2): a world-1 plan over
  // the full graph with heads / world heads; Q, K, V, dY, LSE are scattered by head group (all-to-all,
  // rows of this rank -> all rows of this rank's heads), Y, LSE, dQ, dK, dV gathered back.  The head
  // slices of Q, K, V and LSE are retained from gt_attn_fwd for gt_attn_bwd.
  gt_plan_s* sub = nullptr;
  int heads_l = 0;
  int64_t csc_base = 0;            // first entry of the owned columns in the global CSC
  gt::DevBuf d_hq, d_hk, d_hv, d_hy, d_hlse, d_hdy, d_hdq, d_hdk, d_hdv;   // [n, heads_l, d] ([n, heads_l])
  gt::DevBuf d_stage[3];                                                  // [world][n_local] head-group rows
  std::vector<int64_t> a2a_loc_off, a2a_loc_cnt, a2a_glob_off, a2a_glob_cnt;  // per peer, in rows

  // end-to-end host staging (gt_attn_fwd_bwd_host): copy streams and their ordering events
  gt::DevBuf h2d[9];
  cudaStream_t e2e_in = nullptr, e2e_out = nullptr;
  cudaEvent_t e2e_ev[5] = {}, ev_dq = nullptr;
  // streamed world-1 gt_attn_fwd_bwd_host: C row (column) chunks - item bounds t, row bounds r, heavy-id
  // bounds h of the row list [0] and the column list [1] - and one event per chunk and stage
  int e2e_c = 0;
  std::vector<int64_t> e2e_t[2], e2e_r[2], e2e_h[2];
  std::vector<cudaEvent_t> e2e_cev;
  cudaEvent_t ev_dq_ready = nullptr;  // when set, gt_attn_bwd records it once dQ is complete

  // CUDA-graph replay (gt_opts.cuda_graphs, world 1): executable graphs keyed by the tensor pointers
  bool graphs = false, fwd_warm = false, bwd_warm = false;
  typedef std::array<const void*, 11> GraphKey;
  struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> gfwd, gbwd;

  gt_plan_info info{};
  cudaStream_t side = nullptr;

  // stage profiling (opts.profile)
  bool profile = false;
  struct Rec { int stage; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t take_event();
  // fp8 K||V storage (gt_opts.kv_fp8): quantised table, its row bytes, {E_k, E_v}, and the k, v it holds
  bool kv_fp8 = false;
  gt::DevBuf d_kv8, d_kvref;
  int64_t kv8_row = 0;
  const void* kv8_tag[2] = {nullptr, nullptr};
  int reserve_sms = 16;            // gt_opts.reserve_sms: SMs left to NCCL during the forward's overlap
  // hot-column table (gt_opts.hot_cols, world 1): packed [k | v] rows of the top in-degree columns
  int64_t n_hot = 0, hot_entries = 0;
  gt::DevBuf d_hot, d_hot_idx;
  const void* hot_tag[2] = {nullptr, nullptr};
  nvtxRangeId_t nvtx_id[5] = {0, 0, 0, 0, 0};   // open NVTX range per stage
  void mark_begin(int stage, cudaStream_t st, cudaEvent_t* a);
  void mark_end(int stage, cudaStream_t st, cudaEvent_t a);
  ~gt_plan_s();
};

namespace gt {
// attention kernels (attn.cu)
gt_status launch_fwd(gt_plan_s* P, const void* q, const void* k, const void* v, const void* halo_kv, void* y,
                     float* lse, cudaStream_t st, cudaEvent_t halo_ready);
// column pass with the fused peer-gather transport (remote in-neighbour rows read from the owners)
gt_status launch_bwd_cols_peer(gt_plan_s* P, const void* q, const void* k, const void* v, const void* dy, void* dk,
                               void* dv, cudaStream_t st);
// forward with the fused peer-gather transport
gt_status launch_fwd_peer(gt_plan_s* P, const void* q, const void* k, const void* v, void* y, float* lse,
                          cudaStream_t st);
// use_logits: read the forward's stored logits (false: recompute q.k; the stored ones belong to
// another forward)
gt_status launch_pass_range(gt_plan_s* P, int pass, const void* q, const void* k, const void* v, const void* y,
                            const float* lse, const void* dy, void* out_a, void* out_b, cudaStream_t st, int64_t t0,
                            int64_t t1, int64_t h0, int64_t h1, bool fill);
gt_status launch_bwd_rows(gt_plan_s* P, const void* q, const void* k, const void* v, const void* y,
                          const void* halo_kv, const float* lse, const void* dy, void* dq, cudaStream_t st,
                          bool use_logits = true);
gt_status launch_bwd_cols(gt_plan_s* P, const void* q, const void* k, const void* v, const void* dy,
                          const void* halo_qd, const void* halo_st, void* dk, void* dv, cudaStream_t st,
                          cudaEvent_t side_ready);
// reduce-scatter backward: partials of the halo columns summed per slot into d_rs_send (st)
// Column-first backward (world 1, stored logits; EntryState::mode 1): cols = (LSE2, D) of every row, then
// the column pass (dK, dV, and dS per entry in CSR order); rows = the row pass gathering k_j alone (dQ).
gt_status launch_bwd_cf_cols(gt_plan_s* P, const void* q, const void* k, const void* v, const void* y,
                             const float* lse, const void* dy, void* dk, void* dv, cudaStream_t st);
gt_status launch_bwd_cf_rows(gt_plan_s* P, const void* q, const void* k, const void* v, const float* lse,
                             const void* dy, void* dq, cudaStream_t st);
// (LSE2, D) [n][sb bytes] of every row: LSE2 = lse log2(e), D = <dY, Y> per head
gt_status row_stats(int dtype, int H, int D, const void* y, const void* dy, const float* lse, int64_t n,
                    float* stats, int sb, cudaStream_t st);
gt_status launch_bwd_halo_cols(gt_plan_s* P, const void* q, const void* dy, cudaStream_t st);
// reduce-scatter backward: owned columns from owned rows; merged columns completed after `recv_ready`
gt_status launch_bwd_cols_rs(gt_plan_s* P, const void* q, const void* k, const void* v, const void* dy, void* dk,
                             void* dv, cudaStream_t st, cudaEvent_t recv_ready);
bool shape_supported(int heads, int d, int dtype);
int launches_fwd(const gt_plan_s* P);
int launches_bwd(const gt_plan_s* P);

// Materialised per-entry state of the ES kernels (all null: recompute kernels).
struct EntryState {
  float* out = nullptr;          // fwd: s2 [nnz_local][heads] | rowb: (P, dS) [nnz_local][heads] (bf16x2 | f32x2)
  const float* in = nullptr;     // rowb: s2 | colb: (P, dS)
  const int32_t* src = nullptr;  // colb: entry -> local CSR entry (-1: remote row)
  // column pass over another entry list (the halo columns of the reduce-scatter backward)
  const int32_t* nbr = nullptr;  // neighbour (row) ids of the entries; null: the plan's CSC slice
  int64_t nnbr = 0;
  int64_t own_stride = 0;        // bytes between own rows (0: one feature row)
  const void* own_c = nullptr;   // rowb: Y (D_i = <dY_i, Y_i>)
  // L2 access-policy window (persisting) for the launch: the hot-column table (gt_opts.hot_cols)
  const void* win = nullptr;
  int64_t win_bytes = 0;
  // fp8 K||V gathers (gt_opts.kv_fp8): the quantised table, its row bytes and {E_k, E_v}
  const void* kv8 = nullptr;
  int64_t kv8_row = 0;
  const int* kvref = nullptr;
  // 1: column-first backward (world 1, stored logits): the column pass computes dP = <dY_i, v_j> with
  // its own v_j, P from the forward's logit (gathered through the CSC -> CSR map) and (LSE2, D) of
  // row i, and stores dS per entry in CSR order; the row pass then gathers k_j only (launch_bwd_colfirst)
  int mode = 0;
};
gt_status quantize_kv(int H, int D, const void* k, const void* v, int64_t n, void* out, int gr, int* ref,
                      cudaStream_t st);
// Item range [t0, t1) of the work list (t1 < 0: to its end); fill: also write the outputs of the list's
// rows (columns) without entries.
struct ItemRange {
  int64_t t0 = 0, t1 = -1;
  bool fill = true;
};
gt_status pipe_pass(gt_plan_s* P, int pass, const WorkList& w, const ChunkTable& ct, float* part, const void* own_a,
                    const void* own_b, const float* lse, const void* gather_a, const void* gather_b, const void* halo,
                    const void* halo_s, void* out_a, void* out_b, float* out_f, cudaStream_t st, int reserve_sms,
                    const EntryState& es = EntryState(), const ItemRange& range = ItemRange());

// pack kernels (comm.cu)
gt_status pack_kv(const void* k, const void* v, const int32_t* idx, int64_t rows, int64_t D, int elt,
                  void* out, cudaStream_t st);
gt_status pack_stats(const float* stats, const int32_t* idx, int64_t rows, int64_t row_bytes, void* out,
                     cudaStream_t st);

// GP-A2A head-group transposes (comm.cu); gb = bytes of one head group of a row
gt_status a2a_pack(const void* src, int64_t rows, int groups, int64_t gb, int self, void* dst, void* dst_self,
                   cudaStream_t st);
gt_status a2a_unpack(const void* src, const void* src_self, int64_t rows, int groups, int64_t gb, int self, void* dst,
                     cudaStream_t st);

// graph (graph.cu)
// d_src (optional, int32[nnz]): CSR entry index of each CSC position
gt_status build_csc_device(const int64_t* d_row_ptr, const int32_t* d_col, int64_t n, int64_t nnz,
                           int64_t* d_col_ptr, int32_t* d_row, int32_t* d_src, cudaStream_t st);
// d_out[p - p_lo] = src[p] - e_lo for CSC positions p in [p_lo, p_hi) whose CSR entry is in [e_lo, e_hi), else -1
gt_status build_local_src(const int32_t* d_src, int64_t p_lo, int64_t p_hi, int64_t e_lo, int64_t e_hi,
                          int32_t* d_out, cudaStream_t st);

// host helpers (host.cpp)
gt_status validate_csr(const int64_t* row_ptr, const int32_t* col_idx, int64_t n, int64_t nnz);
void partition_rows(int64_t n, const int64_t* row_ptr, int p, int mode, int64_t* bounds);
std::vector<int32_t> halo_set(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t lo, int64_t hi,
                              bool inward);
// Rows this rank (owning [lo, hi)) sends to the rank owning [blo, bhi):
//   inward = 0 (forward): owned columns referenced by rows in [blo, bhi)   = H_peer  n [lo, hi)
//   inward = 1 (backward): owned rows with an entry in a column of [blo, bhi) = H_peer^in n [lo, hi)
std::vector<int32_t> send_set(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t lo, int64_t hi,
                              int64_t blo, int64_t bhi, bool inward);
// Builds the work lists of a pass: segs(r, out) lists row r's entry segments in entry order; a
// segment longer than `threshold` is cut into equal chunks; a row with exactly one piece becomes a
// whole-row item, otherwise every piece is a chunk of `t` (merged in entry order).  Rows without
// entries become empty items in phase 0 (their outputs are written as empty rows).
// force(r) (optional): r is always listed in the chunk table (all its pieces, possibly none, are chunks),
// for outputs that are completed by a merge with contributions from elsewhere.
void build_work(int64_t count, const std::function<void(int64_t, std::vector<Segment>&)>& segs, int64_t threshold,
                int nphase, WorkList* phases, ChunkTable* t, const std::function<bool(int64_t)>& force = nullptr);
}  // namespace gt
