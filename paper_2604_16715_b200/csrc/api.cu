// C ABI entry points of libgt.so (include/gt.h): plan construction, forward, backward, exports.
#include <cuda_runtime.h>
#include <omp.h>
#include <stdint.h>

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "gt_internal.h"

namespace gt {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
gt_status fail(gt_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

gt_status DevBuf::alloc(size_t n) {
  release();
  if (n == 0) return GT_OK;
  cudaError_t e = cudaMalloc(&p, n);
  if (e != cudaSuccess) {
    p = nullptr;
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? GT_ENOMEM : GT_ECUDA,
                std::string("cudaMalloc(") + std::to_string(n) + "): " + cudaGetErrorString(e));
  }
  bytes = n;
  return GT_OK;
}

void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

template <typename V>
static gt_status upload(DevBuf& b, const V* src, size_t count) {
  GT_TRY(b.alloc(std::max<size_t>(count, 1) * sizeof(V)));
  if (count) GT_CUDA_TRY(cudaMemcpy(b.p, src, count * sizeof(V), cudaMemcpyHostToDevice));
  return GT_OK;
}

static gt_status upload_work(WorkList& w) {
  GT_TRY(upload(w.d_beg, w.beg.data(), w.beg.size()));
  GT_TRY(upload(w.d_end, w.end.data(), w.end.size()));
  GT_TRY(upload(w.d_own, w.own.data(), w.own.size()));
  GT_TRY(upload(w.d_empty, w.empty.data(), w.empty.size()));
  GT_TRY(w.d_counter.alloc(sizeof(unsigned long long)));
  return GT_OK;
}

static gt_status upload_chunks(ChunkTable& t) {
  if (t.nchunks() == 0) return GT_OK;
  GT_TRY(upload(t.d_ids, t.ids.data(), t.ids.size()));
  GT_TRY(upload(t.d_first, t.first.data(), t.first.size()));
  GT_TRY(upload(t.d_lo, t.chunk_lo.data(), t.chunk_lo.size()));
  GT_TRY(upload(t.d_hi, t.chunk_hi.data(), t.chunk_hi.size()));
  GT_TRY(upload(t.d_owner, t.chunk_owner.data(), t.chunk_owner.size()));
  return GT_OK;
}

static int owner_of(const std::vector<int64_t>& bounds, int64_t j) {
  // last r with bounds[r] <= j among non-empty ranges
  int r = (int)(std::upper_bound(bounds.begin(), bounds.end(), j) - bounds.begin()) - 1;
  return r;
}

// Remaps a global id to this rank's gathered-row index space: owned -> id - lo;
// remote -> n_local + slot in the receive table (halo: position in the sorted halo list;
// all-gather: owner * n_max + offset within the owner's block).
static void remap_ids(int32_t* ids, int64_t count, const gt_plan_s* P, const std::vector<int32_t>& halo, bool ag) {
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < count; ++e) {
    int64_t j = ids[e];
    int64_t out;
    if (j >= P->lo && j < P->hi) {
      out = j - P->lo;
    } else if (ag) {
      int o = owner_of(P->bounds, j);
      out = P->n_local + (int64_t)o * P->n_max + (j - P->bounds[o]);
    } else {
      out = P->n_local + (std::lower_bound(halo.begin(), halo.end(), (int32_t)j) - halo.begin());
    }
    ids[e] = (int32_t)out;
  }
}

// rows of `ids` (ascending global ids) grouped by owner: offsets/counts per rank
static void group_by_owner(const std::vector<int32_t>& ids, const std::vector<int64_t>& bounds,
                           std::vector<int64_t>& off, std::vector<int64_t>& cnt) {
  const int w = (int)bounds.size() - 1;
  off.assign(w, 0);
  cnt.assign(w, 0);
  for (int s = 0; s < w; ++s) {
    auto a = std::lower_bound(ids.begin(), ids.end(), (int32_t)bounds[s]);
    auto b = std::lower_bound(ids.begin(), ids.end(), (int32_t)bounds[s + 1]);
    off[s] = a - ids.begin();
    cnt[s] = b - a;
  }
}

struct Pattern {  // one exchange: rows to send per peer (local ids) and rows to receive per peer
  std::vector<int64_t> send_off, send_cnt, recv_off, recv_cnt;
  std::vector<int32_t> send_idx;  // local ids, concatenated in peer order
  int64_t recv_rows = 0;
};

static void make_halo_pattern(const gt_plan_s* P, const std::vector<std::vector<int32_t>>& send,
                              const std::vector<int32_t>& recv_ids, Pattern& pt) {
  const int w = P->world;
  pt.send_off.assign(w, 0);
  pt.send_cnt.assign(w, 0);
  pt.send_idx.clear();
  for (int s = 0; s < w; ++s) {
    pt.send_off[s] = (int64_t)pt.send_idx.size();
    pt.send_cnt[s] = (int64_t)send[s].size();
    for (int32_t j : send[s]) pt.send_idx.push_back((int32_t)(j - P->lo));
  }
  group_by_owner(recv_ids, P->bounds, pt.recv_off, pt.recv_cnt);
  pt.recv_rows = (int64_t)recv_ids.size();
}

static void make_ag_pattern(const gt_plan_s* P, Pattern& pt) {
  const int w = P->world;
  pt.send_off.assign(w, 0);
  pt.send_cnt.assign(w, P->n_max);
  pt.recv_off.resize(w);
  pt.recv_cnt.assign(w, P->n_max);
  for (int s = 0; s < w; ++s) pt.recv_off[s] = (int64_t)s * P->n_max;
  pt.recv_cnt[P->rank] = 0;
  pt.send_idx.resize(P->n_local);
  std::iota(pt.send_idx.begin(), pt.send_idx.end(), 0);
  pt.recv_rows = (int64_t)w * P->n_max;
}

static int64_t round16(int64_t x) { return (x + 15) / 16 * 16; }

// Measured-beta profile (gt_opts.beta_profile; Fig. 2 / Alg. 3, reading Z14): a JSON object
// {"allgather": B, "halo": B, "a2a": B, "row_bytes": R} where B is seconds per exchanged row of R bytes
// (R absent: this plan's K||V row), either a number or an object keyed by the GPU count
// ({"2": b2, "8": b8}, as written by paper_2604_16715_b200.agp --profile-out).
// Returns NaN for a strategy the file does not give (that candidate is probed instead).
static double profile_beta(const std::string& text, const char* name, int world) {
  const std::string key = std::string("\"") + name + "\"";
  size_t at = text.find(key);
  if (at == std::string::npos) return NAN;
  at = text.find(':', at + key.size());
  if (at == std::string::npos) return NAN;
  ++at;
  while (at < text.size() && std::isspace((unsigned char)text[at])) ++at;
  if (at < text.size() && text[at] == '{') {  // per GPU count
    const size_t end = text.find('}', at);
    const std::string obj = text.substr(at, end == std::string::npos ? std::string::npos : end - at);
    const std::string wk = "\"" + std::to_string(world) + "\"";
    size_t w = obj.find(wk);
    if (w == std::string::npos) return NAN;
    w = obj.find(':', w + wk.size());
    if (w == std::string::npos) return NAN;
    return std::strtod(obj.c_str() + w + 1, nullptr);
  }
  char* endp = nullptr;
  const double v = std::strtod(text.c_str() + at, &endp);
  return endp == text.c_str() + at ? NAN : v;
}

// The forward pattern reversed, for the reduce-scatter backward: every received row (halo slot, or
// padded all-gather block row) goes back to its owner as an fp32 partial.  send_idx of the result
// holds, per received row, the local column it belongs to (-1: all-gather padding).
static Pattern reverse_pattern(const gt_plan_s* P, const Pattern& f, bool ag) {
  const int w = P->world;
  Pattern r;
  r.send_off = f.recv_off;
  r.send_cnt = f.recv_cnt;
  r.recv_off.assign(w, 0);
  r.recv_cnt.assign(w, 0);
  if (ag) {
    r.send_idx.assign((size_t)w * P->n_max, -1);
    for (int s = 0; s < w; ++s) {
      r.recv_off[s] = (int64_t)s * P->n_max;
      r.recv_cnt[s] = s == P->rank ? 0 : P->n_max;
      if (s == P->rank) continue;
      for (int64_t k = 0; k < P->n_local; ++k) r.send_idx[(size_t)(s * P->n_max + k)] = (int32_t)k;
    }
    r.recv_rows = (int64_t)w * P->n_max;
  } else {
    r.recv_off = f.send_off;
    r.recv_cnt = f.send_cnt;
    r.send_idx = f.send_idx;
    r.recv_rows = (int64_t)f.send_idx.size();
  }
  return r;
}

}  // namespace gt

using namespace gt;

cudaEvent_t gt_plan_s::take_event() {
  if (!ev_pool.empty()) {
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
// NVTX ranges (header-only NVTX3: no-ops unless a profiler injects itself) per stage, named like
// gt_plan_timings' stages, plus one per entry point (NvtxScope).
static const char* const kStageNames[5] = {"gt.fwd_exchange", "gt.fwd", "gt.bwd_rows", "gt.bwd_exchange",
                                           "gt.bwd_cols"};
void gt_plan_s::mark_begin(int stage, cudaStream_t st, cudaEvent_t* a) {
  *a = nullptr;
  if (stage >= 0 && stage < 5) nvtx_id[stage] = nvtxRangeStartA(kStageNames[stage]);
  if (!profile) return;
  *a = take_event();
  cudaEventRecord(*a, st);
}
void gt_plan_s::mark_end(int stage, cudaStream_t st, cudaEvent_t a) {
  if (stage >= 0 && stage < 5 && nvtx_id[stage]) {
    nvtxRangeEnd(nvtx_id[stage]);
    nvtx_id[stage] = 0;
  }
  if (!profile || !a) return;
  cudaEvent_t b = take_event();
  cudaEventRecord(b, st);
  recs.push_back({stage, a, b});
}

gt_plan_s::~gt_plan_s() {
  for (cudaEvent_t e : {ev_bwd0, ev_rows, ev_side, ev_fwd0, ev_halo})
    if (e) cudaEventDestroy(e);
  for (auto& r : recs) { ev_pool.push_back(r.a); ev_pool.push_back(r.b); }
  for (auto e : ev_pool) cudaEventDestroy(e);
  if (side) cudaStreamDestroy(side);
  if (e2e_in) cudaStreamDestroy(e2e_in);
  if (e2e_out) cudaStreamDestroy(e2e_out);
  for (cudaEvent_t e : e2e_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : e2e_cev)
    if (e) cudaEventDestroy(e);
  if (ev_dq) cudaEventDestroy(ev_dq);
  for (auto* c : {&gfwd, &gbwd})
    for (auto& e : *c) cudaGraphExecDestroy(e.exec);
  if (comm && own_comm) delete comm;
  delete sub;
}

static bool ag_of(const gt_plan_s* P) { return P->strategy == GT_ALLGATHER; }

// Reduce-scatter backward structures (reading Z11):
//  * halo columns: the local CSR's remote-column entries grouped by receive slot, rows ascending
//    (d_hrow local row, d_hsrc local CSR entry); one work item per <= T-entry piece, all chunks;
//  * owned columns over owned-row entries; a column with remote in-edges is always merged;
//  * the reversed forward pattern, and per merged column the fixed-order list of rows to sum
//    (its own pieces, then the received partials in rank order).
static gt_status build_reduce_backward(gt_plan_s* P, const gt_csr* csr, const std::vector<int64_t>& rp_local,
                                       const std::vector<int32_t>& cols, const DevBuf& full_row, int64_t c0, bool ag,
                                       const Pattern& f, int64_t T, cudaStream_t st) {
  (void)st;
  const int64_t D = (int64_t)P->heads * P->d;
  const int64_t nl = P->n_local;
  P->rs_row_bytes = 2 * D * 4;
  const int64_t nslots = f.recv_rows;
  P->n_slots = nslots;
  std::vector<int64_t> hptr((size_t)nslots + 1, 0);
  for (int32_t c : cols)
    if (c >= nl) ++hptr[(size_t)(c - nl) + 1];
  for (int64_t s = 0; s < nslots; ++s) hptr[s + 1] += hptr[s];
  P->n_hent = hptr[nslots];
  std::vector<int32_t> hrow((size_t)P->n_hent), hsrc((size_t)P->n_hent);
  std::vector<int64_t> fill(hptr.begin(), hptr.end() - 1);
  for (int64_t r = 0; r < nl; ++r)
    for (int64_t e = rp_local[r]; e < rp_local[r + 1]; ++e) {
      const int32_t c = cols[(size_t)e];
      if (c < nl) continue;
      const int64_t k = fill[(size_t)(c - nl)]++;
      hrow[(size_t)k] = (int32_t)r;
      hsrc[(size_t)k] = (int32_t)e;
    }
  GT_TRY(upload(P->d_hrow, hrow.data(), hrow.size()));
  GT_TRY(upload(P->d_hsrc, hsrc.data(), hsrc.size()));
  build_work(nslots, [&](int64_t s, std::vector<Segment>& o) { o.push_back({hptr[s], hptr[s + 1], 0}); }, T, 1,
             &P->w_hcols, &P->hcol_chunks, [](int64_t) { return true; });
  // owned columns, owned-row entries [e0 + a, e0 + b) (CSC rows ascend within a column)
  std::vector<int32_t> grow((size_t)P->nnz_in_local);
  if (P->nnz_in_local)
    GT_CUDA_TRY(cudaMemcpy(grow.data(), full_row.as<int32_t>() + c0, grow.size() * sizeof(int32_t),
                           cudaMemcpyDeviceToHost));
  std::vector<int64_t> la((size_t)nl), lb((size_t)nl);
  for (int64_t c = 0; c < nl; ++c) {
    const int32_t* r0 = grow.data() + P->h_col_ptr[c];
    const int32_t* r1 = grow.data() + P->h_col_ptr[c + 1];
    la[c] = std::lower_bound(r0, r1, (int32_t)P->lo) - r0;
    lb[c] = std::lower_bound(r0, r1, (int32_t)P->hi) - r0;
  }
  build_work(nl,
             [&](int64_t c, std::vector<Segment>& o) {
               o.push_back({P->h_col_ptr[c] + la[c], P->h_col_ptr[c] + lb[c], 0});
             },
             T, 1, &P->w_colrs, &P->rs_chunks,
             [&](int64_t c) { return la[c] > 0 || lb[c] < P->h_col_ptr[c + 1] - P->h_col_ptr[c]; });
  for (ChunkTable* t : {&P->hcol_chunks, &P->rs_chunks}) {  // ids / first even when there are no pieces
    GT_TRY(upload(t->d_ids, t->ids.data(), t->ids.size()));
    GT_TRY(upload(t->d_first, t->first.data(), t->first.size()));
    GT_TRY(upload(t->d_lo, t->chunk_lo.data(), t->chunk_lo.size()));
    GT_TRY(upload(t->d_hi, t->chunk_hi.data(), t->chunk_hi.size()));
    GT_TRY(upload(t->d_owner, t->chunk_owner.data(), t->chunk_owner.size()));
  }
  GT_TRY(upload_work(P->w_hcols));
  GT_TRY(upload_work(P->w_colrs));
  // reversed pattern and merge lists
  const Pattern rev = reverse_pattern(P, f, ag);
  P->rs_send_off = rev.send_off; P->rs_send_cnt = rev.send_cnt;
  P->rs_recv_off = rev.recv_off; P->rs_recv_cnt = rev.recv_cnt;
  P->rs_recv_rows = rev.recv_rows;
  const int64_t nrc = P->rs_chunks.nchunks();
  std::vector<int64_t> rptr((size_t)nl + 1, 0);
  for (int32_t col : rev.send_idx)
    if (col >= 0) ++rptr[(size_t)col + 1];
  for (int64_t c = 0; c < nl; ++c) rptr[c + 1] += rptr[c];
  std::vector<int64_t> rrows((size_t)rptr[nl]);
  {
    std::vector<int64_t> at(rptr.begin(), rptr.end() - 1);
    for (int64_t k = 0; k < (int64_t)rev.send_idx.size(); ++k)  // ascending k = ascending rank
      if (rev.send_idx[(size_t)k] >= 0) rrows[(size_t)at[(size_t)rev.send_idx[(size_t)k]]++] = k;
  }
  const auto& ids = P->rs_chunks.ids;
  std::vector<int64_t> mptr(ids.size() + 1, 0), midx;
  for (size_t x = 0; x < ids.size(); ++x) {
    for (int32_t ch = P->rs_chunks.first[x]; ch < P->rs_chunks.first[x + 1]; ++ch) midx.push_back(ch);
    for (int64_t k = rptr[(size_t)ids[x]]; k < rptr[(size_t)ids[x] + 1]; ++k) midx.push_back(nrc + rrows[(size_t)k]);
    mptr[x + 1] = (int64_t)midx.size();
  }
  GT_TRY(upload(P->d_mptr, mptr.data(), mptr.size()));
  GT_TRY(upload(P->d_midx, midx.data(), midx.size()));
  GT_TRY(P->d_part_h.alloc((size_t)std::max<int64_t>(P->hcol_chunks.nchunks(), 1) * P->rs_row_bytes));
  GT_TRY(P->d_rs_send.alloc((size_t)std::max<int64_t>(nslots, 1) * P->rs_row_bytes));
  GT_TRY(P->d_part_rs.alloc((size_t)std::max<int64_t>(nrc + rev.recv_rows, 1) * P->rs_row_bytes));
  (void)csr;
  return GT_OK;
}

extern "C" {
static gt_status plan_impl(const gt_csr* csr, int64_t n, int64_t nnz, int heads, int d, int world,
                           const gt_opts* opts, gt_plan_t* out);
}

static void fill_info(gt_plan_s* P, int64_t nrc, int64_t ncc) {
  const bool single = P->world == 1;
  gt_plan_info& I = P->info;
  I.world = P->world; I.rank = P->rank; I.strategy = P->strategy; I.dtype = P->dtype; I.heads = P->heads;
  I.d = P->d; I.scale = P->scale; I.n = P->n; I.nnz = P->nnz; I.row_lo = P->lo; I.row_hi = P->hi;
  I.n_local = P->n_local; I.nnz_local = P->nnz_local; I.nnz_in_local = P->nnz_in_local;
  I.halo_out_rows = single ? 0 : (P->strategy == GT_ALLGATHER ? (int64_t)(P->world - 1) * P->n_max : (int64_t)P->halo_out.size());
  I.halo_in_rows = single ? 0 : (P->strategy == GT_ALLGATHER ? (int64_t)(P->world - 1) * P->n_max : (int64_t)P->halo_in.size());
  I.heavy_rows = (int64_t)P->heavy_rows.ids.size();
  I.heavy_row_chunks = nrc;
  I.heavy_cols = (int64_t)P->heavy_cols.ids.size();
  I.heavy_col_chunks = ncc;
  I.launches_fwd = launches_fwd(P) + (single ? 0 : 1);
  I.launches_bwd = launches_bwd(P) + (single ? 0 : (P->bwd_reduce ? 0 : 1));
  I.bwd_mode = P->bwd_reduce ? 1 : 0;
  I.transport = P->peer ? 1 : 0;
  if (P->peer) I.launches_fwd = launches_fwd(P) + 1;  // + the publish pack
  I.kv_fp8 = P->kv_fp8 ? 1 : 0;
  I.kv_fp8_bytes = P->kv_fp8 ? P->n_local * P->kv8_row : 0;
  if (P->kv_fp8) I.launches_fwd += 1;                   // + the quantisation
  I.hot_cols = P->n_hot;
  I.hot_entries = P->hot_entries;
  if (P->n_hot) I.launches_fwd += 1;                    // + the hot-table pack
  // column-first backward (a backward of the last forward, world 1): + the (LSE2, D) kernel
  I.bwd_colfirst = single && P->colfirst && P->es_logits && !P->kv_fp8 && !P->n_hot &&
                   P->heads * (P->dtype == GT_F32 ? 4 : 2) >= 4;
  if (I.bwd_colfirst) I.launches_bwd += 1;
  int64_t dev = 0;
  for (const DevBuf* b : {&P->d_row_ptr, &P->d_col, &P->d_col_ptr, &P->d_row, &P->d_stats, &P->d_part_fwd,
                          &P->d_part_rowb, &P->d_part_colb, &P->d_send_out_idx, &P->d_send_in_idx, &P->d_send_buf,
                          &P->d_recv_kv, &P->d_recv_qd, &P->d_recv_st, &P->d_send_st, &P->d_s2, &P->d_pd, &P->d_src,
                          &P->d_hrow, &P->d_hsrc, &P->d_part_h, &P->d_rs_send, &P->d_part_rs, &P->d_mptr, &P->d_midx,
                          &P->d_hq, &P->d_hk, &P->d_hv, &P->d_hy, &P->d_hlse, &P->d_hdy, &P->d_hdq, &P->d_hdk,
                          &P->d_hdv, &P->d_stage[0], &P->d_stage[1], &P->d_stage[2], &P->d_pub, &P->d_iota, &P->d_pub_qd,
                          &P->d_kv8, &P->d_kvref, &P->d_hot, &P->d_hot_idx})
    dev += (int64_t)b->bytes;
  if (P->strategy == GT_A2A && P->sub) {  // the world-1 plan over all rows with heads / world heads
    const gt_plan_info& S = P->sub->info;
    dev += S.device_bytes;
    I.heavy_rows = S.heavy_rows; I.heavy_row_chunks = S.heavy_row_chunks;
    I.heavy_cols = S.heavy_cols; I.heavy_col_chunks = S.heavy_col_chunks;
    I.launches_fwd = S.launches_fwd + 5;   // 3 packs + 2 unpacks (Y, LSE)
    I.launches_bwd = S.launches_bwd + 5;   // 2 packs (dY, LSE) + 3 unpacks
    I.edge_state = S.edge_state; I.edge_state_bytes = S.edge_state_bytes;
    const int64_t gb = (int64_t)P->heads_l * P->d * (P->dtype == GT_F32 ? 4 : 2);
    const int64_t remote = P->n - P->n_local;
    I.exch_fwd_bytes = remote * (3 * gb + P->heads_l * 4) + (P->world - 1) * P->n_local * (gb + P->heads_l * 4);
    I.exch_bwd_bytes = remote * (gb + P->heads_l * 4) + (P->world - 1) * P->n_local * 3 * gb;
  }
  I.device_bytes = dev;
}

// GP-A2A: the world-1 plan over the full graph with heads / world heads, head-slice buffers and the
// two all-to-all patterns (rows in head-group units: local block -> all rows of the rank's heads).
static gt_status build_a2a(gt_plan_s* P, const gt_csr* csr, int64_t n, int64_t nnz, int d, const gt_opts* opts) {
  const int w = P->world;
  P->heads_l = P->heads / w;
  gt_opts so = *opts;
  so.rank = 0;
  so.comm_kind = GT_COMM_NONE;
  so.comm = nullptr;
  so.strategy = GT_SINGLE;
  so.bwd_mode = 0;
  so.validate = 0;  // validated by the caller
  so.device = P->device;
  so.scale = P->scale;  // 1 / sqrt(heads d) of the full problem, not of the head slice
  gt_plan_t sub = nullptr;
  GT_TRY(plan_impl(csr, n, nnz, P->heads_l, d, 1, &so, &sub));
  P->sub = sub;
  const int elt = P->dtype == GT_F32 ? 4 : 2;
  const int64_t gb = (int64_t)P->heads_l * d * elt;
  const size_t nn = (size_t)std::max<int64_t>(n, 1);
  for (DevBuf* b : {&P->d_hq, &P->d_hk, &P->d_hv, &P->d_hy, &P->d_hdy, &P->d_hdq, &P->d_hdk, &P->d_hdv})
    GT_TRY(b->alloc(nn * gb));
  GT_TRY(P->d_hlse.alloc(nn * P->heads_l * sizeof(float)));
  for (DevBuf& b : P->d_stage)
    GT_TRY(b.alloc((size_t)std::max<int64_t>(P->n_local, 1) * P->heads * d * elt));
  P->a2a_loc_off.resize(w); P->a2a_loc_cnt.resize(w); P->a2a_glob_off.resize(w); P->a2a_glob_cnt.resize(w);
  for (int s = 0; s < w; ++s) {
    P->a2a_loc_off[s] = (int64_t)s * P->n_local;
    P->a2a_loc_cnt[s] = s == P->rank ? 0 : P->n_local;
    P->a2a_glob_off[s] = P->bounds[s];
    P->a2a_glob_cnt[s] = s == P->rank ? 0 : P->bounds[s + 1] - P->bounds[s];
  }
  return GT_OK;
}

// Scatter of a row-partitioned tensor [n_local][heads groups of gb bytes] into the head slice
// [n][gb] of this rank (stage: [world][n_local][gb]); gather is the reverse.
static gt_status a2a_scatter(gt_plan_s* P, const void* src, int64_t gb, void* stage, void* slice, cudaStream_t st) {
  GT_TRY(a2a_pack(src, P->n_local, P->world, gb, P->rank, stage, (char*)slice + P->lo * gb, st));
  return P->comm->exchange(stage, P->a2a_loc_off.data(), P->a2a_loc_cnt.data(), slice, P->a2a_glob_off.data(),
                           P->a2a_glob_cnt.data(), gb, st);
}
static gt_status a2a_gather(gt_plan_s* P, const void* slice, int64_t gb, void* stage, void* dst, cudaStream_t st) {
  GT_TRY(P->comm->exchange(slice, P->a2a_glob_off.data(), P->a2a_glob_cnt.data(), stage, P->a2a_loc_off.data(),
                           P->a2a_loc_cnt.data(), gb, st));
  return a2a_unpack(stage, (const char*)slice + P->lo * gb, P->n_local, P->world, gb, P->rank, dst, st);
}

extern "C" {

const char* gt_last_error(void) { return g_err.c_str(); }

const char* gt_version(void) {
  return "libgt 0.1 (sm_100a; fused SDDMM+softmax+SpMM fwd, row/column backward; NCCL/loopback exchange)";
}

void gt_default_opts(gt_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->dtype = GT_BF16;
  o->strategy = GT_AUTO;
  o->validate = 1;
  o->device = -1;
}

static gt_status plan_impl(const gt_csr* csr, int64_t n, int64_t nnz, int heads, int d, int world,
                           const gt_opts* opts, gt_plan_t* out) {
  if (!csr || !out || !opts) return fail(GT_EINVAL, "gt_plan: null argument");
  *out = nullptr;
  if (n < 0 || nnz < 0 || n >= (1ll << 31) - 128 || nnz >= (1ll << 31) - 128)  // kernels index entries in 32 bits
    return fail(GT_EINVAL, "gt_plan: n and nnz must be in [0, 2^31 - 128)");
  if (!csr->row_ptr || (nnz > 0 && !csr->col_idx)) return fail(GT_EINVAL, "gt_plan: null CSR arrays");
  if (heads <= 0 || d <= 0) return fail(GT_EINVAL, "gt_plan: heads and d must be positive");
  if (!shape_supported(heads, d, opts->dtype))
    return fail(GT_ECONFIG, "gt_plan: unsupported shape: need heads in {1,2,4,8}, heads*d in {64,128,256,512}, "
                            "dtype f32|bf16; got heads=" + std::to_string(heads) + " d=" + std::to_string(d));
  if (world < 1 || opts->rank < 0 || opts->rank >= world) return fail(GT_EINVAL, "gt_plan: bad world/rank");
  if (world > 1 && (!opts->comm || (opts->comm_kind != GT_COMM_NCCL && opts->comm_kind != GT_COMM_LOOPBACK &&
                                    opts->comm_kind != GT_COMM_HOSTIPC)))
    return fail(GT_EINVAL, "gt_plan: world > 1 needs a communicator");
  if (opts->strategy < GT_AUTO || opts->strategy > GT_A2A) return fail(GT_EINVAL, "gt_plan: unknown strategy");
  if (world == 1 && (opts->strategy == GT_ALLGATHER || opts->strategy == GT_HALO || opts->strategy == GT_A2A))
    return fail(GT_ECONFIG, "gt_plan: multi-GPU strategy requested with world == 1");
  if (world > 1 && opts->strategy == GT_A2A && (heads % world != 0 || !shape_supported(heads / world, d, opts->dtype)))
    return fail(GT_ECONFIG, "gt_plan: GP-A2A needs heads % world == 0 and a supported (heads / world, d) shape");
  if (opts->partition != 0 && opts->partition != 1) return fail(GT_EINVAL, "gt_plan: partition must be 0 or 1");
  if (opts->bwd_mode != 0 && opts->bwd_mode != 1) return fail(GT_EINVAL, "gt_plan: bwd_mode must be 0 or 1");
  if (opts->transport != 0 && opts->transport != 1) return fail(GT_EINVAL, "gt_plan: transport must be 0 or 1");
  if (world > 1 && opts->transport == 1 && (world > 8 || opts->bwd_mode == 1))
    return fail(GT_ECONFIG, "gt_plan: the peer-gather transport needs world <= 8 and the transposed-owner backward");
  if (!(opts->scale >= 0.f) || std::isinf(opts->scale)) return fail(GT_EINVAL, "gt_plan: bad scale");
  if (opts->kv_fp8 != 0 && opts->kv_fp8 != 1) return fail(GT_EINVAL, "gt_plan: kv_fp8 must be 0 or 1");
  if (opts->hot_cols < 0) return fail(GT_EINVAL, "gt_plan: hot_cols must be >= 0");
  if (opts->reserve_sms < -1) return fail(GT_EINVAL, "gt_plan: reserve_sms must be >= -1");
  if (opts->hot_cols > 0 && (world != 1 || opts->kv_fp8))
    return fail(GT_ECONFIG, "gt_plan: hot_cols needs world == 1 and kv_fp8 == 0");
  if (opts->kv_fp8 && (world != 1 || opts->dtype != GT_BF16 || (int64_t)heads * d < 128 || opts->edge_state < 0))
    return fail(GT_ECONFIG, "gt_plan: kv_fp8 needs world == 1, a bf16 plan, heads * d >= 128 and the entry state");
  if (opts->validate) GT_TRY(validate_csr(csr->row_ptr, csr->col_idx, n, nnz));
  else if (csr->row_ptr[n] != nnz) return fail(GT_EGRAPH, "row_ptr[n] != nnz");

  if (opts->device >= 0) GT_CUDA_TRY(cudaSetDevice(opts->device));
  auto P = std::make_unique<gt_plan_s>();
  GT_CUDA_TRY(cudaGetDevice(&P->device));
  GT_CUDA_TRY(cudaStreamCreateWithFlags(&P->side, cudaStreamNonBlocking));
  cudaStream_t st = P->side;
  P->world = world;
  P->rank = opts->rank;
  P->heads = heads;
  P->d = d;
  P->dtype = opts->dtype;
  P->n = n;
  P->nnz = nnz;
  P->scale = opts->scale > 0.f ? opts->scale : (float)(1.0 / std::sqrt((double)heads * d));
  P->heavy_threshold = opts->heavy_threshold > 0 ? opts->heavy_threshold : 512;  // A/B-tuned on C3
  P->reserve_sms = opts->reserve_sms == 0 ? 16 : (opts->reserve_sms < 0 ? 0 : opts->reserve_sms);
  P->profile = opts->profile != 0;
  P->bwd_reduce = world > 1 && opts->bwd_mode == 1;
  P->graphs = opts->cuda_graphs != 0;
  P->stats_stride = (int)((8 * heads + 15) / 16 * 16 / 4);
  const int64_t D = (int64_t)heads * d;
  const int elt = opts->dtype == GT_F32 ? 4 : 2;
  P->kv_row_bytes = 2 * D * elt;
  P->st_row_bytes = round16(8 * heads);
  P->in_row_bytes = P->kv_row_bytes + P->st_row_bytes;

  gt_status cst = GT_OK;
  if (world > 1) {
    P->comm = opts->comm_kind == GT_COMM_NCCL       ? make_nccl_comm(opts->comm, world, opts->rank, &cst)
              : opts->comm_kind == GT_COMM_HOSTIPC ? make_hostipc_comm((gt_hostipc_t)opts->comm, world, opts->rank, &cst)
                                                   : make_loopback_comm((gt_loopback_t)opts->comm, world, opts->rank, &cst);
    if (!P->comm) return cst;
  }

  // ---- partition (reading Z9) ----
  P->bounds.resize(world + 1);
  partition_rows(n, csr->row_ptr, world, opts->partition, P->bounds.data());
  P->lo = P->bounds[P->rank];
  P->hi = P->bounds[P->rank + 1];
  P->n_local = P->hi - P->lo;
  P->nnz_local = csr->row_ptr[P->hi] - csr->row_ptr[P->lo];
  for (int r = 0; r < world; ++r) P->n_max = std::max(P->n_max, P->bounds[r + 1] - P->bounds[r]);

  // ---- full graph on device, A^T (CSC) ----
  DevBuf full_rp, full_col_tmp, full_cp, full_row;
  GT_TRY(upload(full_rp, csr->row_ptr, (size_t)n + 1));
  const bool single = world == 1;
  DevBuf* full_col = single ? &P->d_col : &full_col_tmp;
  GT_TRY(upload(*full_col, csr->col_idx, (size_t)nnz));
  DevBuf* cp = single ? &P->d_col_ptr : &full_cp;
  DevBuf* rw = single ? &P->d_row : &full_row;
  GT_TRY(cp->alloc(((size_t)n + 1) * sizeof(int64_t)));
  GT_TRY(rw->alloc(std::max<size_t>((size_t)nnz, 1) * sizeof(int32_t)));
  DevBuf full_src;  // CSR entry of each CSC position (for the entry-state permutation)
  GT_TRY(full_src.alloc(std::max<size_t>((size_t)nnz, 1) * sizeof(int32_t)));
  GT_TRY(build_csc_device(full_rp.as<int64_t>(), full_col->as<int32_t>(), n, nnz, cp->as<int64_t>(),
                          rw->as<int32_t>(), full_src.as<int32_t>(), st));
  std::vector<int64_t> col_ptr_full((size_t)n + 1);
  GT_CUDA_TRY(cudaMemcpy(col_ptr_full.data(), cp->p, ((size_t)n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));

  // ---- local row slice (row pass) ----
  std::vector<int64_t> rp_local((size_t)P->n_local + 1);
  for (int64_t i = 0; i <= P->n_local; ++i) rp_local[i] = csr->row_ptr[P->lo + i] - csr->row_ptr[P->lo];
  GT_TRY(upload(P->d_row_ptr, rp_local.data(), rp_local.size()));
  // ---- local column slice (column pass) ----
  const int64_t c0 = col_ptr_full[P->lo], c1 = col_ptr_full[P->hi];
  P->nnz_in_local = c1 - c0;
  P->csc_base = c0;
  P->h_col_ptr.resize((size_t)P->n_local + 1);
  for (int64_t j = 0; j <= P->n_local; ++j) P->h_col_ptr[j] = col_ptr_full[P->lo + j] - c0;

  // ---- multi-rank: halo sets, send lists, strategy ----
  Pattern pf_halo, pb_halo, pf_ag, pb_ag;
  if (!single) {
    const int w = world;
    const int64_t lo = P->lo, hi = P->hi;
    const int64_t* rp = csr->row_ptr;
    const int32_t* ci = csr->col_idx;
    P->halo_out = halo_set(n, rp, ci, lo, hi, false);
    P->halo_in = halo_set(n, rp, ci, lo, hi, true);
    P->send_out.assign(w, {});
    P->send_in.assign(w, {});
    for (int s = 0; s < w; ++s) {
      if (s == P->rank) continue;
      P->send_out[s] = send_set(n, rp, ci, lo, hi, P->bounds[s], P->bounds[s + 1], false);
      P->send_in[s] = send_set(n, rp, ci, lo, hi, P->bounds[s], P->bounds[s + 1], true);
    }
    make_halo_pattern(P.get(), P->send_out, P->halo_out, pf_halo);
    make_halo_pattern(P.get(), P->send_in, P->halo_in, pb_halo);
    make_ag_pattern(P.get(), pf_ag);
    make_ag_pattern(P.get(), pb_ag);

    int strategy = opts->strategy;
    // cost model (Eq. 6-8 generalised): t_c = alpha (E_r + N_r) + t_exchange,c
    const double alpha = 3200.0 / (0.6 * 6.45e12);  // s per (edge + row): gather-model bytes / 60% HBM
    double units = (double)(P->nnz_local + P->nnz_in_local) / 2 + (double)P->n_local;
    double t_compute = alpha * units;
    GT_TRY(P->comm->max_host(&t_compute, st));
    const double t_iter1 = alpha * (double)(nnz + n);
    P->info.alpha_s_per_unit = alpha;
    size_t free_b = 0, total_b = 0;
    GT_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    const int64_t rs_bytes = 2 * D * 4;  // one fp32 partial dK || dV row (reduce-scatter backward)
    std::string prof;
    if (opts->beta_profile && opts->beta_profile[0]) {
      FILE* fp = std::fopen(opts->beta_profile, "rb");
      if (!fp) return fail(GT_EINVAL, std::string("gt_plan: cannot read beta_profile ") + opts->beta_profile);
      char buf[4096];
      size_t got;
      while ((got = std::fread(buf, 1, sizeof(buf), fp)) > 0) prof.append(buf, got);
      std::fclose(fp);
    }
    for (int c : {(int)GT_ALLGATHER, (int)GT_HALO}) {
      const Pattern& f = c == GT_ALLGATHER ? pf_ag : pf_halo;
      const Pattern rev = P->bwd_reduce ? reverse_pattern(P.get(), f, c == GT_ALLGATHER) : Pattern();
      const Pattern& b = P->bwd_reduce ? rev : (c == GT_ALLGATHER ? pb_ag : pb_halo);
      const int64_t b_row = P->bwd_reduce ? rs_bytes : P->in_row_bytes;
      int64_t need = f.recv_rows * P->kv_row_bytes + b.recv_rows * b_row +
                     (P->bwd_reduce ? f.recv_rows * 2 * rs_bytes
                                    : std::max((int64_t)f.send_idx.size() * P->kv_row_bytes,
                                               (int64_t)b.send_idx.size() * P->in_row_bytes) +
                                          (c == GT_ALLGATHER ? P->n_max * (P->kv_row_bytes + P->in_row_bytes) : 0));
      double misfit = (double)need < 0.85 * (double)free_b ? 0.0 : 1.0;
      GT_TRY(P->comm->max_host(&misfit, st));  // every rank must agree (the probe below is collective)
      const double fits = misfit > 0 ? 0.0 : 1.0;
      double t_ex = INFINITY;
      const double pb = prof.empty() ? NAN : profile_beta(prof, c == GT_ALLGATHER ? "allgather" : "halo", world);
      if (strategy == GT_AUTO && fits > 0 && std::isfinite(pb)) {
        // profiled beta x rows moved (Eq. 7 term).  A profile that states the row size it was measured at
        // ("row_bytes", agp.py) is rescaled to this plan's rows (bandwidth regime: time ~ bytes); without
        // it the profile is taken to be at this plan's K||V row size.
        const double rb = prof.empty() ? NAN : profile_beta(prof, "row_bytes", world);
        const double sf = (std::isfinite(rb) && rb > 0) ? (double)P->kv_row_bytes / rb : 1.0;
        const double sb = (std::isfinite(rb) && rb > 0) ? (double)b_row / rb : 1.0;
        t_ex = pb * ((double)f.recv_rows * sf + (double)b.recv_rows * sb);
      } else if (strategy == GT_AUTO && fits > 0) {
        // measure the forward and backward exchanges of this pattern (2 warm-up + 3 timed)
        DevBuf sb, rf, rb;
        int64_t sbytes = std::max({(int64_t)f.send_idx.size() * P->kv_row_bytes,
                                   P->bwd_reduce ? f.recv_rows * rs_bytes : (int64_t)b.send_idx.size() * P->in_row_bytes,
                                   c == GT_ALLGATHER ? P->n_max * P->in_row_bytes : 0, (int64_t)16});
        GT_TRY(sb.alloc((size_t)sbytes));
        GT_TRY(rf.alloc((size_t)std::max<int64_t>(f.recv_rows * P->kv_row_bytes, 16)));
        GT_TRY(rb.alloc((size_t)std::max<int64_t>(b.recv_rows * b_row, 16)));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float ms_best = 1e30f;
        for (int it = 0; it < 5; ++it) {
          GT_TRY(P->comm->barrier(st));
          cudaEventRecord(e0, st);
          if (c == GT_ALLGATHER) GT_TRY(P->comm->all_gather(sb.p, rf.p, P->n_max, P->kv_row_bytes, st));
          else
            GT_TRY(P->comm->exchange(sb.p, f.send_off.data(), f.send_cnt.data(), rf.p, f.recv_off.data(),
                                     f.recv_cnt.data(), P->kv_row_bytes, st));
          if (c == GT_ALLGATHER && !P->bwd_reduce)
            GT_TRY(P->comm->all_gather(sb.p, rb.p, P->n_max, P->in_row_bytes, st));
          else
            GT_TRY(P->comm->exchange(sb.p, b.send_off.data(), b.send_cnt.data(), rb.p, b.recv_off.data(),
                                     b.recv_cnt.data(), b_row, st));
          cudaEventRecord(e1, st);
          GT_CUDA_TRY(cudaEventSynchronize(e1));
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          if (it >= 2) ms_best = std::min(ms_best, ms);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        t_ex = ms_best * 1e-3;
        GT_TRY(P->comm->max_host(&t_ex, st));
      }
      double rows = (double)(f.recv_rows + b.recv_rows);
      P->info.beta_s_per_row[c] = std::isfinite(t_ex) && rows > 0 ? t_ex / rows : 0.0;
      P->info.predicted_ms[c] = std::isfinite(t_ex) ? (t_compute + t_ex) * 1e3 : INFINITY;
      // Eq. 14 with beta_c * N replaced by the measured exchange time: p t_comm / (p - 1) <= t_iter(1)
      P->info.agp_score[c] = std::isfinite(t_ex) ? world * t_ex / (world - 1) * 1e3 : INFINITY;
      P->info.agp_feasible[c] = std::isfinite(t_ex) && world * t_ex / (world - 1) <= t_iter1;
      if (!fits && strategy == c) return fail(GT_ENOMEM, "gt_plan: strategy buffers do not fit in device memory");
    }
    P->info.predicted_ms[GT_SINGLE] = t_iter1 * 1e3;
    // GP-A2A (Alg. 2; Table 1 volume 8 N d / p): every rank does heads / world of all
    // the work; 4 all-to-alls of head groups per direction (Q, K, V in + Y out; dY in + dQ, dK, dV out)
    P->info.predicted_ms[GT_A2A] = INFINITY;
    P->info.agp_score[GT_A2A] = INFINITY;
    if (heads % world == 0 && shape_supported(heads / world, d, opts->dtype) &&
        (strategy == GT_AUTO || strategy == GT_A2A)) {
      const int64_t gb = (int64_t)(heads / world) * d * elt;
      const int64_t sub_bytes = nnz * (12 + (int64_t)(heads / world) * 12) + n * 40;   // graph + entry state
      const int64_t need = 9 * n * gb + 3 * P->n_max * D * elt + sub_bytes;
      size_t free_a = 0, total_a = 0;
      GT_CUDA_TRY(cudaMemGetInfo(&free_a, &total_a));
      double misfit = (double)need < 0.85 * (double)free_a ? 0.0 : 1.0;
      GT_TRY(P->comm->max_host(&misfit, st));
      if (misfit > 0 && strategy == GT_A2A) return fail(GT_ENOMEM, "gt_plan: GP-A2A buffers do not fit in device memory");
      const double pa = prof.empty() ? NAN : profile_beta(prof, "a2a", world);
      if (misfit == 0 && strategy == GT_AUTO && std::isfinite(pa)) {
        const double rb = profile_beta(prof, "row_bytes", world);  // head-group rows are gb bytes
        const double t_ex = pa * 8.0 * (double)(n - P->n_local) * ((std::isfinite(rb) && rb > 0) ? (double)gb / rb : 1.0);
        P->info.beta_s_per_row[GT_A2A] = pa;
        P->info.predicted_ms[GT_A2A] = (t_iter1 / world + t_ex) * 1e3;
        P->info.agp_score[GT_A2A] = world * t_ex / (world - 1) * 1e3;
        P->info.agp_feasible[GT_A2A] = world * t_ex / (world - 1) <= t_iter1;
      } else if (misfit == 0 && strategy == GT_AUTO) {
        std::vector<int64_t> loff(world), lcnt(world), goff(world), gcnt(world);
        for (int s = 0; s < world; ++s) {
          loff[s] = (int64_t)s * P->n_local;
          lcnt[s] = s == P->rank ? 0 : P->n_local;
          goff[s] = P->bounds[s];
          gcnt[s] = s == P->rank ? 0 : P->bounds[s + 1] - P->bounds[s];
        }
        DevBuf sb, rb;
        GT_TRY(sb.alloc((size_t)std::max<int64_t>(world * P->n_local * gb, 16)));
        GT_TRY(rb.alloc((size_t)std::max<int64_t>(n * gb, 16)));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float ms_best = 1e30f;
        for (int it = 0; it < 5; ++it) {
          GT_TRY(P->comm->barrier(st));
          cudaEventRecord(e0, st);
          for (int x = 0; x < 8; ++x)
            GT_TRY(P->comm->exchange(sb.p, loff.data(), lcnt.data(), rb.p, goff.data(), gcnt.data(), gb, st));
          cudaEventRecord(e1, st);
          GT_CUDA_TRY(cudaEventSynchronize(e1));
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          if (it >= 2) ms_best = std::min(ms_best, ms);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        double t_ex = ms_best * 1e-3;
        GT_TRY(P->comm->max_host(&t_ex, st));
        const double rows = 8.0 * (double)(n - P->n_local);
        P->info.beta_s_per_row[GT_A2A] = rows > 0 ? t_ex / rows : 0.0;
        P->info.predicted_ms[GT_A2A] = (t_iter1 / world + t_ex) * 1e3;
        P->info.agp_score[GT_A2A] = world * t_ex / (world - 1) * 1e3;
        P->info.agp_feasible[GT_A2A] = world * t_ex / (world - 1) <= t_iter1;
      }
    }
    if (strategy == GT_AUTO) {
      int32_t pick = P->info.predicted_ms[GT_HALO] < P->info.predicted_ms[GT_ALLGATHER] ? GT_HALO : GT_ALLGATHER;
      if (P->info.predicted_ms[GT_A2A] < P->info.predicted_ms[pick]) pick = GT_A2A;
      GT_TRY(P->comm->broadcast_host(&pick, sizeof(pick), st));  // rank 0 decides
      strategy = pick;
    }
    P->strategy = strategy;
  } else {
    P->strategy = GT_SINGLE;
    // ---- hot-column table (opts.hot_cols): the K||V rows of the most referenced columns, packed per
    // forward and read under a persisting L2 access-policy window; their CSR entries point into it ----
    if (opts->hot_cols > 0 && nnz > 0) {
      const int64_t H = std::min<int64_t>(opts->hot_cols, n);
      std::vector<int32_t> order((size_t)n);
      std::iota(order.begin(), order.end(), 0);
      std::partial_sort(order.begin(), order.begin() + H, order.end(), [&](int32_t a, int32_t b) {
        const int64_t da = col_ptr_full[a + 1] - col_ptr_full[a], db = col_ptr_full[b + 1] - col_ptr_full[b];
        return da != db ? da > db : a < b;
      });
      order.resize((size_t)H);
      std::vector<int32_t> slot((size_t)n, -1);
      for (int64_t x = 0; x < H; ++x) slot[(size_t)order[(size_t)x]] = (int32_t)x;
      std::vector<int32_t> cols((size_t)nnz);
      int64_t hits = 0;
      for (int64_t e = 0; e < nnz; ++e) {
        const int32_t j = csr->col_idx[e], sl = slot[(size_t)j];
        cols[(size_t)e] = sl >= 0 ? (int32_t)(n + sl) : j;
        hits += sl >= 0;
      }
      GT_TRY(upload(P->d_col, cols.data(), cols.size()));
      GT_TRY(upload(P->d_hot_idx, order.data(), order.size()));
      GT_TRY(P->d_hot.alloc((size_t)H * P->kv_row_bytes));
      P->n_hot = H;
      P->hot_entries = hits;
      int maxp = 0;
      GT_CUDA_TRY(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, P->device));
      if (maxp > 0)
        GT_CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize,
                                       (size_t)std::min<int64_t>(maxp, (int64_t)P->d_hot.bytes)));
    }
  }
  if (P->strategy == GT_A2A) {
    GT_TRY(build_a2a(P.get(), csr, n, nnz, d, opts));
    fill_info(P.get(), 0, 0);
    *out = P.release();
    return GT_OK;
  }

  // ---- remapped local CSR columns and CSC rows ----
  std::vector<int32_t> cols;  // remapped local CSR columns (kept for the reduce-scatter halo columns)
  if (!single) {
    const bool ag = P->strategy == GT_ALLGATHER;
    cols.assign(csr->col_idx + csr->row_ptr[P->lo], csr->col_idx + csr->row_ptr[P->hi]);
    P->peer = opts->transport == 1 && P->strategy != GT_A2A;
    if (P->peer) {  // remote column j -> n_local + (owner << shift) + (j - bounds[owner])
      while ((int64_t(1) << P->peer_shift) < std::max<int64_t>(P->n_max, 2)) ++P->peer_shift;
      if (P->n_local + ((int64_t)world << P->peer_shift) >= (int64_t(1) << 31))
        return fail(GT_ECONFIG, "gt_plan: peer-gather ids do not fit in 32 bits");
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < (int64_t)cols.size(); ++e) {
        const int64_t j = cols[(size_t)e];
        if (j >= P->lo && j < P->hi) {
          cols[(size_t)e] = (int32_t)(j - P->lo);
        } else {
          const int o = owner_of(P->bounds, j);
          cols[(size_t)e] = (int32_t)(P->n_local + ((int64_t)o << P->peer_shift) + (j - P->bounds[o]));
        }
      }
    } else {
      remap_ids(cols.data(), (int64_t)cols.size(), P.get(), P->halo_out, ag);
    }
    GT_TRY(upload(P->d_col, cols.data(), cols.size()));
    std::vector<int32_t> rows((size_t)P->nnz_in_local);
    if (P->nnz_in_local)
      GT_CUDA_TRY(cudaMemcpy(rows.data(), full_row.as<int32_t>() + c0, rows.size() * sizeof(int32_t),
                             cudaMemcpyDeviceToHost));
    if (P->peer) {  // remote row i -> n_local + (owner << shift) + (i - bounds[owner])
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < (int64_t)rows.size(); ++e) {
        const int64_t i = rows[(size_t)e];
        if (i >= P->lo && i < P->hi) {
          rows[(size_t)e] = (int32_t)(i - P->lo);
        } else {
          const int o = owner_of(P->bounds, i);
          rows[(size_t)e] = (int32_t)(P->n_local + ((int64_t)o << P->peer_shift) + (i - P->bounds[o]));
        }
      }
    } else {
      remap_ids(rows.data(), (int64_t)rows.size(), P.get(), P->halo_in, ag);
    }
    GT_TRY(upload(P->d_row, rows.data(), rows.size()));
    GT_TRY(upload(P->d_col_ptr, P->h_col_ptr.data(), P->h_col_ptr.size()));
    const Pattern& f = ag ? pf_ag : pf_halo;
    const Pattern& b = ag ? pb_ag : pb_halo;
    P->so_off = f.send_off; P->so_cnt = f.send_cnt; P->ro_off = f.recv_off; P->ro_cnt = f.recv_cnt;
    P->si_off = b.send_off; P->si_cnt = b.send_cnt; P->ri_off = b.recv_off; P->ri_cnt = b.recv_cnt;
    P->halo_out_rows = f.recv_rows;
    P->halo_in_rows = b.recv_rows;
    P->n_send_out = (int64_t)f.send_idx.size();
    P->n_send_in = (int64_t)b.send_idx.size();
    GT_TRY(upload(P->d_send_out_idx, f.send_idx.data(), f.send_idx.size()));
    GT_TRY(upload(P->d_send_in_idx, b.send_idx.data(), b.send_idx.size()));
    int64_t sbytes = std::max((int64_t)f.send_idx.size(), (int64_t)b.send_idx.size()) * P->kv_row_bytes;
    if (ag) sbytes = P->n_max * P->kv_row_bytes;
    GT_TRY(P->d_send_buf.alloc((size_t)std::max<int64_t>(sbytes, 16)));
    if (P->peer) {
      GT_TRY(P->d_pub.alloc((size_t)std::max<int64_t>(P->n_local, 1) * P->kv_row_bytes));
      std::vector<int32_t> iota((size_t)P->n_local);
      std::iota(iota.begin(), iota.end(), 0);
      GT_TRY(upload(P->d_iota, iota.data(), iota.size()));
      GT_TRY(P->comm->share_pointers(P->d_pub.p, P->peer_base, st));
      GT_TRY(P->d_pub_qd.alloc((size_t)std::max<int64_t>(P->n_local, 1) * P->kv_row_bytes));
      GT_TRY(P->comm->share_pointers(P->d_pub_qd.p, P->peer_qd, st));
      GT_TRY(P->d_recv_kv.alloc(16));
    } else {
      GT_TRY(P->d_recv_kv.alloc((size_t)std::max<int64_t>(f.recv_rows * P->kv_row_bytes, 16)));
    }
    if (!P->bwd_reduce && !P->peer) {  // transposed-owner backward: [q | dy] and (LSE2, D) rows of the in-halo
      GT_TRY(P->d_recv_qd.alloc((size_t)std::max<int64_t>(b.recv_rows * P->kv_row_bytes, 16)));
      GT_TRY(P->d_recv_st.alloc((size_t)std::max<int64_t>(b.recv_rows * P->st_row_bytes, 16)));
      GT_TRY(P->d_send_st.alloc((size_t)std::max<int64_t>((ag ? P->n_max : (int64_t)b.send_idx.size()) * P->st_row_bytes, 16)));
    }
    GT_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_bwd0, cudaEventDisableTiming));
    GT_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_rows, cudaEventDisableTiming));
    GT_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_side, cudaEventDisableTiming));
    int64_t recv_f = 0, recv_b = 0, send_f = 0, send_b = 0;
    for (int s = 0; s < world; ++s) {
      if (s == P->rank) continue;
      recv_f += f.recv_cnt[s]; recv_b += b.recv_cnt[s];
      send_f += f.send_cnt[s]; send_b += b.send_cnt[s];
    }
    P->info.exch_fwd_bytes = recv_f * P->kv_row_bytes;
    P->info.exch_bwd_bytes = recv_b * P->in_row_bytes;
    P->info.send_fwd_bytes = send_f * P->kv_row_bytes;
    P->info.send_bwd_bytes = send_b * P->in_row_bytes;
    if (P->bwd_reduce) {
      const Pattern rev = reverse_pattern(P.get(), f, ag);
      int64_t rs_recv = 0, rs_send = 0;
      for (int s = 0; s < world; ++s) {
        if (s == P->rank) continue;
        rs_recv += rev.recv_cnt[s];
        rs_send += rev.send_cnt[s];
      }
      P->info.exch_bwd_bytes = rs_recv * 2 * D * 4;
      P->info.send_bwd_bytes = rs_send * 2 * D * 4;
    }
  }

  // ---- degree binning and work lists (rows / columns split into chunks) ----
  {
    const int64_t T = P->heavy_threshold;
    build_work(P->n_local, [&](int64_t r, std::vector<Segment>& o) { o.push_back({rp_local[r], rp_local[r + 1], 0}); },
               T, 1, &P->w_rows, &P->heavy_rows);
    build_work(P->n_local,
               [&](int64_t c, std::vector<Segment>& o) { o.push_back({P->h_col_ptr[c], P->h_col_ptr[c + 1], 0}); }, T,
               1, &P->w_cols, &P->heavy_cols);
    if (!single) {
      // forward split: entries [e0, a) and [b, e1) of a row have remote columns (global column < lo or
      // >= hi; columns are sorted), [a, b) owned columns
      P->fwd_split = true;
      const int64_t lo = P->lo, hi = P->hi;
      build_work(P->n_local,
                 [&](int64_t r, std::vector<Segment>& o) {
                   const int64_t g0 = csr->row_ptr[lo + r], g1 = csr->row_ptr[lo + r + 1];
                   const int32_t* c0 = csr->col_idx + g0;
                   const int32_t* c1 = csr->col_idx + g1;
                   const int64_t a = std::lower_bound(c0, c1, (int32_t)lo) - c0;
                   const int64_t b = std::lower_bound(c0, c1, (int32_t)hi) - c0;
                   const int64_t base = rp_local[r];
                   o.push_back({base, base + a, 1});
                   o.push_back({base + a, base + b, 0});
                   o.push_back({base + b, base + (g1 - g0), 1});
                 },
                 T, 2, P->w_fwd, &P->fwd_chunks);
      GT_TRY(upload_chunks(P->fwd_chunks));
      for (auto* w : {&P->w_fwd[0], &P->w_fwd[1]}) GT_TRY(upload_work(*w));
      GT_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_fwd0, cudaEventDisableTiming));
      GT_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_halo, cudaEventDisableTiming));
    }
    // ---- materialised entry state (opts.edge_state) ----
    if (opts->edge_state < -1 || opts->edge_state > 1) return fail(GT_EINVAL, "gt_plan: edge_state must be -1, 0 or 1");
    if (opts->edge_state >= 0) {
      const char* lg = std::getenv("GT_ES_LOGITS");  // logits half of the state (A/B switch; default on)
      const bool logits = !(lg && lg[0] == '0');
      // per entry and head: the logit (f32) and (P, dS) (bf16x2 for bf16 plans, f32x2 for f32 plans)
      const int64_t pdb = P->dtype == GT_F32 ? 8 : 4;
      const int64_t es_bytes = P->nnz_local * heads * ((logits ? 4 : 0) + pdb) + P->nnz_in_local * 4;
      size_t free_b = 0, total_b = 0;
      GT_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
      double misfit = (double)es_bytes < 0.85 * (double)free_b ? 0.0 : 1.0;
      if (!single) GT_TRY(P->comm->max_host(&misfit, st));  // the column-pass split must agree across ranks
      if (misfit > 0 && opts->edge_state == 1) return fail(GT_ENOMEM, "gt_plan: entry state does not fit in device memory");
      P->es = misfit == 0;
      P->es_logits = P->es && logits;
      P->info.edge_state_bytes = P->es ? es_bytes : 0;
      const char* cf = std::getenv("GT_COLFIRST");  // backward order at world 1 (A/B switch; default column-first)
      P->colfirst = !(cf && cf[0] == '0');
    }
    if (P->es) {
      if (P->es_logits) GT_TRY(P->d_s2.alloc(std::max<size_t>((size_t)P->nnz_local, 1) * heads * sizeof(float)));
      GT_TRY(P->d_pd.alloc(std::max<size_t>((size_t)P->nnz_local, 1) * heads * (P->dtype == GT_F32 ? 8 : 4)));
      GT_TRY(P->d_src.alloc(std::max<size_t>((size_t)P->nnz_in_local, 1) * sizeof(int32_t)));
      GT_TRY(build_local_src(full_src.as<int32_t>(), c0, c1, csr->row_ptr[P->lo], csr->row_ptr[P->hi],
                             P->d_src.as<int32_t>(), st));
      if (!single && !P->bwd_reduce) {
        // column split: CSC rows ascend within a column, so entries [e0, a) and [b, e1) have remote
        // rows (global row < lo or >= hi), [a, b) owned rows
        P->col_split = true;
        std::vector<int32_t> grow((size_t)P->nnz_in_local);
        if (P->nnz_in_local)
          GT_CUDA_TRY(cudaMemcpy(grow.data(), full_row.as<int32_t>() + c0, grow.size() * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost));
        const int64_t lo = P->lo, hi = P->hi;
        build_work(P->n_local,
                   [&](int64_t c, std::vector<Segment>& o) {
                     const int64_t e0 = P->h_col_ptr[c], e1 = P->h_col_ptr[c + 1];
                     const int32_t* r0 = grow.data() + e0;
                     const int32_t* r1 = grow.data() + e1;
                     const int64_t a = std::lower_bound(r0, r1, (int32_t)lo) - r0;
                     const int64_t b = std::lower_bound(r0, r1, (int32_t)hi) - r0;
                     o.push_back({e0, e0 + a, 1});
                     o.push_back({e0 + a, e0 + b, 0});
                     o.push_back({e0 + b, e1, 1});
                   },
                   T, 2, P->w_colp, &P->col_chunks);
        GT_TRY(upload_chunks(P->col_chunks));
        for (auto* w : {&P->w_colp[0], &P->w_colp[1]}) GT_TRY(upload_work(*w));
      }
    }
    // ---- fp8 K||V table (opts.kv_fp8) ----
    if (opts->kv_fp8) {
      if (!P->es) return fail(GT_ECONFIG, "gt_plan: kv_fp8 needs the entry state, which does not fit");
      P->kv_fp8 = true;
      P->kv8_row = (2 * D + 8 * heads + 15) / 16 * 16;
      GT_TRY(P->d_kv8.alloc((size_t)std::max<int64_t>(P->n_local, 1) * P->kv8_row));
      GT_CUDA_TRY(cudaMemset(P->d_kv8.p, 0, P->d_kv8.bytes));   // row padding stays zero
      GT_TRY(P->d_kvref.alloc(2 * sizeof(int)));
    }
    // ---- reduce-scatter backward (opts.bwd_mode = 1) ----
    if (P->bwd_reduce) GT_TRY(build_reduce_backward(P.get(), csr, rp_local, cols, full_row, c0, ag_of(P.get()),
                                                    P->strategy == GT_ALLGATHER ? pf_ag : pf_halo, T, st));
    P->info.edge_state = P->es ? 1 : 0;
    GT_TRY(upload_chunks(P->heavy_rows));
    GT_TRY(upload_chunks(P->heavy_cols));
    GT_TRY(upload_work(P->w_rows));
    GT_TRY(upload_work(P->w_cols));
  }
  const int64_t nrc = P->heavy_rows.nchunks(), ncc = P->col_split ? P->col_chunks.nchunks() : P->heavy_cols.nchunks();
  const int64_t nfc = P->fwd_split ? P->fwd_chunks.nchunks() : nrc;
  GT_TRY(P->d_part_fwd.alloc((size_t)std::max<int64_t>(nfc, 1) * (D + 2 * heads) * sizeof(float)));
  GT_TRY(P->d_part_rowb.alloc((size_t)std::max<int64_t>(nrc, 1) * D * sizeof(float)));
  GT_TRY(P->d_part_colb.alloc((size_t)std::max<int64_t>(ncc, 1) * (2 * D) * sizeof(float)));
  GT_TRY(P->d_stats.alloc((size_t)std::max<int64_t>(P->n_local, 1) * P->stats_stride * sizeof(float)));
  if (P->peer) GT_TRY(P->comm->share_pointers(P->d_stats.p, P->peer_st, st));  // read by the peers' column pass
  GT_CUDA_TRY(cudaStreamSynchronize(st));

  fill_info(P.get(), nrc, ncc);
  *out = P.release();
  return GT_OK;
}

struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};

gt_status gt_plan(const gt_csr* csr, int64_t n, int64_t nnz, int heads, int d, int world, const gt_opts* opts,
                  gt_plan_t* out) {
  NvtxScope nvtx("gt_plan");
  gt_opts def;
  if (!opts) {
    gt_default_opts(&def);
    opts = &def;
  }
  try {
    return plan_impl(csr, n, nnz, heads, d, world, opts, out);
  } catch (const std::bad_alloc&) {
    return fail(GT_ENOMEM, "gt_plan: host allocation failed");
  } catch (...) {
    return fail(GT_EINVAL, "gt_plan: unexpected exception");
  }
}

gt_status gt_plan_info_get(gt_plan_t P, gt_plan_info* out) {
  if (!P || !out) return fail(GT_EINVAL, "gt_plan_info_get: null argument");
  *out = P->info;
  out->fwd_gen = (int64_t)P->fwd_gen;
  out->stale_bwds = P->stale_bwds;
  return GT_OK;
}

gt_status gt_plan_export(gt_plan_t P, int what, int peer, void* dst, int64_t cap, int64_t* len) {
  if (!P || !len) return fail(GT_EINVAL, "gt_plan_export: null argument");
  const void* src = nullptr;
  int64_t count = 0, esz = 4;
  std::vector<int32_t> tmp32;
  switch (what) {
    case GT_EXPORT_BOUNDS: src = P->bounds.data(); count = (int64_t)P->bounds.size(); esz = 8; break;
    case GT_EXPORT_HALO_OUT: src = P->halo_out.data(); count = (int64_t)P->halo_out.size(); break;
    case GT_EXPORT_HALO_IN: src = P->halo_in.data(); count = (int64_t)P->halo_in.size(); break;
    case GT_EXPORT_SEND_OUT:
    case GT_EXPORT_SEND_IN: {
      if (peer < 0 || peer >= P->world) return fail(GT_EINVAL, "gt_plan_export: bad peer");
      if (P->world > 1) {
        const auto& v = what == GT_EXPORT_SEND_OUT ? P->send_out[peer] : P->send_in[peer];
        src = v.data();
        count = (int64_t)v.size();
      }
      break;
    }
    case GT_EXPORT_CSC_PTR: src = P->h_col_ptr.data(); count = (int64_t)P->h_col_ptr.size(); esz = 8; break;
    case GT_EXPORT_CSC_IDX: {
      count = P->nnz_in_local;
      tmp32.resize((size_t)count);
      // GP-A2A keeps the CSC only in its full-graph plan (global row ids): the owned-column slice
      const int32_t* rows = P->sub ? P->sub->d_row.as<int32_t>() + P->csc_base : P->d_row.as<int32_t>();
      if (count) {
        cudaError_t e = cudaMemcpy(tmp32.data(), rows, (size_t)count * 4, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return fail(GT_ECUDA, cudaGetErrorString(e));
      }
      if (P->world > 1 && !P->sub) {  // undo the remap: report global row ids
        for (auto& x : tmp32) {
          int64_t i = x;
          if (i < P->n_local) x = (int32_t)(i + P->lo);
          else if (P->peer) {
            const int64_t slot = i - P->n_local;
            x = (int32_t)(P->bounds[slot >> P->peer_shift] + (slot & ((int64_t(1) << P->peer_shift) - 1)));
          } else if (P->strategy == GT_ALLGATHER) {
            int64_t s = (i - P->n_local) / P->n_max, off = (i - P->n_local) % P->n_max;
            x = (int32_t)(P->bounds[s] + off);
          } else {
            x = P->halo_in[i - P->n_local];
          }
        }
      }
      src = tmp32.data();
      break;
    }
    case GT_EXPORT_HEAVY_ROWS: src = P->heavy_rows.ids.data(); count = (int64_t)P->heavy_rows.ids.size(); break;
    case GT_EXPORT_HEAVY_COLS: src = P->heavy_cols.ids.data(); count = (int64_t)P->heavy_cols.ids.size(); break;
    case GT_EXPORT_KV8: {
      esz = 1;
      count = P->kv_fp8 ? P->n_local * P->kv8_row : 0;
      if (dst && count) {
        if (cap < count) return fail(GT_EINVAL, "gt_plan_export: cap too small");
        GT_CUDA_TRY(cudaDeviceSynchronize());
        GT_CUDA_TRY(cudaMemcpy(dst, P->d_kv8.p, (size_t)count, cudaMemcpyDeviceToHost));
      }
      *len = count;
      return GT_OK;
    }
    default: return fail(GT_EINVAL, "gt_plan_export: unknown table");
  }
  *len = count;
  if (dst) {
    if (cap < count) return fail(GT_EINVAL, "gt_plan_export: cap too small");
    if (count) std::memcpy(dst, src, (size_t)(count * esz));
  }
  return GT_OK;
}

static gt_status check_ptrs(gt_plan_t P, std::initializer_list<const void*> ps) {
  if (!P) return fail(GT_EINVAL, "null plan");
  if (P->n_local == 0) return GT_OK;
  for (const void* p : ps) {
    if (!p) return fail(GT_EINVAL, "null tensor pointer");
    if (((uintptr_t)p) & 15) return fail(GT_EINVAL, "tensor pointer not 16-byte aligned");
  }
  return GT_OK;
}

// K||V rows of the forward halo (pack + all-gather / all-to-all-v) on the side stream, ordered after the
// work already on `st`; ev_halo marks their arrival.  Collective.
static gt_status fwd_exchange(gt_plan_t P, const void* k, const void* v, cudaStream_t st) {
  const int elt = P->dtype == GT_F32 ? 4 : 2;
  const int64_t D = (int64_t)P->heads * P->d;
  cudaEvent_t ev2 = nullptr;
  GT_CUDA_TRY(cudaEventRecord(P->ev_fwd0, st));
  GT_CUDA_TRY(cudaStreamWaitEvent(P->side, P->ev_fwd0, 0));
  P->mark_begin(0, P->side, &ev2);
  GT_TRY(pack_kv(k, v, P->d_send_out_idx.as<int32_t>(), P->n_send_out, D, elt, P->d_send_buf.p, P->side));
  if (P->strategy == GT_ALLGATHER)
    GT_TRY(P->comm->all_gather(P->d_send_buf.p, P->d_recv_kv.p, P->n_max, P->kv_row_bytes, P->side));
  else
    GT_TRY(P->comm->exchange(P->d_send_buf.p, P->so_off.data(), P->so_cnt.data(), P->d_recv_kv.p, P->ro_off.data(),
                             P->ro_cnt.data(), P->kv_row_bytes, P->side));
  P->mark_end(0, P->side, ev2);
  GT_CUDA_TRY(cudaEventRecord(P->ev_halo, P->side));
  return GT_OK;
}

static void set_fwd_tag(gt_plan_t P, const void* q, const void* k, const void* v, const void* lse) {
  P->kv_tag[0] = k;
  P->kv_tag[1] = v;
  P->kv_valid = true;
  P->lg_tag[0] = q;
  P->lg_tag[1] = k;
  P->lg_tag[2] = v;
  P->lg_tag[3] = lse;
  P->lg_valid = true;
  P->slice_tag[0] = q;
  P->slice_tag[1] = k;
  P->slice_tag[2] = v;
  P->slice_valid = true;
  P->fwd_gen++;
}

// Records `ev` on `st`; under stream capture as an external event node, so that replaying the graph
// records it again (a plain record inside a capture only orders the captured work).
static gt_status record_external(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  GT_CUDA_TRY(cudaStreamIsCapturing(st, &cs));
  if (cs == cudaStreamCaptureStatusActive) GT_CUDA_TRY(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal));
  else GT_CUDA_TRY(cudaEventRecord(ev, st));
  return GT_OK;
}

// Which retained pieces belong to these tensors (gt_plan_s tags).
static bool logits_fresh(gt_plan_t P, const void* q, const void* k, const void* v, const void* lse) {
  return P->lg_valid && P->lg_tag[0] == q && P->lg_tag[1] == k && P->lg_tag[2] == v && P->lg_tag[3] == lse;
}
static bool kv_fresh(gt_plan_t P, const void* k, const void* v) {
  return P->kv_valid && P->kv_tag[0] == k && P->kv_tag[1] == v;
}
static bool slices_fresh(gt_plan_t P, const void* q, const void* k, const void* v) {
  return P->slice_valid && P->slice_tag[0] == q && P->slice_tag[1] == k && P->slice_tag[2] == v;
}

// fp8 K||V table (gt_opts.kv_fp8) of these k, v
static gt_status requantize(gt_plan_t P, const void* k, const void* v, cudaStream_t st) {
  GT_TRY(quantize_kv(P->heads, P->heads * P->d, k, v, P->n_local, P->d_kv8.p, (int)P->kv8_row,
                     P->d_kvref.as<int>(), st));
  P->kv8_tag[0] = k;
  P->kv8_tag[1] = v;
  return GT_OK;
}

// hot-column table (gt_opts.hot_cols) of these k, v
static gt_status repack_hot(gt_plan_t P, const void* k, const void* v, cudaStream_t st) {
  GT_TRY(pack_kv(k, v, P->d_hot_idx.as<int32_t>(), P->n_hot, (int64_t)P->heads * P->d, P->dtype == GT_F32 ? 4 : 2,
                 P->d_hot.p, st));
  P->hot_tag[0] = k;
  P->hot_tag[1] = v;
  return GT_OK;
}

static gt_status attn_fwd_eager(gt_plan_t P, const void* q, const void* k, const void* v, void* y, float* lse,
                                void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  GT_CUDA_TRY(cudaSetDevice(P->device));
  if (P->strategy == GT_A2A) {  // GP-A2A (Alg. 2): scatter Q, K, V by head group, all rows, gather Y, LSE
    const int64_t gb = (int64_t)P->heads_l * P->d * (P->dtype == GT_F32 ? 4 : 2);
    const int64_t lb = (int64_t)P->heads_l * 4;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    P->mark_begin(0, st, &e0);
    GT_TRY(a2a_scatter(P, q, gb, P->d_stage[0].p, P->d_hq.p, st));
    GT_TRY(a2a_scatter(P, k, gb, P->d_stage[1].p, P->d_hk.p, st));
    GT_TRY(a2a_scatter(P, v, gb, P->d_stage[2].p, P->d_hv.p, st));
    P->mark_end(0, st, e0);
    GT_TRY(gt_attn_fwd(P->sub, P->d_hq.p, P->d_hk.p, P->d_hv.p, P->d_hy.p, P->d_hlse.as<float>(), stream));
    P->mark_begin(0, st, &e1);
    GT_TRY(a2a_gather(P, P->d_hy.p, gb, P->d_stage[0].p, y, st));
    GT_TRY(a2a_gather(P, P->d_hlse.p, lb, P->d_stage[1].p, lse, st));
    P->mark_end(0, st, e1);
    set_fwd_tag(P, q, k, v, lse);
    return GT_OK;
  }
  const void* halo = nullptr;
  cudaEvent_t ev = nullptr;
  if (P->peer) {  // fused peer gather: no exchange, the kernels read remote rows from the owners
    P->mark_begin(1, st, &ev);
    GT_TRY(launch_fwd_peer(P, q, k, v, y, lse, st));
    P->mark_end(1, st, ev);
    set_fwd_tag(P, q, k, v, lse);
    return GT_OK;
  }
  if (P->world > 1) {
    // K||V rows of the halo on the side stream, overlapped with phase A (owned-column entries)
    GT_TRY(fwd_exchange(P, k, v, st));
    halo = P->d_recv_kv.p;
  }
  P->mark_begin(1, st, &ev);
  if (P->kv_fp8) GT_TRY(requantize(P, k, v, st));
  if (P->n_hot) {
    GT_TRY(repack_hot(P, k, v, st));
    halo = P->d_hot.p;
  }
  GT_TRY(launch_fwd(P, q, k, v, halo, y, lse, st, P->world > 1 ? P->ev_halo : nullptr));
  P->mark_end(1, st, ev);
  set_fwd_tag(P, q, k, v, lse);
  return GT_OK;
}

// fresh: the stored logits belong to this backward's (q, k, v, lse) (logits_fresh).  Retained rows /
// head slices that belong to other tensors are re-fetched (and re-tagged) here; stale logits are
// recomputed by the row pass instead of read.
static gt_status attn_bwd_eager(gt_plan_t P, const void* q, const void* k, const void* v, const void* y,
                                const float* lse, const void* dy, void* dq, void* dk, void* dv, void* stream,
                                bool fresh) {
  cudaStream_t st = (cudaStream_t)stream;
  GT_CUDA_TRY(cudaSetDevice(P->device));
  bool stale = !fresh && P->es_logits;
  if (P->strategy == GT_A2A) {  // GP-A2A: scatter dY and LSE, all rows for this rank's heads, gather grads
    const int64_t gb = (int64_t)P->heads_l * P->d * (P->dtype == GT_F32 ? 4 : 2);
    const int64_t lb = (int64_t)P->heads_l * 4;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    P->mark_begin(3, st, &e0);
    if (!slices_fresh(P, q, k, v)) {  // the head slices belong to other tensors: scatter these
      GT_TRY(a2a_scatter(P, q, gb, P->d_stage[0].p, P->d_hq.p, st));
      GT_TRY(a2a_scatter(P, k, gb, P->d_stage[1].p, P->d_hk.p, st));
      GT_TRY(a2a_scatter(P, v, gb, P->d_stage[2].p, P->d_hv.p, st));
      P->slice_tag[0] = q;
      P->slice_tag[1] = k;
      P->slice_tag[2] = v;
      P->slice_valid = true;
      stale = true;
    }
    // the sub-plan's stored logits are those of the last forward through this plan
    if (!fresh) P->sub->lg_valid = false;
    stale = stale || !fresh;
    if (stale) P->stale_bwds++;
    GT_TRY(a2a_scatter(P, dy, gb, P->d_stage[0].p, P->d_hdy.p, st));
    GT_TRY(a2a_scatter(P, y, gb, P->d_stage[2].p, P->d_hy.p, st));
    GT_TRY(a2a_scatter(P, lse, lb, P->d_stage[1].p, P->d_hlse.p, st));
    P->mark_end(3, st, e0);
    GT_TRY(gt_attn_bwd(P->sub, P->d_hq.p, P->d_hk.p, P->d_hv.p, P->d_hy.p, P->d_hlse.as<float>(), P->d_hdy.p,
                       P->d_hdq.p, P->d_hdk.p, P->d_hdv.p, stream));
    P->mark_begin(3, st, &e1);
    GT_TRY(a2a_gather(P, P->d_hdq.p, gb, P->d_stage[0].p, dq, st));
    GT_TRY(a2a_gather(P, P->d_hdk.p, gb, P->d_stage[1].p, dk, st));
    GT_TRY(a2a_gather(P, P->d_hdv.p, gb, P->d_stage[2].p, dv, st));
    P->mark_end(3, st, e1);
    return GT_OK;
  }
  // remote K || V rows: the received table, or (peer gather) the owners' published rows; world 1 with
  // gt_opts.hot_cols: the hot-column table (re-packed when it holds another forward's k, v)
  const void* halo_kv = P->world > 1 ? (P->peer ? P->d_pub.p : P->d_recv_kv.p) : (P->n_hot ? P->d_hot.p : nullptr);
  if (P->n_hot && (P->hot_tag[0] != k || P->hot_tag[1] != v)) {
    GT_TRY(repack_hot(P, k, v, st));
    if (!fresh) stale = true;
  }
  cudaEvent_t ev = nullptr, ev2 = nullptr;
  const bool multi = P->world > 1;
  const bool ag = P->strategy == GT_ALLGATHER;
  if (multi && !kv_fresh(P, k, v)) {
    stale = true;
    P->kv_tag[0] = k;
    P->kv_tag[1] = v;
    P->kv_valid = true;
    if (P->peer) {  // publish these k, v once every peer is done with the rows published before
      const int elt = P->dtype == GT_F32 ? 4 : 2;
      GT_TRY(P->comm->stream_barrier(st));
      GT_TRY(pack_kv(k, v, P->d_iota.as<int32_t>(), P->n_local, (int64_t)P->heads * P->d, elt, P->d_pub.p, st));
    } else {        // the forward's exchange again, for these k, v
      GT_TRY(fwd_exchange(P, k, v, st));
      GT_CUDA_TRY(cudaStreamWaitEvent(st, P->ev_halo, 0));
    }
  }
  if (P->kv_fp8 && (P->kv8_tag[0] != k || P->kv8_tag[1] != v)) {  // the table holds another forward's k, v
    GT_TRY(requantize(P, k, v, st));
    stale = true;
  }
  if (stale) P->stale_bwds++;
  if (multi && P->bwd_reduce) {
    // Reduce-scatter backward (reading Z11): row pass; fp32 partials of the halo columns, sent to their
    // owners on the side stream while the owned columns run; then the fixed-order merge.
    P->mark_begin(2, st, &ev);
    GT_TRY(launch_bwd_rows(P, q, k, v, y, halo_kv, lse, dy, dq, st, fresh));
    if (P->ev_dq_ready) GT_TRY(record_external(P->ev_dq_ready, st));
    GT_TRY(launch_bwd_halo_cols(P, q, dy, st));
    P->mark_end(2, st, ev);
    GT_CUDA_TRY(cudaEventRecord(P->ev_rows, st));
    GT_CUDA_TRY(cudaStreamWaitEvent(P->side, P->ev_rows, 0));
    P->mark_begin(3, P->side, &ev2);
    char* recv = (char*)P->d_part_rs.p + P->rs_chunks.nchunks() * P->rs_row_bytes;
    GT_TRY(P->comm->exchange(P->d_rs_send.p, P->rs_send_off.data(), P->rs_send_cnt.data(), recv,
                             P->rs_recv_off.data(), P->rs_recv_cnt.data(), P->rs_row_bytes, P->side));
    P->mark_end(3, P->side, ev2);
    GT_CUDA_TRY(cudaEventRecord(P->ev_side, P->side));
    P->mark_begin(4, st, &ev);
    GT_TRY(launch_bwd_cols_rs(P, q, k, v, dy, dk, dv, st, P->ev_side));
    P->mark_end(4, st, ev);
    return GT_OK;
  }
  if (multi && P->peer) {
    // Fused peer gather, backward: publish [q | dy] (known at entry) once every peer is done with the
    // previous step's rows, row pass (its (LSE2, D) stats are read in place by the peers), owned-row
    // column entries, a device-side barrier, then the remote-row column entries read from the owners.
    const int elt = P->dtype == GT_F32 ? 4 : 2;
    P->mark_begin(2, st, &ev);
    GT_TRY(P->comm->stream_barrier(st));
    GT_TRY(pack_kv(q, dy, P->d_iota.as<int32_t>(), P->n_local, (int64_t)P->heads * P->d, elt, P->d_pub_qd.p, st));
    GT_TRY(launch_bwd_rows(P, q, k, v, y, halo_kv, lse, dy, dq, st, fresh));
    if (P->ev_dq_ready) GT_TRY(record_external(P->ev_dq_ready, st));
    P->mark_end(2, st, ev);
    P->mark_begin(4, st, &ev);
    GT_TRY(launch_bwd_cols_peer(P, q, k, v, dy, dk, dv, st));
    P->mark_end(4, st, ev);
    return GT_OK;
  }
  if (!multi && P->colfirst && P->es_logits && fresh && !stale && !P->kv_fp8 && !P->n_hot &&
      P->heads * (P->dtype == GT_F32 ? 4 : 2) >= 4) {
    // Column-first order (world 1, this forward's logits stored): the column pass computes dP with its own
    // v_j and stores dS, so the row pass gathers k_j alone (2 KB -> 1.5 KB of gathered rows per entry)
    P->mark_begin(4, st, &ev);
    GT_TRY(launch_bwd_cf_cols(P, q, k, v, y, lse, dy, dk, dv, st));
    P->mark_end(4, st, ev);
    P->mark_begin(2, st, &ev);
    GT_TRY(launch_bwd_cf_rows(P, q, k, v, lse, dy, dq, st));
    if (P->ev_dq_ready) GT_TRY(record_external(P->ev_dq_ready, st));
    P->mark_end(2, st, ev);
    return GT_OK;
  }
  if (multi) {
    // Side stream, overlapped with the row pass: [q | dy] rows of the in-halo are known at entry.
    // Both messages go on the side stream so the communicator sees one ordered sequence.
    const int elt = P->dtype == GT_F32 ? 4 : 2;
    const int64_t D = (int64_t)P->heads * P->d;
    GT_CUDA_TRY(cudaEventRecord(P->ev_bwd0, st));
    GT_CUDA_TRY(cudaStreamWaitEvent(P->side, P->ev_bwd0, 0));
    P->mark_begin(3, P->side, &ev2);
    GT_TRY(pack_kv(q, dy, P->d_send_in_idx.as<int32_t>(), P->n_send_in, D, elt, P->d_send_buf.p, P->side));
    if (ag)
      GT_TRY(P->comm->all_gather(P->d_send_buf.p, P->d_recv_qd.p, P->n_max, P->kv_row_bytes, P->side));
    else
      GT_TRY(P->comm->exchange(P->d_send_buf.p, P->si_off.data(), P->si_cnt.data(), P->d_recv_qd.p,
                               P->ri_off.data(), P->ri_cnt.data(), P->kv_row_bytes, P->side));
    P->mark_end(3, P->side, ev2);
  }
  P->mark_begin(2, st, &ev);
  GT_TRY(launch_bwd_rows(P, q, k, v, y, halo_kv, lse, dy, dq, st, fresh));
  if (P->ev_dq_ready) GT_TRY(record_external(P->ev_dq_ready, st));
  P->mark_end(2, st, ev);
  if (multi) {
    // (LSE2, D) blocks of the in-halo rows: written by the row pass on their owners
    GT_CUDA_TRY(cudaEventRecord(P->ev_rows, st));
    GT_CUDA_TRY(cudaStreamWaitEvent(P->side, P->ev_rows, 0));
    P->mark_begin(3, P->side, &ev2);
    GT_TRY(pack_stats(P->d_stats.as<float>(), P->d_send_in_idx.as<int32_t>(), P->n_send_in, P->st_row_bytes,
                      P->d_send_st.p, P->side));
    if (ag)
      GT_TRY(P->comm->all_gather(P->d_send_st.p, P->d_recv_st.p, P->n_max, P->st_row_bytes, P->side));
    else
      GT_TRY(P->comm->exchange(P->d_send_st.p, P->si_off.data(), P->si_cnt.data(), P->d_recv_st.p,
                               P->ri_off.data(), P->ri_cnt.data(), P->st_row_bytes, P->side));
    P->mark_end(3, P->side, ev2);
    GT_CUDA_TRY(cudaEventRecord(P->ev_side, P->side));
    if (!P->col_split) GT_CUDA_TRY(cudaStreamWaitEvent(st, P->ev_side, 0));
  }
  P->mark_begin(4, st, &ev);
  GT_TRY(launch_bwd_cols(P, q, k, v, dy, multi ? P->d_recv_qd.p : nullptr, multi ? P->d_recv_st.p : nullptr, dk,
                         dv, st, multi ? P->ev_side : nullptr));
  P->mark_end(4, st, ev);
  return GT_OK;
}

// CUDA-graph replay of a world-1 plan's launch sequence (gt_opts.cuda_graphs): the first call of a
// direction runs eagerly (kernel attributes, grid sizes), later calls are captured once per set of
// tensor pointers and replayed (a few launches instead of ~10 driver calls; helps small graphs,
// whose steps are launch-bound).  Not used for the legacy default stream, with profiling, or when
// world > 1 (host-side protocol steps).
static bool graph_ok(gt_plan_t P, cudaStream_t st, bool warm) {
  return P->graphs && P->world == 1 && !P->profile && warm && st != nullptr && st != cudaStreamLegacy &&
         st != cudaStreamPerThread;
}

}  // extern "C" (the template below has C++ linkage)
template <typename F>
static gt_status graph_run(gt_plan_t P, std::vector<gt_plan_s::GraphEntry>& cache, const gt_plan_s::GraphKey& key,
                           cudaStream_t st, F&& eager) {
  for (auto& e : cache)
    if (e.key == key) {
      GT_CUDA_TRY(cudaGraphLaunch(e.exec, st));
      return GT_OK;
    }
  cudaGraph_t g = nullptr;
  GT_CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const gt_status s = eager();
  const cudaError_t ce = cudaStreamEndCapture(st, &g);
  if (s != GT_OK) {
    if (g) cudaGraphDestroy(g);
    return s;
  }
  if (ce != cudaSuccess) return fail(GT_ECUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(ce));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  if (ie != cudaSuccess) return fail(GT_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ie));
  if (cache.size() >= 4) {  // a few pointer sets (allocator reuse makes steps repeat them)
    cudaGraphExecDestroy(cache.front().exec);
    cache.erase(cache.begin());
  }
  cache.push_back({key, exec});
  GT_CUDA_TRY(cudaGraphLaunch(exec, st));
  return GT_OK;
}
extern "C" {

gt_status gt_attn_fwd(gt_plan_t P, const void* q, const void* k, const void* v, void* y, float* lse, void* stream) {
  NvtxScope nvtx("gt_attn_fwd");
  GT_TRY(check_ptrs(P, {q, k, v, y, lse}));
  cudaStream_t st = (cudaStream_t)stream;
  if (graph_ok(P, st, P->fwd_warm)) {
    GT_CUDA_TRY(cudaSetDevice(P->device));
    const gt_plan_s::GraphKey key = {q, k, v, y, lse, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    GT_TRY(graph_run(P, P->gfwd, key, st, [&] { return attn_fwd_eager(P, q, k, v, y, lse, stream); }));
    set_fwd_tag(P, q, k, v, lse);
    return GT_OK;
  }
  GT_TRY(attn_fwd_eager(P, q, k, v, y, lse, stream));
  P->fwd_warm = true;
  return GT_OK;
}

gt_status gt_attn_bwd(gt_plan_t P, const void* q, const void* k, const void* v, const void* y, const float* lse,
                      const void* dy, void* dq, void* dk, void* dv, void* stream) {
  NvtxScope nvtx("gt_attn_bwd");
  GT_TRY(check_ptrs(P, {q, k, v, y, lse, dy, dq, dk, dv}));
  const bool fresh = logits_fresh(P, q, k, v, lse);
  cudaStream_t st = (cudaStream_t)stream;
  if (graph_ok(P, st, P->bwd_warm)) {
    GT_CUDA_TRY(cudaSetDevice(P->device));
    const gt_plan_s::GraphKey key = {q, k, v, y, lse, dy, dq, dk, dv, P->ev_dq_ready,
                                     fresh ? (const void*)1 : nullptr};
    return graph_run(P, P->gbwd, key, st,
                     [&] { return attn_bwd_eager(P, q, k, v, y, lse, dy, dq, dk, dv, stream, fresh); });
  }
  GT_TRY(attn_bwd_eager(P, q, k, v, y, lse, dy, dq, dk, dv, stream, fresh));
  P->bwd_warm = true;
  return GT_OK;
}

}  // extern "C"

// Chunk bounds of a work list for the streamed host path: C contiguous ranges of about equal entry
// counts, cut only at items of whole rows (columns) so a heavy row's chunks stay in one range;
// t = item bounds, r = row (column) bounds, h = bounds in the heavy ids of `ct`.
static void stream_bounds(const WorkList& w, const ChunkTable& ct, int64_t n_local, int C, std::vector<int64_t>& t,
                          std::vector<int64_t>& r, std::vector<int64_t>& h) {
  t.assign(1, 0);
  r.assign(1, 0);
  const int64_t E = w.n ? w.end[(size_t)w.n - 1] - w.beg[0] : 0;
  int64_t x = 0;
  for (int c = 1; c < C && w.n; ++c) {
    const int64_t target = w.beg[0] + E * c / C;
    x = std::max<int64_t>(x, t.back() + 1);
    while (x < w.n && (w.beg[(size_t)x] < target || w.own[(size_t)x] < 0)) ++x;
    if (x >= w.n) break;
    t.push_back(x);
    r.push_back(w.own[(size_t)x]);
  }
  t.push_back(w.n);
  r.push_back(n_local);
  h.clear();
  for (int64_t b : r) h.push_back(std::lower_bound(ct.ids.begin(), ct.ids.end(), (int32_t)b) - ct.ids.begin());
}

// World-1 gt_attn_fwd_bwd_host, streamed in C row (column) chunks so that the host<->device copies
// overlap the passes and each other (PCIe is full duplex): K, V go in first; then Q chunk c feeds
// forward chunk c, whose Y / LSE rows leave at once; dY chunk c feeds row-pass chunk c, whose dQ rows
// leave at once; the column pass (it needs every row's (P, dS)) runs in column chunks whose dK / dV
// rows leave as they finish.  The arithmetic is that of gt_attn_fwd + gt_attn_bwd.
static gt_status fwd_bwd_host_streamed(gt_plan_t P, const void* q, const void* k, const void* v, const void* dy,
                                       void* y, float* lse, void* dq, void* dk, void* dv, cudaStream_t st) {
  const int elt = P->dtype == GT_F32 ? 4 : 2;
  const int64_t rb = (int64_t)P->heads * P->d * elt, lb = (int64_t)P->heads * 4;
  if (!P->e2e_c) {
    const char* env = std::getenv("GT_E2E_CHUNKS");
    P->e2e_c = std::max(1, std::min(64, env ? std::atoi(env) : 8));
    stream_bounds(P->w_rows, P->heavy_rows, P->n_local, P->e2e_c, P->e2e_t[0], P->e2e_r[0], P->e2e_h[0]);
    stream_bounds(P->w_cols, P->heavy_cols, P->n_local, P->e2e_c, P->e2e_t[1], P->e2e_r[1], P->e2e_h[1]);
    P->e2e_cev.assign(4 * (size_t)P->e2e_c + 4, nullptr);
    for (auto& e : P->e2e_cev) GT_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const int Cr = (int)P->e2e_t[0].size() - 1, Cc = (int)P->e2e_t[1].size() - 1;
  const auto& R = P->e2e_r[0];
  const auto& Rc = P->e2e_r[1];
  cudaEvent_t* ev = P->e2e_cev.data();            // [0, C) q in, [C, 2C) dy in, [2C, 3C) fwd, [3C, 4C) row pass
  cudaEvent_t ev_start = P->e2e_ev[0], ev_kv = P->e2e_ev[1];
  const int C = P->e2e_c;
  char* q_d = (char*)P->h2d[0].p;
  char* k_d = (char*)P->h2d[1].p;
  char* v_d = (char*)P->h2d[2].p;
  char* dy_d = (char*)P->h2d[3].p;
  char* y_d = (char*)P->h2d[4].p;
  float* lse_d = P->h2d[5].as<float>();
  char* dq_d = (char*)P->h2d[6].p;
  char* dk_d = (char*)P->h2d[7].p;
  char* dv_d = (char*)P->h2d[8].p;
  auto h2d = [&](char* dst, const void* src, int64_t r0, int64_t r1, int64_t row) -> gt_status {
    if (r1 > r0)
      GT_CUDA_TRY(cudaMemcpyAsync(dst + r0 * row, (const char*)src + r0 * row, (size_t)((r1 - r0) * row),
                                  cudaMemcpyHostToDevice, P->e2e_in));
    return GT_OK;
  };
  auto d2h = [&](void* dst, const char* src, int64_t r0, int64_t r1, int64_t row) -> gt_status {
    if (dst && r1 > r0)
      GT_CUDA_TRY(cudaMemcpyAsync((char*)dst + r0 * row, src + r0 * row, (size_t)((r1 - r0) * row),
                                  cudaMemcpyDeviceToHost, P->e2e_out));
    return GT_OK;
  };
  GT_CUDA_TRY(cudaEventRecord(ev_start, st));  // staging buffers are free once earlier work on `st` is done
  GT_CUDA_TRY(cudaStreamWaitEvent(P->e2e_in, ev_start, 0));
  GT_CUDA_TRY(cudaStreamWaitEvent(P->e2e_out, ev_start, 0));
  GT_TRY(h2d(k_d, k, 0, P->n_local, rb));
  GT_TRY(h2d(v_d, v, 0, P->n_local, rb));
  GT_CUDA_TRY(cudaEventRecord(ev_kv, P->e2e_in));
  for (int c = 0; c < Cr; ++c) {
    GT_TRY(h2d(q_d, q, R[c], R[c + 1], rb));
    GT_CUDA_TRY(cudaEventRecord(ev[c], P->e2e_in));
  }
  for (int c = 0; c < Cr; ++c) {
    GT_TRY(h2d(dy_d, dy, R[c], R[c + 1], rb));
    GT_CUDA_TRY(cudaEventRecord(ev[C + c], P->e2e_in));
  }
  // forward, in row chunks
  GT_CUDA_TRY(cudaStreamWaitEvent(st, ev_kv, 0));
  if (P->kv_fp8) GT_TRY(requantize(P, k_d, v_d, st));
  if (P->n_hot) GT_TRY(repack_hot(P, k_d, v_d, st));
  for (int c = 0; c < Cr; ++c) {
    GT_CUDA_TRY(cudaStreamWaitEvent(st, ev[c], 0));
    GT_TRY(launch_pass_range(P, 0, q_d, k_d, v_d, nullptr, lse_d, nullptr, y_d, nullptr, st, P->e2e_t[0][c],
                             P->e2e_t[0][c + 1], P->e2e_h[0][c], P->e2e_h[0][c + 1], c == 0));
    GT_CUDA_TRY(cudaEventRecord(ev[2 * C + c], st));
  }
  set_fwd_tag(P, q_d, k_d, v_d, lse_d);
  // row pass, in row chunks
  for (int c = 0; c < Cr; ++c) {
    GT_CUDA_TRY(cudaStreamWaitEvent(st, ev[C + c], 0));
    GT_TRY(launch_pass_range(P, 1, q_d, k_d, v_d, y_d, lse_d, dy_d, dq_d, nullptr, st, P->e2e_t[0][c], P->e2e_t[0][c + 1],
                             P->e2e_h[0][c], P->e2e_h[0][c + 1], c == 0));
    GT_CUDA_TRY(cudaEventRecord(ev[3 * C + c], st));
  }
  // outputs of the forward and the row pass leave while the column pass runs
  for (int c = 0; c < Cr; ++c) {
    GT_CUDA_TRY(cudaStreamWaitEvent(P->e2e_out, ev[2 * C + c], 0));
    GT_TRY(d2h(y, y_d, R[c], R[c + 1], rb));
    GT_TRY(d2h(lse, (const char*)lse_d, R[c], R[c + 1], lb));
  }
  for (int c = 0; c < Cr; ++c) {
    GT_CUDA_TRY(cudaStreamWaitEvent(P->e2e_out, ev[3 * C + c], 0));
    GT_TRY(d2h(dq, dq_d, R[c], R[c + 1], rb));
  }
  // column pass, in column chunks (reusing the forward's events, whose waits are already enqueued)
  for (int c = 0; c < Cc; ++c) {
    GT_TRY(launch_pass_range(P, 2, q_d, k_d, v_d, nullptr, nullptr, dy_d, dk_d, dv_d, st, P->e2e_t[1][c],
                             P->e2e_t[1][c + 1], P->e2e_h[1][c], P->e2e_h[1][c + 1], c == 0));
    GT_CUDA_TRY(cudaEventRecord(ev[4 * C + (c & 3)], st));
    GT_CUDA_TRY(cudaStreamWaitEvent(P->e2e_out, ev[4 * C + (c & 3)], 0));
    GT_TRY(d2h(dk, dk_d, Rc[c], Rc[c + 1], rb));
    GT_TRY(d2h(dv, dv_d, Rc[c], Rc[c + 1], rb));
  }
  GT_CUDA_TRY(cudaStreamSynchronize(P->e2e_out));
  GT_CUDA_TRY(cudaStreamSynchronize(st));
  return GT_OK;
}

extern "C" {

gt_status gt_attn_fwd_bwd_host(gt_plan_t P, const void* q, const void* k, const void* v, const void* dy, void* y,
                               float* lse, void* dq, void* dk, void* dv, void* stream) {
  if (!P || !q || !k || !v || !dy) return fail(GT_EINVAL, "gt_attn_fwd_bwd_host: null input");
  cudaStream_t st = (cudaStream_t)stream;
  GT_CUDA_TRY(cudaSetDevice(P->device));
  const int elt = P->dtype == GT_F32 ? 4 : 2;
  const size_t tb = (size_t)std::max<int64_t>(P->n_local, 1) * P->heads * P->d * elt;
  const size_t lb = (size_t)std::max<int64_t>(P->n_local, 1) * P->heads * sizeof(float);
  // staging: 0 q, 1 k, 2 v, 3 dy, 4 y, 5 lse, 6 dq, 7 dk, 8 dv
  for (int i = 0; i < 9; ++i)
    if (!P->h2d[i].p) GT_TRY(P->h2d[i].alloc(i == 5 ? lb : tb));
  const size_t nb = (size_t)P->n_local * P->heads * P->d * elt;
  const size_t nl = (size_t)P->n_local * P->heads * sizeof(float);
  // Copies overlap the compute on two copy streams (PCIe is full duplex): K, V, Q in; the forward
  // starts when they are resident while dY is still arriving; Y, LSE go out during the backward, dQ
  // during the column pass, dK, dV last.
  if (!P->e2e_in) {
    GT_CUDA_TRY(cudaStreamCreateWithFlags(&P->e2e_in, cudaStreamNonBlocking));
    GT_CUDA_TRY(cudaStreamCreateWithFlags(&P->e2e_out, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&P->e2e_ev[0], &P->e2e_ev[1], &P->e2e_ev[2], &P->e2e_ev[3], &P->e2e_ev[4], &P->ev_dq})
      GT_CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  const char* sm = std::getenv("GT_E2E_STREAM");  // A/B switch: "0" = the unchunked schedule below
  if (P->world == 1 && !P->graphs && !(sm && sm[0] == '0'))
    return fwd_bwd_host_streamed(P, q, k, v, dy, y, lse, dq, dk, dv, st);
  cudaEvent_t ev_start = P->e2e_ev[0], ev_qkv = P->e2e_ev[1], ev_dy = P->e2e_ev[2], ev_fwd = P->e2e_ev[3],
              ev_bwd = P->e2e_ev[4];
  GT_CUDA_TRY(cudaEventRecord(ev_start, st));  // staging buffers are free once earlier work on `stream` is
  GT_CUDA_TRY(cudaStreamWaitEvent(P->e2e_in, ev_start, 0));
  const void* in[4] = {k, v, q, dy};
  const int in_idx[4] = {1, 2, 0, 3};
  for (int i = 0; i < 4; ++i) {
    if (nb) GT_CUDA_TRY(cudaMemcpyAsync(P->h2d[in_idx[i]].p, in[i], nb, cudaMemcpyHostToDevice, P->e2e_in));
    if (i == 2) GT_CUDA_TRY(cudaEventRecord(ev_qkv, P->e2e_in));
  }
  GT_CUDA_TRY(cudaEventRecord(ev_dy, P->e2e_in));
  GT_CUDA_TRY(cudaStreamWaitEvent(st, ev_qkv, 0));
  GT_TRY(gt_attn_fwd(P, P->h2d[0].p, P->h2d[1].p, P->h2d[2].p, P->h2d[4].p, P->h2d[5].as<float>(), stream));
  GT_CUDA_TRY(cudaEventRecord(ev_fwd, st));
  GT_CUDA_TRY(cudaStreamWaitEvent(st, ev_dy, 0));
  P->ev_dq_ready = P->ev_dq;
  gt_status bs = gt_attn_bwd(P, P->h2d[0].p, P->h2d[1].p, P->h2d[2].p, P->h2d[4].p, P->h2d[5].as<float>(),
                             P->h2d[3].p, P->h2d[6].p, P->h2d[7].p, P->h2d[8].p, stream);
  P->ev_dq_ready = nullptr;
  GT_TRY(bs);
  if (P->strategy == GT_A2A) GT_CUDA_TRY(cudaEventRecord(P->ev_dq, st));  // dQ arrives with dK, dV there
  GT_CUDA_TRY(cudaEventRecord(ev_bwd, st));
  GT_CUDA_TRY(cudaStreamWaitEvent(P->e2e_out, ev_fwd, 0));
  if (y && nb) GT_CUDA_TRY(cudaMemcpyAsync(y, P->h2d[4].p, nb, cudaMemcpyDeviceToHost, P->e2e_out));
  if (lse && nl) GT_CUDA_TRY(cudaMemcpyAsync(lse, P->h2d[5].p, nl, cudaMemcpyDeviceToHost, P->e2e_out));
  GT_CUDA_TRY(cudaStreamWaitEvent(P->e2e_out, P->ev_dq, 0));
  if (dq && nb) GT_CUDA_TRY(cudaMemcpyAsync(dq, P->h2d[6].p, nb, cudaMemcpyDeviceToHost, P->e2e_out));
  GT_CUDA_TRY(cudaStreamWaitEvent(P->e2e_out, ev_bwd, 0));
  if (dk && nb) GT_CUDA_TRY(cudaMemcpyAsync(dk, P->h2d[7].p, nb, cudaMemcpyDeviceToHost, P->e2e_out));
  if (dv && nb) GT_CUDA_TRY(cudaMemcpyAsync(dv, P->h2d[8].p, nb, cudaMemcpyDeviceToHost, P->e2e_out));
  GT_CUDA_TRY(cudaStreamSynchronize(P->e2e_out));
  GT_CUDA_TRY(cudaStreamSynchronize(st));
  return GT_OK;
}

gt_status gt_plan_timings(gt_plan_t P, double* ms, int64_t* calls) {
  if (!P || !ms) return fail(GT_EINVAL, "gt_plan_timings: null argument");
  for (int i = 0; i < 5; ++i) {
    ms[i] = 0;
    if (calls) calls[i] = 0;
  }
  for (auto& r : P->recs) {
    GT_CUDA_TRY(cudaEventSynchronize(r.b));
    float t = 0;
    GT_CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.stage] += t;
    if (calls) calls[r.stage]++;
    P->ev_pool.push_back(r.a);
    P->ev_pool.push_back(r.b);
  }
  P->recs.clear();
  if (P->sub) {  // GP-A2A: the head-slice plan's stages
    double sm[5];
    int64_t sc[5];
    GT_TRY(gt_plan_timings(P->sub, sm, sc));
    for (int i = 0; i < 5; ++i) {
      ms[i] += sm[i];
      if (calls) calls[i] += sc[i];
    }
  }
  return GT_OK;
}

void gt_free(gt_plan_t P) {
  if (!P) return;
  cudaSetDevice(P->device);
  cudaDeviceSynchronize();
  delete P;
}

}  // extern "C"
