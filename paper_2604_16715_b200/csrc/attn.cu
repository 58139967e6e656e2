// Pass launchers and the partial-state merge kernels (K6) for rows/columns split into chunks.
//
// The three passes themselves are the pipelined kernels in attn_pipe.cu (Eq. 2/4/5 and
// Section 2.2).  A row (column) with more than `heavy_threshold` entries is processed as
// several chunks by different warps; each chunk leaves a partial state in an fp32 workspace and the
// merge kernels below combine them in chunk order (deterministic, no atomics):
//   forward   (m_c, l_c, acc_c):  M = max m_c, L = sum l_c 2^(m_c - M), y = sum acc_c 2^(m_c - M) / L,
//                                 LSE = (M + log2 L) ln 2          (log-sum-exp merge of online softmax)
//   row pass  A_c = sum dS k:     dQ = scale sum A_c   (D_i = <dY_i, Y_i> is known to every chunk)
//   col pass  (dK_c, dV_c):       dK = scale sum dK_c,  dV = sum dV_c
// (The first-round register-gather kernels are superseded by attn_pipe.cu; their measurements are
// in profiles/r01 and DESIGN.md.)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "gt_internal.h"

namespace gt {
namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kBlock = 256;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int H>
constexpr int kSBF = (8 * H + 15) / 16 * 4;  // floats per row of the (LSE2, D) stats array

// One warp per heavy row/column; lane l owns elements [l * EPL, (l + 1) * EPL) of a row.
template <typename T, int H, int D>
struct Cfg {
  static constexpr int EPL = D / 32;
  static constexpr int LPH = 32 / H;
  static_assert(D % 32 == 0 && 32 % H == 0, "unsupported shape");
};

template <typename T, int EPL>
__device__ __forceinline__ void store_row(char* row, int lane, const float (&f)[EPL]) {
  if constexpr (sizeof(T) == 4) {
    float* p = reinterpret_cast<float*>(row) + lane * EPL;
#pragma unroll
    for (int i = 0; i < EPL; ++i) p[i] = f[i];
  } else {
    __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(row) + lane * (EPL / 2);
#pragma unroll
    for (int i = 0; i < EPL / 2; ++i) p[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  }
}

struct MergeArgs {
  int64_t nids;
  const int32_t* ids;      // heavy row/column local ids
  const int32_t* first;    // chunk range per id
  const float* part;
  char* y;                 // forward outputs
  float* lse;
  char* dq;                // row-pass outputs
  float* stats;
  const float* lse_in;
  char* dk;                // column-pass outputs
  char* dv;
  float scale;
};

template <typename T, int H, int D>
__global__ void __launch_bounds__(kBlock) fwd_merge_kernel(MergeArgs a) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL, LPH = C::LPH;
  const int lane = threadIdx.x & 31;
  const int head = lane / LPH;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < a.nids; x += nw) {
    const int64_t row = a.ids[x];
    const int c0 = a.first[x], c1 = a.first[x + 1];
    float M = -INFINITY;
    for (int c = c0; c < c1; ++c) M = fmaxf(M, a.part[(int64_t)c * (D + 2 * H) + D + 2 * head]);
    float L = 0.f, acc[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
    for (int c = c0; c < c1; ++c) {
      const float* pp = a.part + (int64_t)c * (D + 2 * H);
      const float f = ex2(pp[D + 2 * head] - M);
      L = fmaf(pp[D + 2 * head + 1], f, L);
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] = fmaf(pp[lane * EPL + i], f, acc[i]);
    }
    const float inv = 1.f / L;
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] *= inv;
    store_row<T, EPL>(a.y + row * (int64_t)(D * sizeof(T)), lane, acc);
    if (lane % LPH == 0) a.lse[row * H + head] = (M + __log2f(L)) * kLn2;
  }
}

template <typename T, int H, int D>
__global__ void __launch_bounds__(kBlock) rowb_merge_kernel(MergeArgs a) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL, LPH = C::LPH;
  const int lane = threadIdx.x & 31;
  const int head = lane / LPH;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < a.nids; x += nw) {
    const int64_t row = a.ids[x];
    const int c0 = a.first[x], c1 = a.first[x + 1];
    float A[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) A[i] = 0.f;
    for (int c = c0; c < c1; ++c) {
      const float* pp = a.part + (int64_t)c * D;
#pragma unroll
      for (int i = 0; i < EPL; ++i) A[i] += pp[lane * EPL + i];
    }
#pragma unroll
    for (int i = 0; i < EPL; ++i) A[i] *= a.scale;
    store_row<T, EPL>(a.dq + row * (int64_t)(D * sizeof(T)), lane, A);
  }
}

template <typename T, int H, int D>
__global__ void __launch_bounds__(kBlock) colb_merge_kernel(MergeArgs a) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < a.nids; x += nw) {
    const int64_t col = a.ids[x];
    const int c0 = a.first[x], c1 = a.first[x + 1];
    float dK[EPL], dV[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) { dK[i] = 0.f; dV[i] = 0.f; }
    for (int c = c0; c < c1; ++c) {
      const float* pp = a.part + (int64_t)c * (2 * D);
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        dK[i] += pp[lane * EPL + i];
        dV[i] += pp[D + lane * EPL + i];
      }
    }
#pragma unroll
    for (int i = 0; i < EPL; ++i) dK[i] *= a.scale;
    store_row<T, EPL>(a.dk + col * (int64_t)(D * sizeof(T)), lane, dK);
    store_row<T, EPL>(a.dv + col * (int64_t)(D * sizeof(T)), lane, dV);
  }
}

// Reduce-scatter backward, sender side: row `slot` of `out` = sum of the partial rows of its pieces
// [first[slot], first[slot + 1]) in piece order (zeros for a slot without entries).  Rows: 2 D fp32.
__global__ void __launch_bounds__(kBlock) sum_slots_kernel(int64_t nslots, const int32_t* first, const float4* part,
                                                           int64_t row4, float4* out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < nslots; x += nw) {
    const int c0 = first[x], c1 = first[x + 1];
    for (int64_t i = lane; i < row4; i += 32) {
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int c = c0; c < c1; ++c) {
        const float4 v = part[(int64_t)c * row4 + i];
        s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
      }
      out[x * row4 + i] = s;
    }
  }
}

// Reduce-scatter backward, owner side: column ids[x] = the sum, in list order, of rows idx[ptr[x] ..
// ptr[x + 1]) of `part` (its owned-row pieces first, then the partials received from each peer in
// rank order): dK = scale * sum dK_c, dV = sum dV_c.
template <typename T, int H, int D>
__global__ void __launch_bounds__(kBlock) colb_merge_list_kernel(int64_t nids, const int32_t* ids, const int64_t* ptr,
                                                                 const int64_t* idx, const float* part, char* dk,
                                                                 char* dv, float scale) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < nids; x += nw) {
    const int64_t col = ids[x];
    float K[EPL], V[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) { K[i] = 0.f; V[i] = 0.f; }
    for (int64_t k = ptr[x]; k < ptr[x + 1]; ++k) {
      const float* pp = part + idx[k] * (int64_t)(2 * D);
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        K[i] += pp[lane * EPL + i];
        V[i] += pp[D + lane * EPL + i];
      }
    }
#pragma unroll
    for (int i = 0; i < EPL; ++i) K[i] *= scale;
    store_row<T, EPL>(dk + col * (int64_t)(D * sizeof(T)), lane, K);
    store_row<T, EPL>(dv + col * (int64_t)(D * sizeof(T)), lane, V);
  }
}

template <typename K>
int merge_grid(K, int64_t ids) {  // one warp per heavy row, at most 4 blocks per SM (tiny kernels)
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);  // per call: plans may use several devices
  const int64_t cap = (int64_t)std::max(sms, 1) * 4;
  return (int)std::max<int64_t>(1, std::min<int64_t>(cap, (ids * 32 + kBlock - 1) / kBlock));
}

MergeArgs merge_args(const ChunkTable& ht, const DevBuf& part, float scale) {
  MergeArgs m{};
  m.nids = (int64_t)ht.ids.size();
  m.ids = ht.d_ids.as<int32_t>();
  m.first = ht.d_first.as<int32_t>();
  m.part = part.as<float>();
  m.scale = scale;
  return m;
}

template <typename T, int H, int D>
struct Merges {
  static gt_status run_list(int64_t nids, const int32_t* ids, const int64_t* ptr, const int64_t* idx,
                            const float* part, char* dk, char* dv, float scale, cudaStream_t st) {
    colb_merge_list_kernel<T, H, D><<<merge_grid(colb_merge_list_kernel<T, H, D>, nids), kBlock, 0, st>>>(
        nids, ids, ptr, idx, part, dk, dv, scale);
    GT_CUDA_TRY(cudaGetLastError());
    return GT_OK;
  }
  static gt_status run(int pass, const MergeArgs& m, cudaStream_t st) {
    if (pass == 0) fwd_merge_kernel<T, H, D><<<merge_grid(fwd_merge_kernel<T, H, D>, m.nids), kBlock, 0, st>>>(m);
    else if (pass == 1)
      rowb_merge_kernel<T, H, D><<<merge_grid(rowb_merge_kernel<T, H, D>, m.nids), kBlock, 0, st>>>(m);
    else colb_merge_kernel<T, H, D><<<merge_grid(colb_merge_kernel<T, H, D>, m.nids), kBlock, 0, st>>>(m);
    GT_CUDA_TRY(cudaGetLastError());
    return GT_OK;
  }
};

gt_status merge_list(int dtype, int H, int D, int64_t nids, const int32_t* ids, const int64_t* ptr,
                     const int64_t* idx, const float* part, char* dk, char* dv, float scale, cudaStream_t st) {
#define GT_CASE(TT, HH, DD) \
  if (H == HH && D == DD) return Merges<TT, HH, DD>::run_list(nids, ids, ptr, idx, part, dk, dv, scale, st);
#define GT_HCASES(TT)                                                                              \
  GT_CASE(TT, 1, 64) GT_CASE(TT, 2, 64) GT_CASE(TT, 4, 64) GT_CASE(TT, 8, 64)                        \
  GT_CASE(TT, 1, 128) GT_CASE(TT, 1, 256) GT_CASE(TT, 1, 512) GT_CASE(TT, 2, 128) GT_CASE(TT, 2, 256) \
  GT_CASE(TT, 2, 512) GT_CASE(TT, 4, 128) GT_CASE(TT, 4, 256) GT_CASE(TT, 4, 512) GT_CASE(TT, 8, 128) \
  GT_CASE(TT, 8, 256) GT_CASE(TT, 8, 512)
  if (dtype == GT_F32) { GT_HCASES(float) }
  else { GT_HCASES(__nv_bfloat16) }
#undef GT_HCASES
#undef GT_CASE
  return fail(GT_ECONFIG, "unsupported (dtype, heads, heads*d)");
}

gt_status merge(int dtype, int H, int D, int pass, const MergeArgs& m, cudaStream_t st) {
#define GT_CASE(TT, HH, DD) \
  if (H == HH && D == DD) return Merges<TT, HH, DD>::run(pass, m, st);
#define GT_HCASES(TT)                                                                              \
  GT_CASE(TT, 1, 64) GT_CASE(TT, 2, 64) GT_CASE(TT, 4, 64) GT_CASE(TT, 8, 64)                        \
  GT_CASE(TT, 1, 128) GT_CASE(TT, 1, 256) GT_CASE(TT, 1, 512) GT_CASE(TT, 2, 128) GT_CASE(TT, 2, 256) \
  GT_CASE(TT, 2, 512) GT_CASE(TT, 4, 128) GT_CASE(TT, 4, 256) GT_CASE(TT, 4, 512) GT_CASE(TT, 8, 128) \
  GT_CASE(TT, 8, 256) GT_CASE(TT, 8, 512)
  if (dtype == GT_F32) { GT_HCASES(float) }
  else { GT_HCASES(__nv_bfloat16) }
#undef GT_HCASES
#undef GT_CASE
  return fail(GT_ECONFIG, "unsupported (dtype, heads, heads*d)");
}

}  // namespace

bool shape_supported(int heads, int d, int dtype) {
  const int D = heads * d;
  if (dtype != GT_F32 && dtype != GT_BF16) return false;
  if (heads != 1 && heads != 2 && heads != 4 && heads != 8) return false;
  return D == 64 || D == 128 || D == 256 || D == 512;
}

static int fills(const WorkList& w) { return w.empty.empty() ? 0 : 1; }

int launches_fwd(const gt_plan_s* P) {
  if (P->fwd_split)
    return (P->w_fwd[0].n > 0 ? 1 : 0) + (P->w_fwd[1].n > 0 ? 1 : 0) + (P->fwd_chunks.nchunks() > 0 ? 1 : 0) +
           fills(P->w_fwd[0]);
  return (P->w_rows.n > 0 ? 1 : 0) + (P->heavy_rows.nchunks() > 0 ? 1 : 0) + fills(P->w_rows);
}
int launches_bwd(const gt_plan_s* P) {
  const int rows = (P->w_rows.n > 0 ? 1 : 0) + (P->heavy_rows.nchunks() > 0 ? 1 : 0) + fills(P->w_rows);
  if (P->bwd_reduce)
    return rows + (P->w_hcols.n > 0 ? 1 : 0) + (P->n_slots > 0 ? 1 : 0) + (P->w_colrs.n > 0 ? 1 : 0) +
           fills(P->w_colrs) +
           (P->rs_chunks.ids.empty() ? 0 : 1);
  if (P->col_split)
    return rows + (P->w_colp[0].n > 0 ? 1 : 0) + (P->w_colp[1].n > 0 ? 1 : 0) + (P->col_chunks.nchunks() > 0 ? 1 : 0) +
           fills(P->w_colp[0]);
  return rows + (P->w_cols.n > 0 ? 1 : 0) + (P->heavy_cols.nchunks() > 0 ? 1 : 0) + fills(P->w_cols);
}

// Entry-state arguments of a pass (Table 1 keeps Z and U per edge): the forward
// stores base-2 logits and the row pass (P, dS) per entry in local CSR order; the row pass reads the
// logits in the same order, the column pass reads (P, dS) through the CSC -> CSR map.
static EntryState entry_state(gt_plan_s* P, int pass, bool use_logits = true) {
  EntryState e;
  if (P->n_hot && pass < 2) {  // hot-column table read under a persisting L2 window (gt_opts.hot_cols)
    e.win = P->d_hot.p;
    e.win_bytes = (int64_t)P->d_hot.bytes;
  }
  if (!P->es) return e;
  if (P->kv_fp8 && pass < 2) {  // fp8 K||V gathers (gt_opts.kv_fp8)
    e.kv8 = P->d_kv8.p;
    e.kv8_row = P->kv8_row;
    e.kvref = P->d_kvref.as<int>();
  }
  if (pass == 0) {
    if (P->es_logits) e.out = P->d_s2.as<float>();
  } else if (pass == 1) {
    if (P->es_logits && use_logits) e.in = P->d_s2.as<float>();
    e.out = P->d_pd.as<float>();
  } else if (pass == 2) {
    e.in = P->d_pd.as<float>();
    e.src = P->d_src.as<int32_t>();
  }
  return e;
}

// Forward.  world == 1: one pass over all rows.  world > 1: phase A (owned-column entries) runs while
// the K||V halo is in flight on the side stream, leaving a few SMs to the communication kernels;
// phase B (remote-column entries) waits for `halo_ready`; rows split across phases are merged.
gt_status launch_fwd(gt_plan_s* P, const void* q, const void* k, const void* v, const void* halo_kv, void* y,
                     float* lse, cudaStream_t st, cudaEvent_t halo_ready) {
  float* part = P->d_part_fwd.as<float>();
  const ChunkTable& ct = P->fwd_split ? P->fwd_chunks : P->heavy_rows;
  if (!P->fwd_split) {
    GT_TRY(pipe_pass(P, 0, P->w_rows, ct, part, q, nullptr, nullptr, k, v, halo_kv, nullptr, y, nullptr, lse, st, 0,
                     entry_state(P, 0)));
  } else {
    GT_TRY(pipe_pass(P, 0, P->w_fwd[0], ct, part, q, nullptr, nullptr, k, v, halo_kv, nullptr, y, nullptr, lse, st,
                     P->reserve_sms, entry_state(P, 0)));
    if (halo_ready) GT_CUDA_TRY(cudaStreamWaitEvent(st, halo_ready, 0));
    GT_TRY(pipe_pass(P, 0, P->w_fwd[1], ct, part, q, nullptr, nullptr, k, v, halo_kv, nullptr, y, nullptr, lse, st, 0,
                     entry_state(P, 0)));
  }
  if (ct.nchunks() > 0) {
    MergeArgs m = merge_args(ct, P->d_part_fwd, P->scale);
    m.y = (char*)y;
    m.lse = lse;
    GT_TRY(merge(P->dtype, P->heads, P->heads * P->d, 0, m, st));
  }
  return GT_OK;
}

// Column pass with the fused peer-gather transport: owned-row entries first (split plans) or nothing,
// a device-side barrier (every rank's [q | dy] rows are published and its row pass has written the
// (LSE2, D) blocks), then the entries with remote rows, read from the owners.
gt_status launch_bwd_cols_peer(gt_plan_s* P, const void* q, const void* k, const void* v, const void* dy, void* dk,
                               void* dv, cudaStream_t st) {
  const ChunkTable& ct = P->col_split ? P->col_chunks : P->heavy_cols;
  float* part = P->d_part_colb.as<float>();
  const void* mark = P->d_pub_qd.p;  // non-null: selects the remote-row (peer) kernel
  if (!P->col_split) {
    GT_TRY(P->comm->stream_barrier(st));
    GT_TRY(pipe_pass(P, 2, P->w_cols, ct, part, k, v, nullptr, q, dy, mark, mark, dk, dv, nullptr, st, 0,
                     entry_state(P, 2)));
  } else {
    GT_TRY(pipe_pass(P, 2, P->w_colp[0], ct, part, k, v, nullptr, q, dy, nullptr, nullptr, dk, dv, nullptr, st, 0,
                     entry_state(P, 2)));
    GT_TRY(P->comm->stream_barrier(st));
    GT_TRY(pipe_pass(P, 2, P->w_colp[1], ct, part, k, v, nullptr, q, dy, mark, mark, dk, dv, nullptr, st, 0));
  }
  if (ct.nchunks() > 0) {
    MergeArgs m = merge_args(ct, P->d_part_colb, P->scale);
    m.dk = (char*)dk;
    m.dv = (char*)dv;
    GT_TRY(merge(P->dtype, P->heads, P->heads * P->d, 2, m, st));
  }
  return GT_OK;
}

// Forward with the fused peer-gather transport: own rows published, owned-column entries (phase A)
// while the peers publish, a device-side barrier, then remote-column entries (phase B) reading the
// owners' rows over NVLink.  The first barrier keeps a rank from overwriting its published rows while
// peers may still read them (their previous row pass).
gt_status launch_fwd_peer(gt_plan_s* P, const void* q, const void* k, const void* v, void* y, float* lse,
                          cudaStream_t st) {
  const int elt = P->dtype == GT_F32 ? 4 : 2;
  float* part = P->d_part_fwd.as<float>();
  const ChunkTable& ct = P->fwd_chunks;
  GT_TRY(P->comm->stream_barrier(st));
  GT_TRY(pack_kv(k, v, P->d_iota.as<int32_t>(), P->n_local, (int64_t)P->heads * P->d, elt, P->d_pub.p, st));
  GT_TRY(pipe_pass(P, 0, P->w_fwd[0], ct, part, q, nullptr, nullptr, k, v, nullptr, nullptr, y, nullptr, lse, st, 0,
                   entry_state(P, 0)));
  GT_TRY(P->comm->stream_barrier(st));
  GT_TRY(pipe_pass(P, 0, P->w_fwd[1], ct, part, q, nullptr, nullptr, k, v, P->d_pub.p, nullptr, y, nullptr, lse, st,
                   0, entry_state(P, 0)));
  if (ct.nchunks() > 0) {
    MergeArgs m = merge_args(ct, P->d_part_fwd, P->scale);
    m.y = (char*)y;
    m.lse = lse;
    GT_TRY(merge(P->dtype, P->heads, P->heads * P->d, 0, m, st));
  }
  return GT_OK;
}

// Streamed world-1 pass (gt_attn_fwd_bwd_host): work items [t0, t1) of the row (column) list - a
// contiguous range of rows (columns) with every heavy row's chunks inside it - and the merges of the
// heavy rows (columns) h0 .. h1 - 1 of the plan's chunk table among them.  fill: also the outputs of the
// rows (columns) without entries.  pass 0: y, lse; 1: dq (+ the (LSE2, D) stats); 2: dk, dv.
gt_status launch_pass_range(gt_plan_s* P, int pass, const void* q, const void* k, const void* v, const void* y,
                            const float* lse, const void* dy, void* out_a, void* out_b, cudaStream_t st, int64_t t0,
                            int64_t t1, int64_t h0, int64_t h1, bool fill) {
  const ItemRange rg{t0, t1, fill};
  const ChunkTable& ct = pass == 2 ? P->heavy_cols : P->heavy_rows;
  const DevBuf& part = pass == 0 ? P->d_part_fwd : (pass == 1 ? P->d_part_rowb : P->d_part_colb);
  const void* hot = P->n_hot ? P->d_hot.p : nullptr;  // hot-column table (gt_opts.hot_cols)
  if (pass == 0) {
    GT_TRY(pipe_pass(P, 0, P->w_rows, ct, part.as<float>(), q, nullptr, nullptr, k, v, hot, nullptr, out_a,
                     nullptr, const_cast<float*>(lse), st, 0, entry_state(P, 0), rg));
  } else if (pass == 1) {
    EntryState e = entry_state(P, 1, true);
    e.own_c = y;
    GT_TRY(pipe_pass(P, 1, P->w_rows, ct, part.as<float>(), q, dy, lse, k, v, hot, nullptr, out_a, nullptr,
                     P->d_stats.as<float>(), st, 0, e, rg));
  } else {
    GT_TRY(pipe_pass(P, 2, P->w_cols, ct, part.as<float>(), k, v, nullptr, q, dy, nullptr, nullptr, out_a, out_b,
                     nullptr, st, 0, entry_state(P, 2), rg));
  }
  if (h1 > h0) {
    MergeArgs m = merge_args(ct, part, P->scale);
    m.ids += h0;
    m.first += h0;
    m.nids = h1 - h0;
    if (pass == 0) {
      m.y = (char*)out_a;
      m.lse = const_cast<float*>(lse);
    } else if (pass == 1) {
      m.dq = (char*)out_a;
    } else {
      m.dk = (char*)out_a;
      m.dv = (char*)out_b;
    }
    GT_TRY(merge(P->dtype, P->heads, P->heads * P->d, pass, m, st));
  }
  return GT_OK;
}

gt_status launch_bwd_rows(gt_plan_s* P, const void* q, const void* k, const void* v, const void* y,
                          const void* halo_kv, const float* lse, const void* dy, void* dq, cudaStream_t st,
                          bool use_logits) {
  EntryState e = entry_state(P, 1, use_logits);
  e.own_c = y;
  GT_TRY(pipe_pass(P, 1, P->w_rows, P->heavy_rows, P->d_part_rowb.as<float>(), q, dy, lse, k, v, halo_kv, nullptr,
                   dq, nullptr, P->d_stats.as<float>(), st, 0, e));
  if (P->heavy_rows.nchunks() > 0) {
    MergeArgs m = merge_args(P->heavy_rows, P->d_part_rowb, P->scale);
    m.dq = (char*)dq;
    GT_TRY(merge(P->dtype, P->heads, P->heads * P->d, 1, m, st));
  }
  return GT_OK;
}

// Column pass.  With entry state and world > 1 the owned-row entries (phase A, stored (P, dS)) run
// before `side_ready` (the in-halo [q | dy] rows and stats) is waited on; the remote-row entries
// (phase B) recompute p and dP; columns split across the phases are merged.
gt_status launch_bwd_cols(gt_plan_s* P, const void* q, const void* k, const void* v, const void* dy,
                          const void* halo_qd, const void* halo_st, void* dk, void* dv, cudaStream_t st,
                          cudaEvent_t side_ready) {
  const ChunkTable& ct = P->col_split ? P->col_chunks : P->heavy_cols;
  float* part = P->d_part_colb.as<float>();
  if (!P->col_split) {
    if (side_ready) GT_CUDA_TRY(cudaStreamWaitEvent(st, side_ready, 0));
    GT_TRY(pipe_pass(P, 2, P->w_cols, ct, part, k, v, nullptr, q, dy, halo_qd, halo_st, dk, dv, nullptr, st, 0,
                     entry_state(P, 2)));
  } else {
    GT_TRY(pipe_pass(P, 2, P->w_colp[0], ct, part, k, v, nullptr, q, dy, nullptr, nullptr, dk, dv, nullptr, st, 0,
                     entry_state(P, 2)));
    if (side_ready) GT_CUDA_TRY(cudaStreamWaitEvent(st, side_ready, 0));
    GT_TRY(pipe_pass(P, 2, P->w_colp[1], ct, part, k, v, nullptr, q, dy, halo_qd, halo_st, dk, dv, nullptr, st, 0));
  }
  if (ct.nchunks() > 0) {
    MergeArgs m = merge_args(ct, P->d_part_colb, P->scale);
    m.dk = (char*)dk;
    m.dv = (char*)dv;
    GT_TRY(merge(P->dtype, P->heads, P->heads * P->d, 2, m, st));
  }
  return GT_OK;
}

// Column-first backward, column half: (LSE2, D) of every row, then the column pass over A^T computing
// dP = <dY_i, v_j> with its own v_j (the row pass of the row-first order gathers v_j for it), P from the
// forward's logit, dS; it stores dS per entry in CSR order for the row half.  Bytes per entry: q_i, dY_i,
// (LSE2, D)_i, the logit; the row half then gathers k_j and dS alone.
gt_status launch_bwd_cf_cols(gt_plan_s* P, const void* q, const void* k, const void* v, const void* y,
                             const float* lse, const void* dy, void* dk, void* dv, cudaStream_t st) {
  GT_TRY(row_stats(P->dtype, P->heads, P->heads * P->d, y, dy, lse, P->n_local, P->d_stats.as<float>(),
                   (int)P->st_row_bytes, st));
  EntryState e;
  e.mode = 1;
  e.in = P->d_s2.as<float>();
  e.out = P->d_pd.as<float>();
  e.src = P->d_src.as<int32_t>();
  GT_TRY(pipe_pass(P, 2, P->w_cols, P->heavy_cols, P->d_part_colb.as<float>(), k, v, nullptr, q, dy, nullptr, nullptr,
                   dk, dv, nullptr, st, 0, e));
  if (P->heavy_cols.nchunks() > 0) {
    MergeArgs m = merge_args(P->heavy_cols, P->d_part_colb, P->scale);
    m.dk = (char*)dk;
    m.dv = (char*)dv;
    GT_TRY(merge(P->dtype, P->heads, P->heads * P->d, 2, m, st));
  }
  return GT_OK;
}

// Column-first backward, row half: dQ_i = scale sum_e dS_e k_j with the column half's dS.
gt_status launch_bwd_cf_rows(gt_plan_s* P, const void* q, const void* k, const void* v, const float* lse,
                             const void* dy, void* dq, cudaStream_t st) {
  EntryState e;
  e.mode = 1;
  e.in = P->d_pd.as<float>();
  GT_TRY(pipe_pass(P, 1, P->w_rows, P->heavy_rows, P->d_part_rowb.as<float>(), q, dy, lse, k, v, nullptr, nullptr, dq,
                   nullptr, P->d_stats.as<float>(), st, 0, e));
  if (P->heavy_rows.nchunks() > 0) {
    MergeArgs m = merge_args(P->heavy_rows, P->d_part_rowb, P->scale);
    m.dq = (char*)dq;
    GT_TRY(merge(P->dtype, P->heads, P->heads * P->d, 1, m, st));
  }
  return GT_OK;
}

// Reduce-scatter backward, sender side: the column pass over the halo columns (local rows' entries
// with remote columns, grouped by slot; own k, v = the [k | v] rows received in the forward), every
// piece a chunk partial, then summed per slot into the send rows.
gt_status launch_bwd_halo_cols(gt_plan_s* P, const void* q, const void* dy, cudaStream_t st) {
  const int elt = P->dtype == GT_F32 ? 4 : 2;
  const int64_t RB = (int64_t)P->heads * P->d * elt;
  if (P->w_hcols.n > 0) {
    EntryState e;
    if (P->es) {
      e.in = P->d_pd.as<float>();
      e.src = P->d_hsrc.as<int32_t>();
    }
    e.nbr = P->d_hrow.as<int32_t>();
    e.nnbr = P->n_hent;
    e.own_stride = 2 * RB;
    const char* kv = (const char*)P->d_recv_kv.p;
    GT_TRY(pipe_pass(P, 2, P->w_hcols, P->hcol_chunks, P->d_part_h.as<float>(), kv, kv + RB, nullptr, q, dy, nullptr,
                     nullptr, nullptr, nullptr, nullptr, st, 0, e));
  }
  if (P->n_slots > 0) {
    const int64_t row4 = 2 * (int64_t)P->heads * P->d / 4;
    sum_slots_kernel<<<merge_grid(sum_slots_kernel, P->n_slots), kBlock, 0, st>>>(
        P->n_slots, P->hcol_chunks.d_first.as<int32_t>(), (const float4*)P->d_part_h.p, row4, (float4*)P->d_rs_send.p);
    GT_CUDA_TRY(cudaGetLastError());
  }
  return GT_OK;
}

// Reduce-scatter backward, owner side: owned columns over owned-row entries (columns with remote
// in-edges leave chunk partials), then, once the partials of the peers are in (`recv_ready`), the
// fixed-order merge of those columns.
gt_status launch_bwd_cols_rs(gt_plan_s* P, const void* q, const void* k, const void* v, const void* dy, void* dk,
                             void* dv, cudaStream_t st, cudaEvent_t recv_ready) {
  EntryState e;
  if (P->es) {
    e.in = P->d_pd.as<float>();
    e.src = P->d_src.as<int32_t>();
  }
  GT_TRY(pipe_pass(P, 2, P->w_colrs, P->rs_chunks, P->d_part_rs.as<float>(), k, v, nullptr, q, dy, nullptr, nullptr,
                   dk, dv, nullptr, st, 0, e));
  if (recv_ready) GT_CUDA_TRY(cudaStreamWaitEvent(st, recv_ready, 0));
  const int64_t nids = (int64_t)P->rs_chunks.ids.size();
  if (nids > 0)
    GT_TRY(merge_list(P->dtype, P->heads, P->heads * P->d, nids, P->rs_chunks.d_ids.as<int32_t>(),
                      P->d_mptr.as<int64_t>(), P->d_midx.as<int64_t>(), P->d_part_rs.as<float>(), (char*)dk,
                      (char*)dv, P->scale, st));
  return GT_OK;
}

}  // namespace gt
