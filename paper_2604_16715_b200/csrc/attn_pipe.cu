// Pipelined sparse-attention kernels for sm_100a: asynchronous gathers (cp.async / LDGSTS) of
// neighbour rows into per-warp shared-memory stage rings.
//
// Mathematics (Eq. 2/4/5, Section 2.2), base-2 softmax with fp32 accumulation:
//   pass 0 (fwd):  per row i:    s_e = scale <q_i,k_j>, online softmax, y_i = sum p_e v_j / l, LSE
//   pass 1 (rowb): per row i:    p_e = exp(s_e - LSE_i), dP_e = <dY_i, v_j>, D_i = sum p dP,
//                                dQ_i = scale (sum p dP k_j - D_i sum p k_j)
//   pass 2 (colb): per column j: dV_j = sum p dY_i, dK_j = scale sum p (dP - D_i) q_i
//
// Entry state (template bits ES; Table 1 keeps Z and U per edge): with bit 2 the
// forward stores each entry's base-2 logit and the row pass reads it instead of q.k; with bit 1 the
// row pass stores (p, dS) per entry and the column pass reads them (through the CSC -> CSR map)
// instead of recomputing q.k and dY.v.  Stores go through a per-warp shared-memory transpose: one
// coalesced, predicated store per stage.  Without entry state the column pass recomputes p and dP
// from (q_i, dY_i, LSE_i, D_i) and its own k_j, v_j.
//
// Remote rows (HALO kernels, world > 1) come from a received table, or (peer transport) straight
// from the owners' published buffers through a per-rank base table (NVLink peer loads).
//
// Execution model.  Persistent CTAs; every warp owns a ring of kS stages in shared memory, each
// holding up to U neighbours (two feature rows, plus the neighbour's (LSE2, D) pair in pass 2, plus
// the stage's entry state), and an "own" slot per stage for the data of the row (column) an item
// starts.  Warps grab kG consecutive work items (rows, or chunks of heavy rows, in row order) per
// atomicAdd (kG = 2, A/B-tuned on C3 and C5), so the resident warps sweep the graph in a narrow window of rows and
// the neighbours they gather stay in L2 (community locality); consecutive items have contiguous
// entry ranges, streamed through a 32-entry register window of neighbour ids with the next window
// prefetched.  Rows with more than the plan's threshold of entries are split into chunks whose fp32
// partial states are merged in chunk order by attn.cu (deterministic).
//
// The warp is its own producer.  Lane l issues cp.async copies of ITS 16-byte slice of every
// gathered row (a whole 512-byte row is one coalesced request per warp) and later reads back only
// those same bytes, so completion needs no barrier or cross-lane synchronisation: one
// cp.async.commit_group per stage and cp.async.wait_group(kS - 1) before consuming the oldest
// stage.  kS * U neighbours (8 KB at D = 256 bf16) stay in flight per warp, across row boundaries,
// without occupying registers.  (Measured alternatives - a TMA cp.async.bulk variant, lane-group
// producers, half-warp rows - are in DESIGN.md section 6.)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "gt_internal.h"

namespace gt {
namespace pipe {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxDevices = 64;
#ifndef GT_PIPE_WARPS
#define GT_PIPE_WARPS 4
#endif
#ifndef GT_PIPE_STAGES
#define GT_PIPE_STAGES 2
#endif
#ifndef GT_PIPE_GRAB
#define GT_PIPE_GRAB 2
#endif
#ifndef GT_RT_STRIDE
#define GT_RT_STRIDE 1
#endif
#ifndef GT_PIPE_TMA
#define GT_PIPE_TMA 0  // measured slower on C3; kept for A/B builds
#endif
#ifndef GT_PIPE_MMA
#define GT_PIPE_MMA 0  // tensor-core (mma.sync) consumer for the products shape, bit p = pass p (measured slower: DESIGN.md section 6)
#endif
constexpr int kWarps = GT_PIPE_WARPS;   // warps per CTA
#ifndef GT_COLB_STAGES
#define GT_COLB_STAGES 2
#endif
// stages per warp: 2 (measured best: more resident warps).  A third stage for the stored-state column
// pass alone measured 8.45 -> 8.54 ms on C3 (3 stages for every pass: column pass -4 %, row pass +15 %)
template <int PASS, int ES>
constexpr int stages_of() { return (PASS == 2 && (ES & 1)) ? GT_COLB_STAGES : GT_PIPE_STAGES; }
constexpr int kG = GT_PIPE_GRAB;        // items per grab

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 16-byte copy that zero-fills the destination instead of reading when !valid (no branch)
__device__ __forceinline__ void cp_async16z(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async4z(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(su32(dst)), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async8z(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(su32(dst)), "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}

template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(su32(dst)), "l"(src), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---- mbarrier + TMA (sm_100a) ----
__device__ __forceinline__ void mbar_init(void* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(void* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                 : "=r"(ok) : "r"(su32(bar)), "r"(parity) : "memory");
  } while (!ok);
}
// 4 rows (r0..r3) of a 2-D tensor map, columns [c, c + box), into dst (rows contiguous); completion is
// counted in bytes on `bar`.  Rows outside the tensor are zero-filled.
__device__ __forceinline__ void tma_gather4(const void* map, void* dst, void* bar, int c, int r0, int r1, int r2,
                                            int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(dst)), "l"(map), "r"(su32(bar)), "r"(c), "r"(r0),
      "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct TmaMaps {   // tensor maps of the two gathered tables (k | q, v | dY): [rows][D] elements
  CUtensorMap a, b;
};

// predicated global store (no branch, so the warp stays provably converged for the shuffles)
__device__ __forceinline__ void st_pred(float* p, float x, bool on) {
  asm volatile("{.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f32 [%0], %1;}" ::"l"(p), "f"(x),
               "r"((int)on) : "memory");
}

__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

template <typename T, int H, int D, int PASS, int ES>
struct PC {
  // ES bit 4: fp8 K||V gathers (gt_opts.kv_fp8; forward and row pass): the gathered table is the plan's
  // quantised one, a row [k8 (D B) | v8 (D B) | 2^ek f32[H] | 2^ev f32[H]] (e4m3 with power-of-two
  // scales per (row, head), quantize_kv_kernel)
  static constexpr bool F8 = (ES & 4) != 0;
  static constexpr int GR = F8 ? (2 * D + 8 * H + 15) / 16 * 16 : 0;   // bytes of a gathered fp8 row
  static constexpr int LB8 = D / 32;                                    // bytes per lane of its fp8 slices
  static constexpr int RB = D * (int)sizeof(T);          // bytes of one feature row
  static constexpr int EPL = D / 32;                      // elements per lane
  static constexpr int LB = EPL * (int)sizeof(T);         // bytes per lane of one row (8..64)
  static constexpr int W = LB / 4;                        // 32-bit words per lane slice
  static constexpr int LPH = 32 / H;                      // lanes per head
  static constexpr int SB = (8 * H + 15) / 16 * 16;       // (LSE2, D) row of the stats array, padded
  static constexpr int PDB = sizeof(T) == 2 ? 4 : 8;      // stored (P, dS) of one entry and head: bf16x2 | f32x2
  // the recompute column pass gathers each in-neighbour's (LSE2, D) block; with stored (P, dS) it does not
  static constexpr bool STATS = PASS == 2 && !(ES & 1);
  // ES bit 8: column-first backward (PArgs::mode 1, launch_bwd_colfirst): the column pass gathers q_i,
  // dY_i and (LSE2, D)_i, reads the forward's logit through the CSC -> CSR map, computes dP with its own
  // v_j and stores dS per entry (CSR order); the row pass then gathers k_j alone and reads that dS
  static constexpr bool CF = (ES & 8) != 0;
  static constexpr int ESZ = (int)sizeof(T);              // bytes of a stored dS (column-first)
  // own slot: fwd q | rowb [q] dY Y lse | colb [k v]   (the row pass recomputing q.k needs q; with
  // stored (P, dS) the column pass needs no own-column data)
  static constexpr int OWN_DY = PASS == 1 ? ((ES & 2) ? 0 : RB) : 0;
  static constexpr int OWN_Y = OWN_DY + RB;
  static constexpr int OWN_LSE = OWN_Y + RB;   // the row's LSE of the lane's head, one 4-byte slot per lane
  static constexpr int OWN = PASS == 0 ? RB : (PASS == 1 ? (CF ? 0 : OWN_LSE + 4 * 32) : ((ES & 1) ? 0 : (CF ? RB : 2 * RB)));
#ifdef GT_PIPE_U  // tuning override (A/B builds)
  static constexpr int U = RB >= 2048 ? 1 : (RB >= 1024 ? 2 : (GT_PIPE_U * H <= 32 ? GT_PIPE_U : 32 / H));
#else
  // neighbours per stage (fp8: 4; 8 in two butterfly groups measured slower on C3 / C5: fwd 10.7 -> 11.1 /
  // 31.7 -> 40.3 ms)
  static constexpr int U = F8 ? 4 : (RB >= 2048 ? 1 : (RB >= 1024 ? 2 : 4));
#endif
  // per-stage entry state gathered into the stage (ES): rowb s2[U][H] f32 (the forward's logits),
  // colb (P, dS)[U][H] (the row pass's)
  // (column-first: rowb dS[U][H] (T); colb s2[U][H] f32 + the U entries' CSR positions)
  static constexpr int AUX = PASS == 1 ? (CF ? U * H * ESZ : ((ES & 2) ? U * H * 4 : 0))
                                       : ((PASS == 2 && (ES & 1)) ? U * H * PDB : ((PASS == 2 && CF) ? U * H * 4 + U * 4 : 0));
  // TMA gathers (sm_100 cp.async.bulk.tensor tile::gather4: 4 rows of a 2-D tensor map per instruction)
  // for the two feature rows of every neighbour when the stage holds exactly 4 neighbours; the
  // stage then keeps the 4 first rows (k | q) contiguous, then the 4 second rows (v | dY), then stats
  static constexpr bool TMA = GT_PIPE_TMA && U == 4 && !F8 && !CF;
  // Tensor-core consumer (Mma below): the stage's dot products and SpMM updates as mma.sync m16n8k16
  // products for the products shape (bf16, 4 heads of 64, 4 neighbours per stage) - the forward, the
  // row pass reading the forward's logits and the column pass reading the stored (P, dS)
  static constexpr bool MMA = ((GT_PIPE_MMA >> PASS) & 1) && sizeof(T) == 2 && H == 4 && D == 256 && U == 4 && !F8 && !TMA &&
                              (PASS == 0 || (PASS == 1 && (ES & 2)) || (PASS == 2 && (ES & 1)));
  // bytes per neighbour in a stage; the tensor-core layout pads it to 32 mod 128 so that the 8 rows one
  // ldmatrix phase reads (4 neighbours x 2 heads) fall in 8 distinct 16-byte bank groups
  static constexpr int EB = (F8 ? GR : ((PASS == 1 && CF) ? RB : 2 * RB + (STATS ? SB : 0))) + (MMA ? 32 : 0);
  static constexpr int STAGE = (U * EB + AUX + 127) / 128 * 128;   // 128-byte aligned TMA destinations
  static constexpr int OWNP = (OWN + 15) / 16 * 16;
  // ES transpose scratch of the per-stage store: fwd s2[U][H], rowb (P, dS)[U][H]
  // (the tensor-core consumer stores them from the registers of the lanes holding them: no scratch)
  static constexpr int XS = MMA ? 0 : (PASS == 0 ? ((ES & 2) ? U * H * 4 : 0)
                                                 : ((PASS == 1 && (ES & 1)) ? U * H * PDB : ((PASS == 2 && CF) ? U * H * ESZ : 0)));
  static constexpr int kS = stages_of<PASS, ES>();                   // stages per warp
  static constexpr int MB = TMA ? kS * 8 : 0;                       // one mbarrier per stage
  static constexpr int WARP_SMEM = (kS * (STAGE + OWNP + XS) + MB + 127) / 128 * 128;
  // byte offsets in a stage of neighbour u's first row, second row and (LSE2, D) block (tma: the kernel
  // gathers with TMA; kernels with remote rows keep the interleaved per-lane-copy layout)
  template <bool TM> static __device__ __forceinline__ int koff(int u) { return TM ? u * RB : u * EB; }
  template <bool TM> static __device__ __forceinline__ int voff(int u) {
    return TM ? U * RB + u * RB : u * EB + (F8 ? D : RB);
  }
  template <bool TM> static __device__ __forceinline__ int soff(int u) { return TM ? 2 * U * RB + u * SB : u * EB + 2 * RB; }
  static_assert(LB == 4 || LB == 8 || LB % 16 == 0, "lane slice must be 4, 8 or a multiple of 16 bytes");
  static_assert(U * H <= 32, "entry-state copies: one lane per (neighbour, head)");
  static_assert(!F8 || (sizeof(T) == 2 && PASS < 2 && LB8 >= 4 && 32 / H >= 4), "fp8 gathers: bf16 plans, D >= 128");
};

struct PArgs {
  const int64_t* ibeg;   // [nitems] entry range [ibeg, iend) of each item in the neighbour array
  const int64_t* iend;
  const int32_t* iown;   // [nitems]: >= 0 row/column id, < 0 chunk -1 - c
  const int32_t* cown;   // chunk -> row/column id
  const int32_t* nbr;    // neighbour ids in entry order (remapped: < n_local local, else halo slot)
  int64_t nnbr;          // entries in nbr
  int64_t nitems;
  unsigned long long* counter;
  const char* ga;        // local tensor gathered first  (k | k | q)
  const char* gb;        // local tensor gathered second (v | v | dy)
  const char* gs;        // local (LSE2, D) rows [n_local][SB bytes] (pass 2)
  const char* halo;      // packed remote rows: [k | v] (passes 0, 1) or [q | dy] (pass 2)
  const char* peer[8];   // fused peer gather (peer_shift > 0): rank s's published rows, [k | v] (passes 0,
  const char* peer_s[8]; //   1) or [q | dy] (pass 2), and (pass 2) rank s's (LSE2, D) blocks
  int peer_shift;        //   remote slot = (owner << peer_shift) + offset
  const char* halo_s;    // pass 2: remote (LSE2, D) blocks [rows][SB bytes]
  int64_t halo_stride;
  int64_t n_local;
  const char* oa;        // own tensor A (q | q | k)
  const char* ob;        // own tensor B (- | dy | v)
  const char* oc;        // own tensor C (- | y | -): the row pass takes D_i = <dY_i, Y_i>
  int64_t own_stride;    // bytes between own rows of the column pass (a feature row, or 2 of them when
                         // the own rows are the [k | v] rows received in the forward)
  const float* lse;      // pass 1: caller's LSE [n_local][H] (natural log)
  char* out_a;           // y | dq | dk
  char* out_b;           // - | - | dv
  float* out_f;          // lse (pass 0) | stats [n_local][SB/4] (pass 1)
  float* part;           // chunk partials
  float qscale, scale;
  // materialised entry state (ES kernels; Table 1 keeps U per edge)
  float* es_out;         // fwd: s2 [nnz_local][H] base-2 logits | rowb: (P, dS) [nnz_local][H] (bf16x2 for
                         // bf16 plans, f32x2 for f32 plans), both in local CSR entry order
  const float* es_in;    // rowb: s2 | colb: (P, dS)
  const int32_t* src;    // colb: local CSC position -> local CSR entry (read through a window like nbr)
  const int* kvref;      // fp8 gathers: {E_k, E_v} = max exponent of the K / V scales over the table
  const void* win;       // persisting L2 access-policy window of the launch (hot-column table), or null
  int64_t win_bytes;
  int mode;              // 1: column-first backward (EntryState::mode; selects the ES bit 8 kernels)
  uint32_t rb, rb2, sb;  // row strides (bytes) of the gathered tables as run-time values: a row address is
                         // then one IMAD.WIDE.U32 (an immediate power-of-two stride becomes shift + high +
                         // two 64-bit adds)
};

// lane slice copy of one row: LB bytes at byte offset lane * LB
template <int LB>
__device__ __forceinline__ void cp_slice(char* dst_row, const char* src_row, int lane) {
  if constexpr (LB == 4) {
    cp_async<4>(dst_row + lane * 4, src_row + lane * 4);
  } else if constexpr (LB == 8) {
    cp_async<8>(dst_row + lane * 8, src_row + lane * 8);
  } else {
#pragma unroll
    for (int i = 0; i < LB / 16; ++i) cp_async<16>(dst_row + lane * LB + 16 * i, src_row + lane * LB + 16 * i);
  }
}

// base + idx * stride with one mad.wide.u32 (64-bit result)
__device__ __forceinline__ const char* row_addr(const char* base, uint32_t idx, uint32_t stride) {
  const char* r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(idx), "r"(stride), "l"(base));
  return r;
}

// this lane's LB bytes: dst and src already point at the lane's slice
template <int LB>
__device__ __forceinline__ void cp_lane_z(char* dst, const char* src, bool valid) {
  if constexpr (LB == 4) {
    cp_async4z(dst, src, valid);
  } else if constexpr (LB == 8) {
    cp_async8z(dst, src, valid);
  } else {
#pragma unroll
    for (int i = 0; i < LB / 16; ++i) cp_async16z(dst + 16 * i, src + 16 * i, valid);
  }
}

template <typename T, int EPL>
__device__ __forceinline__ void lds_f32(const char* p, float (&f)[EPL]) {
  constexpr int W = EPL * (int)sizeof(T) / 4;
  uint32_t w[W];
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int i = 0; i < W / 4; ++i) {
      uint4 x = *reinterpret_cast<const uint4*>(p + 16 * i);
      w[4 * i] = x.x; w[4 * i + 1] = x.y; w[4 * i + 2] = x.z; w[4 * i + 3] = x.w;
    }
  } else if constexpr (W == 2) {
    uint2 x = *reinterpret_cast<const uint2*>(p);
    w[0] = x.x; w[1] = x.y;
  } else {
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  }
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < EPL; ++i) f[i] = __uint_as_float(w[i]);
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
}

template <typename T, int EPL>
__device__ __forceinline__ void stg_f32(char* p, const float (&f)[EPL]) {
  constexpr int W = EPL * (int)sizeof(T) / 4;
  uint32_t w[W];
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < EPL; ++i) w[i] = __float_as_uint(f[i]);
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) {
      __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&b);
    }
  }
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int i = 0; i < W / 4; ++i)
      reinterpret_cast<uint4*>(p)[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
  } else if constexpr (W == 2) {
    *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
  } else {
    *reinterpret_cast<uint32_t*>(p) = w[0];
  }
}

template <int EPL>
__device__ __forceinline__ float dot(const float (&a)[EPL], const float (&b)[EPL]) {
  float2 s = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < EPL; i += 2) s = f2fma(make_float2(a[i], a[i + 1]), make_float2(b[i], b[i + 1]), s);
  return s.x + s.y;
}

template <int EPL>
__device__ __forceinline__ void axpy(float p, const float (&x)[EPL], float (&acc)[EPL]) {
  const float2 pp = make_float2(p, p);
#pragma unroll
  for (int i = 0; i < EPL; i += 2) {
    float2 r = f2fma(pp, make_float2(x[i], x[i + 1]), make_float2(acc[i], acc[i + 1]));
    acc[i] = r.x;
    acc[i + 1] = r.y;
  }
}

template <int EPL>
__device__ __forceinline__ void scale2(float c, float (&acc)[EPL]) {
  const float2 cc = make_float2(c, c);
#pragma unroll
  for (int i = 0; i < EPL; i += 2) {
    float2 r = f2fma(cc, make_float2(acc[i], acc[i + 1]), make_float2(0.f, 0.f));
    acc[i] = r.x;
    acc[i + 1] = r.y;
  }
}

template <int W>
__device__ __forceinline__ void lds_raw(const char* p, uint32_t (&w)[W]) {
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int i = 0; i < W / 4; ++i) {
      uint4 x = *reinterpret_cast<const uint4*>(p + 16 * i);
      w[4 * i] = x.x; w[4 * i + 1] = x.y; w[4 * i + 2] = x.z; w[4 * i + 3] = x.w;
    }
  } else if constexpr (W == 2) {
    uint2 x = *reinterpret_cast<const uint2*>(p);
    w[0] = x.x; w[1] = x.y;
  } else {
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  }
}

__device__ __forceinline__ float fma_bf16(uint16_t a, uint16_t b, float c) {
  float d;
  asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}

// <a, b> of two rows held as raw storage words, accumulated in fp32.  bf16: FHFMA.BF16 reads the
// two halves of each word in place (exact products, fp32 sums) - no unpacking.
template <typename T, int W>
__device__ __forceinline__ float dot_raw(const uint32_t (&a)[W], const uint32_t (&b)[W]) {
  if constexpr (sizeof(T) == 2) {
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      uint16_t al, ah, bl, bh;
      asm("mov.b32 {%0, %1}, %2;" : "=h"(al), "=h"(ah) : "r"(a[i]));
      asm("mov.b32 {%0, %1}, %2;" : "=h"(bl), "=h"(bh) : "r"(b[i]));
      s0 = fma_bf16(al, bl, s0);
      s1 = fma_bf16(ah, bh, s1);
    }
    return s0 + s1;
  } else {
    float2 s = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < W; i += 2)
      s = f2fma(make_float2(__uint_as_float(a[i]), __uint_as_float(a[i + 1])),
                make_float2(__uint_as_float(b[i]), __uint_as_float(b[i + 1])), s);
    return s.x + s.y;
  }
}

// Weight of an accumulation acc += w x, as the 32-bit word that is broadcast between lanes: bf16 plans
// round it to bf16 (low half; the products w x are then exact in fp32 and summed in fp32, as
// FlashAttention rounds P and dS before its P V and dS K products), f32 plans keep the fp32 bits.
template <typename T>
__device__ __forceinline__ uint32_t wpack(float x) {
  if constexpr (sizeof(T) == 2) {
    uint16_t b;
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(b) : "f"(x));
    return (uint32_t)b;
  } else {
    return __float_as_uint(x);
  }
}

// (P, dS) of one entry and head as stored by the row pass: bf16x2 {lo = P, hi = dS} (bf16 plans)
__device__ __forceinline__ uint32_t pack_pd_bf16(float p, float ds) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(ds), "f"(p));
  return r;
}

// acc += w x over this lane's raw slice x (W storage words).  bf16: w is the bf16 in half HI of wb
// (FHFMA.BF16 reads both halves of the row words in place: no unpacking); f32: w = the float wb.
template <typename T, int W, int EPL, bool HI = false>
__device__ __forceinline__ void accum(uint32_t wb, const uint32_t (&x)[W], float (&acc)[EPL]) {
  if constexpr (sizeof(T) == 2) {
    uint16_t wl, wh;
    asm("mov.b32 {%0, %1}, %2;" : "=h"(wl), "=h"(wh) : "r"(wb));
    const uint16_t w = HI ? wh : wl;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      uint16_t xl, xh;
      asm("mov.b32 {%0, %1}, %2;" : "=h"(xl), "=h"(xh) : "r"(x[i]));
      acc[2 * i] = fma_bf16(w, xl, acc[2 * i]);
      acc[2 * i + 1] = fma_bf16(w, xh, acc[2 * i + 1]);
    }
  } else {
    const float w = __uint_as_float(wb);
    const float2 ww = make_float2(w, w);
#pragma unroll
    for (int i = 0; i < W; i += 2) {
      const float2 r = f2fma(ww, make_float2(__uint_as_float(x[i]), __uint_as_float(x[i + 1])),
                             make_float2(acc[i], acc[i + 1]));
      acc[i] = r.x;
      acc[i + 1] = r.y;
    }
  }
}

// ---- fp8 (e4m3) gathers: decoded to f16 and multiplied by f16 operands with fp32 accumulation ----
__device__ __forceinline__ float fma_f16(uint16_t a, uint16_t b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}
__device__ __forceinline__ uint32_t f16x2_of(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint16_t f16_of(float x) {   // saturating: |x| > 65504 -> +-65504
  uint16_t r;
  asm("cvt.rn.satfinite.f16.f32 %0, %1;" : "=h"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ uint32_t e4m3x2_to_f16x2(uint32_t x16) {
  uint32_t r;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(r) : "h"((uint16_t)x16));
  return r;
}
// 2^e for e in [-126, 127] (exact)
__device__ __forceinline__ float exp2i(int e) { return __int_as_float((e + 127) << 23); }
// floor(log2 |x|) of a positive normal float, clamped to [-126, 126] (x == 0: 0)
__device__ __forceinline__ int ilog2f(float x) {
  const int e = ((__float_as_int(x) >> 23) & 0xff) - 127;
  return x > 0.f ? max(-126, min(126, e)) : 0;
}
// the lane's EPL fp8 elements (EPL / 4 words) from shared memory
template <int EPL>
__device__ __forceinline__ void lds_f8(const char* p, uint32_t (&w)[EPL / 4]) {
  constexpr int NW = EPL / 4;
  if constexpr (NW == 4) {
    const uint4 x = *reinterpret_cast<const uint4*>(p);
    w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
  } else if constexpr (NW == 2) {
    const uint2 x = *reinterpret_cast<const uint2*>(p);
    w[0] = x.x; w[1] = x.y;
  } else {
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  }
}
// <o, x> with o the lane's EPL elements as f16x2 words and x its EPL fp8 elements
template <int EPL>
__device__ __forceinline__ float dot_f8(const uint32_t (&o)[EPL / 2], const uint32_t (&x)[EPL / 4]) {
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int i = 0; i < EPL / 4; ++i) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const uint32_t f = e4m3x2_to_f16x2(hh ? x[i] >> 16 : x[i] & 0xffffu);  // elements 4i + 2hh, +1
      uint16_t fl, fh, ol, oh;
      asm("mov.b32 {%0, %1}, %2;" : "=h"(fl), "=h"(fh) : "r"(f));
      asm("mov.b32 {%0, %1}, %2;" : "=h"(ol), "=h"(oh) : "r"(o[2 * i + hh]));
      s0 = fma_f16(ol, fl, s0);
      s1 = fma_f16(oh, fh, s1);
    }
  }
  return s0 + s1;
}
// acc += w x over the lane's EPL fp8 elements, w an f16
template <int EPL>
__device__ __forceinline__ void accum_f8(uint16_t w, const uint32_t (&x)[EPL / 4], float (&acc)[EPL]) {
#pragma unroll
  for (int i = 0; i < EPL / 4; ++i) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const uint32_t f = e4m3x2_to_f16x2(hh ? x[i] >> 16 : x[i] & 0xffffu);
      uint16_t fl, fh;
      asm("mov.b32 {%0, %1}, %2;" : "=h"(fl), "=h"(fh) : "r"(f));
      acc[4 * i + 2 * hh] = fma_f16(w, fl, acc[4 * i + 2 * hh]);
      acc[4 * i + 2 * hh + 1] = fma_f16(w, fh, acc[4 * i + 2 * hh + 1]);
    }
  }
}

// The lane's EPL bf16 elements (raw words) scaled by 2^-e, e = floor(log2 max |x|) over the lane's head
// (the largest is then in [1, 2): exact in f16 unless 2^14 times smaller than the max), as f16x2 words.
template <int EPL, int LPH>
__device__ __forceinline__ int to_f16_norm(const uint32_t (&w)[EPL / 2], uint32_t (&o)[EPL / 2]) {
  float f[EPL];
#pragma unroll
  for (int i = 0; i < EPL / 2; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
  float am = 0.f;
#pragma unroll
  for (int i = 0; i < EPL; ++i) am = fmaxf(am, fabsf(f[i]));
#pragma unroll
  for (int o2 = LPH / 2; o2 >= 1; o2 >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o2));
  const int e = ilog2f(am);
  const float sc = exp2i(-e);
#pragma unroll
  for (int i = 0; i < EPL / 2; ++i) o[i] = f16x2_of(f[2 * i] * sc, f[2 * i + 1] * sc);
  return e;
}

// predicated 32-bit shared store (generic address of a shared location)
__device__ __forceinline__ void sts_pred_u32(void* p, uint32_t x, bool on) {
  asm volatile("{.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.b32 [%0], %1;}" ::"r"(su32(p)), "r"(x),
               "r"((int)on) : "memory");
}
// predicated 16-bit global store of raw bits
__device__ __forceinline__ void st_pred_u16(void* p, uint16_t x, bool on) {
  asm volatile("{.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.b16 [%0], %1;}" ::"l"(p), "h"(x),
               "r"((int)on) : "memory");
}

// predicated 32-bit global store of raw bits
__device__ __forceinline__ void st_pred_u32(uint32_t* p, uint32_t x, bool on) {
  asm volatile("{.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.b32 [%0], %1;}" ::"l"(p), "r"(x),
               "r"((int)on) : "memory");
}

template <int LPH>
__device__ __forceinline__ float head_sum(float x) {
#pragma unroll
  for (int o = LPH / 2; o >= 1; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

// Transposed (reduce-scatter) butterfly of 4 per-lane partial sums over a head's LPH lanes (LPH >= 4):
// the two top lane bits of the head pick the neighbour, g = 2 b_top + b_top-1, whose full sum the lane
// ends with (the lower levels are plain xor-sums).  bfly_src(u) is a lane holding neighbour u's sum.
template <int LPH>
struct Bfly {
  static constexpr int TOP = LPH == 32 ? 4 : (LPH == 16 ? 3 : (LPH == 8 ? 2 : 1));
  static_assert(LPH >= 4 && (1 << (TOP + 1)) == LPH, "butterfly needs 4..32 lanes per head");
  static __device__ __forceinline__ int group(int lane) { return 2 * ((lane >> TOP) & 1) + ((lane >> (TOP - 1)) & 1); }
  static __device__ __forceinline__ int src(int lane, int u) {
    return (lane & ~(LPH - 1)) | ((u >> 1) << TOP) | ((u & 1) << (TOP - 1));
  }
  static __device__ __forceinline__ float reduce(const float (&v)[4], int lane) {
    const bool bh = (lane >> TOP) & 1, bl = (lane >> (TOP - 1)) & 1;
    float a0 = bh ? v[2] : v[0], a1 = bh ? v[3] : v[1];
    const float t0 = bh ? v[0] : v[2], t1 = bh ? v[1] : v[3];
    a0 += __shfl_xor_sync(0xffffffffu, t0, 1 << TOP);
    a1 += __shfl_xor_sync(0xffffffffu, t1, 1 << TOP);
    float r = bl ? a1 : a0;
    r += __shfl_xor_sync(0xffffffffu, bl ? a0 : a1, 1 << (TOP - 1));
#pragma unroll
    for (int o = (1 << (TOP - 1)) >> 1; o >= 1; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    return r;
  }
  // sum (or max) over the 4 neighbour groups of a per-group value
  static __device__ __forceinline__ float all_sum(float x) {
    x += __shfl_xor_sync(0xffffffffu, x, 1 << (TOP - 1));
    return x + __shfl_xor_sync(0xffffffffu, x, 1 << TOP);
  }
  static __device__ __forceinline__ float all_max(float x) {
    x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 1 << (TOP - 1)));
    return fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 1 << TOP));
  }
};

// ---- tensor-core consumer: mma.sync m16n8k16 (bf16 operands, exact products, fp32 accumulation) ----
__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr) : "memory");
}
__device__ __forceinline__ void ldsm4t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr) : "memory");
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t bf16x2_of(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void st_pred_bf16(char* p, float x, bool on) {
  asm volatile("{.reg .pred q;\n\t.reg .b16 h;\n\tsetp.ne.b32 q, %2, 0;\n\tcvt.rn.bf16.f32 h, %1;\n\t"
               "@q st.global.b16 [%0], h;}" ::"l"(p), "f"(x), "r"((int)on) : "memory");
}

// Lane geometry of the tensor-core consumer (H = 4 heads of 64 elements, U = 4 neighbours per stage,
// lane = 4 g + t).
//  * Dot products (q.k in the forward, dY.v in the row pass): per 16-element chunk c of the heads one
//    m16n8k16 product D = A B with A[m = 4h + u][k] = neighbour u's head-h chunk c (ldmatrix of the
//    staged rows; the two 8-element halves swapped for odd h, which puts the 8 rows of an ldmatrix
//    phase in 8 bank groups given the 32-mod-128 neighbour stride) and B[k][n = h] = the own row's
//    head h in the same element order (registers, once per row; B[.][n >= 4] = 0).  Only the diagonal
//    D[4h + u][h] is used: lane 4g + t, t < 2 ("holder"), ends with entry (h = 2t + g/4, u = g % 4).
//  * SpMM (y += p v, dQ += dS k, dV += P dY, dK += dS q): the transposed product D'[i][n] +=
//    A'[i][k] B'[k][n] with A'[i][4h + u] = neighbour u's head-h element tau_h(c, i) (ldmatrix.trans)
//    and B'[4h + u][n] = w(u, h) for n = h, else 0 (block diagonal: 2 registers from 4 shuffles).
//    Holder lane 4g + t accumulates heads 2t, 2t + 1: acc[c] = {y_2t[16c + g], y_2t+1[16c + 8 + g],
//    y_2t[16c + 8 + g], y_2t+1[16c + g]}.
//  Products are exact (bf16 x bf16) and summed in fp32, as in the FHFMA.BF16 consumer; the weights
//  p, dS, P are rounded to bf16 first, as there.
struct Mma {
  int g, t;
  bool holder;             // t < 2: holds one (head, neighbour) product
  int h, u;                // holder: its entry's head and neighbour
  int src_e;               // lane holding the product of entry-state slot `lane` = 4 u' + h' (u' < 4)
  bool b0on, b1on;         // B' registers this lane supplies (heads t/2 and 2 + t/2)
  uint32_t off_dot, off_sp;  // byte offsets (within a stage's first row block) of the ldmatrix rows
  template <int EB>
  __device__ __forceinline__ void init(int lane) {
    g = lane >> 2;
    t = lane & 3;
    holder = t < 2;
    h = (2 * t + (g >> 2)) & 3;
    u = g & 3;
    const int eh = lane & 3, eu = (lane >> 2) & 3;
    src_e = 16 * (eh & 1) + 4 * eu + (eh >> 1);
    b0on = g == (t >> 1);
    b1on = g == 2 + (t >> 1);
    const int j = lane >> 3, r = lane & 7;
    const int hd = 2 * (j & 1) + (r >> 2), hs = 2 * (j >> 1) + (r >> 2);
    off_dot = (uint32_t)((r & 3) * EB + hd * 128 + 16 * (((j >> 1) + hd) & 1));
    off_sp = (uint32_t)((r & 3) * EB + hs * 128 + 16 * (((j & 1) + hs) & 1));
  }
  // B fragments of the own row (512-byte bf16 row at shared address `o`): b[2c], b[2c + 1]
  __device__ __forceinline__ void load_b(const char* o, uint32_t (&b)[8]) const {
    const int gg = g & 3;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(o);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int e0 = gg * 64 + 16 * c + 8 * (gg & 1) + 2 * t, e1 = gg * 64 + 16 * c + 8 * ((gg + 1) & 1) + 2 * t;
      b[2 * c] = g < 4 ? w[e0 >> 1] : 0u;
      b[2 * c + 1] = g < 4 ? w[e1 >> 1] : 0u;
    }
  }
  // the 16 dot products of a stage (rows at shared address `rows` + off_dot); holder lanes' value is theirs
  __device__ __forceinline__ float dot(uint32_t rows, const uint32_t (&b)[8]) const {
    float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t a0[4], a1[4];
    ldsm4(rows, a0);
    ldsm4(rows + 32, a1);
    mma16816(d0, a0, b[0], b[1]);
    mma16816(d1, a1, b[2], b[3]);
    ldsm4(rows + 64, a0);
    ldsm4(rows + 96, a1);
    mma16816(d0, a0, b[4], b[5]);
    mma16816(d1, a1, b[6], b[7]);
    const bool lo = g < 4, odd = t & 1;
    const float x0 = odd ? (lo ? d0[2] : d0[3]) : (lo ? d0[0] : d0[1]);
    const float x1 = odd ? (lo ? d1[2] : d1[3]) : (lo ? d1[0] : d1[1]);
    return x0 + x1;
  }
  // B' registers of the weights w held by the holder lanes (rounded to bf16)
  __device__ __forceinline__ void weights(float w, int lane, uint32_t& b0, uint32_t& b1) const {
    const float wn = __shfl_sync(kFull, w, (lane + 4) & 31);   // neighbour u + 1 of the same head
    const uint32_t pair = bf16x2_of(w, wn);
    const uint32_t w0 = __shfl_sync(kFull, pair, 8 * t), w1 = __shfl_sync(kFull, pair, 8 * t + 1);
    b0 = b0on ? w0 : 0u;
    b1 = b1on ? w1 : 0u;
  }
  // acc[c] += A'(rows at shared address `rows` + off_sp) B'
  __device__ __forceinline__ void spmm(uint32_t rows, uint32_t b0, uint32_t b1, float (&acc)[4][4]) const {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t a[4];
      ldsm4t(rows + 32 * c, a);
      mma16816(acc[c], a, b0, b1);
    }
  }
  // element index (within a 256-element row) of acc[c][i]
  __device__ __forceinline__ int elem(int c, int i) const {
    const int hh = 2 * t + (i & 1);
    return hh * 64 + 16 * c + ((i == 1 || i == 2) ? 8 : 0) + g;
  }
  __device__ __forceinline__ void store_bf16(char* row, const float (&acc)[4][4], float fe, float fo) const {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int i = 0; i < 4; ++i) st_pred_bf16(row + 2 * elem(c, i), acc[c][i] * ((i & 1) ? fo : fe), holder);
  }
  __device__ __forceinline__ void store_f32(float* row, const float (&acc)[4][4]) const {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int i = 0; i < 4; ++i) st_pred(row + elem(c, i), acc[c][i], holder);
  }
  __device__ __forceinline__ void scale(float (&acc)[4][4], float fe, float fo) const {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      acc[c][0] *= fe;
      acc[c][1] *= fo;
      acc[c][2] *= fe;
      acc[c][3] *= fo;
    }
  }
};
constexpr float kRescale = 8.f;  // forward (tensor-core consumer): the running reference max of a head is
                                 // raised only when a score exceeds it by more than 2^8 (weights <= 256)

struct Meta {      // warp-uniform description of one filled stage
  int32_t e0;      // entry index (in `nbr` order) of the stage's first neighbour (nnz < 2^31)
  int32_t own;     // row/column id, or chunk -1 - c
  int32_t cnt;     // neighbours in the stage (0 = no work left)
  bool first, last;
};

// ------------------------------------------------------------------ kernel --
// Minimum resident CTAs per SM (register cap) of the backward passes where the lane slice is small
// enough not to spill (A/B-tuned with tools/build_variants.py; 5 CTAs = 20 warps <= 96 registers).
#ifndef GT_ROWB_MINB
#define GT_ROWB_MINB 1
#endif
#ifndef GT_COLB_MINB
#define GT_COLB_MINB 1
#endif
#ifndef GT_FWD_MINB  // forward: 6 CTAs/SM (<= 80 registers, no spills) with the full shared-memory carveout
#define GT_FWD_MINB 6
#endif
#ifndef GT_CARVEOUT  // preferred shared-memory carveout (percent of the unified L1/shared array); -1 = driver's
#define GT_CARVEOUT 100
#endif
#ifndef GT_MMA_BWD_MINB  // tensor-core backward passes: resident CTAs per SM (register cap)
#define GT_MMA_BWD_MINB 5
#endif
#ifndef GT_CF_COLB_MINB  // column-first column pass: resident CTAs per SM (register cap)
#define GT_CF_COLB_MINB 4   // A/B: 4 (96 registers, still 5 CTAs by shared memory) vs 5 (87, rematerialised lane constants): column pass -6 %
#endif
template <typename T, int H, int D, int PASS, int ES>
constexpr int min_ctas() {
  constexpr int EPL = D / 32;
  return EPL > 8 ? 1
                 : ((ES & 8) && PASS == 2) ? GT_CF_COLB_MINB
                 : ((ES & 4) ? 5
                             : (PASS == 0 ? GT_FWD_MINB
                                          : (PC<T, H, D, PASS, ES>::MMA ? GT_MMA_BWD_MINB
                                                                       : (PASS == 1 ? GT_ROWB_MINB : GT_COLB_MINB))));
}

template <typename T, int H, int D, int PASS, bool HALO, int ES>
__global__ void __launch_bounds__(kWarps * 32, (min_ctas<T, H, D, PASS, ES>()))
    pipe_kernel(const PArgs a, const __grid_constant__ TmaMaps tm) {
  static_assert(!((ES & 1) && PASS == 2 && HALO), "the ES column pass reads local rows only");
  using C = PC<T, H, D, PASS, ES>;
  constexpr int EPL = C::EPL, LPH = C::LPH, RB = C::RB, EB = C::EB, U = C::U, LB = C::LB;
#ifndef GT_FWD_BFLY
#define GT_FWD_BFLY 1
#endif
  constexpr bool kBfly = GT_FWD_BFLY && PASS == 0 && LPH >= 4 && U == 4;  // forward butterfly (see below)
#ifndef GT_ROWB_BFLY
#define GT_ROWB_BFLY 1
#endif
  constexpr bool kBflyR = GT_ROWB_BFLY && PASS == 1 && (ES & 2) && LPH >= 4 && U == 4;  // row-pass butterfly
  extern __shared__ __align__(128) char smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int head = lane / LPH;
  constexpr int kS = C::kS;
  char* const stages = smem + (size_t)wid * C::WARP_SMEM;   // kS * STAGE
  char* const owns = stages + kS * C::STAGE;                 // kS * OWNP
  char* const xs = owns + kS * C::OWNP;                      // kS * XS
  char* const mbar = xs + kS * C::XS;                        // kS mbarriers (TMA)
  constexpr bool kTma = C::TMA && !HALO;
  uint32_t phase = 0;                                        // parity of each stage's next mbarrier phase
  if constexpr (kTma) {
    if (lane == 0) {
      for (int s = 0; s < kS; ++s) mbar_init(mbar + 8 * s, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      fence_proxy_async();
    }
    __syncwarp();
  }

  // ---------------- producer state (warp-uniform; per-lane only the tables) ----------------
  const int32_t nitems = (int32_t)a.nitems;
  const int32_t nnbr = (int32_t)a.nnbr;
  // entry and item indices are 32-bit (gt_plan: n, nnz < 2^31 - 1)
  int32_t t_next = 0, t_end = 0, batch_t0 = 0;
  int32_t my_beg = 0, my_end = 0;    // lane k < kG: entry range of item batch_t0 + k
  int32_t my_own = 0;                // lane k < kG: owner of item batch_t0 + k
  bool done = false;
  int32_t pe = 0, pe_end = 0;        // current item's remaining edge range
  int32_t cur_own = 0;
  bool cur_first = false;
  int32_t win_base = -(1 << 30);     // lane l holds nbr[win_base + l] in win, nbr[win_base + 32 + l] in win_next
  int32_t win = 0, win_next = 0;
  int32_t wsrc = 0, wsrc_next = 0;   // ES column pass: src[] over the same window
  // this lane's slice of row 0 of every gathered table: a row address is one mad.wide.u32
  const char* const ga_l = a.ga + lane * LB;
  const char* const g8_l = C::F8 ? a.ga + lane * C::LB8 : nullptr;       // fp8: the lane's k8 slice
  const char* const gs8_l = C::F8 ? a.ga + 2 * D + lane * 16 : nullptr;  // fp8: 16 B of the scales
  const char* const gb_l = a.gb + lane * LB;
  const char* const h_l = HALO ? a.halo + lane * LB : nullptr;
  const char* const gs_l = PASS == 2 ? a.gs + lane * 16 : nullptr;
  const char* const hs_l = (PASS == 2 && HALO) ? a.halo_s + lane * 16 : nullptr;
  const uint32_t n_loc = (uint32_t)a.n_local;
#if GT_RT_STRIDE
  const uint32_t sRB = a.rb, sRB2 = a.rb2, sSB = a.sb;
#else
  constexpr uint32_t sRB = RB, sRB2 = 2 * RB, sSB = C::SB;
#endif

  auto finalize_empty = [&](int64_t r) {  // a row (column) with no entries
    float z[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) z[i] = 0.f;
    stg_f32<T, EPL>(a.out_a + r * RB + lane * LB, z);
    if constexpr (PASS == 0) {
      a.out_f[r * H + head] = -INFINITY;
    } else if constexpr (PASS == 1) {
      reinterpret_cast<float2*>(reinterpret_cast<char*>(a.out_f) + r * C::SB)[head] = make_float2(-INFINITY, 0.f);
    } else {
      stg_f32<T, EPL>(a.out_b + r * RB + lane * LB, z);
    }
  };

  auto load_window = [&](int32_t base) {
    win_base = base;
    win = (base + lane < nnbr) ? __ldg(a.nbr + base + lane) : 0;
    win_next = (base + 32 + lane < nnbr) ? __ldg(a.nbr + base + 32 + lane) : 0;
    if constexpr ((ES & 9) && PASS == 2) {
      wsrc = (base + lane < nnbr) ? __ldg(a.src + base + lane) : 0;
      wsrc_next = (base + 32 + lane < nnbr) ? __ldg(a.src + base + 32 + lane) : 0;
    }
  };

  // Advances to the next non-empty item; false when the grid's work is exhausted.
  auto next_item = [&]() -> bool {
    for (;;) {
      if (t_next >= t_end) {
        if (done) return false;
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(a.counter, (unsigned long long)kG);
        b = __shfl_sync(kFull, b, 0);
        if ((int64_t)b >= nitems) {
          done = true;
          return false;
        }
        batch_t0 = (int32_t)b;
        t_end = min(batch_t0 + kG, nitems);
        t_next = batch_t0;
        const int32_t k = batch_t0 + lane;
        const bool in = lane < kG && k < nitems;
        my_beg = in ? (int32_t)__ldg(a.ibeg + k) : 0;
        my_end = in ? (int32_t)__ldg(a.iend + k) : 0;
        my_own = in ? __ldg(a.iown + k) : 0;
      }
      const int k = (int)(t_next - batch_t0);
      const int32_t e0 = __shfl_sync(kFull, my_beg, k);
      const int32_t e1 = __shfl_sync(kFull, my_end, k);
      const int32_t own = __shfl_sync(kFull, my_own, k);
      ++t_next;
      if (e1 == e0) {
        finalize_empty(own);
        continue;
      }
      pe = e0;
      pe_end = e1;
      cur_own = own;
      cur_first = true;
      // items of a list need not be contiguous (split forward; new batch): reload the window.  Done
      // unconditionally: with a data-dependent test (or lane-conditional stores, see below) ptxas can
      // no longer prove the warp converged and emulates every shuffle (WARPSYNC.COLLECTIVE) - measured
      // 3-8 % slower per pass on C3.  Per-head values are therefore stored by all lanes of the head
      // (identical bytes, one sector) instead of under `if (lane % LPH == 0)`.
      load_window(pe);
      return true;
    }
  };

  // Fills stage `s` with the next group of neighbours (this lane's slices) and returns its meta.
  auto produce = [&](int s) -> Meta {
    Meta md;
    md.e0 = 0;
    md.cnt = 0;
    md.own = 0;
    md.first = md.last = false;
    if (pe >= pe_end && !next_item()) return md;
    if (pe == win_base + 32) {  // slide the neighbour window; prefetch the one after
      win_base += 32;
      win = win_next;
      win_next = (win_base + 32 + lane < nnbr) ? __ldg(a.nbr + win_base + 32 + lane) : 0;
      if constexpr ((ES & 9) && PASS == 2) {
        wsrc = wsrc_next;
        wsrc_next = (win_base + 32 + lane < nnbr) ? __ldg(a.src + win_base + 32 + lane) : 0;
      }
    }
    const int off = (int)(pe - win_base);
    const int cnt = min(min((int)(pe_end - pe), 32 - off), U);
    char* st = stages + s * C::STAGE;
    if constexpr (kTma) {
      // one lane issues two gather4 copies (the 4 neighbours' first and second rows); masked neighbours
      // get an out-of-range row (zero-filled by the TMA unit).  The stage was just read with generic
      // loads by the whole warp: order those before the async-proxy writes.
      int id[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int cv = __shfl_sync(kFull, win, off + u);
        id[u] = u < cnt ? cv : (int)n_loc;
      }
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();
        mbar_expect_tx(mbar + 8 * s, 2 * U * RB);
        tma_gather4(&tm.a, st, mbar + 8 * s, 0, id[0], id[1], id[2], id[3]);
        tma_gather4(&tm.b, st + U * RB, mbar + 8 * s, 0, id[0], id[1], id[2], id[3]);
      }
      if constexpr (C::STATS) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (lane < C::SB / 16)
            cp_async16z(st + C::template soff<kTma>(u) + lane * 16, row_addr(gs_l, (uint32_t)(u < cnt ? id[u] : id[0]), C::SB),
                        u < cnt);
      }
    } else if constexpr (C::F8) {
      // fp8 K||V rows: the lane's k8 and v8 slices off one row address, the scales by the first lanes
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool valid = u < cnt;
        const uint32_t cv = (uint32_t)__shfl_sync(kFull, win, off + u);
        const char* pr = row_addr(g8_l, cv, sRB);
        char* dst = st + u * EB + lane * C::LB8;
        cp_lane_z<C::LB8>(dst, pr, valid);
        cp_lane_z<C::LB8>(dst + D, pr + D, valid);
        if (lane < (8 * H + 15) / 16) cp_async16z(st + u * EB + 2 * D + lane * 16, row_addr(gs8_l, cv, sRB), valid);
      }
    } else {
#pragma unroll
    for (int u = 0; u < U; ++u) {  // branch-free: neighbours u >= cnt are zero-filled, not read
      const bool valid = u < cnt;
      // shfl.idx reads the low 5 bits of the lane index; masked neighbours fetch some valid id
      const uint32_t cv = (uint32_t)__shfl_sync(kFull, win, off + u);
      const char *pa, *pb, *ps = nullptr;
      if constexpr (HALO) {
        const bool loc = cv < n_loc;
        const char* hrow;
        const char* srow = nullptr;
        if (a.peer_shift) {  // NVLink peer load of the owner's published row (kernel param: uniform)
          const uint32_t slot = cv - n_loc;
          const uint32_t own = (slot >> a.peer_shift) & 7, off = slot & ((1u << a.peer_shift) - 1);
          hrow = row_addr(a.peer[own] + lane * LB, off, sRB2);
          if constexpr (PASS == 2) srow = row_addr(a.peer_s[own] + lane * 16, off, C::SB);
        } else {
          hrow = row_addr(h_l, cv - n_loc, sRB2);
          if constexpr (PASS == 2) srow = row_addr(hs_l, cv - n_loc, C::SB);
        }
        pa = loc ? row_addr(ga_l, cv, sRB) : hrow;
        pb = loc ? row_addr(gb_l, cv, sRB) : hrow + RB;
        if constexpr (PASS == 2) ps = loc ? row_addr(gs_l, cv, sSB) : srow;
      } else {
        pa = row_addr(ga_l, cv, sRB);
        pb = row_addr(gb_l, cv, sRB);
        if constexpr (PASS == 2) ps = row_addr(gs_l, cv, sSB);
      }
      char* dst = st + u * EB + lane * LB;
      cp_lane_z<LB>(dst, pa, valid);
      if constexpr (!(PASS == 1 && C::CF)) cp_lane_z<LB>(dst + RB, pb, valid);
      // (LSE2, D) block of the neighbour (remote-row kernels): SB / 16 lanes copy 16 bytes each (read by
      // all lanes of a head after the stage's wait + __syncwarp)
      if constexpr (C::STATS && HALO) {
        if (lane < C::SB / 16) cp_async16z(st + u * EB + 2 * RB + lane * 16, ps, valid);
      }
    }
    if constexpr (C::STATS && !HALO) {
      // the stage's (LSE2, D) blocks in one copy: lane l < U SB/16 takes 16 bytes of neighbour l / (SB/16)
      // (one row address per lane and stage instead of one per neighbour)
      constexpr int LS = C::SB / 16;
      const int su = lane / LS, sp = lane % LS;
      const uint32_t sv = (uint32_t)__shfl_sync(kFull, win, off + su);
      if (lane < U * LS) cp_async16z(st + su * EB + 2 * RB + sp * 16, row_addr(a.gs + sp * 16, sv, sSB), su < cnt);
    }
    }
    if constexpr ((ES & 2) && PASS == 1) {  // s2 of the stage's entries (contiguous), stored by the forward
      const bool kv = lane < cnt * H;
      if (lane < U * H)
        cp_async4z(st + U * EB + lane * 4, row_addr(reinterpret_cast<const char*>(a.es_in), (uint32_t)pe * H + (kv ? lane : 0), 4), kv);
    }
    if constexpr ((ES & 1) && PASS == 2) {  // (P, dS) of the stage's entries, stored in CSR order by the row pass
      const int ku = lane / H, kh = lane % H;
      const uint32_t ke = (uint32_t)__shfl_sync(kFull, wsrc, off + ku);
      // window entries past the item may be remote rows (src -1): masked, and read entry 0 instead
      const char* src = row_addr(reinterpret_cast<const char*>(a.es_in) + kh * C::PDB, ku < cnt ? ke : 0u, H * C::PDB);
      if (lane < U * H) {
        if constexpr (C::PDB == 8) cp_async8z(st + U * EB + lane * 8, src, ku < cnt);
        else cp_async4z(st + U * EB + lane * 4, src, ku < cnt);
      }
    }
    if constexpr (C::CF && PASS == 1) {  // dS of the stage's entries (contiguous, CSR order), stored by the column pass
      constexpr int EW = H * C::ESZ / 4;   // words per entry (the host selects these kernels for H * ESZ >= 4)
      const bool kv = lane < cnt * EW;
      if (lane < U * EW)
        cp_async4z(st + U * EB + lane * 4,
                   row_addr(reinterpret_cast<const char*>(a.es_in), (uint32_t)pe * EW + (kv ? lane : 0), 4), kv);
    }
    if constexpr (C::CF && PASS == 2) {
      // the forward's base-2 logits of the stage's entries through the CSC -> CSR map, and (plain shared
      // stores, ordered before the consumer by its __syncwarp) the entries' CSR positions for the dS store
      const int ku = lane / H, kh = lane % H;
      const uint32_t ke = (uint32_t)__shfl_sync(kFull, wsrc, off + ku);
      const char* src = row_addr(reinterpret_cast<const char*>(a.es_in) + kh * 4, ku < cnt ? ke : 0u, H * 4);
      if (lane < U * H) cp_async4z(st + U * EB + lane * 4, src, ku < cnt);
      const uint32_t pu = (uint32_t)__shfl_sync(kFull, wsrc, off + (lane & (U - 1)));
      sts_pred_u32(st + U * EB + U * H * 4 + lane * 4, pu, lane < U);
    }
    md.e0 = pe;
    md.cnt = cnt;
    md.own = cur_own;
    md.first = cur_first;
    md.last = pe + cnt == pe_end;
    if (cur_first) {
      char* o = owns + s * C::OWNP;
      const int64_t r = cur_own >= 0 ? cur_own : a.cown[-1 - (int64_t)cur_own];
      if constexpr (PASS == 0) {
        cp_slice<LB>(o, a.oa + r * RB, lane);
      } else if constexpr (PASS == 1) {
        if constexpr (!C::CF) {  // (the column-first row pass needs no own-row data)
          if constexpr (!(ES & 2)) cp_slice<LB>(o, a.oa + r * RB, lane);
          cp_slice<LB>(o + C::OWN_DY, a.ob + r * RB, lane);
          cp_slice<LB>(o + C::OWN_Y, a.oc + r * RB, lane);
          cp_async<4>(o + C::OWN_LSE + lane * 4, a.lse + r * H + head);  // distinct slots: no same-address writes
        }
      } else if constexpr (C::CF) {  // column-first column pass: v_j (dP = <dY_i, v_j>)
        cp_slice<LB>(o, a.ob + r * a.own_stride, lane);
      } else if constexpr (!(ES & 1)) {
        cp_slice<LB>(o, a.oa + r * a.own_stride, lane);
        cp_slice<LB>(o + RB, a.ob + r * a.own_stride, lane);
      }
      cur_first = false;
    }
    pe += cnt;
    return md;
  };

  // ---------------- consumer state ----------------
  constexpr int W = C::W;
  float acc[EPL], acc2[EPL];  // fwd: y | rowb: dQ (unscaled) | colb: dK (unscaled), dV (acc2)
  uint32_t ow[W];             // raw own-row words: q (fwd), dY (rowb), k (colb recompute)
  uint32_t ow2[W];            // rowb recompute: q; colb recompute: v
  float m = 0.f, l = 0.f;     // fwd: running max / sum (base 2) | rowb: lse2 (m), D (l)
  // fp8 gathers: own row as normalised f16 (fwd q', rowb dY' and, without stored logits, q') and its
  // factors (fwd: qscale 2^eq; rowb: 2^e_dy, qscale 2^eq); table references 2^E_k, 2^E_v
  uint32_t oh[C::F8 ? EPL / 2 : 1], oq[(C::F8 && PASS == 1 && !(ES & 2)) ? EPL / 2 : 1];
  float fo = 1.f, ifo = 1.f, fq = 1.f;
  const float rk = C::F8 ? exp2i(__ldg(a.kvref)) : 1.f, rv = C::F8 ? exp2i(__ldg(a.kvref + 1)) : 1.f;
  const float irk = 1.f / rk, irv = 1.f / rv;
  // column-first column pass, butterfly layout: per-lane constants (byte offsets in a stage of the lane
  // group's (LSE2, D) and logit, the dS store's source lane, CSR-position slot and head offset)
  int cf_ug = 0, cf_sd = 0, cf_s2 = 0, cf_src = 0, cf_pos = 0, cf_eo = 0;
  int cf_w[4] = {0, 0, 0, 0};
  if constexpr (C::CF && PASS == 2 && U == 4 && LPH >= 4) {
    cf_ug = Bfly<LPH>::group(lane);
    cf_sd = cf_ug * EB + 2 * RB + head * 8;
    cf_s2 = U * EB + (cf_ug * H + head) * 4;
    const int f = lane < U * H ? lane : 0;
    cf_src = Bfly<LPH>::src(LPH * (f % H), f / H);
    cf_pos = U * EB + U * H * 4 + (f / H) * 4;
    cf_eo = (f % H) * C::ESZ;
#pragma unroll
    for (int u = 0; u < 4; ++u) cf_w[u] = Bfly<LPH>::src(lane, u);
  }
  // tensor-core consumer: lane geometry, own-row B fragments, accumulators (Mma)
  Mma mg;
  if constexpr (C::MMA) mg.init<EB>(lane);
  uint32_t bq[C::MMA ? 8 : 1];
  float macc[C::MMA ? 4 : 1][4], macc2[(C::MMA && PASS == 2) ? 4 : 1][4];
  float mh = 0.f, dh = 0.f;   // row pass: the holder's (LSE2, D) of its head
  const uint32_t st_sh = su32(stages);

  Meta md[kS];
#pragma unroll
  for (int s = 0; s < kS; ++s) {
    md[s] = produce(s);
    cp_commit();
  }
  for (;;) {
#pragma unroll
    for (int s = 0; s < kS; ++s) {
      cp_wait<kS - 1>();
      if constexpr (PASS == 2 || (PASS == 1 && ((ES & 2) || C::CF)) || C::F8 || C::MMA) __syncwarp();  // blocks copied by other lanes
      const Meta cur = md[s];
      if (cur.cnt == 0) return;  // stages are consumed in order: nothing after an empty one (no copy in flight)
      if constexpr (kTma) {
        mbar_wait(mbar + 8 * s, (phase >> s) & 1u);
        phase ^= 1u << s;
      }
      const char* st = stages + s * C::STAGE;
      if (cur.first) {
        const char* o = owns + s * C::OWNP;
        if constexpr (C::MMA) {
          if constexpr (PASS == 0) {
            mg.load_b(o, bq);   // q
            m = -INFINITY;      // per holder lane: its head's reference max; l its entry group's sum
            l = 0.f;
          } else if constexpr (PASS == 1) {
            lds_raw<W>(o + C::OWN_DY + lane * LB, ow);
            uint32_t yw[W];
            lds_raw<W>(o + C::OWN_Y + lane * LB, yw);
            // D_i = <dY_i, Y_i> (Sum_e P_e = 1); (m, l) = (LSE2, D) of head lane / LPH
            l = head_sum<LPH>(dot_raw<T, W>(ow, yw));
            m = reinterpret_cast<const float*>(o + C::OWN_LSE)[lane] * kLog2e;
            mh = __shfl_sync(kFull, m, LPH * mg.h);
            dh = __shfl_sync(kFull, l, LPH * mg.h);
            mg.load_b(o + C::OWN_DY, bq);   // dY
          }
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int i = 0; i < 4; ++i) macc[c][i] = 0.f;
          if constexpr (PASS == 2) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int i = 0; i < 4; ++i) macc2[(PASS == 2) ? c : 0][i] = 0.f;
          }
        } else if constexpr (PASS == 0) {
          lds_raw<W>(o + lane * LB, ow);
          if constexpr (C::F8) fo = a.qscale * exp2i(to_f16_norm<EPL, LPH>(ow, oh));
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
          m = -INFINITY;
          l = 0.f;
        } else if constexpr (PASS == 1 && C::CF) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
        } else if constexpr (PASS == 1) {
          if constexpr (!(ES & 2)) lds_raw<W>(o + lane * LB, ow2);
          lds_raw<W>(o + C::OWN_DY + lane * LB, ow);
          uint32_t yw[W];
          lds_raw<W>(o + C::OWN_Y + lane * LB, yw);
          // D_i = sum_e P_e dP_e = <dY_i, sum_e P_e v_j> = <dY_i, Y_i> (Sum_e P_e = 1)
          l = head_sum<LPH>(dot_raw<T, W>(ow, yw));
          m = reinterpret_cast<const float*>(o + C::OWN_LSE)[lane] * kLog2e;
          if constexpr (C::F8) {
            const int e = to_f16_norm<EPL, LPH>(ow, oh);
            fo = exp2i(e);
            ifo = exp2i(-e);
            if constexpr (!(ES & 2)) fq = a.qscale * exp2i(to_f16_norm<EPL, LPH>(ow2, oq));
          }
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
        } else {
          if constexpr (C::CF) {
            lds_raw<W>(o + lane * LB, ow2);      // v_j
          } else if constexpr (!(ES & 1)) {
            lds_raw<W>(o + lane * LB, ow);       // k_j
            lds_raw<W>(o + RB + lane * LB, ow2); // v_j
          }
#pragma unroll
          for (int i = 0; i < EPL; ++i) { acc[i] = 0.f; acc2[i] = 0.f; }
        }
      }
      const int cnt = cur.cnt;
      if constexpr (C::MMA && PASS == 0) {
        // Forward on the tensor cores (Mma): s = qscale <q_i, k_j> for the stage's 16 (head, neighbour)
        // pairs, base-2 online softmax against a per-head reference max m (raised only when a score
        // exceeds it by 2^kRescale: the warp-uniform rescale is rare), y += p v
        const uint32_t sa = st_sh + s * C::STAGE;
        const float sv = mg.dot(sa + mg.off_dot, bq) * a.qscale;
        const float sl = mg.holder ? (mg.u < cnt ? sv : -INFINITY) : 0.f;
        if constexpr (ES & 2)  // s2[entry e0 + u][head] for the row pass: one coalesced store per stage
          st_pred(a.es_out + (int64_t)cur.e0 * H + lane, __shfl_sync(kFull, sv, mg.src_e), lane < cnt * H);
        float smax = fmaxf(sl, __shfl_xor_sync(kFull, sl, 4));
        smax = fmaxf(smax, __shfl_xor_sync(kFull, smax, 8));
        const bool grow = smax > m + kRescale;
        if (__any_sync(kFull, grow)) {
          const float mn = grow ? smax : m;
          const float corr = ex2(m - mn);
          l *= corr;
          mg.scale(macc, __shfl_sync(kFull, corr, mg.t), __shfl_sync(kFull, corr, 16 + mg.t));
          m = mn;
        }
        const float p = ex2(sl - m);   // 0 for masked neighbours
        l += p;
        uint32_t b0, b1;
        mg.weights(p, lane, b0, b1);
        mg.spmm(sa + RB + mg.off_sp, b0, b1, macc);
      } else if constexpr (C::MMA && PASS == 1) {
        // Row pass on the tensor cores: dP = <dY_i, v_j>, p = 2^(s2 - LSE2_i) from the forward's logit,
        // dS = p (dP - D_i), (p, dS) stored per entry, dQ += dS k_j
        const uint32_t sa = st_sh + s * C::STAGE;
        const float dp = mg.dot(sa + RB + mg.off_dot, bq);
        const float s_ = reinterpret_cast<const float*>(st + U * EB)[mg.u * H + mg.h];
        const float p = mg.u < cnt ? ex2(s_ - mh) : 0.f;
        const float ds = p * (dp - dh);
        if constexpr (ES & 1)
          st_pred_u32(reinterpret_cast<uint32_t*>(a.es_out) + (int64_t)cur.e0 * H + lane,
                      __shfl_sync(kFull, pack_pd_bf16(p, ds), mg.src_e), lane < cnt * H);
        uint32_t b0, b1;
        mg.weights(ds, lane, b0, b1);
        mg.spmm(sa + mg.off_sp, b0, b1, macc);
      } else if constexpr (C::MMA && PASS == 2) {
        // Column pass on the tensor cores: dV_j += P dY_i, dK_j += dS q_i with the row pass's (P, dS)
        // (bf16x2 {lo P, hi dS}; zero-filled for masked neighbours) as block-diagonal B' registers
        const uint32_t sa = st_sh + s * C::STAGE;
        const uint32_t* aux = reinterpret_cast<const uint32_t*>(st + U * EB);
        const int hb = mg.t >> 1, u0 = 2 * (mg.t & 1);
        const uint32_t wa = aux[u0 * H + hb], wb = aux[(u0 + 1) * H + hb];
        const uint32_t wc = aux[u0 * H + hb + 2], wd = aux[(u0 + 1) * H + hb + 2];
        const uint32_t p0 = mg.b0on ? __byte_perm(wa, wb, 0x5410) : 0u, p1 = mg.b1on ? __byte_perm(wc, wd, 0x5410) : 0u;
        const uint32_t d0 = mg.b0on ? __byte_perm(wa, wb, 0x7632) : 0u, d1 = mg.b1on ? __byte_perm(wc, wd, 0x7632) : 0u;
        mg.spmm(sa + RB + mg.off_sp, p0, p1, macc2);
        mg.spmm(sa + mg.off_sp, d0, d1, macc);
      } else if constexpr (C::CF && PASS == 1) {
        // Column-first row pass: dQ_i += dS_e k_j with the column pass's dS (masked neighbours: zero-filled
        // rows and weights)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          uint32_t kw[W];
          lds_raw<W>(st + u * EB + lane * LB, kw);
          uint32_t w;
          if constexpr (sizeof(T) == 2) w = reinterpret_cast<const uint16_t*>(st + U * EB)[u * H + head];
          else w = reinterpret_cast<const uint32_t*>(st + U * EB)[u * H + head];
          accum<T, W, EPL>(w, kw, acc);
        }
      } else if constexpr (C::CF && PASS == 2) {
        // Column-first column pass: dP_e = <dY_i, v_j> with the column's own v_j,
        // P_e = 2^(s2_e - LSE2_i) from the forward's logit, dS_e = P_e (dP_e - D_i); dV_j += P_e dY_i,
        // dK_j += dS_e q_i (unscaled; weights rounded to T as in the stored-state pass); dS_e is stored at
        // the entry's CSR position for the row pass (rounded to T: the row pass's dQ weight)
        const float* s2x = reinterpret_cast<const float*>(st + U * EB);
        const uint32_t* pos = reinterpret_cast<const uint32_t*>(st + U * EB + U * H * 4);
        T* xd = reinterpret_cast<T*>(xs + s * C::XS);
        if constexpr (U == 4 && LPH >= 4) {
          using B = Bfly<LPH>;
          float part[4];
          uint32_t gws[4][W];   // dY_i slices, kept for dV (no second load)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            lds_raw<W>(st + C::template voff<false>(u) + lane * LB, gws[u]);
            part[u] = dot_raw<T, W>(gws[u], ow2);
          }
          const float dpl = B::reduce(part, lane);
          const float2 sd = *reinterpret_cast<const float2*>(st + cf_sd);
          const float pl = cf_ug < cnt ? ex2(*reinterpret_cast<const float*>(st + cf_s2) - sd.x) : 0.f;
          const float dsl = pl * (dpl - sd.y);
          {  // dS of the stage's entries to their CSR positions: lane f = u H + h, from a lane holding it
            const float x = __shfl_sync(kFull, dsl, cf_src);
            char* dst = const_cast<char*>(row_addr(reinterpret_cast<const char*>(a.es_out) + cf_eo,
                                                   *reinterpret_cast<const uint32_t*>(st + cf_pos), H * C::ESZ));
            if constexpr (sizeof(T) == 2)
              st_pred_u16(dst, __bfloat16_as_ushort(__float2bfloat16_rn(x)), lane < cnt * H);
            else
              st_pred_u32(reinterpret_cast<uint32_t*>(dst), __float_as_uint(x), lane < cnt * H);
          }
          if constexpr (sizeof(T) == 2) {
            const uint32_t wl = pack_pd_bf16(pl, dsl);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint32_t e = __shfl_sync(kFull, wl, cf_w[u]);
              uint32_t qw[W];
              lds_raw<W>(st + C::template koff<false>(u) + lane * LB, qw);
              accum<T, W, EPL, false>(e, gws[u], acc2);  // P (low half)
              accum<T, W, EPL, true>(e, qw, acc);        // dS (high half)
            }
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float pu = __shfl_sync(kFull, pl, cf_w[u]);
              const float du = __shfl_sync(kFull, dsl, cf_w[u]);
              uint32_t qw[W];
              lds_raw<W>(st + C::template koff<false>(u) + lane * LB, qw);
              const uint32_t (&gw)[W] = gws[u];
              accum<T, W, EPL>(__float_as_uint(pu), gw, acc2);
              accum<T, W, EPL>(__float_as_uint(du), qw, acc);
            }
          }
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            uint32_t qw[W], gw[W];
            lds_raw<W>(st + C::template koff<false>(u) + lane * LB, qw);
            lds_raw<W>(st + C::template voff<false>(u) + lane * LB, gw);
            const float2 sd = reinterpret_cast<const float2*>(st + C::template soff<false>(u))[head];
            const float dp = head_sum<LPH>(dot_raw<T, W>(gw, ow2));
            const float p = u < cnt ? ex2(s2x[u * H + head] - sd.x) : 0.f;
            const float ds = p * (dp - sd.y);
            xd[u * H + head] = T(ds);   // all lanes of a head write the same value
            if constexpr (sizeof(T) == 2) {
              const uint32_t e = pack_pd_bf16(p, ds);
              accum<T, W, EPL, false>(e, gw, acc2);
              accum<T, W, EPL, true>(e, qw, acc);
            } else {
              accum<T, W, EPL>(__float_as_uint(p), gw, acc2);
              accum<T, W, EPL>(__float_as_uint(ds), qw, acc);
            }
          }
        }
        // (head_sum branch) dS of the stage's entries to their CSR positions: lane f = u H + h stores one
        if constexpr (!(U == 4 && LPH >= 4)) {
          __syncwarp();
          const int f = lane < U * H ? lane : 0;
          if constexpr (sizeof(T) == 2)
            st_pred_u16(reinterpret_cast<uint16_t*>(a.es_out) + (int64_t)pos[f / H] * H + f % H,
                        reinterpret_cast<const uint16_t*>(xd)[f], lane < cnt * H);
          else
            st_pred_u32(reinterpret_cast<uint32_t*>(a.es_out) + (int64_t)pos[f / H] * H + f % H,
                        reinterpret_cast<const uint32_t*>(xd)[f], lane < cnt * H);
        }
      } else if constexpr (C::F8 && PASS == 0) {
        // fp8 forward: s = qscale 2^eq 2^ek_j <q', k8_j>, p~ = 2^(s - m), acc += f16(p~ 2^(ev_j - E_v)) v8_j
        // (y = acc 2^E_v / l); the dots are reduce-scattered by the butterfly as in the bf16 path, in
        // groups of 4 neighbours
        using B = Bfly<LPH>;
#pragma unroll
        for (int g0 = 0; g0 < U; g0 += 4) {
        float part[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint32_t kx[EPL / 4];
          lds_f8<EPL>(st + C::template koff<false>(g0 + u) + lane * C::LB8, kx);
          part[u] = dot_f8<EPL>(oh, kx);
        }
        const float r = B::reduce(part, lane);
        const int ug = g0 + B::group(lane);
        const float* scl = reinterpret_cast<const float*>(st + ug * EB + 2 * D);
        const float sv = r * fo * scl[head];
        const float sl = ug < cnt ? sv : -INFINITY;
        if constexpr (ES & 2) reinterpret_cast<float*>(xs + s * C::XS)[ug * H + head] = sv;
        const float mx = fmaxf(B::all_max(sl), m);
        const float corr = ex2(m - mx);
        l *= corr;
        scale2<EPL>(corr, acc);
        const float pl = ex2(sl - mx);
        l += pl;
        const uint32_t wl = f16_of(pl * scl[H + head] * irv);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t w = __shfl_sync(kFull, wl, B::src(lane, u));
          uint32_t vx[EPL / 4];
          lds_f8<EPL>(st + C::template voff<false>(g0 + u) + lane * C::LB8, vx);
          accum_f8<EPL>((uint16_t)w, vx, acc);
        }
        m = mx;
        }
        if constexpr (ES & 2) {  // s2 of the stage's entries: one coalesced store
          __syncwarp();
          const float* x = reinterpret_cast<const float*>(xs + s * C::XS);
          st_pred(a.es_out + (int64_t)cur.e0 * H + lane, x[lane < U * H ? lane : 0], lane < cnt * H);
        }
      } else if constexpr (C::F8 && PASS == 1) {
        // fp8 row pass: dP = 2^e_dy 2^ev_j <dY', v8_j>, p = 2^(s - lse2), dS = p (dP - D),
        // acc += f16(dS 2^-e_dy 2^(ek_j - E_k)) k8_j   (dQ = scale 2^e_dy 2^E_k acc)
        using B = Bfly<LPH>;
#pragma unroll
        for (int g0 = 0; g0 < U; g0 += 4) {
        float part[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint32_t vx[EPL / 4];
          lds_f8<EPL>(st + C::template voff<false>(g0 + u) + lane * C::LB8, vx);
          part[u] = dot_f8<EPL>(oh, vx);
        }
        const float dr = B::reduce(part, lane);
        const int ug = g0 + B::group(lane);
        const float* scl = reinterpret_cast<const float*>(st + ug * EB + 2 * D);
        const float dpl = dr * fo * scl[H + head];
        float s_;
        if constexpr (ES & 2) {
          s_ = reinterpret_cast<const float*>(st + U * EB)[ug * H + head];  // forward's logit
        } else {
          float pq[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint32_t kx[EPL / 4];
            lds_f8<EPL>(st + C::template koff<false>(g0 + u) + lane * C::LB8, kx);
            pq[u] = dot_f8<EPL>(oq, kx);
          }
          s_ = B::reduce(pq, lane) * fq * scl[head];
        }
        const float pl = ug < cnt ? ex2(s_ - m) : 0.f;
        const float dsl = pl * (dpl - l);
        if constexpr (ES & 1) {
          if constexpr (C::PDB == 4) reinterpret_cast<uint32_t*>(xs + s * C::XS)[ug * H + head] = pack_pd_bf16(pl, dsl);
          else reinterpret_cast<float2*>(xs + s * C::XS)[ug * H + head] = make_float2(pl, dsl);
        }
        const uint32_t wl = f16_of(dsl * ifo * scl[head] * irk);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t w = __shfl_sync(kFull, wl, B::src(lane, u));
          uint32_t kx[EPL / 4];
          lds_f8<EPL>(st + C::template koff<false>(g0 + u) + lane * C::LB8, kx);
          accum_f8<EPL>((uint16_t)w, kx, acc);
        }
        }
        if constexpr (ES & 1) {
          constexpr int NW = U * H * C::PDB / 4;
          constexpr int EW = H * C::PDB / 4;
          __syncwarp();
          const uint32_t* x = reinterpret_cast<const uint32_t*>(xs + s * C::XS);
          uint32_t* dst = reinterpret_cast<uint32_t*>(a.es_out) + (int64_t)cur.e0 * EW;
#pragma unroll
          for (int t = 0; t < (NW + 31) / 32; ++t) {
            const int f = lane + 32 * t;
            st_pred_u32(dst + f, x[f < NW ? f : 0], f < cnt * EW);
          }
        }
      } else if constexpr (PASS == 0 && kBfly) {
        // Transposed (reduce-scatter) butterfly over the head's lanes (Bfly): the 4 per-lane partial dot
        // products of the stage are summed so that each lane group ends up with one neighbour's full
        // score (14 instructions instead of 4 x 6 at 8 lanes per head); max and exp are then taken once
        // per lane, and the 4 weights broadcast back for the SpMM.  l is kept per lane group and summed
        // over the groups at the end of the row.
        float part[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint32_t kw[W];
          lds_raw<W>(st + C::template koff<kTma>(u) + lane * LB, kw);
          part[u] = dot_raw<T, W>(ow, kw);
        }
        using B = Bfly<LPH>;
        const float r = B::reduce(part, lane);
        const int ug = B::group(lane);  // this lane's neighbour
        const float sv = r * a.qscale;
        const float sl = ug < cnt ? sv : -INFINITY;
        if constexpr (ES & 2) {  // s2[entry e0 + u][head] for the row pass: one coalesced store per stage
          reinterpret_cast<float*>(xs + s * C::XS)[ug * H + head] = sv;  // lanes b0 = 0, 1 agree
          __syncwarp();
          const float* x = reinterpret_cast<const float*>(xs + s * C::XS);
          st_pred(a.es_out + (int64_t)cur.e0 * H + lane, x[lane < U * H ? lane : 0], lane < cnt * H);
        }
        const float mx = fmaxf(B::all_max(sl), m);
        const float corr = ex2(m - mx);
        l *= corr;
        scale2<EPL>(corr, acc);
        const float pl = ex2(sl - mx);  // 0 for masked neighbours
        l += pl;
        const uint32_t wl = wpack<T>(pl);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t w = __shfl_sync(kFull, wl, B::src(lane, u));
          uint32_t vw[W];
          lds_raw<W>(st + C::template voff<kTma>(u) + lane * LB, vw);
          accum<T, W, EPL>(w, vw, acc);
        }
        m = mx;
      } else if constexpr (PASS == 0) {
        float sc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          uint32_t kw[W];
          lds_raw<W>(st + C::template koff<kTma>(u) + lane * LB, kw);
          const float sv = head_sum<LPH>(dot_raw<T, W>(ow, kw)) * a.qscale;
          sc[u] = u < cnt ? sv : -INFINITY;
          if constexpr (ES & 2) reinterpret_cast<float*>(xs + s * C::XS)[u * H + head] = sv;  // head lanes agree
        }
        if constexpr (ES & 2) {  // s2[entry e0 + u][head] for the row pass: one coalesced store per stage
          __syncwarp();
          const float* x = reinterpret_cast<const float*>(xs + s * C::XS);
          st_pred(a.es_out + (int64_t)cur.e0 * H + lane, x[lane < U * H ? lane : 0], lane < cnt * H);
        }
        float mx = m;
#pragma unroll
        for (int u = 0; u < U; ++u) mx = fmaxf(mx, sc[u]);
        const float corr = ex2(m - mx);
        l *= corr;
        scale2<EPL>(corr, acc);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float p = ex2(sc[u] - mx);  // 0 for masked neighbours
          l += p;
          uint32_t vw[W];
          lds_raw<W>(st + C::template voff<kTma>(u) + lane * LB, vw);
          accum<T, W, EPL>(wpack<T>(p), vw, acc);
        }
        m = mx;
      } else if constexpr (PASS == 1) {
        // Row pass: p_e = 2^(s2_e - lse2_i), dP_e = <dY_i, v_j>, dS_e = p_e (dP_e - D_i) (unscaled),
        // dQ_i += dS_e k_j; (p, dS) stored per entry for the column pass.
        if constexpr (kBflyR) {
          // the 4 partial dP are reduced by the transposed butterfly (each lane group ends with one
          // neighbour's dP); p and dS are computed once per lane for that neighbour
          float part[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint32_t vw[W];
            lds_raw<W>(st + C::template voff<kTma>(u) + lane * LB, vw);
            part[u] = dot_raw<T, W>(ow, vw);
          }
          using B = Bfly<LPH>;
          const float dpl = B::reduce(part, lane);
          const int ug = B::group(lane);
          const float s_ = reinterpret_cast<const float*>(st + U * EB)[ug * H + head];  // forward's logit
          const float pl = ug < cnt ? ex2(s_ - m) : 0.f;
          const float dsl = pl * (dpl - l);
          if constexpr (ES & 1) {  // lanes b0 = 0, 1 write the same bytes
            if constexpr (C::PDB == 4) reinterpret_cast<uint32_t*>(xs + s * C::XS)[ug * H + head] = pack_pd_bf16(pl, dsl);
            else reinterpret_cast<float2*>(xs + s * C::XS)[ug * H + head] = make_float2(pl, dsl);
          }
          const uint32_t wl = wpack<T>(dsl);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t w = __shfl_sync(kFull, wl, B::src(lane, u));
            uint32_t kw[W];
            lds_raw<W>(st + C::template koff<kTma>(u) + lane * LB, kw);
            accum<T, W, EPL>(w, kw, acc);
          }
        } else {
          float pv[U], dsv[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            uint32_t kw[W], vw[W];
            lds_raw<W>(st + C::template koff<kTma>(u) + lane * LB, kw);
            lds_raw<W>(st + C::template voff<kTma>(u) + lane * LB, vw);
            float s_;
            if constexpr (ES & 2) s_ = reinterpret_cast<const float*>(st + U * EB)[u * H + head];  // forward's logit
            else s_ = head_sum<LPH>(dot_raw<T, W>(ow2, kw)) * a.qscale;
            const float dp = head_sum<LPH>(dot_raw<T, W>(ow, vw));
            pv[u] = u < cnt ? ex2(s_ - m) : 0.f;
            dsv[u] = pv[u] * (dp - l);
            if constexpr (ES & 1) {  // all lanes of a head write the same bytes
              if constexpr (C::PDB == 4)
                reinterpret_cast<uint32_t*>(xs + s * C::XS)[u * H + head] = pack_pd_bf16(pv[u], dsv[u]);
              else reinterpret_cast<float2*>(xs + s * C::XS)[u * H + head] = make_float2(pv[u], dsv[u]);
            }
            accum<T, W, EPL>(wpack<T>(dsv[u]), kw, acc);
          }
        }
        if constexpr (ES & 1) {
          // (P, dS)[entry e0 + u][head] of the stage, transposed through shared memory and written with
          // one coalesced store per 32 words (the stage's scratch is rewritten two stages later, after
          // another __syncwarp).
          constexpr int NW = U * H * C::PDB / 4;   // words of the stage
          constexpr int EW = H * C::PDB / 4;       // words per entry
          __syncwarp();
          const uint32_t* x = reinterpret_cast<const uint32_t*>(xs + s * C::XS);
          uint32_t* dst = reinterpret_cast<uint32_t*>(a.es_out) + (int64_t)cur.e0 * EW;
#pragma unroll
          for (int t = 0; t < (NW + 31) / 32; ++t) {
            const int f = lane + 32 * t;
            st_pred_u32(dst + f, x[f < NW ? f : 0], f < cnt * EW);
          }
        }
      } else {
        // Column pass: dV_j += p_e dY_i, dK_j += dS_e q_i (unscaled), with (p, dS) stored by the row pass
        // or recomputed from q_i, dY_i, (LSE2_i, D_i) and the column's own k_j, v_j.
#pragma unroll
        for (int u = 0; u < U; ++u) {
          uint32_t qw[W], gw[W];
          lds_raw<W>(st + C::template koff<kTma>(u) + lane * LB, qw);
          lds_raw<W>(st + C::template voff<kTma>(u) + lane * LB, gw);
          if constexpr (ES & 1) {  // stored by the row pass; zero-filled for masked neighbours
            if constexpr (C::PDB == 4) {
              const uint32_t e = reinterpret_cast<const uint32_t*>(st + U * EB)[u * H + head];
              accum<T, W, EPL, false>(e, gw, acc2);  // P (low half)
              accum<T, W, EPL, true>(e, qw, acc);    // dS (high half)
            } else {
              const float2 e = reinterpret_cast<const float2*>(st + U * EB)[u * H + head];
              accum<T, W, EPL>(__float_as_uint(e.x), gw, acc2);
              accum<T, W, EPL>(__float_as_uint(e.y), qw, acc);
            }
          } else {
            const float2 sd = reinterpret_cast<const float2*>(st + C::template soff<kTma>(u))[head];
            const float s_ = head_sum<LPH>(dot_raw<T, W>(qw, ow)) * a.qscale;
            const float dp = head_sum<LPH>(dot_raw<T, W>(gw, ow2));
            const float p = u < cnt ? ex2(s_ - sd.x) : 0.f;
            const float ds = p * (dp - sd.y);
            if constexpr (sizeof(T) == 2) {
              const uint32_t e = pack_pd_bf16(p, ds);
              accum<T, W, EPL, false>(e, gw, acc2);
              accum<T, W, EPL, true>(e, qw, acc);
            } else {
              accum<T, W, EPL>(__float_as_uint(p), gw, acc2);
              accum<T, W, EPL>(__float_as_uint(ds), qw, acc);
            }
          }
        }
      }
      if (cur.last) {
        const int32_t own = cur.own;
        const int64_t r = own >= 0 ? own : 0;
        if constexpr (PASS == 1 && !C::CF) {  // (LSE2, D) of the row (every chunk of a heavy row writes the same values)
          const int64_t rr = own >= 0 ? own : a.cown[-1 - (int64_t)own];
          reinterpret_cast<float2*>(reinterpret_cast<char*>(a.out_f) + rr * C::SB)[head] = make_float2(m, l);
        }
        if constexpr (C::MMA) {
          // accumulators from the holder lanes' fragments (Mma::elem); chunks: fp32 partial states in the
          // layout the merge kernels read
          const int64_t ch = own < 0 ? -1 - (int64_t)own : 0;
          if constexpr (PASS == 0) {
            float lt = l + __shfl_xor_sync(kFull, l, 4);   // the head's sum over its 4 entry groups
            lt += __shfl_xor_sync(kFull, lt, 8);
            const bool first_u = mg.holder && mg.u == 0;
            if (own < 0) {
              float* pp = a.part + ch * (int64_t)(D + 2 * H);
              st_pred(pp + D + 2 * mg.h, m, first_u);
              st_pred(pp + D + 2 * mg.h + 1, lt, first_u);
              mg.store_f32(pp, macc);
            } else {
              const float le = __shfl_sync(kFull, lt, mg.t), lo = __shfl_sync(kFull, lt, 16 + mg.t);
              mg.store_bf16(a.out_a + r * RB, macc, 1.f / le, 1.f / lo);
              st_pred(a.out_f + r * H + mg.h, (m + __log2f(lt)) * kLn2, first_u);
            }
          } else if constexpr (PASS == 1) {
            if (own < 0) mg.store_f32(a.part + ch * (int64_t)D, macc);
            else mg.store_bf16(a.out_a + r * RB, macc, a.scale, a.scale);
          } else {
            if (own < 0) {
              float* pp = a.part + ch * (int64_t)(2 * D);
              mg.store_f32(pp, macc);
              mg.store_f32(pp + D, macc2);
            } else {
              mg.store_bf16(a.out_a + r * RB, macc, a.scale, a.scale);
              mg.store_bf16(a.out_b + r * RB, macc2, 1.f, 1.f);
            }
          }
        } else if (own < 0) {  // chunk of a heavy row/column: partial state for the merge kernel
          const int64_t ch = -1 - (int64_t)own;
          if constexpr (PASS == 0 && kBfly) l = Bfly<LPH>::all_sum(l);  // per lane group -> the row's (chunk's) l
          if constexpr (PASS == 0) {
            float* pp = a.part + ch * (int64_t)(D + 2 * H);
#pragma unroll
            for (int i = 0; i < EPL; ++i) pp[lane * EPL + i] = C::F8 ? acc[i] * rv : acc[i];
            { pp[D + 2 * head] = m; pp[D + 2 * head + 1] = l; }
          } else if constexpr (PASS == 1) {
            float* pp = a.part + ch * (int64_t)D;
#pragma unroll
            for (int i = 0; i < EPL; ++i) pp[lane * EPL + i] = C::F8 ? acc[i] * (fo * rk) : acc[i];
          } else {
            float* pp = a.part + ch * (int64_t)(2 * D);
#pragma unroll
            for (int i = 0; i < EPL; ++i) { pp[lane * EPL + i] = acc[i]; pp[D + lane * EPL + i] = acc2[i]; }
          }
        } else {
          if constexpr (PASS == 0 && kBfly) l = Bfly<LPH>::all_sum(l);
          if constexpr (PASS == 0) {
            const float inv = (C::F8 ? rv : 1.f) / l;
#pragma unroll
            for (int i = 0; i < EPL; ++i) acc[i] *= inv;
            stg_f32<T, EPL>(a.out_a + r * RB + lane * LB, acc);
            a.out_f[r * H + head] = (m + __log2f(l)) * kLn2;
          } else if constexpr (PASS == 1) {
            const float f = C::F8 ? a.scale * fo * rk : a.scale;
#pragma unroll
            for (int i = 0; i < EPL; ++i) acc[i] *= f;
            stg_f32<T, EPL>(a.out_a + r * RB + lane * LB, acc);
          } else {
#pragma unroll
            for (int i = 0; i < EPL; ++i) acc[i] *= a.scale;
            stg_f32<T, EPL>(a.out_a + r * RB + lane * LB, acc);
            stg_f32<T, EPL>(a.out_b + r * RB + lane * LB, acc2);
          }
        }
      }
      // stage blocks other lanes read (entry state, stats) are refilled by the lanes that copy them:
      // order those reads before the new copies (formally, under independent thread scheduling)
      if constexpr (PASS == 2 || (PASS == 1 && ((ES & 2) || C::CF)) || C::F8 || C::MMA) __syncwarp();
      md[s] = produce(s);   // refill the stage just consumed
      cp_commit();
    }
  }
}

// Outputs of rows (columns) without entries (reading Z4): Y = 0 and LSE = -inf (pass 0); dQ = 0 and
// (LSE2, D) = (-inf, 0) (pass 1); dK = dV = 0 (pass 2).  One warp per id, grid-stride.
template <int PASS>
__global__ void __launch_bounds__(256) fill_empty_kernel(const int32_t* ids, int64_t n, char* out_a, char* out_b,
                                                         float* out_f, int64_t rb, int heads, int sb) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < n; x += nw) {
    const int64_t r = ids[x];
    for (int64_t c = lane * 16; c < rb; c += 32 * 16) {
      *reinterpret_cast<uint4*>(out_a + r * rb + c) = make_uint4(0, 0, 0, 0);
      if constexpr (PASS == 2) *reinterpret_cast<uint4*>(out_b + r * rb + c) = make_uint4(0, 0, 0, 0);
    }
    if constexpr (PASS == 0) {
      if (lane < heads) out_f[r * heads + lane] = -INFINITY;
    } else if constexpr (PASS == 1) {
      if (lane < heads)
        reinterpret_cast<float2*>(reinterpret_cast<char*>(out_f) + r * sb)[lane] = make_float2(-INFINITY, 0.f);
    }
  }
}

// (LSE2, D) of every row for the column-first backward (D_i = sum_e P_e dP_e =
// <dY_i, Y_i> since sum_e P_e = 1), the values the row pass of the row-first order writes (same products,
// same order); rows without entries get (-inf, 0) (their LSE is -inf, their Y 0).  One warp per row.
template <typename T, int H, int D>
__global__ void __launch_bounds__(256) row_stats_kernel(const char* y, const char* dy, const float* lse, int64_t n,
                                                        char* stats, int sb) {
  using C = PC<T, H, D, 1, 0>;
  constexpr int W = C::W, LB = C::LB, LPH = C::LPH, RB = C::RB;
  const int lane = threadIdx.x & 31, head = lane / LPH;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    uint32_t yw[W], gw[W];
    lds_raw<W>(y + r * RB + lane * LB, yw);
    lds_raw<W>(dy + r * RB + lane * LB, gw);
    const float d = head_sum<LPH>(dot_raw<T, W>(gw, yw));
    if (lane % LPH == 0) reinterpret_cast<float2*>(stats + r * sb)[head] = make_float2(lse[r * H + head] * kLog2e, d);
  }
}

template <typename T, int H, int D>
gt_status row_stats_run(const void* y, const void* dy, const float* lse, int64_t n, float* stats, int sb,
                        cudaStream_t st) {
  if (n <= 0) return GT_OK;
  const int blocks = (int)std::min<int64_t>((n * 32 + 255) / 256, 148 * 8);
  row_stats_kernel<T, H, D><<<blocks, 256, 0, st>>>((const char*)y, (const char*)dy, lse, n, (char*)stats, sb);
  GT_CUDA_TRY(cudaGetLastError());
  return GT_OK;
}

gt_status fill_empty(int pass, const int32_t* ids, int64_t n, char* out_a, char* out_b, float* out_f, int64_t rb,
                     int heads, int sb, cudaStream_t st) {
  if (n <= 0) return GT_OK;
  const int blocks = (int)std::min<int64_t>((n * 32 + 255) / 256, 148 * 8);
  if (pass == 0) fill_empty_kernel<0><<<blocks, 256, 0, st>>>(ids, n, out_a, out_b, out_f, rb, heads, sb);
  else if (pass == 1) fill_empty_kernel<1><<<blocks, 256, 0, st>>>(ids, n, out_a, out_b, out_f, rb, heads, sb);
  else fill_empty_kernel<2><<<blocks, 256, 0, st>>>(ids, n, out_a, out_b, out_f, rb, heads, sb);
  GT_CUDA_TRY(cudaGetLastError());
  return GT_OK;
}

// ------------------------------------------------------------ fp8 K||V table --
// gt_opts.kv_fp8 (NEXT-4): K and V quantised per (row, head) to e4m3 with a power-of-two scale 2^e,
// e the smallest integer with max |x| <= 448 2^e (448 = e4m3's largest finite value), x8 = RNE(x 2^-e)
// (exact scaling, one rounding; reading Z25).  Row layout [k8 | v8 | 2^ek f32[H] | 2^ev f32[H]], padded
// to 16 B; ref = {max ek, max ev} over the table (the kernels' f16 weights are taken relative to it).
template <int H, int D>
__global__ void __launch_bounds__(256) quantize_kv_kernel(const uint32_t* k, const uint32_t* v, int64_t n, char* out,
                                                          int gr, int* ref) {
  constexpr int EPL = D / 32, LPH = 32 / H, W = EPL / 2;
  const int lane = threadIdx.x & 31, head = lane / LPH;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int emax[2] = {-126, -126};
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint32_t* src = (t ? v : k) + r * (D / 2) + lane * W;
      float f[EPL];
#pragma unroll
      for (int i = 0; i < W; ++i) {
        const uint32_t x = __ldg(src + i);
        f[2 * i] = __uint_as_float(x << 16);
        f[2 * i + 1] = __uint_as_float(x & 0xffff0000u);
      }
      float am = 0.f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) am = fmaxf(am, fabsf(f[i]));
#pragma unroll
      for (int o = LPH / 2; o >= 1; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
      int e = -126;
      if (am > 0.f) {
        const int bits = __float_as_int(am);
        const int E = ((bits >> 23) & 0xff) - 127;
        e = (bits & 0x7fffff) <= 0x600000 ? E - 8 : E - 7;   // 1.m 2^E <= 1.75 2^(8 + e), e minimal
        e = max(-126, min(126, e));
      }
      emax[t] = max(emax[t], e);
      const float sc = __int_as_float((127 - e) << 23);    // 2^-e
      uint32_t w8[EPL / 4];
#pragma unroll
      for (int i = 0; i < EPL / 2; ++i) {
        uint16_t b;
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(b) : "f"(f[2 * i + 1] * sc), "f"(f[2 * i] * sc));
        if (i % 2 == 0) w8[i / 2] = b;
        else w8[i / 2] |= (uint32_t)b << 16;
      }
      char* dst = out + r * gr + t * D + lane * (EPL);
      if constexpr (EPL / 4 == 4) *reinterpret_cast<uint4*>(dst) = make_uint4(w8[0], w8[1], w8[2], w8[3]);
      else if constexpr (EPL / 4 == 2) *reinterpret_cast<uint2*>(dst) = make_uint2(w8[0], w8[1]);
      else *reinterpret_cast<uint32_t*>(dst) = w8[0];
      if (lane % LPH == 0)
        reinterpret_cast<float*>(out + r * gr + 2 * D)[t * H + head] = __int_as_float((e + 127) << 23);
    }
  }
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    int x = emax[t];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) atomicMax(ref + t, x);
  }
}

gt_status quantize_kv_impl(int H, int D, const void* k, const void* v, int64_t n, void* out, int gr, int* ref,
                           cudaStream_t st) {
  GT_CUDA_TRY(cudaMemsetAsync(ref, 0x80, 2 * sizeof(int), st));  // INT_MIN-like start for the max
  if (n <= 0) return GT_OK;
  const int blocks = (int)std::min<int64_t>((n * 32 + 255) / 256, 148 * 16);
#define GT_Q(HH, DD)                                                                                         \
  if (H == HH && D == DD) {                                                                                  \
    quantize_kv_kernel<HH, DD><<<blocks, 256, 0, st>>>((const uint32_t*)k, (const uint32_t*)v, n, (char*)out, gr, \
                                                       ref);                                                 \
    GT_CUDA_TRY(cudaGetLastError());                                                                         \
    return GT_OK;                                                                                            \
  }
  GT_Q(1, 128) GT_Q(2, 128) GT_Q(4, 128) GT_Q(8, 128) GT_Q(1, 256) GT_Q(2, 256) GT_Q(4, 256) GT_Q(8, 256)
  GT_Q(1, 512) GT_Q(2, 512) GT_Q(4, 512) GT_Q(8, 512)
#undef GT_Q
  return fail(GT_ECONFIG, "kv_fp8: unsupported (heads, heads * d)");
}

// ----------------------------------------------------------------- launcher --
// Tensor map of a gathered table: `rows` rows of D elements, `stride` bytes apart; box = one row (the
// gather4 instruction supplies 4 row coordinates).  Encoded on the host per launch (pointers change).
static gt_status encode_rows(CUtensorMap* m, const void* base, int64_t rows, int D, int elt, int64_t stride) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!enc) return fail(GT_ECUDA, "cuTensorMapEncodeTiled is not available");
  const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)std::max<int64_t>(rows, 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)stride};
  const cuuint32_t box[2] = {(cuuint32_t)D, 1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, elt == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                         const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(GT_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return GT_OK;
}

template <typename T, int H, int D, int PASS, bool HALO, int ES>
gt_status launch(const PArgs& a, cudaStream_t st, int reserve_sms) {
  using C = PC<T, H, D, PASS, ES>;
  // per device (the smem attribute and the SM count are per device; plans may live on several)
  static std::mutex mu;
  static int grid_of[kMaxDevices] = {}, sms_of[kMaxDevices] = {};
  const size_t smem = (size_t)kWarps * C::WARP_SMEM;
  int dev = 0;
  GT_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(GT_ECONFIG, "device ordinal out of range");
  int grid = 0, sms = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!grid_of[dev]) {
      auto k = pipe_kernel<T, H, D, PASS, HALO, ES>;
      GT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if (GT_CARVEOUT >= 0)
        GT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, GT_CARVEOUT));
      int per = 0;
      GT_CUDA_TRY(cudaDeviceGetAttribute(&sms_of[dev], cudaDevAttrMultiProcessorCount, dev));
      GT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kWarps * 32, smem));
      if (const char* cap = std::getenv("GT_CTAS_PER_SM"))  // tuning: narrower in-flight window of rows
        per = std::min(per, std::max(1, std::atoi(cap)));
      grid_of[dev] = sms_of[dev] * std::max(per, 1);
    }
    grid = grid_of[dev];
    sms = sms_of[dev];
  }
  if (a.nitems <= 0) return GT_OK;
  const int64_t want = (a.nitems + kG - 1) / kG;
  int cap = grid;
  if (reserve_sms > 0)  // leave SMs free for concurrent communication kernels (overlap phases)
    cap = std::max(1, grid - grid / sms * reserve_sms);
  const int g = (int)std::min<int64_t>(cap, (want + kWarps - 1) / kWarps);
  TmaMaps tm;
  std::memset(&tm, 0, sizeof(tm));
  if constexpr (C::TMA && !HALO) {
    GT_TRY(encode_rows(&tm.a, a.ga, a.n_local, D, (int)sizeof(T), C::RB));
    GT_TRY(encode_rows(&tm.b, a.gb, a.n_local, D, (int)sizeof(T), C::RB));
  }
  GT_CUDA_TRY(cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), st));
  if (a.win && a.win_bytes > 0) {  // hot-column table: persisting in L2 for this launch
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(kWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeAccessPolicyWindow;
    at[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(a.win);
    at[0].val.accessPolicyWindow.num_bytes = (size_t)a.win_bytes;
    at[0].val.accessPolicyWindow.hitRatio = 1.0f;
    at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    GT_CUDA_TRY(cudaLaunchKernelEx(&cfg, pipe_kernel<T, H, D, PASS, HALO, ES>, a, tm));
    return GT_OK;
  }
  pipe_kernel<T, H, D, PASS, HALO, ES><<<g, kWarps * 32, smem, st>>>(a, tm);
  GT_CUDA_TRY(cudaGetLastError());
  return GT_OK;
}

template <typename T, int H, int D>
struct Ops {
  // ES bits: 1 = (P, dS) materialised (rowb stores, colb reads), 2 = logits materialised (fwd stores,
  // rowb reads)
  static gt_status run(int pass, const PArgs& a, cudaStream_t st, int rs) {
    if (a.mode == 1) {  // column-first backward (world 1, stored logits; dS rows of >= 4 bytes per entry)
      if constexpr (H * sizeof(T) >= 4) {
        if (pass == 1) return launch<T, H, D, 1, false, 8>(a, st, rs);
        if (pass == 2) return launch<T, H, D, 2, false, 8>(a, st, rs);
      }
      return fail(GT_ECONFIG, "column-first backward: unsupported pass / shape");
    }
    if (a.kvref) {  // fp8 K||V gathers (world 1, bf16, heads * d >= 128)
      if constexpr (sizeof(T) == 2 && D >= 128) {
        if (pass == 0) return a.es_out ? launch<T, H, D, 0, false, 6>(a, st, rs) : launch<T, H, D, 0, false, 4>(a, st, rs);
        if (pass == 1 && a.es_out)
          return a.es_in ? launch<T, H, D, 1, false, 7>(a, st, rs) : launch<T, H, D, 1, false, 5>(a, st, rs);
      }
      return fail(GT_ECONFIG, "kv_fp8: unsupported pass / shape");
    }
    if (pass == 0) {
      if (a.halo) return a.es_out ? launch<T, H, D, 0, true, 2>(a, st, rs) : launch<T, H, D, 0, true, 0>(a, st, rs);
      return a.es_out ? launch<T, H, D, 0, false, 2>(a, st, rs) : launch<T, H, D, 0, false, 0>(a, st, rs);
    }
    if (pass == 1) {
      const int m = (a.es_out ? 1 : 0) | (a.es_in ? 2 : 0);
      if (a.halo) {
        if (m == 3) return launch<T, H, D, 1, true, 3>(a, st, rs);
        if (m == 1) return launch<T, H, D, 1, true, 1>(a, st, rs);
        if (m == 2) return launch<T, H, D, 1, true, 2>(a, st, rs);
        return launch<T, H, D, 1, true, 0>(a, st, rs);
      }
      if (m == 3) return launch<T, H, D, 1, false, 3>(a, st, rs);
      if (m == 1) return launch<T, H, D, 1, false, 1>(a, st, rs);
      if (m == 2) return launch<T, H, D, 1, false, 2>(a, st, rs);
      return launch<T, H, D, 1, false, 0>(a, st, rs);
    }
    if (a.halo) return launch<T, H, D, 2, true, 0>(a, st, rs);
    return a.es_in ? launch<T, H, D, 2, false, 1>(a, st, rs) : launch<T, H, D, 2, false, 0>(a, st, rs);
  }
};

gt_status dispatch(int dtype, int H, int D, int pass, const PArgs& a, cudaStream_t st, int rs) {
#define GT_CASE(TT, HH, DD) \
  if (H == HH && D == DD) return Ops<TT, HH, DD>::run(pass, a, st, rs);
#ifdef GT_QUICK_ONE_SHAPE  // tooling: SASS inspection of the products shape only
#define GT_HCASES(TT) GT_CASE(TT, 4, 256)
#else
#define GT_HCASES(TT)                                                                              \
  GT_CASE(TT, 1, 64) GT_CASE(TT, 2, 64) GT_CASE(TT, 4, 64) GT_CASE(TT, 8, 64)                        \
  GT_CASE(TT, 1, 128) GT_CASE(TT, 1, 256) GT_CASE(TT, 1, 512) GT_CASE(TT, 2, 128) GT_CASE(TT, 2, 256) \
  GT_CASE(TT, 2, 512) GT_CASE(TT, 4, 128) GT_CASE(TT, 4, 256) GT_CASE(TT, 4, 512) GT_CASE(TT, 8, 128) \
  GT_CASE(TT, 8, 256) GT_CASE(TT, 8, 512)
#endif
  if (dtype == GT_F32) { GT_HCASES(float) }
  else { GT_HCASES(__nv_bfloat16) }
#undef GT_HCASES
#undef GT_CASE
  return fail(GT_ECONFIG, "unsupported (dtype, heads, heads*d)");
}

gt_status row_stats_dispatch(int dtype, int H, int D, const void* y, const void* dy, const float* lse, int64_t n,
                             float* stats, int sb, cudaStream_t st) {
#define GT_CASE(TT, HH, DD) \
  if (H == HH && D == DD) return row_stats_run<TT, HH, DD>(y, dy, lse, n, stats, sb, st);
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

}  // namespace pipe

gt_status row_stats(int dtype, int H, int D, const void* y, const void* dy, const float* lse, int64_t n, float* stats,
                    int sb, cudaStream_t st) {
  return pipe::row_stats_dispatch(dtype, H, D, y, dy, lse, n, stats, sb, st);
}

gt_status quantize_kv(int H, int D, const void* k, const void* v, int64_t n, void* out, int gr, int* ref,
                      cudaStream_t st) {
  return pipe::quantize_kv_impl(H, D, k, v, n, out, gr, ref, st);
}

// Runs one pass of the pipelined kernel over the work list `w` (chunks of `ct` write partial states
// to `part`; their merges are launched by the caller).
gt_status pipe_pass(gt_plan_s* P, int pass, const WorkList& w, const ChunkTable& ct, float* part, const void* own_a,
                    const void* own_b, const float* lse, const void* gather_a, const void* gather_b, const void* halo,
                    const void* halo_s, void* out_a, void* out_b, float* out_f, cudaStream_t st, int reserve_sms,
                    const EntryState& es, const ItemRange& range) {
  pipe::PArgs a{};
  const bool rows = pass != 2;
  const int64_t t0 = std::min<int64_t>(range.t0, w.n), t1 = range.t1 < 0 ? w.n : std::min<int64_t>(range.t1, w.n);
  a.ibeg = w.d_beg.as<int64_t>() + t0;
  a.iend = w.d_end.as<int64_t>() + t0;
  a.iown = w.d_own.as<int32_t>() + t0;
  a.nitems = std::max<int64_t>(t1 - t0, 0);
  a.cown = ct.d_owner.as<int32_t>();
  a.nbr = es.nbr ? es.nbr : (rows ? P->d_col : P->d_row).as<int32_t>();
  a.nnbr = es.nbr ? es.nnbr : (rows ? P->nnz_local : P->nnz_in_local);
  a.own_stride = es.own_stride ? es.own_stride : (int64_t)P->heads * P->d * (P->dtype == GT_F32 ? 4 : 2);
  a.counter = w.d_counter.as<unsigned long long>();
  a.ga = (const char*)gather_a;
  a.gb = (const char*)gather_b;
  a.gs = (const char*)P->d_stats.p;
  a.halo = (const char*)halo;
  a.halo_s = (const char*)halo_s;
  a.halo_stride = P->kv_row_bytes;  // [k | v] and [q | dy] rows have the same size
  a.n_local = P->n_local;
  a.oa = (const char*)own_a;
  a.ob = (const char*)own_b;
  a.oc = (const char*)es.own_c;
  a.lse = lse;
  a.out_a = (char*)out_a;
  a.out_b = (char*)out_b;
  a.out_f = out_f;
  a.part = part;
  a.qscale = P->scale * pipe::kLog2e;
  a.scale = P->scale;
  a.peer_shift = (P->peer && halo) ? P->peer_shift : 0;
  a.rb = (uint32_t)((int64_t)P->heads * P->d * (P->dtype == GT_F32 ? 4 : 2));
  a.rb2 = 2 * a.rb;
  a.sb = (uint32_t)P->st_row_bytes;
  for (int s = 0; s < 8; ++s) {
    a.peer[s] = (const char*)(pass < 2 ? P->peer_base[s] : P->peer_qd[s]);
    a.peer_s[s] = (const char*)P->peer_st[s];
  }
  a.es_out = es.out;
  a.es_in = es.in;
  a.src = es.src;
  a.win = es.win;
  a.win_bytes = es.win_bytes;
  a.mode = es.mode;
  if (es.kv8 && pass < 2) {  // fp8 K||V table replaces the two gathered tables
    a.ga = (const char*)es.kv8;
    a.gb = nullptr;
    a.rb = (uint32_t)es.kv8_row;
    a.kvref = es.kvref;
  }
  if (range.fill && !w.empty.empty())
    GT_TRY(pipe::fill_empty(pass, w.d_empty.as<int32_t>(), (int64_t)w.empty.size(), (char*)out_a, (char*)out_b,
                            out_f, (int64_t)P->heads * P->d * (P->dtype == GT_F32 ? 4 : 2), P->heads,
                            (int)P->st_row_bytes, st));
  return pipe::dispatch(P->dtype, P->heads, P->heads * P->d, pass, a, st, reserve_sms);
}

}  // namespace gt
