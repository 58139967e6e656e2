// Fused sparse graph attention kernels for sm_100a (B200).
//
//   K1  fwd_kernel      SDDMM + online edge softmax + SpMM per row (Eq. 2, 4, 5)
//   K3  rowb_kernel     backward row pass: SDDMM dP = <dY_i, v_j>, softmax backward, SpMM dQ
//   K4  colb_kernel     backward column pass over A^T: SpMM dV = U^T dY, SpMM dK = dS^T Q
//   K6  *_merge_kernel  combine the partial states of rows/columns split into chunks
//
// Layout: every feature tensor is [rows, H, d] row-major, D = H * d elements per row.  One warp
// owns one row (or chunk): lane l holds elements [l*EPL, (l+1)*EPL) of the row, EPL = D / 32, so
// a row is one fully coalesced 32 x (EPL * sizeof(T)) byte access and head t is lanes
// [t*LPH, (t+1)*LPH), LPH = 32 / H.  Per-head dot products reduce with log2(LPH) xor-shuffles.
// Neighbour rows are gathered with 128-bit non-coherent loads, U edges per batch.  No tensor
// cores: each edge is an independent d-length dot product and axpy, not a dense contraction.
//
// Softmax runs in base 2: q is pre-multiplied by scale * log2(e), so p = exp2(s - m) with one
// FFMA-free ex2.approx.  LSE is returned in natural-log units (gt.h).  Accumulation is fp32;
// outputs are rounded to the storage dtype with round-to-nearest-even.
//
// Rows (columns) with more than `heavy` entries are split into chunks processed by separate
// warps that write partial states to a workspace; a merge kernel combines them in chunk order
// (deterministic, no atomics anywhere in the numerics).
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
constexpr unsigned kFull = 0xffffffffu;
constexpr int kBlock = 256;
#ifndef GT_BWD_MINB
#define GT_BWD_MINB 1
#endif

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int H>
constexpr int kSBF = (8 * H + 15) / 16 * 4;  // floats per row of the (LSE2, D) stats array

template <typename T, int H, int D>
struct Cfg {
  static constexpr int EPL = D / 32;                        // elements per lane
  static constexpr int LPH = 32 / H;                        // lanes per head
  static constexpr int W = EPL * (int)sizeof(T) / 4;        // 32-bit words per lane
  static constexpr int U = W >= 16 ? 1 : (W >= 8 ? 2 : 4);  // edges gathered per batch
  static_assert(D % 32 == 0 && 32 % H == 0 && W >= 2, "unsupported shape");
};

template <int W>
__device__ __forceinline__ void ld_words(const void* p, uint32_t (&w)[W]) {
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int i = 0; i < W / 4; ++i) {
      uint4 x = ldg_stream(reinterpret_cast<const uint4*>(p) + i);
      w[4 * i] = x.x; w[4 * i + 1] = x.y; w[4 * i + 2] = x.z; w[4 * i + 3] = x.w;
    }
  } else {
    uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
    w[0] = x.x; w[1] = x.y;
  }
}

template <int W>
__device__ __forceinline__ void zero_words(uint32_t (&w)[W]) {
#pragma unroll
  for (int i = 0; i < W; ++i) w[i] = 0u;
}

template <typename T, int EPL, int W>
__device__ __forceinline__ void to_f32(const uint32_t (&w)[W], float (&f)[EPL]) {
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

template <typename T, int EPL, int W>
__device__ __forceinline__ void from_f32(const float (&f)[EPL], uint32_t (&w)[W]) {
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
}

template <int W>
__device__ __forceinline__ void st_words(void* p, const uint32_t (&w)[W]) {
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int i = 0; i < W / 4; ++i)
      reinterpret_cast<uint4*>(p)[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
  } else {
    *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
  }
}

template <typename T, int EPL, int W>
__device__ __forceinline__ void load_f32(const void* row_base, int lane, float (&f)[EPL]) {
  uint32_t w[W];
  ld_words<W>(static_cast<const char*>(row_base) + (size_t)lane * W * 4, w);
  to_f32<T, EPL, W>(w, f);
}

template <typename T, int EPL, int W>
__device__ __forceinline__ void store_f32(void* row_base, int lane, const float (&f)[EPL]) {
  uint32_t w[W];
  from_f32<T, EPL, W>(f, w);
  st_words<W>(static_cast<char*>(row_base) + (size_t)lane * W * 4, w);
}

// Packed fp32 math (FFMA2 / FMUL2 on sm_100a): two lanes of fp32 per instruction.
#ifndef GT_FFMA2
#define GT_FFMA2 1
#endif
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
#if GT_FFMA2
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
#else
  return make_float2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y));
#endif
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
#if GT_FFMA2
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
#else
  return make_float2(a.x * b.x, a.y * b.y);
#endif
}

// acc[i] += p * x[i]  (pairwise)
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
__device__ __forceinline__ void scale_by(float c, float (&acc)[EPL]) {
  const float2 cc = make_float2(c, c);
#pragma unroll
  for (int i = 0; i < EPL; i += 2) {
    float2 r = f2mul(cc, make_float2(acc[i], acc[i + 1]));
    acc[i] = r.x;
    acc[i + 1] = r.y;
  }
}

template <int LPH>
__device__ __forceinline__ float head_sum(float x) {
#pragma unroll
  for (int o = LPH / 2; o >= 1; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

template <int EPL>
__device__ __forceinline__ float dot(const float (&a)[EPL], const float (&b)[EPL]) {
  float2 s = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < EPL; i += 2) s = f2fma(make_float2(a[i], a[i + 1]), make_float2(b[i], b[i + 1]), s);
  return s.x + s.y;
}

// Source of gathered rows: index c < n_local reads the caller's tensors, c >= n_local reads a
// packed halo row (c - n_local) of `halo_stride` bytes whose second tensor starts at `off2`.
struct Src2 {
  const char* a;      // local tensor 1 (row stride row_bytes)
  const char* b;      // local tensor 2
  const char* halo;   // packed halo rows
  int64_t n_local;
  int64_t row_bytes;
  int64_t halo_stride;
  int64_t off2;
  __device__ __forceinline__ void ptrs(int64_t c, const char*& pa, const char*& pb) const {
    if (c < n_local) {
      pa = a + c * row_bytes;
      pb = b + c * row_bytes;
    } else {
      pa = halo + (c - n_local) * halo_stride;
      pb = pa + off2;
    }
  }
};

// Dynamic in-order work distribution.  Items are listed in row (column) order; a row with more
// than `heavy` entries appears as its chunks (item < 0 => chunk -1 - item).  Warps grab kGrab
// consecutive items per atomicAdd, so all resident warps work inside a narrow window of rows and
// the K/V rows their edges gather (community locality) stay resident in L2.
constexpr int kGrab = 2;
struct Work {
  const int32_t* items;
  int64_t nitems;
  unsigned long long* counter;   // zeroed before each launch
};

template <typename F>
__device__ __forceinline__ void for_each_item(const Work& w, int lane, F&& f) {
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(w.counter, (unsigned long long)kGrab);
    base = __shfl_sync(kFull, base, 0);
    if ((int64_t)base >= w.nitems) break;
    const int64_t end = min((int64_t)base + kGrab, w.nitems);
    for (int64_t t = (int64_t)base; t < end; ++t) f(__ldg(w.items + t));
  }
}

// ============================================================== forward (K1) ==
struct FwdArgs {
  const char* q;
  Src2 kv;                 // k, v
  char* y;
  float* lse;
  const int64_t* row_ptr;
  const int32_t* col;
  float qscale;            // scale * log2(e)
  Work work;
  const int64_t* clo;      // chunk entry ranges and owner rows
  const int64_t* chi;
  const int32_t* cown;
  float* part;             // [nchunks, D + 2H]: acc (lane-major), then (m, l) per head
};

template <typename T, int H, int D>
__device__ __forceinline__ void fwd_segment(const FwdArgs& a, int64_t row, int64_t e0, int64_t e1, int lane,
                                            float& m, float& l, float (&acc)[Cfg<T, H, D>::EPL]) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL, W = C::W, U = C::U, LPH = C::LPH;
  float q[EPL];
  load_f32<T, EPL, W>(a.q + row * (int64_t)(D * sizeof(T)), lane, q);
#pragma unroll
  for (int i = 0; i < EPL; ++i) { q[i] *= a.qscale; acc[i] = 0.f; }
  m = -INFINITY;
  l = 0.f;
  for (int64_t base = e0; base < e1; base += 32) {
    const int cnt = (e1 - base) < 32 ? (int)(e1 - base) : 32;
    const int myc = lane < cnt ? __ldg(a.col + base + lane) : 0;
    for (int u0 = 0; u0 < cnt; u0 += U) {
      uint32_t kw[U][W], vw[U][W];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = __shfl_sync(kFull, myc, (u0 + u) & 31);
        if (u0 + u < cnt) {
          const char *pk, *pv;
          a.kv.ptrs(c, pk, pv);
          ld_words<W>(pk + lane * W * 4, kw[u]);
          ld_words<W>(pv + lane * W * 4, vw[u]);
        } else {
          zero_words<W>(kw[u]);
          zero_words<W>(vw[u]);
        }
      }
      float s[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float kf[EPL];
        to_f32<T, EPL, W>(kw[u], kf);
        s[u] = dot<EPL>(q, kf);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) s[u] = head_sum<LPH>(s[u]);
      float mx = m;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u0 + u >= cnt) s[u] = -INFINITY;
        mx = fmaxf(mx, s[u]);
      }
      const float corr = ex2(m - mx);
      l *= corr;
      scale_by<EPL>(corr, acc);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float p = ex2(s[u] - mx);
        l += p;
        float vf[EPL];
        to_f32<T, EPL, W>(vw[u], vf);
        axpy<EPL>(p, vf, acc);
      }
      m = mx;
    }
  }
}

template <typename T, int H, int D>
__global__ void __launch_bounds__(kBlock) fwd_kernel(FwdArgs a) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL, W = C::W, LPH = C::LPH;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int head = lane / LPH;
  (void)warp; (void)nwarps;
  for_each_item(a.work, lane, [&](int32_t it) {
    if (it < 0) {
      const int64_t ch = -1 - (int64_t)it;
      const int64_t row = a.cown[ch];
      float m, l, acc[EPL];
      fwd_segment<T, H, D>(a, row, a.clo[ch], a.chi[ch], lane, m, l, acc);
      float* pp = a.part + ch * (int64_t)(D + 2 * H);
#pragma unroll
      for (int i = 0; i < EPL; ++i) pp[lane * EPL + i] = acc[i];
      if (lane % LPH == 0) {
        pp[D + 2 * head] = m;
        pp[D + 2 * head + 1] = l;
      }
      return;
    }
    const int64_t row = it;
    const int64_t e0 = __ldg(a.row_ptr + row), e1 = __ldg(a.row_ptr + row + 1);
    float m, l, acc[EPL];
    fwd_segment<T, H, D>(a, row, e0, e1, lane, m, l, acc);
    float out[EPL];
    float lse;
    if (e1 == e0) {
#pragma unroll
      for (int i = 0; i < EPL; ++i) out[i] = 0.f;
      lse = -INFINITY;
    } else {
      const float inv = 1.f / l;
#pragma unroll
      for (int i = 0; i < EPL; ++i) out[i] = acc[i] * inv;
      lse = (m + __log2f(l)) * kLn2;
    }
    store_f32<T, EPL, W>(a.y + row * (int64_t)(D * sizeof(T)), lane, out);
    if (lane % LPH == 0) a.lse[row * H + head] = lse;
  });
}

struct MergeArgs {
  int64_t nids;
  const int32_t* ids;      // heavy row/col local ids
  const int32_t* first;    // chunk range per id
  const float* part;
  // forward outputs
  char* y;
  float* lse;
  // backward row outputs
  char* dq;
  float* stats;
  float scale;
  // backward column outputs
  char* dk;
  char* dv;
};

template <typename T, int H, int D>
__global__ void __launch_bounds__(kBlock) fwd_merge_kernel(MergeArgs a) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL, W = C::W, LPH = C::LPH;
  const int lane = threadIdx.x & 31;
  const int head = lane / LPH;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = warp; x < a.nids; x += nwarps) {
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
    store_f32<T, EPL, W>(a.y + row * (int64_t)(D * sizeof(T)), lane, acc);
    if (lane % LPH == 0) a.lse[row * H + head] = (M + __log2f(L)) * kLn2;
  }
}

// ======================================================= backward row pass (K3) ==
// p_e = exp2(s_e - lse2_i), dP_e = <dY_i, v_j>; accumulates A = sum p dP k, C = sum p k,
// Dsum = sum p dP (fp32, in pass);  dQ_i = scale * (A - Dsum * C) = sum_e dS_e k_j.
struct RowbArgs {
  const char* q;
  const char* dy;
  const float* lse;        // natural log, [rows, H]
  Src2 kv;
  char* dq;
  float* stats;            // [rows, H, 2] = (lse * log2e, D)
  const int64_t* row_ptr;
  const int32_t* col;
  float qscale;            // scale * log2(e)
  float scale;
  Work work;
  const int64_t* clo;
  const int64_t* chi;
  const int32_t* cown;
  float* part;             // [nchunks, 2D + H]: A, C (lane-major), Dsum per head
};

template <typename T, int H, int D>
__device__ __forceinline__ void rowb_segment(const RowbArgs& a, int64_t row, int64_t e0, int64_t e1, int lane,
                                             float (&A)[Cfg<T, H, D>::EPL], float (&Cc)[Cfg<T, H, D>::EPL],
                                             float& Dsum) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL, W = C::W, U = C::U, LPH = C::LPH;
  const int head = lane / LPH;
  float q[EPL], g[EPL];
  load_f32<T, EPL, W>(a.q + row * (int64_t)(D * sizeof(T)), lane, q);
  load_f32<T, EPL, W>(a.dy + row * (int64_t)(D * sizeof(T)), lane, g);
#pragma unroll
  for (int i = 0; i < EPL; ++i) { q[i] *= a.qscale; A[i] = 0.f; Cc[i] = 0.f; }
  Dsum = 0.f;
  if (e1 == e0) return;
  const float lse2 = __ldg(a.lse + row * H + head) * kLog2e;
  for (int64_t base = e0; base < e1; base += 32) {
    const int cnt = (e1 - base) < 32 ? (int)(e1 - base) : 32;
    const int myc = lane < cnt ? __ldg(a.col + base + lane) : 0;
    for (int u0 = 0; u0 < cnt; u0 += U) {
      uint32_t kw[U][W], vw[U][W];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = __shfl_sync(kFull, myc, (u0 + u) & 31);
        if (u0 + u < cnt) {
          const char *pk, *pv;
          a.kv.ptrs(c, pk, pv);
          ld_words<W>(pk + lane * W * 4, kw[u]);
          ld_words<W>(pv + lane * W * 4, vw[u]);
        } else {
          zero_words<W>(kw[u]);
          zero_words<W>(vw[u]);
        }
      }
      float s[U], dp[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float kf[EPL], vf[EPL];
        to_f32<T, EPL, W>(kw[u], kf);
        to_f32<T, EPL, W>(vw[u], vf);
        s[u] = dot<EPL>(q, kf);
        dp[u] = dot<EPL>(g, vf);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        s[u] = head_sum<LPH>(s[u]);
        dp[u] = head_sum<LPH>(dp[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float p = (u0 + u < cnt) ? ex2(s[u] - lse2) : 0.f;
        const float pd = p * dp[u];
        Dsum += pd;
        float kf[EPL];
        to_f32<T, EPL, W>(kw[u], kf);
        axpy<EPL>(pd, kf, A);
        axpy<EPL>(p, kf, Cc);
      }
    }
  }
}

template <typename T, int H, int D>
__global__ void __launch_bounds__(kBlock, GT_BWD_MINB) rowb_kernel(RowbArgs a) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL, W = C::W, LPH = C::LPH;
  const int lane = threadIdx.x & 31;
  const int head = lane / LPH;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  (void)warp; (void)nwarps;
  for_each_item(a.work, lane, [&](int32_t it) {
    if (it < 0) {
      const int64_t ch = -1 - (int64_t)it;
      const int64_t row = a.cown[ch];
      float A[EPL], Cc[EPL], Ds;
      rowb_segment<T, H, D>(a, row, a.clo[ch], a.chi[ch], lane, A, Cc, Ds);
      float* pp = a.part + ch * (int64_t)(2 * D + H);
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        pp[lane * EPL + i] = A[i];
        pp[D + lane * EPL + i] = Cc[i];
      }
      if (lane % LPH == 0) pp[2 * D + head] = Ds;
      return;
    }
    const int64_t row = it;
    const int64_t e0 = __ldg(a.row_ptr + row), e1 = __ldg(a.row_ptr + row + 1);
    float A[EPL], Cc[EPL], Ds;
    rowb_segment<T, H, D>(a, row, e0, e1, lane, A, Cc, Ds);
    float out[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) out[i] = a.scale * fmaf(-Ds, Cc[i], A[i]);
    store_f32<T, EPL, W>(a.dq + row * (int64_t)(D * sizeof(T)), lane, out);
    if (lane % LPH == 0) {
      const float lse2 = (e1 == e0) ? -INFINITY : __ldg(a.lse + row * H + head) * kLog2e;
      reinterpret_cast<float2*>(a.stats + row * kSBF<H>)[head] = make_float2(lse2, Ds);
    }
  });
}

template <typename T, int H, int D>
__global__ void __launch_bounds__(kBlock) rowb_merge_kernel(MergeArgs a, const float* lse) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL, W = C::W, LPH = C::LPH;
  const int lane = threadIdx.x & 31;
  const int head = lane / LPH;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = warp; x < a.nids; x += nwarps) {
    const int64_t row = a.ids[x];
    const int c0 = a.first[x], c1 = a.first[x + 1];
    float A[EPL], Cc[EPL], Ds = 0.f;
#pragma unroll
    for (int i = 0; i < EPL; ++i) { A[i] = 0.f; Cc[i] = 0.f; }
    for (int c = c0; c < c1; ++c) {
      const float* pp = a.part + (int64_t)c * (2 * D + H);
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        A[i] += pp[lane * EPL + i];
        Cc[i] += pp[D + lane * EPL + i];
      }
      Ds += pp[2 * D + head];
    }
    float out[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) out[i] = a.scale * fmaf(-Ds, Cc[i], A[i]);
    store_f32<T, EPL, W>(a.dq + row * (int64_t)(D * sizeof(T)), lane, out);
    if (lane % LPH == 0)
      reinterpret_cast<float2*>(a.stats + row * kSBF<H>)[head] = make_float2(__ldg(lse + row * H + head) * kLog2e, Ds);
  }
}

// ==================================================== backward column pass (K4) ==
// For owned column j and in-entry e = (i, j): recompute p_e = exp2(s_e - lse2_i),
// dP_e = <dY_i, v_j>, dS_e = p_e (dP_e - D_i); dV_j += p_e dY_i; dK_j += dS_e q_i; dK *= scale.
struct ColbArgs {
  const char* k;
  const char* v;
  Src2 qg;                 // q, dy (local) / packed halo-in rows [q | dy | stats]
  const float* stats;      // local [rows, H, 2]
  int64_t halo_stats_off;  // byte offset of the stats inside a packed halo-in row
  char* dk;
  char* dv;
  const int64_t* col_ptr;
  const int32_t* row;      // in-neighbour row ids (remapped)
  float qscale;
  float scale;
  Work work;
  const int64_t* clo;
  const int64_t* chi;
  const int32_t* cown;
  float* part;             // [nchunks, 2D]: dK (unscaled), dV
};

template <typename T, int H, int D>
__device__ __forceinline__ void colb_segment(const ColbArgs& a, int64_t col, int64_t e0, int64_t e1, int lane,
                                             float (&dK)[Cfg<T, H, D>::EPL], float (&dV)[Cfg<T, H, D>::EPL]) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL, W = C::W, U = C::U, LPH = C::LPH;
  const int head = lane / LPH;
  float kj[EPL], vj[EPL];
  load_f32<T, EPL, W>(a.k + col * (int64_t)(D * sizeof(T)), lane, kj);
  load_f32<T, EPL, W>(a.v + col * (int64_t)(D * sizeof(T)), lane, vj);
#pragma unroll
  for (int i = 0; i < EPL; ++i) { kj[i] *= a.qscale; dK[i] = 0.f; dV[i] = 0.f; }
  const int64_t nl = a.qg.n_local;
  for (int64_t base = e0; base < e1; base += 32) {
    const int cnt = (e1 - base) < 32 ? (int)(e1 - base) : 32;
    const int myr = lane < cnt ? __ldg(a.row + base + lane) : 0;
    for (int u0 = 0; u0 < cnt; u0 += U) {
      uint32_t qw[U][W], gw[U][W];
      float2 st[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = __shfl_sync(kFull, myr, (u0 + u) & 31);
        if (u0 + u < cnt) {
          const char *pq, *pg;
          a.qg.ptrs(r, pq, pg);
          ld_words<W>(pq + lane * W * 4, qw[u]);
          ld_words<W>(pg + lane * W * 4, gw[u]);
          const float2* sp = r < nl ? reinterpret_cast<const float2*>(a.stats + (int64_t)r * kSBF<H>)
                                    : reinterpret_cast<const float2*>(pq + a.halo_stats_off);
          st[u] = __ldg(sp + head);
        } else {
          zero_words<W>(qw[u]);
          zero_words<W>(gw[u]);
          st[u] = make_float2(0.f, 0.f);
        }
      }
      float s[U], dp[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float qf[EPL], gf[EPL];
        to_f32<T, EPL, W>(qw[u], qf);
        to_f32<T, EPL, W>(gw[u], gf);
        s[u] = dot<EPL>(qf, kj);
        dp[u] = dot<EPL>(gf, vj);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        s[u] = head_sum<LPH>(s[u]);
        dp[u] = head_sum<LPH>(dp[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float p = (u0 + u < cnt) ? ex2(s[u] - st[u].x) : 0.f;
        const float ds = p * (dp[u] - st[u].y);
        float qf[EPL], gf[EPL];
        to_f32<T, EPL, W>(qw[u], qf);
        to_f32<T, EPL, W>(gw[u], gf);
        axpy<EPL>(p, gf, dV);
        axpy<EPL>(ds, qf, dK);
      }
    }
  }
}

template <typename T, int H, int D>
__global__ void __launch_bounds__(kBlock, GT_BWD_MINB) colb_kernel(ColbArgs a) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL, W = C::W;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  (void)warp; (void)nwarps;
  for_each_item(a.work, lane, [&](int32_t it) {
    if (it < 0) {
      const int64_t ch = -1 - (int64_t)it;
      const int64_t col = a.cown[ch];
      float dK[EPL], dV[EPL];
      colb_segment<T, H, D>(a, col, a.clo[ch], a.chi[ch], lane, dK, dV);
      float* pp = a.part + ch * (int64_t)(2 * D);
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        pp[lane * EPL + i] = dK[i];
        pp[D + lane * EPL + i] = dV[i];
      }
      return;
    }
    const int64_t col = it;
    const int64_t e0 = __ldg(a.col_ptr + col), e1 = __ldg(a.col_ptr + col + 1);
    float dK[EPL], dV[EPL];
    colb_segment<T, H, D>(a, col, e0, e1, lane, dK, dV);
#pragma unroll
    for (int i = 0; i < EPL; ++i) dK[i] *= a.scale;
    store_f32<T, EPL, W>(a.dk + col * (int64_t)(D * sizeof(T)), lane, dK);
    store_f32<T, EPL, W>(a.dv + col * (int64_t)(D * sizeof(T)), lane, dV);
  });
}

template <typename T, int H, int D>
__global__ void __launch_bounds__(kBlock) colb_merge_kernel(MergeArgs a) {
  using C = Cfg<T, H, D>;
  constexpr int EPL = C::EPL, W = C::W;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = warp; x < a.nids; x += nwarps) {
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
    store_f32<T, EPL, W>(a.dk + col * (int64_t)(D * sizeof(T)), lane, dK);
    store_f32<T, EPL, W>(a.dv + col * (int64_t)(D * sizeof(T)), lane, dV);
  }
}

// ================================================================= dispatch ==
template <typename K>
int persistent_grid(K kernel, int64_t items) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, 0);
  if (per_sm < 1) per_sm = 1;
  const int64_t want = ((items + kGrab - 1) / kGrab * 32 + kBlock - 1) / kBlock;  // <= one warp per grab
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * per_sm));
}

template <typename T, int H, int D>
struct Launcher {
  static MergeArgs merge_args(const ChunkTable& ht, const DevBuf& part) {
    MergeArgs m{};
    m.nids = (int64_t)ht.ids.size();
    m.ids = ht.d_ids.as<int32_t>();
    m.first = ht.d_first.as<int32_t>();
    m.part = part.as<float>();
    return m;
  }

  static gt_status fwd(gt_plan_s* P, const void* q, const void* k, const void* v, const void* halo, void* y,
                       float* lse, cudaStream_t st) {
    const auto& ht = P->heavy_rows;
    FwdArgs a{};
    a.q = (const char*)q;
    a.kv = Src2{(const char*)k, (const char*)v, (const char*)halo, P->n_local, (int64_t)(D * sizeof(T)),
                P->kv_row_bytes, (int64_t)(D * sizeof(T))};
    a.y = (char*)y;
    a.lse = lse;
    a.row_ptr = P->d_row_ptr.as<int64_t>();
    a.col = P->d_col.as<int32_t>();
    a.qscale = P->scale * kLog2e;
    a.work = Work{P->d_items_rows.as<int32_t>(), P->n_items_rows, P->d_counters.as<unsigned long long>()};
    a.clo = ht.d_lo.as<int64_t>();
    a.chi = ht.d_hi.as<int64_t>();
    a.cown = ht.d_owner.as<int32_t>();
    a.part = P->d_part_fwd.as<float>();
    if (P->kernel == 2) {
      GT_TRY(pipe_pass(P, 0, q, nullptr, nullptr, k, v, halo, y, nullptr, lse, st));
    } else if (P->n_items_rows > 0) {
      GT_CUDA_TRY(cudaMemsetAsync(a.work.counter, 0, sizeof(unsigned long long), st));
      fwd_kernel<T, H, D><<<persistent_grid(fwd_kernel<T, H, D>, P->n_items_rows), kBlock, 0, st>>>(a);
    }
    if (ht.nchunks() > 0) {
      MergeArgs m = merge_args(ht, P->d_part_fwd);
      m.y = (char*)y;
      m.lse = lse;
      fwd_merge_kernel<T, H, D><<<persistent_grid(fwd_merge_kernel<T, H, D>, m.nids), kBlock, 0, st>>>(m);
    }
    GT_CUDA_TRY(cudaGetLastError());
    return GT_OK;
  }

  static gt_status rowb(gt_plan_s* P, const void* q, const void* k, const void* v, const void* halo,
                        const float* lse, const void* dy, void* dq, cudaStream_t st) {
    const auto& ht = P->heavy_rows;
    RowbArgs a{};
    a.q = (const char*)q;
    a.dy = (const char*)dy;
    a.lse = lse;
    a.kv = Src2{(const char*)k, (const char*)v, (const char*)halo, P->n_local, (int64_t)(D * sizeof(T)),
                P->kv_row_bytes, (int64_t)(D * sizeof(T))};
    a.dq = (char*)dq;
    a.stats = P->d_stats.as<float>();
    a.row_ptr = P->d_row_ptr.as<int64_t>();
    a.col = P->d_col.as<int32_t>();
    a.qscale = P->scale * kLog2e;
    a.scale = P->scale;
    a.work = Work{P->d_items_rows.as<int32_t>(), P->n_items_rows, P->d_counters.as<unsigned long long>() + 1};
    a.clo = ht.d_lo.as<int64_t>();
    a.chi = ht.d_hi.as<int64_t>();
    a.cown = ht.d_owner.as<int32_t>();
    a.part = P->d_part_rowb.as<float>();
    if (P->kernel == 2) {
      GT_TRY(pipe_pass(P, 1, q, dy, lse, k, v, halo, dq, nullptr, P->d_stats.as<float>(), st));
    } else if (P->n_items_rows > 0) {
      GT_CUDA_TRY(cudaMemsetAsync(a.work.counter, 0, sizeof(unsigned long long), st));
      rowb_kernel<T, H, D><<<persistent_grid(rowb_kernel<T, H, D>, P->n_items_rows), kBlock, 0, st>>>(a);
    }
    if (ht.nchunks() > 0) {
      MergeArgs m = merge_args(ht, P->d_part_rowb);
      m.dq = (char*)dq;
      m.stats = P->d_stats.as<float>();
      m.scale = P->scale;
      rowb_merge_kernel<T, H, D><<<persistent_grid(rowb_merge_kernel<T, H, D>, m.nids), kBlock, 0, st>>>(m, lse);
    }
    GT_CUDA_TRY(cudaGetLastError());
    return GT_OK;
  }

  static gt_status colb(gt_plan_s* P, const void* q, const void* k, const void* v, const void* dy,
                        const void* halo_in, void* dk, void* dv, cudaStream_t st) {
    const auto& ht = P->heavy_cols;
    ColbArgs a{};
    a.k = (const char*)k;
    a.v = (const char*)v;
    a.qg = Src2{(const char*)q, (const char*)dy, (const char*)halo_in, P->n_local, (int64_t)(D * sizeof(T)),
                P->in_row_bytes, (int64_t)(D * sizeof(T))};
    a.stats = P->d_stats.as<float>();
    a.halo_stats_off = 2 * (int64_t)(D * sizeof(T));
    a.dk = (char*)dk;
    a.dv = (char*)dv;
    a.col_ptr = P->d_col_ptr.as<int64_t>();
    a.row = P->d_row.as<int32_t>();
    a.qscale = P->scale * kLog2e;
    a.scale = P->scale;
    a.work = Work{P->d_items_cols.as<int32_t>(), P->n_items_cols, P->d_counters.as<unsigned long long>() + 2};
    a.clo = ht.d_lo.as<int64_t>();
    a.chi = ht.d_hi.as<int64_t>();
    a.cown = ht.d_owner.as<int32_t>();
    a.part = P->d_part_colb.as<float>();
    if (P->kernel == 2) {
      GT_TRY(pipe_pass(P, 2, k, v, nullptr, q, dy, halo_in, dk, dv, nullptr, st));
    } else if (P->n_items_cols > 0) {
      GT_CUDA_TRY(cudaMemsetAsync(a.work.counter, 0, sizeof(unsigned long long), st));
      colb_kernel<T, H, D><<<persistent_grid(colb_kernel<T, H, D>, P->n_items_cols), kBlock, 0, st>>>(a);
    }
    if (ht.nchunks() > 0) {
      MergeArgs m = merge_args(ht, P->d_part_colb);
      m.dk = (char*)dk;
      m.dv = (char*)dv;
      m.scale = P->scale;
      colb_merge_kernel<T, H, D><<<persistent_grid(colb_merge_kernel<T, H, D>, m.nids), kBlock, 0, st>>>(m);
    }
    GT_CUDA_TRY(cudaGetLastError());
    return GT_OK;
  }
};

template <template <typename, int, int> class F, typename... Args>
gt_status dispatch(int dtype, int H, int D, Args... args) {
#define GT_CASE(TT, HH, DD) \
  if (H == HH && D == DD) return F<TT, HH, DD>::run(args...);
#define GT_HCASES(TT)                                                                              \
  GT_CASE(TT, 1, 128) GT_CASE(TT, 1, 256) GT_CASE(TT, 1, 512) GT_CASE(TT, 2, 128) GT_CASE(TT, 2, 256) \
  GT_CASE(TT, 2, 512) GT_CASE(TT, 4, 128) GT_CASE(TT, 4, 256) GT_CASE(TT, 4, 512) GT_CASE(TT, 8, 128) \
  GT_CASE(TT, 8, 256) GT_CASE(TT, 8, 512)
  if (dtype == GT_F32) { GT_HCASES(float) }
  else { GT_HCASES(__nv_bfloat16) }
#undef GT_HCASES
#undef GT_CASE
  return fail(GT_ECONFIG, "unsupported (dtype, heads, heads*d)");
}

template <typename T, int H, int D>
struct FwdOp {
  template <typename... A> static gt_status run(A... a) { return Launcher<T, H, D>::fwd(a...); }
};
template <typename T, int H, int D>
struct RowbOp {
  template <typename... A> static gt_status run(A... a) { return Launcher<T, H, D>::rowb(a...); }
};
template <typename T, int H, int D>
struct ColbOp {
  template <typename... A> static gt_status run(A... a) { return Launcher<T, H, D>::colb(a...); }
};

}  // namespace

bool shape_supported(int heads, int d, int dtype) {
  const int D = heads * d;
  if (dtype != GT_F32 && dtype != GT_BF16) return false;
  if (heads != 1 && heads != 2 && heads != 4 && heads != 8) return false;
  return D == 128 || D == 256 || D == 512;
}

int launches_fwd(const gt_plan_s* P) {
  return (P->n_items_rows > 0 ? 1 : 0) + (P->heavy_rows.nchunks() > 0 ? 1 : 0);
}
int launches_bwd(const gt_plan_s* P) {
  return (P->n_items_rows > 0 ? 1 : 0) + (P->n_items_cols > 0 ? 1 : 0) + (P->heavy_rows.nchunks() > 0 ? 1 : 0) +
         (P->heavy_cols.nchunks() > 0 ? 1 : 0);
}

gt_status launch_fwd(gt_plan_s* P, const void* q, const void* k, const void* v, const void* halo_kv, void* y,
                     float* lse, cudaStream_t st) {
  return dispatch<FwdOp>(P->dtype, P->heads, P->heads * P->d, P, q, k, v, halo_kv, y, lse, st);
}
gt_status launch_bwd_rows(gt_plan_s* P, const void* q, const void* k, const void* v, const void* halo_kv,
                          const float* lse, const void* dy, void* dq, cudaStream_t st) {
  return dispatch<RowbOp>(P->dtype, P->heads, P->heads * P->d, P, q, k, v, halo_kv, lse, dy, dq, st);
}
gt_status launch_bwd_cols(gt_plan_s* P, const void* q, const void* k, const void* v, const void* dy,
                          const void* halo_in, void* dk, void* dv, cudaStream_t st) {
  return dispatch<ColbOp>(P->dtype, P->heads, P->heads * P->d, P, q, k, v, dy, halo_in, dk, dv, st);
}

}  // namespace gt
