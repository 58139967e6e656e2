// Pipelined sparse-attention kernels for sm_100a: TMA bulk-copy gathers into per-warp shared-memory
// stage rings, completion on mbarriers (UBLKCP + SYNCS in SASS).
//
// Same mathematics as attn.cu (Eq. 2/4/5 and Section 2.2):
//   pass 0 (fwd):  per row i:    s_e = scale <q_i,k_j>, online softmax, y_i = sum p_e v_j / l, LSE
//   pass 1 (rowb): per row i:    p_e = exp(s_e - LSE_i), dP_e = <dY_i, v_j>, D_i = sum p dP,
//                                dQ_i = scale (sum p dP k_j - D_i sum p k_j)
//   pass 2 (colb): per column j: p_e, dP_e recomputed from (q_i, dY_i, LSE_i, D_i);
//                                dV_j = sum p dY_i, dK_j = scale sum p (dP - D_i) q_i
//
// Execution model.  Persistent CTAs of kWarps warps; every warp owns a ring of S stages in shared
// memory, each stage holding up to U gathered neighbours (2 rows of D*sizeof(T) bytes each, plus the
// neighbour's (LSE, D) block in pass 2) and an "own" slot with the row/column's own data.  The warp
// grabs batches of G consecutive work items (rows, or chunks of heavy rows, in row order) with one
// atomicAdd; because items are consecutive their edge ranges form one contiguous span of the
// neighbour array, streamed through a 32-entry register window.  The warp is its own producer: lane u
// issues cp.async.bulk copies of neighbour u's rows straight from global memory into the stage
// (one instruction per 512-byte row) and lane 0 posts the byte count on the stage's mbarrier; then
// the warp consumes the oldest stage (LDS of the lane's 16-byte slice) and refills it.  S*U
// neighbours (16 KB) are in flight per warp without holding registers, across row boundaries.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "gt_internal.h"

namespace gt {
namespace pipe {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarps = 4;     // warps per CTA
constexpr int kS = 4;         // stages per warp
constexpr int kG = 4;         // items per grab

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void bar_init(void* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(1));
}
__device__ __forceinline__ void bar_expect(void* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(void* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
        : "=r"(done)
        : "r"(su32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, void* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

template <typename T, int H, int D, int PASS>
struct PC {
  static constexpr int RB = D * (int)sizeof(T);          // bytes of one feature row
  static constexpr int EPL = D / 32;                      // elements per lane
  static constexpr int LB = EPL * (int)sizeof(T);         // bytes per lane of one row
  static constexpr int W = LB / 4;                        // 32-bit words per lane
  static constexpr int LPH = 32 / H;                      // lanes per head
  static constexpr int SB = (8 * H + 15) / 16 * 16;       // (LSE2, D) block per row, 16-byte padded
  static constexpr int LSEB = (4 * H + 15) / 16 * 16;     // lse block copied for the own row (pass 1)
  static constexpr int EB = 2 * RB + (PASS == 2 ? SB : 0);                        // bytes per neighbour
  static constexpr int OWN = PASS == 0 ? RB : (PASS == 1 ? 2 * RB + LSEB : 2 * RB);
  static constexpr int U = RB >= 2048 ? 1 : (RB >= 1024 ? 2 : 4);                  // neighbours per stage
  static constexpr int STAGE = U * EB;
  static constexpr int WARP_SMEM = kS * (STAGE + OWN) + kS * 16 + kS * 8;
  static_assert(W == 2 || W % 4 == 0, "lane slice must be 8 bytes or a multiple of 16");
};

struct PArgs {
  const int64_t* iptr;   // [nitems + 1] edge range of each item
  const int32_t* iown;   // [nitems]: >= 0 row/column id, < 0 chunk -1 - c
  const int32_t* cown;   // chunk -> row/column id
  const int32_t* nbr;    // neighbour ids in edge order (remapped: < n_local local, else halo slot)
  int64_t nitems;
  unsigned long long* counter;
  const char* ga;        // local tensor gathered first  (k | k | q)
  const char* gb;        // local tensor gathered second (v | v | dy)
  const char* gs;        // local (LSE2, D) blocks [n_local][SB] (pass 2)
  const char* halo;      // packed remote rows
  int64_t halo_stride;
  int64_t n_local;
  const char* oa;        // own tensor A (q | q | k)
  const char* ob;        // own tensor B (- | dy | v)
  const float* lse;      // pass 1: caller's LSE [n_local][H] (natural log)
  char* out_a;           // y | dq | dk
  char* out_b;           // - | - | dv
  float* out_f;          // lse (pass 0) | stats [n_local][SB/4] (pass 1)
  float* part;           // chunk partials
  float qscale, scale;
};

struct Meta {
  int32_t own;           // item id (row/col) or chunk (-1 - c)
  int16_t cnt;
  int8_t first, last;
  int32_t slot, pad;
};

template <int W>
__device__ __forceinline__ void lds_words(const char* p, uint32_t (&w)[W]) {
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int i = 0; i < W / 4; ++i) {
      uint4 x = *reinterpret_cast<const uint4*>(p + 16 * i);
      w[4 * i] = x.x; w[4 * i + 1] = x.y; w[4 * i + 2] = x.z; w[4 * i + 3] = x.w;
    }
  } else {
    uint2 x = *reinterpret_cast<const uint2*>(p);
    w[0] = x.x; w[1] = x.y;
  }
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

template <typename T, int EPL>
__device__ __forceinline__ void lds_f32(const char* p, float (&f)[EPL]) {
  constexpr int W = EPL * (int)sizeof(T) / 4;
  uint32_t w[W];
  lds_words<W>(p, w);
  to_f32<T, EPL, W>(w, f);
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
  } else {
    *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
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

template <int LPH>
__device__ __forceinline__ float head_sum(float x) {
#pragma unroll
  for (int o = LPH / 2; o >= 1; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

// ------------------------------------------------------------------ kernel --
template <typename T, int H, int D, int PASS>
__global__ void __launch_bounds__(kWarps * 32) pipe_kernel(PArgs a) {
  using C = PC<T, H, D, PASS>;
  constexpr int EPL = C::EPL, LPH = C::LPH, RB = C::RB, EB = C::EB, U = C::U;
  extern __shared__ __align__(128) char smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int head = lane / LPH;
  char* wbase = smem + (size_t)wid * C::WARP_SMEM;
  char* stages = wbase;                                   // kS * STAGE
  char* owns = stages + kS * C::STAGE;                    // kS * OWN
  Meta* meta = reinterpret_cast<Meta*>(owns + kS * C::OWN);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(meta) + kS * 16);
  if (lane == 0)
    for (int s = 0; s < kS; ++s) bar_init(&bars[s]);
  __syncwarp();
  fence_async_smem();

  // ---------------- producer state (warp-uniform except lane-distributed tables) ----------------
  int64_t t_next = 0, t_end = 0;     // items of the current batch not yet started
  int64_t my_ptr = 0;                // lane k (< kG): iptr[t0 + k]; lane kG: iptr[t0 + kG] (batch end)
  int32_t my_own = 0;                // lane k: iown[t0 + k]
  int64_t batch_t0 = 0;
  bool done = false;
  int64_t pe = 0, pe_end = 0;        // current item's remaining edge range
  int32_t cur_own = 0;
  int cur_first = 0;
  int64_t win_base = 0;              // neighbour window: lane l holds nbr[win_base + l]
  int32_t win = 0;
  int32_t item_seq = 0;
  int64_t batch_e1 = 0;

  auto finalize_empty = [&](int32_t own) {
    // rows with no entries: Y = 0, LSE = -inf / dQ = 0, stats (-inf, 0) / dK = dV = 0
    float z[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) z[i] = 0.f;
    const int64_t r = own;
    if constexpr (PASS == 0) {
      stg_f32<T, EPL>(a.out_a + r * RB + lane * C::LB, z);
      if (lane % LPH == 0) a.out_f[r * H + head] = -INFINITY;
    } else if constexpr (PASS == 1) {
      stg_f32<T, EPL>(a.out_a + r * RB + lane * C::LB, z);
      if (lane % LPH == 0)
        reinterpret_cast<float2*>(reinterpret_cast<char*>(a.out_f) + r * C::SB)[head] = make_float2(-INFINITY, 0.f);
    } else {
      stg_f32<T, EPL>(a.out_a + r * RB + lane * C::LB, z);
      stg_f32<T, EPL>(a.out_b + r * RB + lane * C::LB, z);
    }
  };

  // Advances to the next non-empty item; returns false when the grid's work is exhausted.
  auto next_item = [&]() -> bool {
    for (;;) {
      if (t_next >= t_end) {
        if (done) return false;
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(a.counter, (unsigned long long)kG);
        b = __shfl_sync(kFull, b, 0);
        if ((int64_t)b >= a.nitems) {
          done = true;
          return false;
        }
        batch_t0 = (int64_t)b;
        t_end = min(batch_t0 + kG, a.nitems);
        t_next = batch_t0;
        const int64_t k = batch_t0 + lane;
        my_ptr = (lane <= kG && k <= a.nitems) ? __ldg(a.iptr + k) : 0;
        my_own = (lane < kG && k < a.nitems) ? __ldg(a.iown + k) : 0;
        batch_e1 = __shfl_sync(kFull, my_ptr, (int)(t_end - batch_t0));
        win_base = -1000000000000ll;
      }
      const int k = (int)(t_next - batch_t0);
      const int64_t e0 = __shfl_sync(kFull, my_ptr, k);
      const int64_t e1 = __shfl_sync(kFull, my_ptr, k + 1);
      const int32_t own = __shfl_sync(kFull, my_own, k);
      ++t_next;
      if (e1 == e0) {
        finalize_empty(own);
        continue;
      }
      pe = e0;
      pe_end = e1;
      cur_own = own;
      cur_first = 1;
      return true;
    }
  };

  // Fills stage `s` with the next group of neighbours; returns false if no work is left.
  auto produce = [&](int s) -> bool {
    if (pe >= pe_end && !next_item()) return false;
    if (pe < win_base || pe >= win_base + 32) {
      win_base = pe;
      win = (pe + lane < batch_e1) ? __ldg(a.nbr + pe + lane) : 0;
    }
    int64_t lim = pe_end - pe;
    if (win_base + 32 - pe < lim) lim = win_base + 32 - pe;
    const int cnt = lim < U ? (int)lim : U;
    const int slot = item_seq % kS;
    const bool first = cur_first != 0;
    const bool last = pe + cnt == pe_end;
    if (lane == 0) {
      Meta m;
      m.own = cur_own;
      m.cnt = (int16_t)cnt;
      m.first = first;
      m.last = last;
      m.slot = slot;
      m.pad = 0;
      meta[s] = m;
      uint32_t bytes = (uint32_t)(cnt * (2 * RB + (PASS == 2 ? C::SB : 0)));
      if (first) bytes += (uint32_t)(PASS == 0 ? RB : (PASS == 1 ? 2 * RB + C::LSEB : 2 * RB));
      bar_expect(&bars[s], bytes);
    }
    __syncwarp();
    fence_async_smem();
    const int32_t c = __shfl_sync(kFull, win, (int)((pe - win_base + lane) & 31));
    char* st = stages + s * C::STAGE;
    if (lane < cnt) {
      const char *pa, *pb, *ps = nullptr;
      const int64_t ci = c;
      if (ci < a.n_local) {
        pa = a.ga + ci * RB;
        pb = a.gb + ci * RB;
        if constexpr (PASS == 2) ps = a.gs + ci * C::SB;
      } else {
        pa = a.halo + (ci - a.n_local) * a.halo_stride;
        pb = pa + RB;
        if constexpr (PASS == 2) ps = pa + 2 * RB;
      }
      char* dst = st + lane * EB;
      bulk_g2s(dst, pa, RB, &bars[s]);
      bulk_g2s(dst + RB, pb, RB, &bars[s]);
      if constexpr (PASS == 2) bulk_g2s(dst + 2 * RB, ps, C::SB, &bars[s]);
    }
    if (first) {
      char* o = owns + slot * C::OWN;
      const int64_t r = cur_own >= 0 ? cur_own : a.cown[-1 - (int64_t)cur_own];
      if (lane == 0) bulk_g2s(o, a.oa + r * RB, RB, &bars[s]);
      if constexpr (PASS >= 1) {
        if (lane == 1) bulk_g2s(o + RB, a.ob + r * RB, RB, &bars[s]);
      }
      if constexpr (PASS == 1) {
        if (lane == 2) {
          const char* lp = reinterpret_cast<const char*>(a.lse) + r * H * 4;
          bulk_g2s(o + 2 * RB, reinterpret_cast<const char*>((uintptr_t)lp & ~(uintptr_t)15), C::LSEB, &bars[s]);
        }
      }
      ++item_seq;
      cur_first = 0;
    }
    pe += cnt;
    return true;
  };

  // ---------------- consumer state ----------------
  float q[EPL], g[EPL], acc[EPL], acc2[EPL];
  float m = 0.f, l = 0.f, aux = 0.f;   // fwd: running max / sum; rowb: lse2 (m), D (l)

  int issued = 0;
  for (int s = 0; s < kS; ++s) {
    if (!produce(s)) break;
    ++issued;
  }
  for (int c = 0; c < issued; ++c) {
    const int s = c % kS;
    bar_wait(&bars[s], (uint32_t)((c / kS) & 1));
    const Meta md = meta[s];
    const char* st = stages + s * C::STAGE;
    if (md.first) {
      const char* o = owns + md.slot * C::OWN;
      if constexpr (PASS == 0) {
        lds_f32<T, EPL>(o + lane * C::LB, q);
#pragma unroll
        for (int i = 0; i < EPL; ++i) { q[i] *= a.qscale; acc[i] = 0.f; }
        m = -INFINITY;
        l = 0.f;
      } else if constexpr (PASS == 1) {
        lds_f32<T, EPL>(o + lane * C::LB, q);
        lds_f32<T, EPL>(o + RB + lane * C::LB, g);
        const int64_t r = md.own >= 0 ? md.own : a.cown[-1 - (int64_t)md.own];
        const int off = (H * 4 >= 16) ? 0 : (int)((r * H * 4) & 15);
        m = reinterpret_cast<const float*>(o + 2 * RB + off)[head] * kLog2e;
#pragma unroll
        for (int i = 0; i < EPL; ++i) { q[i] *= a.qscale; acc[i] = 0.f; acc2[i] = 0.f; }
        l = 0.f;
      } else {
        lds_f32<T, EPL>(o + lane * C::LB, q);      // k_j
        lds_f32<T, EPL>(o + RB + lane * C::LB, g); // v_j
#pragma unroll
        for (int i = 0; i < EPL; ++i) { q[i] *= a.qscale; acc[i] = 0.f; acc2[i] = 0.f; }
      }
    }
    const int cnt = md.cnt;
    if constexpr (PASS == 0) {
      float sc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u < cnt) {
          float kf[EPL];
          lds_f32<T, EPL>(st + u * EB + lane * C::LB, kf);
          sc[u] = head_sum<LPH>(dot<EPL>(q, kf));
        } else {
          sc[u] = -INFINITY;
        }
      }
      float mx = m;
#pragma unroll
      for (int u = 0; u < U; ++u) mx = fmaxf(mx, sc[u]);
      const float corr = ex2(m - mx);
      l *= corr;
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] *= corr;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u < cnt) {
          const float p = ex2(sc[u] - mx);
          l += p;
          float vf[EPL];
          lds_f32<T, EPL>(st + u * EB + RB + lane * C::LB, vf);
          axpy<EPL>(p, vf, acc);
        }
      }
      m = mx;
    } else if constexpr (PASS == 1) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u < cnt) {
          float kf[EPL], vf[EPL];
          lds_f32<T, EPL>(st + u * EB + lane * C::LB, kf);
          lds_f32<T, EPL>(st + u * EB + RB + lane * C::LB, vf);
          const float s_ = head_sum<LPH>(dot<EPL>(q, kf));
          const float dp = head_sum<LPH>(dot<EPL>(g, vf));
          const float p = ex2(s_ - m);
          const float pd = p * dp;
          l += pd;
          axpy<EPL>(pd, kf, acc);
          axpy<EPL>(p, kf, acc2);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u < cnt) {
          float qf[EPL], gf[EPL];
          lds_f32<T, EPL>(st + u * EB + lane * C::LB, qf);
          lds_f32<T, EPL>(st + u * EB + RB + lane * C::LB, gf);
          const float2 sd = reinterpret_cast<const float2*>(st + u * EB + 2 * RB)[head];
          const float s_ = head_sum<LPH>(dot<EPL>(qf, q));
          const float dp = head_sum<LPH>(dot<EPL>(gf, g));
          const float p = ex2(s_ - sd.x);
          const float ds = p * (dp - sd.y);
          axpy<EPL>(p, gf, acc2);   // dV
          axpy<EPL>(ds, qf, acc);   // dK (unscaled)
        }
      }
    }
    if (md.last) {
      const int32_t own = md.own;
      if (own < 0) {  // chunk of a heavy row/column: partial state
        const int64_t ch = -1 - (int64_t)own;
        if constexpr (PASS == 0) {
          float* pp = a.part + ch * (int64_t)(D + 2 * H);
#pragma unroll
          for (int i = 0; i < EPL; ++i) pp[lane * EPL + i] = acc[i];
          if (lane % LPH == 0) { pp[D + 2 * head] = m; pp[D + 2 * head + 1] = l; }
        } else if constexpr (PASS == 1) {
          float* pp = a.part + ch * (int64_t)(2 * D + H);
#pragma unroll
          for (int i = 0; i < EPL; ++i) { pp[lane * EPL + i] = acc[i]; pp[D + lane * EPL + i] = acc2[i]; }
          if (lane % LPH == 0) pp[2 * D + head] = l;
        } else {
          float* pp = a.part + ch * (int64_t)(2 * D);
#pragma unroll
          for (int i = 0; i < EPL; ++i) { pp[lane * EPL + i] = acc[i]; pp[D + lane * EPL + i] = acc2[i]; }
        }
      } else {
        const int64_t r = own;
        if constexpr (PASS == 0) {
          const float inv = 1.f / l;
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] *= inv;
          stg_f32<T, EPL>(a.out_a + r * RB + lane * C::LB, acc);
          if (lane % LPH == 0) a.out_f[r * H + head] = (m + __log2f(l)) * kLn2;
        } else if constexpr (PASS == 1) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] = a.scale * fmaf(-l, acc2[i], acc[i]);
          stg_f32<T, EPL>(a.out_a + r * RB + lane * C::LB, acc);
          if (lane % LPH == 0)
            reinterpret_cast<float2*>(reinterpret_cast<char*>(a.out_f) + r * C::SB)[head] = make_float2(m, l);
        } else {
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] *= a.scale;
          stg_f32<T, EPL>(a.out_a + r * RB + lane * C::LB, acc);
          stg_f32<T, EPL>(a.out_b + r * RB + lane * C::LB, acc2);
        }
      }
    }
    __syncwarp();
    if (produce(s)) ++issued;
  }
  // every issued stage was consumed; produce() returned false only once the work was exhausted
  // (next_item() finalised any empty rows on the way)
}

// ----------------------------------------------------------------- launcher --
template <typename T, int H, int D, int PASS>
gt_status launch(const PArgs& a, cudaStream_t st) {
  using C = PC<T, H, D, PASS>;
  static int grid = 0;
  const size_t smem = (size_t)kWarps * C::WARP_SMEM;
  if (!grid) {
    auto k = pipe_kernel<T, H, D, PASS>;
    GT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    GT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kWarps * 32, smem));
    grid = sms * std::max(per, 1);
  }
  if (a.nitems <= 0) return GT_OK;
  const int64_t want = (a.nitems + kG - 1) / kG;
  const int g = (int)std::min<int64_t>(grid, (want + kWarps - 1) / kWarps);
  GT_CUDA_TRY(cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), st));
  pipe_kernel<T, H, D, PASS><<<g, kWarps * 32, smem, st>>>(a);
  GT_CUDA_TRY(cudaGetLastError());
  return GT_OK;
}

template <typename T, int H, int D>
struct Ops {
  static gt_status run(int pass, const PArgs& a, cudaStream_t st) {
    if (pass == 0) return launch<T, H, D, 0>(a, st);
    if (pass == 1) return launch<T, H, D, 1>(a, st);
    return launch<T, H, D, 2>(a, st);
  }
};

gt_status dispatch(int dtype, int H, int D, int pass, const PArgs& a, cudaStream_t st) {
#define GT_CASE(TT, HH, DD) \
  if (H == HH && D == DD) return Ops<TT, HH, DD>::run(pass, a, st);
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

}  // namespace pipe

// Entry points used by launch_* in attn.cu when the pipelined kernels are selected.
gt_status pipe_pass(gt_plan_s* P, int pass, const void* own_a, const void* own_b, const float* lse,
                    const void* gather_a, const void* gather_b, const void* halo, void* out_a, void* out_b,
                    float* out_f, cudaStream_t st) {
  pipe::PArgs a{};
  const bool rows = pass != 2;
  a.iptr = (rows ? P->d_iptr_rows : P->d_iptr_cols).as<int64_t>();
  a.iown = (rows ? P->d_items_rows : P->d_items_cols).as<int32_t>();
  a.cown = (rows ? P->heavy_rows : P->heavy_cols).d_owner.as<int32_t>();
  a.nbr = (rows ? P->d_col : P->d_row).as<int32_t>();
  a.nitems = rows ? P->n_items_rows : P->n_items_cols;
  a.counter = P->d_counters.as<unsigned long long>() + pass;
  a.ga = (const char*)gather_a;
  a.gb = (const char*)gather_b;
  a.gs = (const char*)P->d_stats.p;
  a.halo = (const char*)halo;
  a.halo_stride = rows ? P->kv_row_bytes : P->in_row_bytes;
  a.n_local = P->n_local;
  a.oa = (const char*)own_a;
  a.ob = (const char*)own_b;
  a.lse = lse;
  a.out_a = (char*)out_a;
  a.out_b = (char*)out_b;
  a.out_f = out_f;
  a.part = (pass == 0 ? P->d_part_fwd : pass == 1 ? P->d_part_rowb : P->d_part_colb).as<float>();
  a.qscale = P->scale * pipe::kLog2e;
  a.scale = P->scale;
  return pipe::dispatch(P->dtype, P->heads, P->heads * P->d, pass, a, st);
}

}  // namespace gt
