// Host-side planning logic of libgt.so: CSR validation, row partition, halo sets, heavy
// row/column chunking, and the paper's cost model / AGP selector (Eq. 6-14, Alg. 3).
// Plan-time only; none of this runs inside gt_attn_fwd / gt_attn_bwd.
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "gt_internal.h"

namespace gt {

gt_status validate_csr(const int64_t* row_ptr, const int32_t* col_idx, int64_t n, int64_t nnz) {
  if (row_ptr[0] != 0) return fail(GT_EGRAPH, "row_ptr[0] != 0");
  if (row_ptr[n] != nnz) return fail(GT_EGRAPH, "row_ptr[n] != nnz");
  std::atomic<int64_t> bad_row{-1};
  std::atomic<int> kind{0};
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i) {
    int64_t a = row_ptr[i], b = row_ptr[i + 1];
    int k = 0;
    if (b < a || a < 0 || b > nnz) k = 1;
    else
      for (int64_t e = a; e < b; ++e) {
        int32_t c = col_idx[e];
        if (c < 0 || c >= n) { k = 2; break; }
        if (e > a && col_idx[e - 1] >= c) { k = 3; break; }
      }
    if (k) {
      int64_t cur = bad_row.load();
      while ((cur < 0 || i < cur) && !bad_row.compare_exchange_weak(cur, i)) {}
      if (bad_row.load() == i) kind.store(k);
    }
  }
  if (bad_row.load() >= 0) {
    static const char* what[] = {"", "row_ptr not nondecreasing", "column index out of range",
                                 "columns not strictly increasing (duplicate or unsorted)"};
    return fail(GT_EGRAPH, std::string("CSR invalid at row ") + std::to_string(bad_row.load()) + ": " +
                               what[kind.load()]);
  }
  return GT_OK;
}

// Reading Z9: W(i) = row_ptr[i] + i; bounds[r] = min{ i : W(i) >= ceil(r (E + N) / p) }.
// W is strictly increasing, so the minimum is found by binary search (the oracle scans).
void partition_rows(int64_t n, const int64_t* row_ptr, int p, int mode, int64_t* bounds) {
  if (mode == 1) {  // first n mod p ranks get one extra row
    int64_t base = n / p, rem = n % p, pos = 0;
    for (int r = 0; r < p; ++r) {
      bounds[r] = pos;
      pos += base + (r < rem ? 1 : 0);
    }
    bounds[p] = n;
    return;
  }
  const __int128 total = (__int128)row_ptr[n] + n;
  bounds[0] = 0;
  for (int r = 1; r < p; ++r) {
    int64_t target = (int64_t)((total * r + p - 1) / p);
    int64_t a = 0, b = n;  // smallest i in [0, n] with row_ptr[i] + i >= target
    while (a < b) {
      int64_t m = a + (b - a) / 2;
      if (row_ptr[m] + m >= target) b = m; else a = m + 1;
    }
    bounds[r] = a;
  }
  bounds[p] = n;
}

// Halo of one owned range [lo, hi): bitmap mark over N, then an ordered compaction.
std::vector<int32_t> halo_set(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t lo, int64_t hi,
                              bool inward) {
  const int64_t words = (n + 63) / 64;
  std::vector<uint64_t> bits((size_t)std::max<int64_t>(words, 1), 0);
  uint64_t* B = bits.data();
  if (!inward) {
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = lo; i < hi; ++i)
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        int64_t j = col_idx[e];
        if (j < lo || j >= hi) __atomic_fetch_or(&B[j >> 6], 1ull << (j & 63), __ATOMIC_RELAXED);
      }
  } else {
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
      if (i >= lo && i < hi) continue;
      const int32_t* c0 = col_idx + row_ptr[i];
      const int32_t* c1 = col_idx + row_ptr[i + 1];
      const int32_t* it = std::lower_bound(c0, c1, (int32_t)lo);  // columns are sorted
      if (it != c1 && *it < hi) __atomic_fetch_or(&B[i >> 6], 1ull << (i & 63), __ATOMIC_RELAXED);
    }
  }
  // ordered compaction: per-word popcounts, prefix, then fill
  std::vector<int64_t> off((size_t)words + 1, 0);
  for (int64_t w = 0; w < words; ++w) off[w + 1] = off[w] + __builtin_popcountll(B[w]);
  std::vector<int32_t> out((size_t)off[words]);
#pragma omp parallel for schedule(static)
  for (int64_t w = 0; w < words; ++w) {
    uint64_t x = B[w];
    int64_t pos = off[w];
    while (x) {
      int b = __builtin_ctzll(x);
      out[pos++] = (int32_t)(w * 64 + b);
      x &= x - 1;
    }
  }
  return out;
}

std::vector<int32_t> send_set(int64_t n, const int64_t* rp, const int32_t* ci, int64_t lo, int64_t hi,
                              int64_t blo, int64_t bhi, bool inward) {
  (void)n;
  const int64_t nl = hi - lo;
  std::vector<uint8_t> mark((size_t)std::max<int64_t>(nl, 1), 0);
  if (!inward) {
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = blo; i < bhi; ++i) {
      const int32_t* a = std::lower_bound(ci + rp[i], ci + rp[i + 1], (int32_t)lo);
      for (const int32_t* x = a; x < ci + rp[i + 1] && *x < hi; ++x) mark[*x - lo] = 1;
    }
  } else {
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = lo; i < hi; ++i) {
      const int32_t* a = std::lower_bound(ci + rp[i], ci + rp[i + 1], (int32_t)blo);
      if (a < ci + rp[i + 1] && *a < bhi) mark[i - lo] = 1;
    }
  }
  std::vector<int32_t> out;
  for (int64_t j = 0; j < nl; ++j)
    if (mark[j]) out.push_back((int32_t)(lo + j));
  return out;
}

void build_work(int64_t count, const std::function<void(int64_t, std::vector<Segment>&)>& segs, int64_t threshold,
                int nphase, WorkList* phases, ChunkTable* t, const std::function<bool(int64_t)>& force) {
  t->ids.clear(); t->first.clear(); t->chunk_lo.clear(); t->chunk_hi.clear(); t->chunk_owner.clear();
  for (int ph = 0; ph < nphase; ++ph) {
    phases[ph].beg.clear(); phases[ph].end.clear(); phases[ph].own.clear(); phases[ph].empty.clear();
  }
  std::vector<Segment> sg, pieces;
  for (int64_t r = 0; r < count; ++r) {
    sg.clear();
    segs(r, sg);
    pieces.clear();
    for (const Segment& s : sg) {
      const int64_t len = s.hi - s.lo;
      if (len <= 0) continue;
      const int64_t nch = (len + threshold - 1) / threshold;  // equal chunks of <= threshold entries
      for (int64_t c = 0; c < nch; ++c)
        pieces.push_back({s.lo + len * c / nch, s.lo + len * (c + 1) / nch, s.phase});
    }
    if (force && force(r)) {
      t->ids.push_back((int32_t)r);
      t->first.push_back((int32_t)t->chunk_lo.size());
      for (const Segment& p : pieces) {
        const int32_t ch = (int32_t)t->chunk_lo.size();
        t->chunk_lo.push_back(p.lo); t->chunk_hi.push_back(p.hi); t->chunk_owner.push_back((int32_t)r);
        WorkList& w = phases[p.phase];
        w.beg.push_back(p.lo); w.end.push_back(p.hi); w.own.push_back(-1 - ch);
      }
    } else if (pieces.empty()) {
      const int64_t at = sg.empty() ? 0 : sg.front().lo;
      (void)at;
      phases[0].empty.push_back((int32_t)r);
    } else if (pieces.size() == 1) {
      WorkList& w = phases[pieces[0].phase];
      w.beg.push_back(pieces[0].lo); w.end.push_back(pieces[0].hi); w.own.push_back((int32_t)r);
    } else {
      t->ids.push_back((int32_t)r);
      t->first.push_back((int32_t)t->chunk_lo.size());
      for (const Segment& p : pieces) {
        const int32_t c = (int32_t)t->chunk_lo.size();
        t->chunk_lo.push_back(p.lo); t->chunk_hi.push_back(p.hi); t->chunk_owner.push_back((int32_t)r);
        WorkList& w = phases[p.phase];
        w.beg.push_back(p.lo); w.end.push_back(p.hi); w.own.push_back(-1 - c);
      }
    }
  }
  t->first.push_back((int32_t)t->chunk_lo.size());
  for (int ph = 0; ph < nphase; ++ph) phases[ph].n = (int64_t)phases[ph].beg.size();
}

}  // namespace gt

using namespace gt;

extern "C" {

gt_status gt_partition(int64_t n, const int64_t* row_ptr, int p, int mode, int64_t* bounds) {
  if (n < 0 || p <= 0 || !bounds || (mode == 0 && !row_ptr) || (mode != 0 && mode != 1))
    return fail(GT_EINVAL, "gt_partition: bad arguments");
  partition_rows(n, row_ptr, p, mode, bounds);
  return GT_OK;
}

gt_status gt_halo(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t lo, int64_t hi, int inward,
                  int32_t* out, int64_t cap, int64_t* len) {
  if (n < 0 || !row_ptr || (!col_idx && row_ptr[n] > 0) || lo < 0 || hi > n || lo > hi || !len)
    return fail(GT_EINVAL, "gt_halo: bad arguments");
  std::vector<int32_t> h = halo_set(n, row_ptr, col_idx, lo, hi, inward != 0);
  *len = (int64_t)h.size();
  if (out) {
    if (cap < (int64_t)h.size()) return fail(GT_EINVAL, "gt_halo: cap too small");
    std::memcpy(out, h.data(), h.size() * sizeof(int32_t));
  }
  return GT_OK;
}

gt_status gt_send_list(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t lo, int64_t hi,
                       int64_t peer_lo, int64_t peer_hi, int inward, int32_t* out, int64_t cap, int64_t* len) {
  if (n < 0 || !row_ptr || (!col_idx && row_ptr[n] > 0) || lo < 0 || hi > n || lo > hi || peer_lo < 0 ||
      peer_hi > n || peer_lo > peer_hi || !len)
    return fail(GT_EINVAL, "gt_send_list: bad arguments");
  std::vector<int32_t> v = send_set(n, row_ptr, col_idx, lo, hi, peer_lo, peer_hi, inward != 0);
  *len = (int64_t)v.size();
  if (out) {
    if (cap < (int64_t)v.size()) return fail(GT_EINVAL, "gt_send_list: cap too small");
    std::memcpy(out, v.data(), v.size() * sizeof(int32_t));
  }
  return GT_OK;
}

// Eq. 7 with Eq. 8: t_iter(p) = alpha(1)/p * E + beta_c(p) * N; beta_c(1) = 0.
double gt_estimate_iter_time(double alpha1, const double* beta, int n_strategies, int P, int c, int p, double N,
                             double E) {
  if (p < 1 || p > P || c < 0 || c >= n_strategies) return NAN;
  double b = (p == 1) ? 0.0 : beta[(size_t)c * (P + 1) + p];
  return alpha1 * E / p + b * N;
}

// Algorithm 3, with the (score, c, i) bookkeeping of reading Z12.
gt_status gt_agp_select(double N, double t_iter1, const double* beta, int n_strategies, int P, int* c_out,
                        int* s_out, double* score_out) {
  if (!beta || !c_out || !s_out || N <= 0 || t_iter1 <= 0 || P < 1 || n_strategies < 1)
    return fail(GT_EINVAL, "gt_agp_select: bad arguments");
  const double k = t_iter1 / N;                    // line 3: k <- t_iter(1) / N
  double best = INFINITY;
  int bc = -1, bs = 1;
  for (int i = 2; i <= P; ++i)                     // line 4
    for (int c = 0; c < n_strategies; ++c) {       // line 5
      double b = beta[(size_t)c * (P + 1) + i];    // line 6: b = beta_c(i)
      double score = i * b / (i - 1);
      if (score <= k && score < best) {            // lines 7-8 (strict < keeps smaller i, then smaller c)
        best = score; bc = c; bs = i;
      }
    }
  *c_out = bc;                                     // line 12: argmin; none feasible => single GPU
  *s_out = bs;
  if (score_out) *score_out = bc >= 0 ? best : 0.0;
  return GT_OK;
}

gt_status gt_fit_beta(const double* x, const double* t, int m, double* beta) {
  if (!x || !t || !beta || m < 2) return fail(GT_EINVAL, "gt_fit_beta: need >= 2 samples");
  double acc = 0;
  for (int i = 0; i < m; ++i) {
    if (!(x[i] > 0) || !(t[i] > 0)) return fail(GT_EINVAL, "gt_fit_beta: non-positive sample");
    acc += std::log(t[i]) - std::log(x[i]);
  }
  *beta = std::exp(acc / m);
  return GT_OK;
}

}  // extern "C"
