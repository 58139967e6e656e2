/*
 * gtgen/csrc/gen.c -- seeded synthetic INPUT generators (graphs and features).
 *
 * This module is shared by the CUDA path's tests/bench and by the CPU oracle's
 * tests.  It holds none of the method's arithmetic (no attention, no softmax,
 * no partitioning): it only draws random numbers and assembles an input graph
 * in canonical CSR form (rows' columns strictly increasing, no duplicates, no
 * self-loops), and i.i.d. N(0,1) feature tensors.
 *
 * Recipes:
 *   - Chung-Lu style sampling: endpoint u ~ w_out, endpoint v ~ w_in (or the
 *     same weights when undirected); optional communities of consecutive ids,
 *     where with probability f_in the second endpoint is drawn inside u's
 *     community.
 *   - R-MAT (Graph500 a,b,c,d) with a seeded label permutation.
 *   - Exactly M unique pairs are kept: the FIRST M unique samples in sample
 *     order (samples are counter-based, so this is independent of threading).
 *
 * RNG: Philox4x32-10 keyed by (seed), counter = (index, stream).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ RNG -- */
static inline uint32_t mulhilo(uint32_t a, uint32_t b, uint32_t* hi) {
  uint64_t p = (uint64_t)a * b;
  *hi = (uint32_t)(p >> 32);
  return (uint32_t)p;
}

/* Philox4x32-10 (Salmon et al., SC'11), standard constants. */
static inline void philox4x32_10(const uint32_t in[4], uint64_t key64, uint32_t out[4]) {
  uint32_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
  uint32_t k0 = (uint32_t)key64, k1 = (uint32_t)(key64 >> 32);
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, hi1;
    uint32_t lo0 = mulhilo(0xD2511F53u, c0, &hi0);
    uint32_t lo1 = mulhilo(0xCD9E8D57u, c2, &hi1);
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static inline void rng4(uint64_t seed, uint32_t stream, uint64_t ctr, uint32_t out[4]) {
  uint32_t in[4] = {(uint32_t)ctr, (uint32_t)(ctr >> 32), stream, 0x6774u /* "gt" */};
  philox4x32_10(in, seed, out);
}

/* 53-bit uniform in the open interval (0,1). */
static inline double u01(uint32_t a, uint32_t b) {
  uint64_t x = ((uint64_t)(a >> 5) << 26) | (uint64_t)(b >> 6);
  return ((double)x + 0.5) * (1.0 / 9007199254740992.0);
}

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* -------------------------------------------------------------- features -- */
/* i.i.d. N(0,1) via Box-Muller; element i of tensor `tensor_id` comes from Philox counter i / 4,
 * so any slice [start, start + n) of the flat tensor can be generated on its own. */
static inline float normal_at(uint64_t seed, uint32_t tensor_id, int64_t i) {
  uint32_t r[4];
  rng4(seed, 0x10000u + tensor_id, (uint64_t)(i >> 2), r);
  int c = (int)(i & 3);
  double u1 = ((double)(r[c < 2 ? 0 : 2] >> 8) + 0.5) * (1.0 / 16777216.0);
  double u2 = ((double)(r[c < 2 ? 1 : 3] >> 8) + 0.5) * (1.0 / 16777216.0);
  double rad = sqrt(-2.0 * log(u1)), th = 6.283185307179586 * u2;
  return (float)((c & 1) ? rad * sin(th) : rad * cos(th));
}

void gen_normal_f32_range(uint64_t seed, uint32_t tensor_id, int64_t start, int64_t n, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = normal_at(seed, tensor_id, start + i);
}

void gen_normal_f32(uint64_t seed, uint32_t tensor_id, int64_t n, float* out) {
  gen_normal_f32_range(seed, tensor_id, 0, n, out);
}

/* fp32 -> bf16 bits, round to nearest even (inputs are finite). */
void gen_f32_to_bf16(const float* in, int64_t n, uint16_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u;
    memcpy(&u, &in[i], 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    out[i] = (uint16_t)(u >> 16);
  }
}

/* ----------------------------------------------------------------- graphs -- */
typedef struct {
  int32_t kind;      /* 0 = Chung-Lu (weights), 1 = R-MAT */
  int32_t directed;  /* 0 = undirected (pairs symmetrised), 1 = directed */
  int64_t n;         /* nodes */
  int64_t m;         /* unique pairs (undirected) or edges (directed) to keep */
  uint64_t seed;
  /* Chung-Lu weights: dist 0 = Pareto(param = gamma), 1 = lognormal(param = sigma), 2 = constant */
  int32_t wdist_out, wdist_in;
  double wparam_out, wmean_out, wcap_out;
  double wparam_in, wmean_in, wcap_in;
  int64_t comm_size; /* communities of consecutive ids of this size (0 = none) */
  double f_in;       /* probability the second endpoint is drawn inside u's community */
  /* R-MAT */
  int32_t scale;
  double a, b, c;
  int32_t permute;   /* apply a seeded label permutation */
  double oversample; /* initial samples = m * oversample */
} gen_params;

static void make_weights(uint64_t seed, uint32_t stream, int64_t n, int dist, double param, double mean,
                         double cap, double* w) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint32_t r[4];
    rng4(seed, stream, (uint64_t)i, r);
    double u = u01(r[0], r[1]);
    double x;
    if (dist == 0) {
      x = pow(u, -1.0 / (param - 1.0));
    } else if (dist == 1) {
      double u2 = u01(r[2], r[3]);
      double z = sqrt(-2.0 * log(u)) * cos(6.283185307179586 * u2);
      x = exp(param * z);
    } else {
      x = 1.0;
    }
    w[i] = x;
  }
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += w[i];
  double f = mean * (double)n / s;
  for (int64_t i = 0; i < n; ++i) {
    double x = w[i] * f;
    w[i] = (cap > 0 && x > cap) ? cap : x;
  }
}

/* cum has n+1 entries; returns index i in [lo,hi) with cum[i] <= x < cum[i+1]. */
static inline int64_t pick(const double* cum, int64_t lo, int64_t hi, double u) {
  double x = cum[lo] + u * (cum[hi] - cum[lo]);
  int64_t a = lo, b = hi - 1;
  while (a < b) {
    int64_t mid = (a + b + 1) >> 1;
    if (cum[mid] <= x) a = mid; else b = mid - 1;
  }
  return a;
}

#define BAD_KEY UINT64_MAX

static void sample_chung_lu(const gen_params* p, const double* cum_out, const double* cum_in, int64_t s0,
                            int64_t s1, uint64_t* keys) {
  const int64_t n = p->n;
#pragma omp parallel for schedule(static)
  for (int64_t s = s0; s < s1; ++s) {
    uint32_t r[4], q[4];
    rng4(p->seed, 1, (uint64_t)s, r);
    rng4(p->seed, 2, (uint64_t)s, q);
    int64_t u = pick(cum_out, 0, n, u01(r[0], r[1]));
    int64_t v;
    if (p->comm_size > 0 && u01(r[2], r[3]) < p->f_in) {
      int64_t c0 = (u / p->comm_size) * p->comm_size;
      int64_t c1 = c0 + p->comm_size < n ? c0 + p->comm_size : n;
      v = pick(cum_in, c0, c1, u01(q[0], q[1]));
    } else {
      v = pick(cum_in, 0, n, u01(q[0], q[1]));
    }
    uint64_t key;
    if (u == v) key = BAD_KEY;
    else if (p->directed) key = ((uint64_t)u << 32) | (uint64_t)v;
    else key = u < v ? (((uint64_t)u << 32) | (uint64_t)v) : (((uint64_t)v << 32) | (uint64_t)u);
    keys[s - s0] = key;
  }
}

static void sample_rmat(const gen_params* p, const int64_t* perm, int64_t s0, int64_t s1, uint64_t* keys) {
  const double a = p->a, ab = p->a + p->b, abc = p->a + p->b + p->c;
  const int sc = p->scale;
#pragma omp parallel for schedule(static)
  for (int64_t s = s0; s < s1; ++s) {
    uint64_t u = 0, v = 0;
    uint32_t r[4] = {0, 0, 0, 0};
    for (int l = 0; l < sc; ++l) {
      if ((l & 3) == 0) rng4(p->seed, 3, (uint64_t)s * 8u + (uint64_t)(l >> 2), r);
      double x = ((double)r[l & 3] + 0.5) * (1.0 / 4294967296.0);
      int bu, bv;
      if (x < a) { bu = 0; bv = 0; }
      else if (x < ab) { bu = 0; bv = 1; }
      else if (x < abc) { bu = 1; bv = 0; }
      else { bu = 1; bv = 1; }
      u = (u << 1) | (uint64_t)bu;
      v = (v << 1) | (uint64_t)bv;
    }
    if (perm) { u = (uint64_t)perm[u]; v = (uint64_t)perm[v]; }
    uint64_t key;
    if (u == v) key = BAD_KEY;
    else if (p->directed) key = (u << 32) | v;
    else key = u < v ? ((u << 32) | v) : ((v << 32) | u);
    keys[s - s0] = key;
  }
}

/* Marks keep[s] = 1 for the first occurrence of each key, scanning in sample
 * order, stopping once m unique keys are marked.  Returns the number marked. */
static int64_t dedup_first_m(const uint64_t* keys, int64_t S, int64_t m, uint8_t* keep) {
  enum { SH_BITS = 12, NSH = 1 << SH_BITS };
  int nt = 1;
#ifdef _OPENMP
  nt = omp_get_max_threads();
#endif
  int64_t* cnt = (int64_t*)calloc((size_t)nt * NSH, sizeof(int64_t));
  int64_t* shard_off = (int64_t*)calloc(NSH + 1, sizeof(int64_t));
  uint32_t* order = (uint32_t*)malloc((size_t)S * sizeof(uint32_t));
  memset(keep, 0, (size_t)S);
  int64_t chunk = (S + nt - 1) / nt;
#pragma omp parallel num_threads(nt)
  {
    int t = 0;
#ifdef _OPENMP
    t = omp_get_thread_num();
#endif
    int64_t a = t * chunk, b = a + chunk < S ? a + chunk : S;
    for (int64_t s = a; s < b; ++s)
      if (keys[s] != BAD_KEY) cnt[(size_t)t * NSH + (mix64(keys[s]) >> (64 - SH_BITS))]++;
  }
  /* offsets: shard-major, then thread-major (thread chunks are in sample order) */
  int64_t pos = 0;
  for (int sh = 0; sh < NSH; ++sh) {
    shard_off[sh] = pos;
    for (int t = 0; t < nt; ++t) {
      int64_t c = cnt[(size_t)t * NSH + sh];
      cnt[(size_t)t * NSH + sh] = pos;
      pos += c;
    }
  }
  shard_off[NSH] = pos;
#pragma omp parallel num_threads(nt)
  {
    int t = 0;
#ifdef _OPENMP
    t = omp_get_thread_num();
#endif
    int64_t a = t * chunk, b = a + chunk < S ? a + chunk : S;
    for (int64_t s = a; s < b; ++s)
      if (keys[s] != BAD_KEY) order[cnt[(size_t)t * NSH + (mix64(keys[s]) >> (64 - SH_BITS))]++] = (uint32_t)s;
  }
#pragma omp parallel for schedule(dynamic, 8)
  for (int sh = 0; sh < NSH; ++sh) {
    int64_t a = shard_off[sh], b = shard_off[sh + 1], k = b - a;
    if (k == 0) continue;
    int64_t cap = 16;
    while (cap < 2 * k) cap <<= 1;
    uint64_t* tab = (uint64_t*)malloc((size_t)cap * sizeof(uint64_t));
    for (int64_t i = 0; i < cap; ++i) tab[i] = BAD_KEY;
    for (int64_t i = a; i < b; ++i) {
      uint32_t s = order[i];
      uint64_t key = keys[s];
      uint64_t h = mix64(key ^ 0x5bd1e995ull) & (uint64_t)(cap - 1);
      for (;;) {
        if (tab[h] == BAD_KEY) { tab[h] = key; keep[s] = 1; break; }
        if (tab[h] == key) break;
        h = (h + 1) & (uint64_t)(cap - 1);
      }
    }
    free(tab);
  }
  int64_t kept = 0;
  for (int64_t s = 0; s < S; ++s) {
    if (!keep[s]) continue;
    if (kept < m) kept++;
    else keep[s] = 0;
  }
  free(cnt); free(shard_off); free(order);
  return kept;
}

static int cmp_i32(const void* x, const void* y) {
  int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
  return (a > b) - (a < b);
}

/* Builds canonical CSR from the kept keys.  Returns nnz. */
static int64_t keys_to_csr(const gen_params* p, const uint64_t* keys, const uint8_t* keep, int64_t S,
                           int64_t** row_ptr_out, int32_t** col_out) {
  const int64_t n = p->n;
  int64_t* rp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t* fill = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < S; ++s) {
    if (!keep[s]) continue;
    uint64_t u = keys[s] >> 32, v = keys[s] & 0xffffffffull;
    __atomic_fetch_add(&rp[u + 1], 1, __ATOMIC_RELAXED);
    if (!p->directed) __atomic_fetch_add(&rp[v + 1], 1, __ATOMIC_RELAXED);
  }
  for (int64_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
  int64_t nnz = rp[n];
  int32_t* col = (int32_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
  memcpy(fill, rp, ((size_t)n + 1) * sizeof(int64_t));
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < S; ++s) {
    if (!keep[s]) continue;
    uint64_t u = keys[s] >> 32, v = keys[s] & 0xffffffffull;
    col[__atomic_fetch_add(&fill[u], 1, __ATOMIC_RELAXED)] = (int32_t)v;
    if (!p->directed) col[__atomic_fetch_add(&fill[v], 1, __ATOMIC_RELAXED)] = (int32_t)u;
  }
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i)
    if (rp[i + 1] - rp[i] > 1) qsort(col + rp[i], (size_t)(rp[i + 1] - rp[i]), sizeof(int32_t), cmp_i32);
  free(fill);
  *row_ptr_out = rp;
  *col_out = col;
  return nnz;
}

/* Generates a graph.  Returns nnz (>= 0) or a negative error code:
 *   -1 bad params, -2 could not reach m unique pairs. */
int64_t gen_graph(const gen_params* p, int64_t** row_ptr, int32_t** col_idx) {
  if (p->n <= 0 || p->m < 0 || p->n >= (1ll << 31)) return -1;
  double* cum_out = NULL;
  double* cum_in = NULL;
  int64_t* perm = NULL;
  if (p->kind == 0) {
    double* w = (double*)malloc((size_t)p->n * sizeof(double));
    cum_out = (double*)malloc(((size_t)p->n + 1) * sizeof(double));
    make_weights(p->seed, 100, p->n, p->wdist_out, p->wparam_out, p->wmean_out, p->wcap_out, w);
    cum_out[0] = 0;
    for (int64_t i = 0; i < p->n; ++i) cum_out[i + 1] = cum_out[i] + w[i];
    if (p->directed) {
      make_weights(p->seed, 101, p->n, p->wdist_in, p->wparam_in, p->wmean_in, p->wcap_in, w);
      cum_in = (double*)malloc(((size_t)p->n + 1) * sizeof(double));
      cum_in[0] = 0;
      for (int64_t i = 0; i < p->n; ++i) cum_in[i + 1] = cum_in[i] + w[i];
    } else {
      cum_in = cum_out;
    }
    free(w);
  } else if (p->kind == 1) {
    if ((1ll << p->scale) != p->n) return -1;
    if (p->permute) {
      perm = (int64_t*)malloc((size_t)p->n * sizeof(int64_t));
      for (int64_t i = 0; i < p->n; ++i) perm[i] = i;
      for (int64_t i = p->n - 1; i > 0; --i) { /* Fisher-Yates, counter-based */
        uint32_t r[4];
        rng4(p->seed, 4, (uint64_t)i, r);
        int64_t j = (int64_t)(u01(r[0], r[1]) * (double)(i + 1));
        if (j > i) j = i;
        int64_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
      }
    }
  } else {
    return -1;
  }
  double os = p->oversample > 1.0 ? p->oversample : 1.1;
  int64_t S = (int64_t)((double)p->m * os) + 1024;
  int64_t rc = -2;
  for (int attempt = 0; attempt < 8; ++attempt) {
    if (S >= (1ll << 32)) break;
    uint64_t* keys = (uint64_t*)malloc((size_t)S * sizeof(uint64_t));
    uint8_t* keep = (uint8_t*)malloc((size_t)S);
    if (p->kind == 0) sample_chung_lu(p, cum_out, cum_in, 0, S, keys);
    else sample_rmat(p, perm, 0, S, keys);
    int64_t kept = dedup_first_m(keys, S, p->m, keep);
    if (kept == p->m) {
      rc = keys_to_csr(p, keys, keep, S, row_ptr, col_idx);
      free(keys); free(keep);
      break;
    }
    free(keys); free(keep);
    S = (int64_t)((double)S * 1.5);
  }
  if (cum_in && cum_in != cum_out) free(cum_in);
  free(cum_out);
  free(perm);
  return rc;
}

void gen_free(void* ptr) { free(ptr); }

int gen_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
