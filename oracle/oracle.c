/*
 * oracle/oracle.c -- CPU fp64 ORACLE for full-graph multi-head sparse graph attention.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  It shares
 * no code with the CUDA path (paper_2604_16715_b200/), and neither imports the other.
 *
 * What it computes is the plain definition in the paper's notation:
 *   Eq. 2  alpha_ij = softmax_j( (W_Q x_i)^T (W_K x_j) / sqrt(d) ), j in N(i)
 *   Eq. 4  Z = (Q K^T) (.) A ,  U = Softmax(Z / sqrt(d))   (over row i's stored entries)
 *   Eq. 5  Y = U V
 *   Section 2.2: the backward of SDDMM/softmax/SpMM = 3 SpMM + 1 SDDMM:
 *       dU = (dY V^T) (.) A                     (SDDMM)
 *       dV = U^T dY                             (SpMM over A^T)
 *       dZ = U (.) (dU - rowsum(dU (.) U))      (softmax backward)  times the scale
 *       dQ = dZ K,  dK = dZ^T Q                 (2 SpMM, the second over A^T)
 *   "scale" is the factor multiplying Q K^T (1/sqrt(d) in Eq. 4; reading Z2 in DESIGN.md:
 *   the caller passes it explicitly).
 *   Multi-head (Alg. 1 shape notes [N,h,d']): every head t is computed independently
 *   on its d' = d slice of the [N, h, d] tensors.
 *
 * Readings: softmax ranges over the stored entries
 * of row i only (Z1); row i of the CSR lists the keys node i attends to (Z3); a row
 * with no entries gives Y = 0, LSE = -inf, dQ = 0 (Z4).
 *
 * Dataflow (deliberately different from the GPU's): two-pass softmax per row-head
 * (max, then sum), P and dS stored per edge in fp64, dK/dV through the oracle's own
 * counting-sort transpose.  All arithmetic is fp64 on inputs upcast exactly from
 * their storage dtype (fp32 or bf16 bit patterns, or fp64 as is).
 *
 * Partition / halo (readings Z9, Z10): contiguous row ranges balancing
 * rows + edges, found by a linear scan; halo sets by mark arrays.
 *
 * Pins: tests/test_oracle_*.py (dense brute force in torch fp64, worked examples,
 * closed forms, invariants, finite differences, hand-computed partitions).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_F32 = 0, OR_BF16 = 1, OR_F64 = 2 };

/* fp64 inputs (OR_F64) are read as they are: used by the SGA-block oracle (oracle/sga.py), whose
 * Q = X W_Q, K, V (Eq. 3) are fp64 products. */
static inline double ld(const void* x, int dt, int64_t i) {
  if (dt == OR_F64) return ((const double*)x)[i];
  if (dt == OR_F32) return (double)((const float*)x)[i];
  uint32_t u = (uint32_t)((const uint16_t*)x)[i] << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

typedef struct {
  int64_t n;
  const int64_t* row_ptr;
  const int32_t* col_idx;
  int heads, d, dtype;
  const void *q, *k, *v, *dy;
  double scale;
} or_problem;

/* s_e = scale * <q_i,t , k_j,t>  (Eq. 4: SDDMM of Q K^T sampled on A, times the scale) */
static double score(const or_problem* P, int64_t i, int64_t j, int t) {
  const int64_t D = (int64_t)P->heads * P->d;
  double acc = 0.0;
  for (int c = 0; c < P->d; ++c)
    acc += ld(P->q, P->dtype, i * D + (int64_t)t * P->d + c) * ld(P->k, P->dtype, j * D + (int64_t)t * P->d + c);
  return P->scale * acc;
}

/* <dY_i,t , v_j,t>  (backward SDDMM: dU = (dY V^T) (.) A) */
static double dscore(const or_problem* P, int64_t i, int64_t j, int t) {
  const int64_t D = (int64_t)P->heads * P->d;
  double acc = 0.0;
  for (int c = 0; c < P->d; ++c)
    acc += ld(P->dy, P->dtype, i * D + (int64_t)t * P->d + c) * ld(P->v, P->dtype, j * D + (int64_t)t * P->d + c);
  return acc;
}

/* Row i, head t: U_e (two-pass softmax over row i's stored entries, Eq. 2/4) into u[deg].
 * Returns lse = m + ln(l); -inf for an empty row. */
static double row_softmax(const or_problem* P, int64_t i, int t, double* u) {
  const int64_t e0 = P->row_ptr[i], e1 = P->row_ptr[i + 1];
  if (e1 == e0) return -INFINITY;
  double m = -INFINITY;
  for (int64_t e = e0; e < e1; ++e) {
    u[e - e0] = score(P, i, P->col_idx[e], t);
    if (u[e - e0] > m) m = u[e - e0];
  }
  double l = 0.0;
  for (int64_t e = e0; e < e1; ++e) l += exp(u[e - e0] - m);
  for (int64_t e = e0; e < e1; ++e) u[e - e0] = exp(u[e - e0] - m) / l;
  return m + log(l);
}

static int64_t max_degree(const or_problem* P) {
  int64_t mx = 0;
  for (int64_t i = 0; i < P->n; ++i)
    if (P->row_ptr[i + 1] - P->row_ptr[i] > mx) mx = P->row_ptr[i + 1] - P->row_ptr[i];
  return mx;
}

/* Forward for one row: Y_i,t = sum_e U_e v_j,t (Eq. 5 SpMM); y has h*d entries, lse h. */
static void row_forward(const or_problem* P, int64_t i, double* u, double* y, double* lse) {
  const int64_t D = (int64_t)P->heads * P->d;
  const int64_t e0 = P->row_ptr[i], e1 = P->row_ptr[i + 1];
  for (int t = 0; t < P->heads; ++t) {
    lse[t] = row_softmax(P, i, t, u);
    for (int c = 0; c < P->d; ++c) {
      double acc = 0.0;
      for (int64_t e = e0; e < e1; ++e) acc += u[e - e0] * ld(P->v, P->dtype, (int64_t)P->col_idx[e] * D + (int64_t)t * P->d + c);
      y[(int64_t)t * P->d + c] = acc;
    }
  }
}

/* Backward stage 1 for one row, all heads: U_e, dU_e = <dY_i, v_j>, Dstat = sum_e U_e dU_e,
 * dZ_e = scale * U_e (dU_e - Dstat)   (softmax backward of Eq. 4 with the scale),
 * dQ_i = sum_e dZ_e k_j               (SpMM dQ = dZ K).
 * Stores u_out[e*h+t] = U_e, ds_out[e*h+t] = dZ_e (indexed relative to row start). */
static void row_backward(const or_problem* P, int64_t i, double* u, double* u_out, double* ds_out, double* dq,
                         double* dstat) {
  const int64_t D = (int64_t)P->heads * P->d;
  const int h = P->heads;
  const int64_t e0 = P->row_ptr[i], e1 = P->row_ptr[i + 1];
  for (int t = 0; t < h; ++t) {
    for (int c = 0; c < P->d; ++c) dq[(int64_t)t * P->d + c] = 0.0;
    dstat[t] = 0.0;
    if (e1 == e0) continue;
    row_softmax(P, i, t, u);
    double Dt = 0.0;
    for (int64_t e = e0; e < e1; ++e) {
      double du = dscore(P, i, P->col_idx[e], t);
      ds_out[(e - e0) * h + t] = du; /* temporarily dU */
      Dt += u[e - e0] * du;
    }
    dstat[t] = Dt;
    for (int64_t e = e0; e < e1; ++e) {
      double ds = P->scale * u[e - e0] * (ds_out[(e - e0) * h + t] - Dt);
      ds_out[(e - e0) * h + t] = ds;
      u_out[(e - e0) * h + t] = u[e - e0];
      int64_t j = P->col_idx[e];
      for (int c = 0; c < P->d; ++c) dq[(int64_t)t * P->d + c] += ds * ld(P->k, P->dtype, j * D + (int64_t)t * P->d + c);
    }
  }
}

/* ------------------------------------------------------------ full graph -- */

/* y: [n,h,d] fp64, lse: [n,h] fp64 */
int oracle_fwd(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int heads, int d, int dtype,
               const void* q, const void* k, const void* v, double scale, double* y, double* lse) {
  or_problem P = {n, row_ptr, col_idx, heads, d, dtype, q, k, v, NULL, scale};
  const int64_t D = (int64_t)heads * d;
  int64_t mx = max_degree(&P);
#pragma omp parallel
  {
    double* u = (double*)malloc((size_t)(mx > 0 ? mx : 1) * sizeof(double));
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) row_forward(&P, i, u, y + i * D, lse + i * heads);
    free(u);
  }
  return 0;
}

/* Oracle's own transpose (plain counting sort over the edge list, stable in edge order):
 * col_ptr[n+1], row_of[nnz] (source row), eid[nnz] (edge id in CSR order). */
void oracle_transpose(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t* col_ptr, int32_t* row_of,
                      int64_t* eid) {
  const int64_t nnz = row_ptr[n];
  for (int64_t j = 0; j <= n; ++j) col_ptr[j] = 0;
  for (int64_t e = 0; e < nnz; ++e) col_ptr[col_idx[e] + 1]++;
  for (int64_t j = 0; j < n; ++j) col_ptr[j + 1] += col_ptr[j];
  int64_t* fill = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  memcpy(fill, col_ptr, (size_t)(n + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      int64_t pos = fill[col_idx[e]]++;
      row_of[pos] = (int32_t)i;
      if (eid) eid[pos] = e;
    }
  free(fill);
}

/* dq, dk, dv: [n,h,d] fp64; dstat: [n,h] fp64 (D_i = sum_e U_e dU_e). */
int oracle_bwd(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int heads, int d, int dtype,
               const void* q, const void* k, const void* v, const void* dy, double scale, double* dq, double* dk,
               double* dv, double* dstat) {
  or_problem P = {n, row_ptr, col_idx, heads, d, dtype, q, k, v, dy, scale};
  const int64_t D = (int64_t)heads * d;
  const int64_t nnz = row_ptr[n];
  int64_t mx = max_degree(&P);
  double* U = (double*)malloc((size_t)(nnz > 0 ? nnz : 1) * heads * sizeof(double));
  double* dS = (double*)malloc((size_t)(nnz > 0 ? nnz : 1) * heads * sizeof(double));
  /* stage 1: rows */
#pragma omp parallel
  {
    double* u = (double*)malloc((size_t)(mx > 0 ? mx : 1) * sizeof(double));
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i)
      row_backward(&P, i, u, U + row_ptr[i] * heads, dS + row_ptr[i] * heads, dq + i * D, dstat + i * heads);
    free(u);
  }
  /* stage 2: columns, via the oracle's own transpose.
   * dV_j = sum_{e=(i,j)} U_e dY_i   (SpMM U^T dY);  dK_j = sum_{e=(i,j)} dZ_e q_i  (SpMM dZ^T Q) */
  int64_t* col_ptr = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  int32_t* row_of = (int32_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
  int64_t* eid = (int64_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int64_t));
  oracle_transpose(n, row_ptr, col_idx, col_ptr, row_of, eid);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t j = 0; j < n; ++j) {
    for (int t = 0; t < heads; ++t)
      for (int c = 0; c < d; ++c) {
        double av = 0.0, ak = 0.0;
        for (int64_t x = col_ptr[j]; x < col_ptr[j + 1]; ++x) {
          int64_t i = row_of[x], e = eid[x];
          av += U[e * heads + t] * ld(dy, dtype, i * D + (int64_t)t * d + c);
          ak += dS[e * heads + t] * ld(q, dtype, i * D + (int64_t)t * d + c);
        }
        dv[j * D + (int64_t)t * d + c] = av;
        dk[j * D + (int64_t)t * d + c] = ak;
      }
  }
  free(col_ptr); free(row_of); free(eid); free(U); free(dS);
  return 0;
}

/* ------------------------------------------------------------- sampled ---- */
/* Same definitions restricted to sampled outputs (for graphs too large for a full
 * fp64 oracle).  rows[nr]: y/lse/dq/dstat for those rows; cols[nc]: dk/dv for those
 * columns.  Any of the output pointers may be NULL to skip that output. */
int oracle_sample(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int heads, int d, int dtype,
                  const void* q, const void* k, const void* v, const void* dy, double scale, int64_t nr,
                  const int64_t* rows, double* y, double* lse, double* dq, double* dstat, int64_t nc,
                  const int64_t* cols, double* dk, double* dv) {
  or_problem P = {n, row_ptr, col_idx, heads, d, dtype, q, k, v, dy, scale};
  const int64_t D = (int64_t)heads * d;
  int64_t mx = max_degree(&P);
#pragma omp parallel
  {
    double* u = (double*)malloc((size_t)(mx > 0 ? mx : 1) * sizeof(double));
    double* uo = (double*)malloc((size_t)(mx > 0 ? mx : 1) * heads * sizeof(double));
    double* so = (double*)malloc((size_t)(mx > 0 ? mx : 1) * heads * sizeof(double));
    double* tq = (double*)malloc((size_t)D * sizeof(double));
    double* td = (double*)malloc((size_t)heads * sizeof(double));
#pragma omp for schedule(dynamic, 1)
    for (int64_t x = 0; x < nr; ++x) {
      int64_t i = rows[x];
      if (y || lse) {
        double* ty = (double*)malloc((size_t)D * sizeof(double));
        double* tl = (double*)malloc((size_t)heads * sizeof(double));
        row_forward(&P, i, u, ty, tl);
        if (y) memcpy(y + x * D, ty, (size_t)D * sizeof(double));
        if (lse) memcpy(lse + x * heads, tl, (size_t)heads * sizeof(double));
        free(ty); free(tl);
      }
      if ((dq || dstat) && dy) {
        row_backward(&P, i, u, uo, so, tq, td);
        if (dq) memcpy(dq + x * D, tq, (size_t)D * sizeof(double));
        if (dstat) memcpy(dstat + x * heads, td, (size_t)heads * sizeof(double));
      }
    }
    free(u); free(uo); free(so); free(tq); free(td);
  }
  if (nc > 0 && (dk || dv) && dy) {
    /* in-edges of the sampled columns, found by scanning the edge list */
    int64_t* slot = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    for (int64_t j = 0; j < n; ++j) slot[j] = -1;
    for (int64_t x = 0; x < nc; ++x) slot[cols[x]] = x;
    if (dk) memset(dk, 0, (size_t)(nc * D) * sizeof(double));
    if (dv) memset(dv, 0, (size_t)(nc * D) * sizeof(double));
    /* rows with at least one edge into a sampled column */
    uint8_t* need = (uint8_t*)calloc((size_t)n, 1);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
        if (slot[col_idx[e]] >= 0) { need[i] = 1; break; }
    int64_t nneed = 0;
    for (int64_t i = 0; i < n; ++i) nneed += need[i];
    int64_t* rl = (int64_t*)malloc((size_t)(nneed > 0 ? nneed : 1) * sizeof(int64_t));
    nneed = 0;
    for (int64_t i = 0; i < n; ++i)
      if (need[i]) rl[nneed++] = i;
    /* Per needed row: stage-1 values U_e, dZ_e.  Collect (column slot, row i, U, dZ)
     * contributions, then reduce per column in ascending row order. */
    int64_t ncontrib = 0;
    for (int64_t x = 0; x < nneed; ++x) {
      int64_t i = rl[x];
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
        if (slot[col_idx[e]] >= 0) ncontrib++;
    }
    int64_t* c_off = (int64_t*)malloc((size_t)(nneed + 1) * sizeof(int64_t));
    c_off[0] = 0;
    for (int64_t x = 0; x < nneed; ++x) {
      int64_t i = rl[x], c = 0;
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
        if (slot[col_idx[e]] >= 0) c++;
      c_off[x + 1] = c_off[x] + c;
    }
    int64_t* c_slot = (int64_t*)malloc((size_t)(ncontrib > 0 ? ncontrib : 1) * sizeof(int64_t));
    int64_t* c_row = (int64_t*)malloc((size_t)(ncontrib > 0 ? ncontrib : 1) * sizeof(int64_t));
    double* c_u = (double*)malloc((size_t)(ncontrib > 0 ? ncontrib : 1) * heads * sizeof(double));
    double* c_s = (double*)malloc((size_t)(ncontrib > 0 ? ncontrib : 1) * heads * sizeof(double));
#pragma omp parallel
    {
      double* u = (double*)malloc((size_t)(mx > 0 ? mx : 1) * sizeof(double));
      double* uo = (double*)malloc((size_t)(mx > 0 ? mx : 1) * heads * sizeof(double));
      double* so = (double*)malloc((size_t)(mx > 0 ? mx : 1) * heads * sizeof(double));
      double* tq = (double*)malloc((size_t)D * sizeof(double));
      double* td = (double*)malloc((size_t)heads * sizeof(double));
#pragma omp for schedule(dynamic, 1)
      for (int64_t x = 0; x < nneed; ++x) {
        int64_t i = rl[x];
        row_backward(&P, i, u, uo, so, tq, td);
        int64_t w = c_off[x];
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
          int64_t s = slot[col_idx[e]];
          if (s < 0) continue;
          c_slot[w] = s;
          c_row[w] = i;
          for (int t = 0; t < heads; ++t) {
            c_u[w * heads + t] = uo[(e - row_ptr[i]) * heads + t];
            c_s[w * heads + t] = so[(e - row_ptr[i]) * heads + t];
          }
          w++;
        }
      }
      free(u); free(uo); free(so); free(tq); free(td);
    }
    for (int64_t w = 0; w < ncontrib; ++w) {
      int64_t s = c_slot[w], i = c_row[w];
      for (int t = 0; t < heads; ++t)
        for (int c = 0; c < d; ++c) {
          int64_t o = s * D + (int64_t)t * d + c;
          if (dv) dv[o] += c_u[w * heads + t] * ld(dy, dtype, i * D + (int64_t)t * d + c);
          if (dk) dk[o] += c_s[w * heads + t] * ld(q, dtype, i * D + (int64_t)t * d + c);
        }
    }
    free(c_off); free(c_slot); free(c_row); free(c_u); free(c_s);
    free(rl); free(need); free(slot);
  }
  return 0;
}

/* ------------------------------------------------------ partition / halo -- */

/* Reading Z9: W(i) = row_ptr[i] + i; bounds[0] = 0, bounds[p] = n,
 * bounds[r] = min{ i : W(i) >= ceil(r (E+N) / p) }  (linear scan).
 * mode 1: SPEC node-balanced rule: first n mod p ranks get one extra row. */
int oracle_partition(int64_t n, const int64_t* row_ptr, int p, int mode, int64_t* bounds) {
  if (p <= 0 || n < 0) return 1;
  if (mode == 1) {
    int64_t base = n / p, rem = n % p, pos = 0;
    for (int r = 0; r < p; ++r) {
      bounds[r] = pos;
      pos += base + (r < rem ? 1 : 0);
    }
    bounds[p] = n;
    return 0;
  }
  const int64_t total = row_ptr[n] + n;
  bounds[0] = 0;
  int64_t i = 0;
  for (int r = 1; r < p; ++r) {
    int64_t target = (int64_t)(((__int128)r * total + p - 1) / p);
    while (i < n && row_ptr[i] + i < target) ++i;
    bounds[r] = i;
  }
  bounds[p] = n;
  return 0;
}

/* Out-halo of rank r: sorted unique columns outside [lo,hi) referenced by rows in [lo,hi).
 * In-halo of rank r: sorted unique rows outside [lo,hi) with an edge into a column in [lo,hi).
 * Returns the count; writes up to cap entries into out (out may be NULL to count only). */
int64_t oracle_halo(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t lo, int64_t hi, int inward,
                    int32_t* out, int64_t cap) {
  uint8_t* mark = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  if (!inward) {
    for (int64_t i = lo; i < hi; ++i)
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        int64_t j = col_idx[e];
        if (j < lo || j >= hi) mark[j] = 1;
      }
  } else {
    for (int64_t i = 0; i < n; ++i) {
      if (i >= lo && i < hi) continue;
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        int64_t j = col_idx[e];
        if (j >= lo && j < hi) { mark[i] = 1; break; }
      }
    }
  }
  int64_t cnt = 0;
  for (int64_t j = 0; j < n; ++j)
    if (mark[j]) {
      if (out && cnt < cap) out[cnt] = (int32_t)j;
      cnt++;
    }
  free(mark);
  return cnt;
}
