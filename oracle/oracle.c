/*
 * oracle.c -- plain CPU oracle (IEEE double) for RelaNN's lifted join-aggregate.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this.  It shares no code
 * with paper_2605_24207_b200/ and never imports it.
 *
 * Each function is the plain definition from the paper, evaluated with nested loops
 * in the order the definition states; no blocking, fusion or reordering.  Library
 * primitives used: qsort (a sort) and bsearch-style binary search.
 *
 * Parity status: every function here is pinned by a -m "not gpu" test in tests/ against
 * something other than itself (brute-force nested-loop joins, dense closed forms, finite
 * differences, adjoint identities, dense matrix powers, published splitmix64 vectors).
 * See DESIGN.md "Oracle pins".  No function is "parity unpinned".
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* O1 step 1: key -> row map as a sorted (key,row) array.  Relations are sets           */
/* ("r is a relation"), so a repeated key is an error.        */
/* ------------------------------------------------------------------------------------ */
typedef struct { int64_t key; int64_t row; } kr_pair;

static int cmp_kr(const void* a, const void* b) {
  int64_t x = ((const kr_pair*)a)->key, y = ((const kr_pair*)b)->key;
  return (x > y) - (x < y);
}

typedef struct { kr_pair* v; int64_t n; } keymap;

static int keymap_build(const int64_t* keys, int64_t n, keymap* m) {
  m->n = n;
  m->v = (kr_pair*)malloc((size_t)(n > 0 ? n : 1) * sizeof(kr_pair));
  if (!m->v) return ORA_ERR_NOMEM;
  for (int64_t i = 0; i < n; ++i) { m->v[i].key = keys[i]; m->v[i].row = i; }
  qsort(m->v, (size_t)n, sizeof(kr_pair), cmp_kr);
  for (int64_t i = 1; i < n; ++i)
    if (m->v[i].key == m->v[i - 1].key) { free(m->v); m->v = NULL; return ORA_ERR_DUPLICATE_KEY; }
  return ORA_OK;
}

static int64_t keymap_find(const keymap* m, int64_t key) {
  int64_t lo = 0, hi = m->n - 1;
  while (lo <= hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (m->v[mid].key == key) return m->v[mid].row;
    if (m->v[mid].key < key) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

/* ------------------------------------------------------------------------------------ */
/* O1: canonical join index                                                              */
/* ------------------------------------------------------------------------------------ */
typedef struct { int64_t t_key; int64_t s_key; int64_t j; int64_t s_row; } jrow;

static int cmp_jrow_edge(const void* a, const void* b) {
  const jrow* x = (const jrow*)a; const jrow* y = (const jrow*)b;
  if (x->t_key != y->t_key) return (x->t_key > y->t_key) - (x->t_key < y->t_key);
  return (x->j > y->j) - (x->j < y->j);
}
static int cmp_jrow_srckey(const void* a, const void* b) {
  const jrow* x = (const jrow*)a; const jrow* y = (const jrow*)b;
  if (x->t_key != y->t_key) return (x->t_key > y->t_key) - (x->t_key < y->t_key);
  if (x->s_key != y->s_key) return (x->s_key > y->s_key) - (x->s_key < y->s_key);
  return (x->j > y->j) - (x->j < y->j);
}

int ora_build_join_index(const int64_t* e_src_key, const int64_t* e_dst_key, int64_t n_e,
                         const int64_t* s_key, int64_t n_s,
                         const int64_t* t_key, int64_t n_t,
                         int within_by_src_key,
                         int64_t* n_join_rows, int64_t* n_groups,
                         int64_t* group_ptr, int64_t* group_key, int32_t* group_dst_row,
                         int32_t* src_row, int32_t* edge_row,
                         int64_t* src_ptr, int32_t* src_pos) {
  if (n_e < 0 || !e_dst_key || (s_key && !e_src_key)) return ORA_ERR_BAD_ARG;
  keymap S = {0, 0}, T = {0, 0};
  int st;
  if (s_key && (st = keymap_build(s_key, n_s, &S)) != ORA_OK) return st;
  if (t_key && (st = keymap_build(t_key, n_t, &T)) != ORA_OK) { free(S.v); return st; }

  /* step 2: J = { j : s_j in S and t_j in T }  (natural join) */
  jrow* J = (jrow*)malloc((size_t)(n_e > 0 ? n_e : 1) * sizeof(jrow));
  if (!J) { free(S.v); free(T.v); return ORA_ERR_NOMEM; }
  int64_t nj = 0;
  for (int64_t j = 0; j < n_e; ++j) {
    int64_t sr = -1;
    if (s_key) { sr = keymap_find(&S, e_src_key[j]); if (sr < 0) continue; }
    if (t_key && keymap_find(&T, e_dst_key[j]) < 0) continue;
    J[nj].t_key = e_dst_key[j];
    J[nj].s_key = e_src_key ? e_src_key[j] : 0;
    J[nj].j = j;
    J[nj].s_row = sr;
    ++nj;
  }
  /* steps 3-4: groups = sorted distinct t (signed ascending); rows ordered by (group, j)
   * or, for the DHN adjacency variant, by (group, s key, j). */
  qsort(J, (size_t)nj, sizeof(jrow), within_by_src_key ? cmp_jrow_srckey : cmp_jrow_edge);
  int64_t G = 0;
  for (int64_t p = 0; p < nj; ++p) {
    if (p == 0 || J[p].t_key != J[p - 1].t_key) {
      group_key[G] = J[p].t_key;
      group_ptr[G] = p;
      group_dst_row[G] = t_key ? (int32_t)keymap_find(&T, J[p].t_key) : -1;
      ++G;
    }
    src_row[p] = (int32_t)J[p].s_row;
    edge_row[p] = (int32_t)J[p].j;
  }
  group_ptr[G] = nj;
  *n_join_rows = nj;
  *n_groups = G;

  /* step 5: source-major order = positions p sorted by (src_row[p], p): a stable counting
   * sort over p ascending.  src_ptr spans all n_s source rows (empty ones included). */
  if (s_key && src_ptr) {
    for (int64_t i = 0; i <= n_s; ++i) src_ptr[i] = 0;
    for (int64_t p = 0; p < nj; ++p) src_ptr[src_row[p] + 1] += 1;
    for (int64_t i = 0; i < n_s; ++i) src_ptr[i + 1] += src_ptr[i];
    int64_t* cur = (int64_t*)malloc((size_t)(n_s > 0 ? n_s : 1) * sizeof(int64_t));
    if (!cur) { free(J); free(S.v); free(T.v); return ORA_ERR_NOMEM; }
    for (int64_t i = 0; i < n_s; ++i) cur[i] = src_ptr[i];
    for (int64_t p = 0; p < nj; ++p) src_pos[cur[src_row[p]]++] = (int32_t)p;
    free(cur);
  }
  free(J); free(S.v); free(T.v);
  return ORA_OK;
}

/* ------------------------------------------------------------------------------------ */
/* O2/O3/O4: forward and backward LJA                                                    */
/* ------------------------------------------------------------------------------------ */
static int present(const ora_operand* o) { return o && o->data; }

static int64_t src_index(const ora_operand* o, const int32_t* src_row, int64_t p) {
  return o->mode == 1 ? p : (int64_t)src_row[p];
}
static int64_t edge_index(const ora_operand* o, const int32_t* edge_row, int64_t p) {
  return o->mode == 1 ? p : (int64_t)edge_row[p];
}
static int64_t dst_index(const ora_operand* o, const int32_t* group_dst_row, int64_t g) {
  return o->mode == 1 ? g : (int64_t)group_dst_row[g];
}
/* value of operand at row r, component c; a dim-1 operand broadcasts as a scalar */
static double at(const ora_operand* o, int64_t r, int c) {
  return o->dim == 1 ? o->data[r * o->ld] : o->data[r * o->ld + c];
}

/* output width implied by (combine, agg, operands); -1 if the combination is invalid */
static int out_dim(int combine, int agg, int heads, const ora_operand* s, const ora_operand* k,
                   const ora_operand* e, const ora_operand* t) {
  if (agg == ORA_AGG_SOFTMAX) {
    if (!present(s) || !present(k) || !present(t) || present(e) || heads < 1) return -1;
    if (s->dim % heads || k->dim % heads || k->dim != t->dim) return -1;
    return s->dim;
  }
  if (combine == ORA_COMBINE_SRC) {
    if (!present(s) || present(t) || (present(e) && e->dim != 1)) return -1;
    return s->dim;
  }
  if (combine == ORA_COMBINE_CONCAT)
    return (present(s) ? s->dim : 0) + (present(e) ? e->dim : 0) + (present(t) ? t->dim : 0);
  if (combine == ORA_COMBINE_MUL || combine == ORA_COMBINE_ADD) {
    int D = 0;
    const ora_operand* ops[3] = {s, e, t};
    for (int i = 0; i < 3; ++i) if (present(ops[i]) && ops[i]->dim > D) D = ops[i]->dim;
    for (int i = 0; i < 3; ++i)
      if (present(ops[i]) && ops[i]->dim != D && ops[i]->dim != 1) return -1;
    return D > 0 ? D : -1;
  }
  return -1;
}

/* per-row combined value v[c], c < D (the transformation T_tau of PAPER.md:444-447) */
static void combine_row(int combine, const ora_operand* s, int64_t rs, const ora_operand* e,
                        int64_t re, const ora_operand* t, int64_t rt, int D, double* v) {
  if (combine == ORA_COMBINE_SRC) {
    double w = present(e) ? e->data[re * e->ld] : 1.0;
    for (int c = 0; c < D; ++c) v[c] = w * s->data[rs * s->ld + c];
    return;
  }
  if (combine == ORA_COMBINE_CONCAT) {
    int o = 0;
    if (present(s)) for (int c = 0; c < s->dim; ++c) v[o++] = s->data[rs * s->ld + c];
    if (present(e)) for (int c = 0; c < e->dim; ++c) v[o++] = e->data[re * e->ld + c];
    if (present(t)) for (int c = 0; c < t->dim; ++c) v[o++] = t->data[rt * t->ld + c];
    return;
  }
  for (int c = 0; c < D; ++c) {
    double acc = combine == ORA_COMBINE_MUL ? 1.0 : 0.0;
    if (present(s)) acc = combine == ORA_COMBINE_MUL ? acc * at(s, rs, c) : acc + at(s, rs, c);
    if (present(e)) acc = combine == ORA_COMBINE_MUL ? acc * at(e, re, c) : acc + at(e, re, c);
    if (present(t)) acc = combine == ORA_COMBINE_MUL ? acc * at(t, rt, c) : acc + at(t, rt, c);
    v[c] = acc;
  }
}

/* score e_{p,i} = scale * < key[s_p, i-block], q[t_g, i-block] >   (Fig. 4) */
static double att_score(const ora_operand* k, int64_t rs, const ora_operand* q, int64_t rt,
                        int i, int dk, double scale) {
  double acc = 0.0;
  for (int c = 0; c < dk; ++c) acc += k->data[rs * k->ld + i * dk + c] * q->data[rt * q->ld + i * dk + c];
  return scale * acc;
}

int ora_lja_fwd(const int64_t* group_ptr, int64_t n_groups,
                const int32_t* src_row, const int32_t* edge_row, const int32_t* group_dst_row,
                int combine, int agg, int heads, double scale,
                const ora_operand* src, const ora_operand* src_key,
                const ora_operand* edge, const ora_operand* dst,
                const int64_t* sel, int64_t n_sel,
                double* out, int64_t ld_out, double* lse) {
  int D = out_dim(combine, agg, heads, src, src_key, edge, dst);
  if (D < 0) return ORA_ERR_BAD_ARG;
  int64_t n = sel ? n_sel : n_groups;
  double* v = (double*)malloc(sizeof(double) * (size_t)(D > 0 ? D : 1));
  if (!v) return ORA_ERR_NOMEM;
  for (int64_t i = 0; i < n; ++i) {
    int64_t g = sel ? sel[i] : i;
    if (g < 0 || g >= n_groups) { free(v); return ORA_ERR_BAD_ARG; }
    int64_t b = group_ptr[g], e = group_ptr[g + 1];
    double* o = out + i * ld_out;
    for (int c = 0; c < D; ++c) o[c] = 0.0;
    if (agg == ORA_AGG_SOFTMAX) {
      /* a = softmax over the rows of the group, per head; out = sum a * value (Fig. 4) */
      int dk = src_key->dim / heads, dv = src->dim / heads;
      int64_t rt = dst_index(dst, group_dst_row, g);
      for (int h = 0; h < heads; ++h) {
        double m = -INFINITY;
        for (int64_t p = b; p < e; ++p) {
          double s = att_score(src_key, src_index(src_key, src_row, p), dst, rt, h, dk, scale);
          if (s > m) m = s;
        }
        double z = 0.0;
        for (int64_t p = b; p < e; ++p)
          z += exp(att_score(src_key, src_index(src_key, src_row, p), dst, rt, h, dk, scale) - m);
        for (int64_t p = b; p < e; ++p) {
          int64_t rs = src_index(src, src_row, p);
          double a = exp(att_score(src_key, src_index(src_key, src_row, p), dst, rt, h, dk, scale) - m) / z;
          for (int c = 0; c < dv; ++c) o[h * dv + c] += a * src->data[rs * src->ld + h * dv + c];
        }
        if (lse) lse[i * heads + h] = m + log(z);
      }
      continue;
    }
    for (int64_t p = b; p < e; ++p) {
      combine_row(combine, src, present(src) ? src_index(src, src_row, p) : -1,
                  edge, present(edge) ? edge_index(edge, edge_row, p) : -1,
                  dst, present(dst) ? dst_index(dst, group_dst_row, g) : -1, D, v);
      for (int c = 0; c < D; ++c) o[c] += v[c];
    }
    if (agg == ORA_AGG_MEAN)   /* one-shot mean over the full multiset */
      for (int c = 0; c < D; ++c) o[c] /= (double)(e - b);
  }
  free(v);
  return ORA_OK;
}

static void zero_fill(double* x, int64_t rows, const ora_operand* o) {
  if (x && present(o)) memset(x, 0, sizeof(double) * (size_t)(rows * o->dim));
}

int ora_lja_bwd(const int64_t* group_ptr, int64_t n_groups,
                const int32_t* src_row, const int32_t* edge_row, const int32_t* group_dst_row,
                int combine, int agg, int heads, double scale,
                const ora_operand* src, const ora_operand* src_key,
                const ora_operand* edge, const ora_operand* dst,
                const double* d_out, int64_t ld_dout,
                int64_t n_src_rows, int64_t n_edge_rows, int64_t n_dst_rows,
                double* d_src, double* d_src_key, double* d_edge, double* d_dst) {
  int D = out_dim(combine, agg, heads, src, src_key, edge, dst);
  if (D < 0) return ORA_ERR_BAD_ARG;
  /* gradient buffers are dense [rows, dim] with ld = dim */
  zero_fill(d_src, n_src_rows, src);
  zero_fill(d_src_key, n_src_rows, src_key);
  zero_fill(d_edge, n_edge_rows, edge);
  zero_fill(d_dst, n_dst_rows, dst);
  for (int64_t g = 0; g < n_groups; ++g) {
    int64_t b = group_ptr[g], e = group_ptr[g + 1];
    const double* dO = d_out + g * ld_dout;
    if (agg == ORA_AGG_SOFTMAX) {
      int dk = src_key->dim / heads, dv = src->dim / heads;
      int64_t rt = dst_index(dst, group_dst_row, g);
      for (int h = 0; h < heads; ++h) {
        double m = -INFINITY, z = 0.0, Dsum = 0.0;
        for (int64_t p = b; p < e; ++p) {
          double s = att_score(src_key, src_index(src_key, src_row, p), dst, rt, h, dk, scale);
          if (s > m) m = s;
        }
        for (int64_t p = b; p < e; ++p)
          z += exp(att_score(src_key, src_index(src_key, src_row, p), dst, rt, h, dk, scale) - m);
        /* D = sum_q a_q da_q with da_p = < dOut_{g,h}, v_p > */
        for (int64_t p = b; p < e; ++p) {
          int64_t rs = src_index(src, src_row, p);
          double a = exp(att_score(src_key, src_index(src_key, src_row, p), dst, rt, h, dk, scale) - m) / z;
          double da = 0.0;
          for (int c = 0; c < dv; ++c) da += dO[h * dv + c] * src->data[rs * src->ld + h * dv + c];
          Dsum += a * da;
        }
        for (int64_t p = b; p < e; ++p) {
          int64_t rs = src_index(src, src_row, p), rk = src_index(src_key, src_row, p);
          double a = exp(att_score(src_key, rk, dst, rt, h, dk, scale) - m) / z;
          double da = 0.0;
          for (int c = 0; c < dv; ++c) da += dO[h * dv + c] * src->data[rs * src->ld + h * dv + c];
          double de = a * (da - Dsum);
          if (d_src)
            for (int c = 0; c < dv; ++c) d_src[rs * src->dim + h * dv + c] += a * dO[h * dv + c];
          if (d_src_key)
            for (int c = 0; c < dk; ++c)
              d_src_key[rk * src_key->dim + h * dk + c] += scale * de * dst->data[rt * dst->ld + h * dk + c];
          if (d_dst)
            for (int c = 0; c < dk; ++c)
              d_dst[rt * dst->dim + h * dk + c] += scale * de * src_key->data[rk * src_key->ld + h * dk + c];
        }
      }
      continue;
    }
    double cg = agg == ORA_AGG_MEAN ? 1.0 / (double)(e - b) : 1.0;
    for (int64_t p = b; p < e; ++p) {
      int64_t rs = present(src) ? src_index(src, src_row, p) : -1;
      int64_t re = present(edge) ? edge_index(edge, edge_row, p) : -1;
      int64_t rt = present(dst) ? dst_index(dst, group_dst_row, g) : -1;
      if (combine == ORA_COMBINE_SRC) {
        double w = present(edge) ? edge->data[re * edge->ld] : 1.0;
        double dw = 0.0;
        for (int c = 0; c < D; ++c) {
          if (d_src) d_src[rs * src->dim + c] += cg * w * dO[c];
          dw += cg * dO[c] * src->data[rs * src->ld + c];
        }
        if (d_edge && present(edge)) d_edge[re] += dw;
      } else if (combine == ORA_COMBINE_CONCAT) {
        int o = 0;
        if (present(src)) { for (int c = 0; c < src->dim; ++c, ++o) if (d_src) d_src[rs * src->dim + c] += cg * dO[o]; }
        if (present(edge)) { for (int c = 0; c < edge->dim; ++c, ++o) if (d_edge) d_edge[re * edge->dim + c] += cg * dO[o]; }
        if (present(dst)) { for (int c = 0; c < dst->dim; ++c, ++o) if (d_dst) d_dst[rt * dst->dim + c] += cg * dO[o]; }
      } else {
        /* MUL / ADD: d(operand X) = G (.) (product of the other operands) for MUL, = G for ADD;
         * a dim-1 operand receives the sum over components. */
        const ora_operand* ops[3] = {src, edge, dst};
        int64_t rows[3] = {rs, re, rt};
        double* grads[3] = {d_src, d_edge, d_dst};
        for (int x = 0; x < 3; ++x) {
          if (!present(ops[x]) || !grads[x]) continue;
          for (int c = 0; c < D; ++c) {
            double other = 1.0;
            if (combine == ORA_COMBINE_MUL)
              for (int y = 0; y < 3; ++y) if (y != x && present(ops[y])) other *= at(ops[y], rows[y], c);
            double gval = cg * dO[c] * other;
            if (ops[x]->dim == 1) grads[x][rows[x]] += gval;
            else grads[x][rows[x] * ops[x]->dim + c] += gval;
          }
        }
      }
    }
  }
  return ORA_OK;
}

/* ------------------------------------------------------------------------------------ */
/* standalone grouped softmax (the ATT relation)                           */
/* ------------------------------------------------------------------------------------ */
int ora_group_softmax(const int64_t* group_ptr, int64_t n_groups, int heads,
                      const double* scores, double* probs) {
  if (heads < 1) return ORA_ERR_BAD_ARG;
  for (int64_t g = 0; g < n_groups; ++g)
    for (int h = 0; h < heads; ++h) {
      double m = -INFINITY, z = 0.0;
      for (int64_t p = group_ptr[g]; p < group_ptr[g + 1]; ++p) if (scores[p * heads + h] > m) m = scores[p * heads + h];
      for (int64_t p = group_ptr[g]; p < group_ptr[g + 1]; ++p) z += exp(scores[p * heads + h] - m);
      for (int64_t p = group_ptr[g]; p < group_ptr[g + 1]; ++p) probs[p * heads + h] = exp(scores[p * heads + h] - m) / z;
    }
  return ORA_OK;
}

int ora_group_softmax_bwd(const int64_t* group_ptr, int64_t n_groups, int heads,
                          const double* probs, const double* d_probs, double* d_scores) {
  if (heads < 1) return ORA_ERR_BAD_ARG;
  for (int64_t g = 0; g < n_groups; ++g)
    for (int h = 0; h < heads; ++h) {
      double dot = 0.0;
      for (int64_t p = group_ptr[g]; p < group_ptr[g + 1]; ++p) dot += probs[p * heads + h] * d_probs[p * heads + h];
      for (int64_t p = group_ptr[g]; p < group_ptr[g + 1]; ++p)
        d_scores[p * heads + h] = probs[p * heads + h] * (d_probs[p * heads + h] - dot);
    }
  return ORA_OK;
}

/* ------------------------------------------------------------------------------------ */
/* O5: dense projection and its backward                                                 */
/* ------------------------------------------------------------------------------------ */
int ora_project(const double* X, int64_t M, int64_t K, int64_t ldx,
                const double* W, int64_t N, int64_t ldw, const double* bias,
                double* Y, int64_t ldy) {
  for (int64_t m = 0; m < M; ++m)
    for (int64_t n = 0; n < N; ++n) {
      double acc = bias ? bias[n] : 0.0;
      for (int64_t k = 0; k < K; ++k) acc += X[m * ldx + k] * W[n * ldw + k];
      Y[m * ldy + n] = acc;
    }
  return ORA_OK;
}

int ora_project_bwd(const double* X, int64_t M, int64_t K, int64_t ldx,
                    const double* W, int64_t N, int64_t ldw,
                    const double* dY, int64_t lddy,
                    double* dX, double* dW, double* db) {
  if (dX)
    for (int64_t m = 0; m < M; ++m)
      for (int64_t k = 0; k < K; ++k) {
        double acc = 0.0;
        for (int64_t n = 0; n < N; ++n) acc += dY[m * lddy + n] * W[n * ldw + k];
        dX[m * K + k] = acc;
      }
  if (dW)
    for (int64_t n = 0; n < N; ++n)
      for (int64_t k = 0; k < K; ++k) {
        double acc = 0.0;
        for (int64_t m = 0; m < M; ++m) acc += dY[m * lddy + n] * X[m * ldx + k];
        dW[n * K + k] = acc;
      }
  if (db)
    for (int64_t n = 0; n < N; ++n) {
      double acc = 0.0;
      for (int64_t m = 0; m < M; ++m) acc += dY[m * lddy + n];
      db[n] = acc;
    }
  return ORA_OK;
}

/* ------------------------------------------------------------------------------------ */
/* O7: GCN normalisation weights                                                         */
/* ------------------------------------------------------------------------------------ */
int ora_gcn_norm(const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                 const int32_t* group_dst_row, int64_t n_nodes, double* w) {
  int64_t* deg = (int64_t*)calloc((size_t)(n_nodes > 0 ? n_nodes : 1), sizeof(int64_t));
  if (!deg) return ORA_ERR_NOMEM;
  for (int64_t g = 0; g < n_groups; ++g) {
    if (group_dst_row[g] < 0) { free(deg); return ORA_ERR_BAD_ARG; }
    deg[group_dst_row[g]] = group_ptr[g + 1] - group_ptr[g];
  }
  for (int64_t g = 0; g < n_groups; ++g)
    for (int64_t p = group_ptr[g]; p < group_ptr[g + 1]; ++p) {
      int64_t ds = deg[src_row[p]], dt = group_ptr[g + 1] - group_ptr[g];
      w[p] = (ds > 0 ? 1.0 / sqrt((double)ds) : 0.0) * (dt > 0 ? 1.0 / sqrt((double)dt) : 0.0);
    }
  free(deg);
  return ORA_OK;
}

/* ------------------------------------------------------------------------------------ */
/* O6: DHN closed-walk aggregates                                                        */
/* ------------------------------------------------------------------------------------ */
typedef struct {
  const int64_t* group_ptr; const int32_t* src_row; const int64_t* node_key;
  const int64_t* grp_of_row;  /* node row -> group id (or -1 if no out-edges) */
} adj_t;

/* number of join rows Edge(x, r): neighbours of x are sorted by key (within_by_src_key) */
static int64_t edge_count(const adj_t* A, int64_t x, int64_t r) {
  int64_t g = A->grp_of_row[x];
  if (g < 0) return 0;
  int64_t key = A->node_key[r], lo = A->group_ptr[g], hi = A->group_ptr[g + 1], cnt = 0;
  /* lower bound */
  int64_t a = lo, b = hi;
  while (a < b) { int64_t m = a + (b - a) / 2; if (A->node_key[A->src_row[m]] < key) a = m + 1; else b = m; }
  while (a < hi && A->node_key[A->src_row[a]] == key) { ++cnt; ++a; }
  return cnt;
}

typedef void (*walk_fn)(void* ctx, const int32_t* v, int64_t mult);

/* enumerate the join rows of the C_k rule rooted at node row r:
 *   k=2: Edge(n,v)                          (one Edge atom, no closing edge)
 *   k=3: Edge(n,v), Edge(v,w), Edge(w,n)
 *   k=4: Edge(n,v), Edge(v,w), Edge(w,p), Edge(p,n)                                     */
static void dhn_walks(const adj_t* A, int k, int64_t g, int32_t r, walk_fn fn, void* ctx) {
  int32_t v[4];
  v[0] = r;
  for (int64_t a = A->group_ptr[g]; a < A->group_ptr[g + 1]; ++a) {
    v[1] = A->src_row[a];
    if (k == 2) { fn(ctx, v, 1); continue; }
    int64_t g1 = A->grp_of_row[v[1]];
    if (g1 < 0) continue;
    for (int64_t b = A->group_ptr[g1]; b < A->group_ptr[g1 + 1]; ++b) {
      v[2] = A->src_row[b];
      if (k == 3) { int64_t m = edge_count(A, v[2], r); if (m) fn(ctx, v, m); continue; }
      int64_t g2 = A->grp_of_row[v[2]];
      if (g2 < 0) continue;
      for (int64_t c = A->group_ptr[g2]; c < A->group_ptr[g2 + 1]; ++c) {
        v[3] = A->src_row[c];
        int64_t m = edge_count(A, v[3], r);
        if (m) fn(ctx, v, m);
      }
    }
  }
}

typedef struct {
  int k, d; const double* const* f; int64_t ldf;
  double* acc;                  /* fwd: [d] accumulator for the root */
  const double* dO;             /* bwd: upstream grad row of the root */
  double* const* d_f;
} dhn_ctx;

static void dhn_fwd_visit(void* vc, const int32_t* v, int64_t mult) {
  dhn_ctx* C = (dhn_ctx*)vc;
  for (int c = 0; c < C->d; ++c) {
    double prod = (double)mult;
    for (int i = 1; i < C->k; ++i) prod *= C->f[i][(int64_t)v[i] * C->ldf + c];
    C->acc[c] += prod;
  }
}

static void dhn_bwd_visit(void* vc, const int32_t* v, int64_t mult) {
  dhn_ctx* C = (dhn_ctx*)vc;
  for (int c = 0; c < C->d; ++c)
    for (int j = 0; j < C->k; ++j) {
      if (!C->d_f[j]) continue;
      double prod = (double)mult * C->dO[c];
      for (int i = 0; i < C->k; ++i) if (i != j) prod *= C->f[i][(int64_t)v[i] * C->ldf + c];
      C->d_f[j][(int64_t)v[j] * C->d + c] += prod;
    }
}

static int64_t* make_grp_of_row(const int32_t* group_dst_row, int64_t n_groups, int64_t n_nodes) {
  int64_t* m = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_nodes > 0 ? n_nodes : 1));
  if (!m) return NULL;
  for (int64_t i = 0; i < n_nodes; ++i) m[i] = -1;
  for (int64_t g = 0; g < n_groups; ++g) m[group_dst_row[g]] = g;
  return m;
}

int ora_dhn_fwd(int k, const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                const int32_t* group_dst_row, const int64_t* node_key, int64_t n_nodes,
                const double* const* f, int64_t ldf, int d,
                const int64_t* sel, int64_t n_sel, double* out, int64_t ld_out) {
  if (k < 2 || k > 4) return ORA_ERR_BAD_ARG;
  int64_t* gor = make_grp_of_row(group_dst_row, n_groups, n_nodes);
  if (!gor) return ORA_ERR_NOMEM;
  adj_t A = {group_ptr, src_row, node_key, gor};
  double* acc = (double*)malloc(sizeof(double) * (size_t)d);
  dhn_ctx C = {k, d, f, ldf, acc, NULL, NULL};
  int64_t n = sel ? n_sel : n_groups;
  for (int64_t i = 0; i < n; ++i) {
    int64_t g = sel ? sel[i] : i;
    int32_t r = group_dst_row[g];
    for (int c = 0; c < d; ++c) acc[c] = 0.0;
    dhn_walks(&A, k, g, r, dhn_fwd_visit, &C);
    for (int c = 0; c < d; ++c) out[i * ld_out + c] = f[0][(int64_t)r * ldf + c] * acc[c];
  }
  free(acc); free(gor);
  return ORA_OK;
}

int ora_dhn_bwd(int k, const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                const int32_t* group_dst_row, const int64_t* node_key, int64_t n_nodes,
                const double* const* f, int64_t ldf, int d,
                const double* d_out, int64_t ld_dout, double* const* d_f) {
  if (k < 2 || k > 4) return ORA_ERR_BAD_ARG;
  int64_t* gor = make_grp_of_row(group_dst_row, n_groups, n_nodes);
  if (!gor) return ORA_ERR_NOMEM;
  for (int j = 0; j < k; ++j) if (d_f[j]) memset(d_f[j], 0, sizeof(double) * (size_t)(n_nodes * d));
  adj_t A = {group_ptr, src_row, node_key, gor};
  dhn_ctx C = {k, d, f, ldf, NULL, NULL, d_f};
  for (int64_t g = 0; g < n_groups; ++g) {
    C.dO = d_out + g * ld_dout;
    dhn_walks(&A, k, g, group_dst_row[g], dhn_bwd_visit, &C);
  }
  free(gor);
  return ORA_OK;
}

/* ------------------------------------------------------------------------------------ */
/* hash partition                                                                        */
/* ------------------------------------------------------------------------------------ */
uint64_t ora_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int ora_hash_partition(const int64_t* keys, int64_t n, int32_t P, uint64_t seed, int32_t* owner) {
  if (P < 1) return ORA_ERR_BAD_ARG;
  for (int64_t i = 0; i < n; ++i) owner[i] = (int32_t)(ora_splitmix64((uint64_t)keys[i] ^ seed) % (uint64_t)P);
  return ORA_OK;
}
