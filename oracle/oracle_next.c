/*
 * oracle_next.c -- plain CPU oracle (IEEE double) for the SURVEY sec 8f rows: node epilogues,
 * the MAX aggregate, the training step's loss and optimiser.  TEST INFRASTRUCTURE ONLY (see
 * oracle.h); shares nothing with the product path.  Plain loops, each function the textbook
 * definition it names.
 *
 *   epilogue  : y = gate * act(x + b) + (1 - gate) * r    (GCN bias + ReLU, PAPER.md:865 / O7;
 *               HGT skip gate sigmoid(skip) over H^{l-1}, PAPER.md:1392-1394 [src-only]);
 *               GELU(x) = x * Phi(x) = x (1 + erf(x / sqrt 2)) / 2
 *   MAX       : projected union with the max aggregate ("sum, mean, or
 *               max"), per output column; ties -> the lowest join position; an empty group
 *               aggregates to 0 (scatter_max convention); the gradient flows to the arg-max
 *               row only (subgradient of max)
 *   loss      : Loss(; CrossEntropyLoss()(Cls(z_p), z_l)), the mean over the
 *               labelled rows of -log softmax(logits)[label]
 *   fit       : ?fit <epochs, lr, weight_decay> -- one Adam step
 *               (Kingma & Ba 2015, bias-corrected) with L2 weight decay added to the gradient
 *               (torch.optim.Adam semantics; the optimiser is not named in the paper)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

static double act_f(int act, double x) {
  if (act == 1) return x > 0.0 ? x : 0.0;
  if (act == 2) return 0.5 * x * (1.0 + erf(x / sqrt(2.0)));
  return x;
}
static double act_d(int act, double x) {
  if (act == 1) return x > 0.0 ? 1.0 : 0.0;
  if (act == 2) return 0.5 * (1.0 + erf(x / sqrt(2.0))) + x * exp(-0.5 * x * x) / 2.5066282746310002;
  return 1.0;
}

int ora_epilogue_fwd(const double* x, int64_t rows, int dim, int64_t ldx, const double* bias,
                     int act, double gate, const double* resid, int64_t ld_resid, double* y,
                     int64_t ldy) {
  if (act < 0 || act > 2 || (resid && (gate < 0.0 || gate > 1.0))) return ORA_ERR_BAD_ARG;
  for (int64_t r = 0; r < rows; ++r)
    for (int c = 0; c < dim; ++c) {
      double v = act_f(act, x[r * ldx + c] + (bias ? bias[c] : 0.0));
      if (resid) v = gate * v + (1.0 - gate) * resid[r * ld_resid + c];
      y[r * ldy + c] = v;
    }
  return ORA_OK;
}

/* dx = dy * g * act'(x + b); d_bias = sum_r dx; d_resid = (1 - g) dy; d_gate = sum dy (act - r)
 * (g = gate with a residual, 1 without).  Outputs nullable, written. */
int ora_epilogue_bwd(const double* dy, const double* x, int64_t rows, int dim, const double* bias,
                     int act, double gate, const double* resid, double* dx, double* d_bias,
                     double* d_resid, double* d_gate) {
  if (act < 0 || act > 2) return ORA_ERR_BAD_ARG;
  const double g = resid ? gate : 1.0;
  if (d_bias) for (int c = 0; c < dim; ++c) d_bias[c] = 0.0;
  if (d_gate) *d_gate = 0.0;
  for (int64_t r = 0; r < rows; ++r)
    for (int c = 0; c < dim; ++c) {
      const int64_t i = r * dim + c;
      const double pre = x[i] + (bias ? bias[c] : 0.0);
      const double d = dy[i] * g * act_d(act, pre);
      if (dx) dx[i] = d;
      if (d_bias) d_bias[c] += d;
      if (d_resid && resid) d_resid[i] = (1.0 - gate) * dy[i];
      if (d_gate && resid) *d_gate += dy[i] * (act_f(act, pre) - resid[i]);
    }
  return ORA_OK;
}

/* MAX aggregate of the SRC combine (w * z_s, w = scalar edge operand or 1) per group and
 * column: out[g, c] = max_p w_p z_s[src_row[p], c]; argmax[g, c] = the lowest position p
 * attaining it (-1 for an empty group, whose out is 0). */
int ora_lja_max_fwd(const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                    const int32_t* edge_row, const double* z, int64_t ldz, int dim,
                    const double* w, int w_by_pos, double* out, int64_t ld_out, int64_t* argmax) {
  for (int64_t g = 0; g < n_groups; ++g)
    for (int c = 0; c < dim; ++c) {
      double best = 0.0;
      int64_t arg = -1;
      for (int64_t p = group_ptr[g]; p < group_ptr[g + 1]; ++p) {
        const double wp = w ? w[w_by_pos ? p : (int64_t)edge_row[p]] : 1.0;
        const double v = wp * z[(int64_t)src_row[p] * ldz + c];
        if (arg < 0 || v > best) { best = v; arg = p; }
      }
      out[g * ld_out + c] = arg < 0 ? 0.0 : best;
      argmax[g * dim + c] = arg;
    }
  return ORA_OK;
}

/* d_z[s, c] = sum over (g, c) whose arg-max row p has src_row[p] = s of w_p d_out[g, c];
 * d_w[p] = sum over columns c with argmax[g, c] = p of d_out[g, c] z[s_p, c].  Written. */
int ora_lja_max_bwd(const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                    const int32_t* edge_row, const double* z, int64_t ldz, int dim,
                    const double* w, int w_by_pos, const int64_t* argmax, const double* d_out,
                    int64_t ld_dout, int64_t n_src_rows, int64_t n_w, double* d_z, double* d_w) {
  if (d_z) memset(d_z, 0, sizeof(double) * (size_t)(n_src_rows * dim));
  if (d_w) memset(d_w, 0, sizeof(double) * (size_t)n_w);
  for (int64_t g = 0; g < n_groups; ++g)
    for (int c = 0; c < dim; ++c) {
      const int64_t p = argmax[g * dim + c];
      if (p < 0) continue;
      const int64_t wi = w_by_pos ? p : (int64_t)edge_row[p];
      const double wp = w ? w[wi] : 1.0;
      const int64_t s = src_row[p];
      if (d_z) d_z[s * dim + c] += wp * d_out[g * ld_dout + c];
      if (d_w && w) d_w[wi] += d_out[g * ld_dout + c] * z[s * ldz + c];
    }
  (void)group_ptr;
  return ORA_OK;
}

/* mean over labelled rows (label >= 0) of -log softmax(logits_i)[label_i]; d_logits =
 * (softmax - onehot) / n_labelled for labelled rows, 0 otherwise. */
int ora_softmax_xent(const double* logits, int64_t n, int C, int64_t ld, const int64_t* label,
                     double* loss, double* d_logits) {
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) m += label[i] >= 0;
  double tot = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double* x = logits + i * ld;
    if (label[i] < 0) {
      if (d_logits) for (int c = 0; c < C; ++c) d_logits[i * C + c] = 0.0;
      continue;
    }
    if (label[i] >= C) return ORA_ERR_BAD_ARG;
    double mx = x[0];
    for (int c = 1; c < C; ++c) if (x[c] > mx) mx = x[c];
    double z = 0.0;
    for (int c = 0; c < C; ++c) z += exp(x[c] - mx);
    tot += -(x[label[i]] - mx - log(z));
    if (d_logits)
      for (int c = 0; c < C; ++c)
        d_logits[i * C + c] = (exp(x[c] - mx) / z - (c == label[i] ? 1.0 : 0.0)) / (double)m;
  }
  *loss = m ? tot / (double)m : 0.0;
  return ORA_OK;
}

/* one Adam step at step number t >= 1 (in place on p, m, v):
 *   g' = g + wd p;  m = b1 m + (1 - b1) g';  v = b2 v + (1 - b2) g'^2;
 *   p -= lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps) */
int ora_adam(double* p, const double* g, double* m, double* v, int64_t n, double lr, double b1,
             double b2, double eps, double wd, int64_t t) {
  if (t < 1) return ORA_ERR_BAD_ARG;
  const double c1 = 1.0 - pow(b1, (double)t), c2 = 1.0 - pow(b2, (double)t);
  for (int64_t i = 0; i < n; ++i) {
    const double gi = g[i] + wd * p[i];
    m[i] = b1 * m[i] + (1.0 - b1) * gi;
    v[i] = b2 * v[i] + (1.0 - b2) * gi * gi;
    p[i] -= lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
  }
  return ORA_OK;
}

/* R-GCN layer with per-join-row transformations, NO pushdown (the per-row T_tau of the join rule,
 * PAPER.md:444; R-GCN PAPER.md:890, :897 -- one weight matrix per relation type):
 *   out[g] = W0 x[t_g] + sum over join rows p of group g of  c_p W_{rel_p} x[s_p],
 *   c_p = 1 / |{p' in g : rel_p' = rel_p}|   (R-GCN's per-relation neighbour normalisation)
 * W [n_rel + 1][d_out][d_in] (W[0] = the self-loop map, W[1 + r] relation r's), x [n, ld_x].
 * Every join row's W_rel x_s is formed and added in double, then the self term. */
int ora_rgcn_fwd(const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                 const int32_t* edge_row, const int32_t* group_dst_row, const int32_t* rel,
                 int n_rel, const double* x, int64_t ldx, int d_in, const double* W, int d_out,
                 double* out, int64_t ld_out) {
  int64_t* cnt = (int64_t*)calloc((size_t)(n_rel > 0 ? n_rel : 1), sizeof(int64_t));
  if (!cnt) return ORA_ERR_NOMEM;
  for (int64_t g = 0; g < n_groups; ++g) {
    double* o = out + g * ld_out;
    for (int k = 0; k < n_rel; ++k) cnt[k] = 0;
    for (int64_t p = group_ptr[g]; p < group_ptr[g + 1]; ++p) {
      const int r = rel[edge_row[p]];
      if (r < 0 || r >= n_rel) { free(cnt); return ORA_ERR_BAD_ARG; }
      cnt[r] += 1;
    }
    const double* xt = x + (int64_t)group_dst_row[g] * ldx;
    for (int i = 0; i < d_out; ++i) {
      double acc = 0.0;
      for (int k = 0; k < d_in; ++k) acc += W[(size_t)i * d_in + k] * xt[k];
      o[i] = acc;
    }
    for (int64_t p = group_ptr[g]; p < group_ptr[g + 1]; ++p) {
      const int r = rel[edge_row[p]];
      const double c = 1.0 / (double)cnt[r];
      const double* Wr = W + (size_t)(1 + r) * d_out * d_in;
      const double* xs = x + (int64_t)src_row[p] * ldx;
      for (int i = 0; i < d_out; ++i) {
        double y = 0.0;                      /* tau_p: W_rel x_s for this join row */
        for (int k = 0; k < d_in; ++k) y += Wr[(size_t)i * d_in + k] * xs[k];
        o[i] += c * y;
      }
    }
  }
  free(cnt);
  return ORA_OK;
}

/* backward of ora_rgcn_fwd: d_x [n, d_in] and d_W [(n_rel + 1) d_out d_in], both written. */
int ora_rgcn_bwd(const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                 const int32_t* edge_row, const int32_t* group_dst_row, const int32_t* rel,
                 int n_rel, const double* x, int64_t ldx, int64_t n_x, int d_in, const double* W,
                 int d_out, const double* d_out_g, int64_t ld_dout, double* d_x, double* d_W) {
  int64_t* cnt = (int64_t*)calloc((size_t)(n_rel > 0 ? n_rel : 1), sizeof(int64_t));
  if (!cnt) return ORA_ERR_NOMEM;
  memset(d_x, 0, sizeof(double) * (size_t)(n_x * d_in));
  memset(d_W, 0, sizeof(double) * (size_t)(n_rel + 1) * d_out * d_in);
  for (int64_t g = 0; g < n_groups; ++g) {
    const double* dO = d_out_g + g * ld_dout;
    for (int k = 0; k < n_rel; ++k) cnt[k] = 0;
    for (int64_t p = group_ptr[g]; p < group_ptr[g + 1]; ++p) cnt[rel[edge_row[p]]] += 1;
    const int64_t t = group_dst_row[g];
    for (int i = 0; i < d_out; ++i)
      for (int k = 0; k < d_in; ++k) {
        d_W[(size_t)i * d_in + k] += dO[i] * x[t * ldx + k];
        d_x[t * d_in + k] += W[(size_t)i * d_in + k] * dO[i];
      }
    for (int64_t p = group_ptr[g]; p < group_ptr[g + 1]; ++p) {
      const int r = rel[edge_row[p]];
      const double c = 1.0 / (double)cnt[r];
      const double* Wr = W + (size_t)(1 + r) * d_out * d_in;
      double* dWr = d_W + (size_t)(1 + r) * d_out * d_in;
      const int64_t s = src_row[p];
      for (int i = 0; i < d_out; ++i)
        for (int k = 0; k < d_in; ++k) {
          dWr[(size_t)i * d_in + k] += c * dO[i] * x[s * ldx + k];
          d_x[s * d_in + k] += c * Wr[(size_t)i * d_in + k] * dO[i];
        }
    }
  }
  free(cnt);
  return ORA_OK;
}
