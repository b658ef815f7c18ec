/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle for the lifted
 * join-aggregate (LJA) of RelaNN's Neuro-Relational Algebra.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load, call or link
 * anything under oracle/.  The product path (librnn.so and its Python
 * binding) never does: the two share no code, header, helper or table.
 *
 * Arithmetic is IEEE double throughout.  Embedding inputs are passed as
 * double arrays (the Python wrapper widens the fp32 bytes exactly), so the
 * oracle is the plain mathematical definition evaluated in fp64.
 *
 * Paper citations (PAPER.md = /root/reference/PAPER.md, LaTeX source):
 *   data model   : PAPER.md:306-309 (sec 2.1) -- relation = content + embedding per tuple
 *   join         : PAPER.md:321-330 (sec 2.2) -- natural join, embeddings concatenated
 *   proj. union  : PAPER.md:332-340 (sec 2.2) -- group by A, aggregate multiset once
 *   transform    : PAPER.md:344-349 (sec 2.2) -- per-tuple differentiable map
 *   join rule    : PAPER.md:438-449 (sec 3.1) -- U_{alpha,x}(T_tau(sigma(R1 |><| ... |><| Rk)))
 *   physical plan: PAPER.md:751-761 (sec 4.2) -- row-index tensors + group-index tensor,
 *                  gradients flow through embeddings only (Fig. 3, :815-817)
 *   HGT attention: PAPER.md:917-927 (Fig. 4), :1343-1409 [appendix, src-only]
 *   DHN patterns : PAPER.md:943-949 (C3 rule), :1481 (closed walks), :1500 (Eq. 3)
 *
 * Every function returns 0 on success or a positive ORA_ERR_* code.
 */
#ifndef RNN_ORACLE_H
#define RNN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORA_OK = 0, ORA_ERR_DUPLICATE_KEY = 1, ORA_ERR_BAD_ARG = 2, ORA_ERR_NOMEM = 3 };

/* combine c(z_s, z_e, z_t) applied per join row (the transformation T_tau of the join rule) */
enum { ORA_COMBINE_SRC = 0,      /* w * z_s, w = scalar edge operand (1 if absent)     */
       ORA_COMBINE_MUL = 1,      /* elementwise product of the present operands        */
       ORA_COMBINE_ADD = 2,      /* elementwise sum of the present operands            */
       ORA_COMBINE_CONCAT = 3 }; /* z_s (+) z_e (+) z_t                   */
/* aggregator alpha of the projected union */
enum { ORA_AGG_SUM = 0, ORA_AGG_MEAN = 1, ORA_AGG_SOFTMAX = 2 };

/* One embedding operand.  data == NULL => operand absent.
 * mode 0: natural row (src: src_row[p]; edge: edge_row[p]; dst: group_dst_row[g])
 * mode 1: positional   (edge: join position p; dst: group id g)                      */
typedef struct {
  const double* data;
  int64_t ld;
  int32_t dim;
  int32_t mode;
} ora_operand;

/* O1: canonical join index.  E(s,t) |><| S(s) |><| T(t), groups by t.
 *   s_key == NULL : S absent (no probe on s, src_row[p] = -1)
 *   t_key == NULL : T absent (groups = distinct e_dst_key, group_dst_row = -1)
 *   within_by_src_key: order rows inside a group by (S key, edge row) instead of edge row.
 * Output arrays are caller-allocated with upper-bound sizes:
 *   group_ptr[n_e+1], group_key[n_e], group_dst_row[n_e], src_row[n_e], edge_row[n_e],
 *   src_ptr[n_s+1], src_pos[n_e].   *n_join_rows, *n_groups receive the sizes. */
int ora_build_join_index(const int64_t* e_src_key, const int64_t* e_dst_key, int64_t n_e,
                         const int64_t* s_key, int64_t n_s,
                         const int64_t* t_key, int64_t n_t,
                         int within_by_src_key,
                         int64_t* n_join_rows, int64_t* n_groups,
                         int64_t* group_ptr, int64_t* group_key, int32_t* group_dst_row,
                         int32_t* src_row, int32_t* edge_row,
                         int64_t* src_ptr, int32_t* src_pos);

/* O2/O3: forward LJA.  out[i, :] for group sel[i] (sel == NULL => all groups, i = g).
 * lse[i, h] (SOFTMAX only, may be NULL) = log sum_p exp(e_{p,h}). */
int ora_lja_fwd(const int64_t* group_ptr, int64_t n_groups,
                const int32_t* src_row, const int32_t* edge_row, const int32_t* group_dst_row,
                int combine, int agg, int heads, double scale,
                const ora_operand* src, const ora_operand* src_key,
                const ora_operand* edge, const ora_operand* dst,
                const int64_t* sel, int64_t n_sel,
                double* out, int64_t ld_out, double* lse);

/* O4: backward LJA.  Gradients are WRITTEN (zero-filled first) into full-size buffers:
 * d_src[n_src_rows, src.dim], d_src_key[n_src_rows, key.dim], d_edge[n_edge_rows or E', edge.dim],
 * d_dst[n_dst_rows or G, dst.dim].  Any may be NULL.  d_out is [G, ld_dout]. */
int ora_lja_bwd(const int64_t* group_ptr, int64_t n_groups,
                const int32_t* src_row, const int32_t* edge_row, const int32_t* group_dst_row,
                int combine, int agg, int heads, double scale,
                const ora_operand* src, const ora_operand* src_key,
                const ora_operand* edge, const ora_operand* dst,
                const double* d_out, int64_t ld_dout,
                int64_t n_src_rows, int64_t n_edge_rows, int64_t n_dst_rows,
                double* d_src, double* d_src_key, double* d_edge, double* d_dst);

/* Standalone grouped softmax over materialised scores [E', heads] in group-major order
 * (the ATT relation) and its backward. */
int ora_group_softmax(const int64_t* group_ptr, int64_t n_groups, int heads,
                      const double* scores, double* probs);
int ora_group_softmax_bwd(const int64_t* group_ptr, int64_t n_groups, int heads,
                          const double* probs, const double* d_probs, double* d_scores);

/* O5: dense per-relation projection (transformation pushed below the join)
 * Y[m,n] = sum_k X[m,k] W[n,k] + b[n]   (W laid out [N, K] like torch.nn.Linear.weight) */
int ora_project(const double* X, int64_t M, int64_t K, int64_t ldx,
                const double* W, int64_t N, int64_t ldw, const double* bias,
                double* Y, int64_t ldy);
int ora_project_bwd(const double* X, int64_t M, int64_t K, int64_t ldx,
                    const double* W, int64_t N, int64_t ldw,
                    const double* dY, int64_t lddy,
                    double* dX /*[M,K] nullable*/, double* dW /*[N,K]*/, double* db /*[N] nullable*/);

/* O7: GCN symmetric normalisation as a per-join-position weight (PyG gcn_norm reading,
 * SURVEY sec 8c ambiguity #1): w_p = deg(s_p)^-1/2 * deg(t_g)^-1/2, deg = in-degree
 * (group size) of the node; S and T are the same node relation (n_nodes rows). */
int ora_gcn_norm(const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                 const int32_t* group_dst_row, int64_t n_nodes, double* w);

/* O6: DHN closed-walk pattern aggregates.
 * Adjacency = a join index built with within_by_src_key over Edge(n, v) grouped by n
 * (group key = root key, src rows = neighbour node rows).  node_key[n_nodes] gives the key of
 * every node row (used for the sorted-membership test n in N(p)).
 * f[i] = position-i operand [n_nodes, d] (ld ldf).  out[i] for group sel[i] (or all groups):
 *   C_k(n) = f0(n) (.) sum_{closed walks n->v1->...->v_{k-1}->n} prod_i f_i(v_i). */
int ora_dhn_fwd(int k, const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                const int32_t* group_dst_row, const int64_t* node_key, int64_t n_nodes,
                const double* const* f, int64_t ldf, int d,
                const int64_t* sel, int64_t n_sel, double* out, int64_t ld_out);
/* backward: d_f[i] [n_nodes, d] written (zero-filled); d_out [G, ld_dout]. */
int ora_dhn_bwd(int k, const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                const int32_t* group_dst_row, const int64_t* node_key, int64_t n_nodes,
                const double* const* f, int64_t ldf, int d,
                const double* d_out, int64_t ld_dout, double* const* d_f);

/* ---- SURVEY sec 8f rows (oracle_next.c) ---- */
/* node epilogue y = gate act(x + b) + (1 - gate) r  (act 0 none, 1 ReLU, 2 GELU; r nullable) */
int ora_epilogue_fwd(const double* x, int64_t rows, int dim, int64_t ldx, const double* bias,
                     int act, double gate, const double* resid, int64_t ld_resid, double* y,
                     int64_t ldy);
int ora_epilogue_bwd(const double* dy, const double* x, int64_t rows, int dim, const double* bias,
                     int act, double gate, const double* resid, double* dx, double* d_bias,
                     double* d_resid, double* d_gate);
/* MAX aggregate of w * z_s; argmax [G, dim] (lowest position, -1 empty) */
int ora_lja_max_fwd(const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                    const int32_t* edge_row, const double* z, int64_t ldz, int dim,
                    const double* w, int w_by_pos, double* out, int64_t ld_out, int64_t* argmax);
int ora_lja_max_bwd(const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                    const int32_t* edge_row, const double* z, int64_t ldz, int dim,
                    const double* w, int w_by_pos, const int64_t* argmax, const double* d_out,
                    int64_t ld_dout, int64_t n_src_rows, int64_t n_w, double* d_z, double* d_w);
/* Loss(; CrossEntropyLoss()(logits, label)) and one Adam step (fit, :554) */
int ora_softmax_xent(const double* logits, int64_t n, int C, int64_t ld, const int64_t* label,
                     double* loss, double* d_logits);
int ora_adam(double* p, const double* g, double* m, double* v, int64_t n, double lr, double b1,
             double b2, double eps, double wd, int64_t t);

/* R-GCN layer, per-join-row transform W_rel x_s with no pushdown:
 * out[g] = W0 x_t + sum_p c_p W_{rel(p)} x_{s(p)}, c_p = 1 / (rows of g with p's relation). */
int ora_rgcn_fwd(const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                 const int32_t* edge_row, const int32_t* group_dst_row, const int32_t* rel,
                 int n_rel, const double* x, int64_t ldx, int d_in, const double* W, int d_out,
                 double* out, int64_t ld_out);
int ora_rgcn_bwd(const int64_t* group_ptr, int64_t n_groups, const int32_t* src_row,
                 const int32_t* edge_row, const int32_t* group_dst_row, const int32_t* rel,
                 int n_rel, const double* x, int64_t ldx, int64_t n_x, int d_in, const double* W,
                 int d_out, const double* d_out_g, int64_t ld_dout, double* d_x, double* d_W);

/* Multi-GPU ownership: owner(key) = splitmix64(key ^ seed) mod P. */
int ora_hash_partition(const int64_t* keys, int64_t n, int32_t P, uint64_t seed, int32_t* owner);
uint64_t ora_splitmix64(uint64_t x);

#ifdef __cplusplus
}
#endif
#endif
