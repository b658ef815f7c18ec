/*
 * rnn.h -- C ABI of librnn.so, the B200-native lifted join-aggregate (LJA) of RelaNN's
 * Neuro-Relational Algebra (arxiv 2605.24207; PAPER.md = /root/reference/PAPER.md).
 *
 * The LJA is the NRA expression a join rule compiles to (sec 3.1):
 *
 *     Out(t; alpha(c(z_s, z_e, z_t))) :- E(s, t; z_e), S(s; z_s), T(t; z_t)
 *     ==  U_{alpha,t}( T_c( E |><| S |><| T ) )
 *
 * - E is the edge / incidence relation (n_edge_rows tuples, content (s, t)), S the gathered
 *   "source" relation keyed by s, T the group-side relation keyed by t.  Each relation is a
 *   set: duplicate keys in S or T are an error.  Rows of E whose s (or t) has
 *   no partner are dropped (natural join).
 * - The join pairs tuples and concatenates embeddings; the combine c is
 *   the per-row transformation T_tau; the projected union groups by t and
 *   aggregates the multiset once.
 * - The paper's physical plan realises this with cuDF merge/groupby index tensors,
 *   torch.index_select and torch_scatter (Fig. 3); this library replaces
 *   them with a key-grouped CSR join index (built once and reused -- "content caching") and
 *   fused gather-combine-reduce kernels, forward and backward (gradients flow through
 *   embeddings only).
 *
 * Conventions (apply to every entry point):
 * - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA memory) unless noted.
 * - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All calls are
 *   asynchronous on `stream` except those marked SYNC.
 * - Ownership: the caller allocates and owns every buffer, including scratch `workspace`
 *   sized by a query; the library never allocates device memory and keeps no global state
 *   besides a thread-local error string.  Inputs are never written.  Outputs must not alias
 *   inputs.  A workspace must not be shared by concurrent calls.
 * - Errors: every function returns rnn_status; nothing throws across the ABI.  Host-side
 *   argument checks are always on.  On error, rnn_last_error() describes it (thread-local,
 *   valid until the next call on the thread).  CUDA launch failures map to RNN_ERR_CUDA.
 * - Embedding operands are fp32, row-major, leading dimension `ld` in elements with
 *   ld % 4 == 0 and a 16-byte aligned base (128-bit loads); 1 <= dim <= 512.
 * - Keys are signed int64 (any value).  Row ids are int32 (relations < 2^31 rows); join-row
 *   counts and CSR pointers are int64.
 * - Determinism: identical inputs give bit-identical outputs (no floating-point atomics on
 *   any path; every reduction has a fixed order) -- except the k = 4 DHN aggregates (A6),
 *   whose hash-table accumulation uses fp32 atomics (rounding order only); the exact
 *   integer walk counts (rnn_dhn_count) are deterministic.
 */
#ifndef RNN_H
#define RNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RNN_ABI_VERSION 1

typedef enum {
  RNN_OK = 0,
  RNN_ERR_INVALID_ARGUMENT = 1,   /* null/misaligned pointer, bad size or flag            */
  RNN_ERR_SHAPE_MISMATCH = 2,     /* operand widths inconsistent      */
  RNN_ERR_INDEX_OUT_OF_RANGE = 3, /* reserved: no entry point returns it in this build --
                                    * the join index is built here (in range by construction),
                                    * DHN root lists are filtered (out-of-range ids ignored),
                                    * gather / scatter row lists are the caller's contract     */
  RNN_ERR_DUPLICATE_KEY = 4,      /* S or T is not a set                   */
  RNN_ERR_UNSUPPORTED = 5,        /* valid request outside this build's limits            */
  RNN_ERR_WORKSPACE_TOO_SMALL = 6,
  RNN_ERR_CUDA = 7                /* a CUDA runtime call failed (detail in last error)    */
} rnn_status;

const char* rnn_status_string(rnn_status s); /* static string, never NULL */
const char* rnn_last_error(void);            /* thread-local detail, never NULL */
int rnn_abi_version(void);

/* ===================================================================================== */
/* A1. Join index (replaces cuDF merge + groupby)                    */
/* ===================================================================================== */

/* Key-grouped CSR of the join rows.  POD; every array is CALLER-owned device memory and is
 * immutable once built, so one index is reused across iterations and streams.
 *   Group-major order: join rows sorted by (group, edge row) -- or (group, S key, edge row)
 *   with RNN_IDX_WITHIN_GROUP_BY_SRC_KEY (DHN adjacency lists).  Groups are the distinct t of
 *   the join rows in ascending signed order (compact output: absent keys have no group).
 *   Source-major order: positions p sorted by (src_row[p], p).
 *   Work schedules: contiguous ranges of positions, each either a run of whole segments
 *   (total <= 2 * rows_per_item rows) or one piece (<= rows_per_item rows) of a longer
 *   segment; they load-balance the kernels over power-law degree skew.                   */
typedef struct {
  int64_t n_edge_rows, n_join_rows, n_groups, n_src_rows, n_dst_rows;
  int64_t* group_ptr;     /* [G+1]  rows of group g are positions [group_ptr[g], group_ptr[g+1])  */
  int64_t* group_key;     /* [G]    t key of group g, strictly ascending                          */
  int32_t* group_dst_row; /* [G]    row of T holding key group_key[g] (-1 when T absent)          */
  int32_t* src_row;       /* [E']   S row of join row p (-1 when S absent)                        */
  int32_t* edge_row;      /* [E']   E row of join row p                                           */
  int32_t* pos_group;     /* [E']   group of group-major position p                               */
  int64_t* src_ptr;       /* [n_src+1] source-major CSR over all S rows (empty rows included)     */
  int32_t* src_pos;       /* [E']   group-major position of the q-th source-major entry           */
  int32_t* src_group;     /* [E']   group of position src_pos[q]                                  */
  int32_t* src_seg;       /* [E']   S row of the q-th source-major entry (= src_row[src_pos[q]])  */
  int64_t n_work;         /* number of group-major work items                                     */
  int64_t* work_ptr;      /* [n_work+1] item boundaries (positions)                               */
  int32_t* work_seg;      /* [n_work] first group an item touches (the one holding work_ptr[i])   */
  int64_t n_src_work;     /* number of source-major work items                                    */
  int64_t* src_work_ptr;  /* [n_src_work+1]                                                       */
  int32_t* src_work_seg;  /* [n_src_work] first source an item touches (empty sources included)   */
} rnn_join_index;

enum {
  RNN_IDX_VALIDATE = 1,                /* check S/T duplicate keys (RNN_ERR_DUPLICATE_KEY)      */
  RNN_IDX_WITHIN_GROUP_BY_SRC_KEY = 2, /* DHN adjacency variant (needs S and T)                 */
  RNN_IDX_NO_TRANSPOSE = 4,            /* skip src_ptr/src_pos/src_group/src_work_ptr           */
  RNN_IDX_DENSE_GROUPS = 8             /* every T row is a group (key order), empty ones too:   */
                                       /* outputs are dense [n_dst, d] in T-key order, so the   */
                                       /* union over several relations with one T is a beta=1   */
                                       /* accumulation; needs T              */
};

/* Build the canonical join index of E(s,t) |><| S(s) |><| T(t) grouped by t.
 *   e_src_key[n_edge_rows], e_dst_key[n_edge_rows] : content columns of E (device).
 *   src_key[n_src] : keys of S, row i <-> embedding row i; NULL => S absent (every E row is
 *                    a join row w.r.t. s and src_row = -1).
 *   dst_key[n_dst] : keys of T; NULL => T absent (groups = distinct e_dst_key).
 *   rows_per_item  : work-schedule granularity (0 => 128).
 * Two phases (SYNC in phase 1):
 *   (1) idx->group_ptr == NULL: computes idx->n_join_rows, idx->n_groups, idx->n_work,
 *       idx->n_src_work and the other counts, and *workspace_bytes; blocks on `stream`.
 *       If workspace == NULL only *workspace_bytes is set (host-only query, no device work).
 *   (2) with every array allocated to those sizes: fills them.  Deterministic: the same
 *       inputs give identical bytes.  Duplicate S/T keys are always detected in phase 1. */
rnn_status rnn_build_join_index(const int64_t* e_src_key, const int64_t* e_dst_key,
                                int64_t n_edge_rows, const int64_t* src_key, int64_t n_src,
                                const int64_t* dst_key, int64_t n_dst, int flags,
                                int64_t rows_per_item, rnn_join_index* idx, void* workspace,
                                size_t* workspace_bytes, void* stream);

/* Selection pushdown (PAPER.md:444 -- the join rule is U(T_tau(sigma(R1 |><| ... |><| Rk))); :1031
 * "selection pushdowns"): the same build over sigma(E), the E rows with
 * e_mask[j] != 0 (uint8 [n_edge_rows], device).  Masked rows are dropped in the probe, before
 * the sort, so the index is exactly the canonical index of the filtered relation (edge_row
 * still refers to rows of the unfiltered E).  Other arguments as rnn_build_join_index. */
rnn_status rnn_build_join_index_sel(const int64_t* e_src_key, const int64_t* e_dst_key,
                                    const uint8_t* e_mask, int64_t n_edge_rows,
                                    const int64_t* src_key, int64_t n_src, const int64_t* dst_key,
                                    int64_t n_dst, int flags, int64_t rows_per_item,
                                    rnn_join_index* idx, void* workspace, size_t* workspace_bytes,
                                    void* stream);
/* Predicate mask over an E attribute column: r_j = attr[j] <op> value, op in {EQ, NE, LT, LE,
 * GT, GE} = 0..5; attr int64 (dtype 0, value truncated to int64) or float32 (dtype 1);
 * combine 0: mask = r, 1: mask &= r, 2: mask |= r (conjunctions / disjunctions of atoms). */
rnn_status rnn_select_mask(const void* attr, int32_t dtype, int64_t n, int32_t op, double value,
                           int32_t combine, uint8_t* mask, void* stream);

/* ===================================================================================== */
/* A3/A4. Fused gather - combine - segmented reduce, forward                             */
/* ===================================================================================== */

typedef enum { RNN_AGG_SUM = 0, RNN_AGG_MEAN = 1, RNN_AGG_SOFTMAX = 2, RNN_AGG_MAX = 3 } rnn_agg;
typedef enum {
  RNN_COMBINE_SRC = 0,   /* w * z_s ; w = scalar edge operand (dim 1) or 1 (GCN norm, a*v)  */
  RNN_COMBINE_MUL = 1,   /* z_s (.) z_e (.) z_t of the present operands (q*k, DHN product)  */
  RNN_COMBINE_ADD = 2,   /* z_s + z_e + z_t of the present operands ("+ z3")   */
  RNN_COMBINE_CONCAT = 3 /* z_s (+) z_e (+) z_t (join default)               */
} rnn_combine;

/* An embedding operand.  data == NULL => absent.
 * mode RNN_BY_ROW: src rows via src_row[p], edge rows via edge_row[p], dst rows via
 *                  group_dst_row[g];  mode RNN_BY_POSITION: edge row = join position p,
 *                  dst row = group id g (src operands must use RNN_BY_ROW).
 * A dim-1 edge operand broadcasts as a scalar (per-row weight). */
enum { RNN_BY_ROW = 0, RNN_BY_POSITION = 1 };
typedef struct {
  const float* data;
  int64_t ld;
  int32_t dim;
  int32_t mode;
} rnn_operand;

typedef struct {
  rnn_combine combine;
  rnn_agg agg;
  int32_t heads;   /* SOFTMAX: number of heads h (dim/h in {4,8,16,32,64}); else 1          */
  float scale;     /* SOFTMAX: score scale (e.g. mu / sqrt(d/h)); else ignored               */
  rnn_operand src;     /* gathered by src_row: values                                         */
  rnn_operand src_key; /* SOFTMAX: keys gathered by src_row                                   */
  rnn_operand edge;    /* gathered by edge_row (or position): edge embedding or scalar weight */
  rnn_operand dst;     /* per group via group_dst_row (or g): group-side factor / queries     */
} rnn_lifted_query;

/* Supported (combine, agg) in this build:
 *   SUM/MEAN x {SRC (edge dim 1 or absent, no dst), MUL, ADD (dims equal, edge may be 1),
 *               CONCAT (total width <= 512)};
 *   SOFTMAX with combine SRC: src/src_key/dst present, edge absent, dim <= 128.
 * out[G, ld_out]: row g = aggregate of group g.  beta = 0 overwrites, beta = 1 accumulates
 * (union over relations, PAPER.md:451-460 / HGT H_tilda sum over phi; SUM/SOFTMAX only).
 * lse[G, heads] (SOFTMAX only, required there): log-sum-exp per group and head, saved for
 * the backward.  workspace: partial states of split groups; size via rnn_lja_workspace_size. */
rnn_status rnn_lja_workspace_size(const rnn_join_index* idx, const rnn_lifted_query* q,
                                  size_t* fwd_bytes, size_t* bwd_bytes);
rnn_status rnn_join_aggregate_fwd(const rnn_join_index* idx, const rnn_lifted_query* q,
                                  float* out, int64_t ld_out, float beta, float* lse,
                                  void* workspace, size_t workspace_bytes, void* stream);

/* Union over relations keeping each relation's own output (HGT: H_tilda(t) = sum_phi O_phi(t),
 * PAPER.md:1408-1409 [src-only], Fig. 4 :917-927).  Computes the aggregate into out exactly as
 * rnn_join_aggregate_fwd with beta = 0 (out and lse are what rnn_join_aggregate_bwd needs:
 * the SOFTMAX backward forms D = <dOut, out> per relation), and in the same pass
 * acc[G, ld_acc] = beta_acc * acc + out (beta_acc 0 for the first relation into a type, 1 for
 * the others).  acc: device, 16-byte aligned, ld_acc % 4 == 0, ld_acc >= width, must not alias
 * out.  Fused into the store of the d = 128 SOFTMAX walker; other (combine, agg) pairs add one
 * pass over [G, width].  MEAN: RNN_ERR_UNSUPPORTED (not decomposable).  Other
 * arguments, layouts and errors: rnn_join_aggregate_fwd. */
rnn_status rnn_join_aggregate_fwd_union(const rnn_join_index* idx, const rnn_lifted_query* q,
                                        float* out, int64_t ld_out, float* lse, float* acc,
                                        int64_t ld_acc, float beta_acc, void* workspace,
                                        size_t workspace_bytes, void* stream);

/* ===================================================================================== */
/* A5. Backward                                                                          */
/* ===================================================================================== */
/* Gradients are WRITTEN (not accumulated) into dense full-relation buffers laid out like
 * their operand (same leading dimension: d_src uses src.ld, d_dst uses dst.ld, ...):
 *   d_src[n_src_rows, src.dim], d_src_key[n_src_rows, src_key.dim],
 *   d_edge[(n_edge_rows or E' for RNN_BY_POSITION), edge.dim],
 *   d_dst[(n_dst_rows or G), dst.dim].  Any may be NULL (not computed).  Rows never
 *   referenced by a join row get 0.  out/lse are the forward's outputs (SOFTMAX only).
 * The source-major pass uses the transposed CSR (no atomics); d_src requires it. */
rnn_status rnn_join_aggregate_bwd(const rnn_join_index* idx, const rnn_lifted_query* q,
                                  const float* out, int64_t ld_out, const float* lse,
                                  const float* d_out, int64_t ld_dout, float* d_src,
                                  float* d_src_key, float* d_edge, float* d_dst,
                                  void* workspace, size_t workspace_bytes, void* stream);
/* As rnn_join_aggregate_bwd, with d_dst = beta_dst * d_dst + (gradient): beta_dst = 1 sums
 * the gradient of a group-side operand shared by several relations (HGT's per-type query
 * QLin<L, tau_t>, reading 12) in place, rows never referenced keeping their value.
 * beta_dst in {0, 1}; beta_dst = 1 is supported where d_dst comes from the SOFTMAX
 * source-major backward (dim 128), else RNN_ERR_UNSUPPORTED. */
rnn_status rnn_join_aggregate_bwd_acc(const rnn_join_index* idx, const rnn_lifted_query* q,
                                      const float* out, int64_t ld_out, const float* lse,
                                      const float* d_out, int64_t ld_dout, float* d_src,
                                      float* d_src_key, float* d_edge, float* d_dst,
                                      float beta_dst, void* workspace, size_t workspace_bytes,
                                      void* stream);

/* MAX aggregate (PAPER.md:209 "sum, mean, or max", :755): agg
 * RNN_AGG_MAX with combine SRC, value w_p * z_s (edge: optional scalar weight, by row or by
 * position).  out[g, c] = max over the group's join rows; argmax[g, c] (int32 [G, ld_arg]) =
 * the LOWEST join position attaining it (ties broken deterministically); an empty group gives
 * out 0 and argmax -1 (scatter_max convention).  Backward (subgradient: everything to the
 * arg-max row): d_src[s, c] = sum of w_p d_out[g, c] over the (g, c) whose arg-max row p has
 * src_row[p] = s (source-major over the transposed CSR, no atomics; rows never referenced
 * get 0), d_edge[p] = sum over c with argmax[g, c] = p of d_out[g, c] z_s[s_p, c] (written;
 * needs the edge weight).  d_src / d_edge use their operand's ld; either may be NULL. */
rnn_status rnn_join_aggregate_max_fwd(const rnn_join_index* idx, const rnn_lifted_query* q,
                                      float* out, int64_t ld_out, int32_t* argmax, int64_t ld_arg,
                                      void* stream);
rnn_status rnn_join_aggregate_max_bwd(const rnn_join_index* idx, const rnn_lifted_query* q,
                                      const int32_t* argmax, int64_t ld_arg, const float* d_out,
                                      int64_t ld_dout, float* d_src, float* d_edge, void* stream);

/* Standalone grouped softmax over materialised scores [E', heads] in group-major order (the
 * ATT relation of Fig. 4), and its backward ds = p (dp - sum_q p dp). */
rnn_status rnn_group_softmax(const rnn_join_index* idx, const float* scores, int32_t heads,
                             float* probs, void* stream);
rnn_status rnn_group_softmax_bwd(const rnn_join_index* idx, const float* probs,
                                 const float* d_probs, int32_t heads, float* d_scores,
                                 void* stream);

/* ===================================================================================== */
/* Node epilogues: bias, activation, gated residual                */
/* ===================================================================================== */
/* The per-node transformation a rule applies after the aggregate or the projection:
 *   y = gate * act(x + bias) + (1 - gate) * resid          (resid == NULL: y = act(x + bias))
 * GCN layers: bias then ReLU (hidden) / bias only (last) -- PyG GCNConv, PAPER.md:865 (O7);
 * the HGT skip connection: gate = sigmoid(skip_tau), resid = the previous layer's H
 * (PAPER.md:1392-1394 [src-only]); GELU for HGT's target-specific aggregation (:1356 ff).
 *   bias  [dim] or NULL;  resid [rows, ld_resid] (row order of x) or NULL;
 *   pre   [rows, ld_pre] or NULL: x + bias saved for the backward (needed for GELU, and for
 *         RELU when resid is given; for RELU without resid the output's sign suffices).   */
typedef enum { RNN_ACT_NONE = 0, RNN_ACT_RELU = 1, RNN_ACT_GELU = 2 } rnn_activation;
typedef struct {
  const float* bias;
  int32_t act;           /* rnn_activation (GELU: x * Phi(x), erf form) */
  float gate;            /* used when resid != NULL, in [0, 1] */
  const float* resid;
  int64_t ld_resid;
  float* pre;
  int64_t ld_pre;
} rnn_epilogue;

/* The forward LJA with the epilogue fused into its final store (the lean SRC/MUL gather path;
 * other paths run the aggregate, then the epilogue in place).  Arguments as
 * rnn_join_aggregate_fwd; beta must be 0 (a union is accumulated first and the epilogue
 * applied once with rnn_epilogue_fwd); SUM / MEAN only. */
rnn_status rnn_join_aggregate_fwd_epi(const rnn_join_index* idx, const rnn_lifted_query* q,
                                      const rnn_epilogue* epi, float* out, int64_t ld_out,
                                      void* workspace, size_t workspace_bytes, void* stream);
/* Standalone epilogue over x [rows, dim] -> y (y may alias x; epi->pre may alias neither). */
rnn_status rnn_epilogue_fwd(const float* x, int64_t ldx, int64_t rows, int32_t dim,
                            const rnn_epilogue* epi, float* y, int64_t ldy, void* stream);
/* Backward of the epilogue: from dy [rows, dim] and the forward's y / epi->pre:
 *   dx = dy * gate * act'(x + bias)   (gate = 1 without resid)   [rows, ld_dx], may alias dy
 *   d_bias = sum over rows of dx      [dim] or NULL   (fixed-order two-stage reduction)
 *   d_resid = (1 - gate) * dy         [rows, ld_dresid] or NULL
 *   d_gate = sum dy * (act(x + bias) - resid)   scalar or NULL (needs pre and resid)
 * workspace: rnn_epilogue_bwd_workspace_size (host-only). */
rnn_status rnn_epilogue_bwd_workspace_size(int64_t rows, int32_t dim, size_t* bytes);
rnn_status rnn_epilogue_bwd(const float* dy, int64_t lddy, const float* y, int64_t ldy,
                            int64_t rows, int32_t dim, const rnn_epilogue* epi, float* dx,
                            int64_t lddx, float* d_bias, float* d_resid, int64_t ld_dresid,
                            float* d_gate, void* workspace, size_t workspace_bytes, void* stream);

/* ===================================================================================== */
/* Training step: the loss relation and the fit optimiser           */
/* ===================================================================================== */
/* Loss(; CrossEntropyLoss()(Cls(z_p), z_l)): loss (device scalar) = mean over
 * the rows with label >= 0 of -log softmax(logits_i)[label_i]; d_logits [n, ld_dlogits]
 * (nullable) = (softmax - onehot) / n_labelled on labelled rows, 0 on the others.  label
 * int64 [n] (device; -1 = unlabelled, < C).  Fixed-order reductions (deterministic).
 * workspace: rnn_softmax_xent_workspace_size (host-only). */
rnn_status rnn_softmax_xent_workspace_size(int64_t n, size_t* bytes);
rnn_status rnn_softmax_xent(const float* logits, int64_t n, int32_t C, int64_t ld,
                            const int64_t* label, float* loss, float* d_logits, int64_t ld_dlogits,
                            void* workspace, size_t workspace_bytes, void* stream);

/* ?fit <lr, weight_decay, ...>: one Adam step on a parameter matrix
 * (Kingma & Ba, bias-corrected; weight decay added to the gradient as L2, torch.optim.Adam):
 *   g' = g + wd p;  m = b1 m + (1 - b1) g';  v = b2 v + (1 - b2) g'^2;
 *   p -= lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
 * param [rows, ld_param] (updated in place), grad [rows, ld_grad], m / v dense [rows, cols]
 * (zero before the first step).  t = *step (device int64, >= 1), advanced once per training
 * step by rnn_adam_tick -- kept on the device so the whole step can be graph-captured. */
typedef struct { float lr, beta1, beta2, eps, weight_decay; } rnn_adam_config;
rnn_status rnn_adam_tick(int64_t* step, void* stream);
rnn_status rnn_adam(float* param, int64_t rows, int32_t cols, int64_t ld_param, const float* grad,
                    int64_t ld_grad, float* m, float* v, const rnn_adam_config* cfg,
                    const int64_t* step, void* stream);

/* ===================================================================================== */
/* A2. Dense per-relation projection on tcgen05 tensor cores                             */
/* ===================================================================================== */
/* The transformation pushed below the join so it runs once per node, not once per edge
 * (PAPER.md:1032).  Y[M, N] = X[M, K] . W^T + b, W laid out [N, K] (torch.nn.Linear).
 * X: ldx % 4 == 0; W: ldw % 4 == 0; Y: ldy % 4 == 0; 16-byte aligned; M < 2^31, K <= 8192,
 * N <= 8192 (tiles of 256 columns; several per-relation projections of one node relation
 * are one GEMM with their weights stacked).  Precision:
 *   RNN_PREC_TF32   : one kind::tf32 MMA per tile (operands truncated to tf32).
 *   RNN_PREC_3XTF32 : split-operand 3xTF32 (hi*hi + hi*lo + lo*hi), ~fp32 accuracy.
 *   RNN_PREC_BF16   : both operands rounded to bf16 (round-to-nearest-even) on chip, exact
 *                     bf16 x bf16 products, fp32 accumulation (north_star's bf16 projection,
 *                     tolerance 1e-2); storage stays fp32 (the embeddings are fp32), so the
 *                     rounded operands run through the kind::tf32 MMA, in which bf16 is exact.
 * Backward: dX = dY . W (may be NULL), dW = dY^T . X (required), db = colsum(dY) (may be NULL),
 * all written.  workspace: dW partials (deterministic split-M reduction). */
typedef enum { RNN_PREC_TF32 = 0, RNN_PREC_3XTF32 = 1, RNN_PREC_BF16 = 2 } rnn_precision;
rnn_status rnn_project(const float* X, int64_t M, int32_t K, int64_t ldx, const float* W,
                       int32_t N, int64_t ldw, const float* bias, float* Y, int64_t ldy,
                       rnn_precision prec, void* stream);
rnn_status rnn_project_bwd_workspace_size(int64_t M, int32_t K, int32_t N, size_t* bytes);
rnn_status rnn_project_bwd(const float* X, int64_t M, int32_t K, int64_t ldx, const float* W,
                           int32_t N, int64_t ldw, const float* dY, int64_t lddy, float* dX,
                           int64_t lddx, float* dW, float* db, rnn_precision prec,
                           void* workspace, size_t workspace_bytes, void* stream);
/* Backward of a projection whose input is the output of a ReLU epilogue, X = ReLU(P) (the
 * hidden layers of the GCN program, H^l = ReLU(A Z + b); rnn_epilogue_fwd with
 * RNN_ACT_RELU): as rnn_project_bwd, but dX (required) receives the gradient at the epilogue's
 * input, dP = (dY . W) (.) [X > 0], and d_in_bias (nullable) receives colsum(dP), the epilogue's
 * bias gradient -- i.e. rnn_project_bwd followed by rnn_epilogue_bwd(relu) on dX, in one pass
 * where dY has <= 128 columns (the mask is applied in the tensor-core kernel's store).  Same
 * workspace as rnn_project_bwd; results equal that two-call sequence up to summation order of
 * d_in_bias (fixed order, deterministic). */
rnn_status rnn_project_bwd_relu(const float* X, int64_t M, int32_t K, int64_t ldx, const float* W,
                                int32_t N, int64_t ldw, const float* dY, int64_t lddy, float* dX,
                                int64_t lddx, float* dW, float* db, float* d_in_bias,
                                rnn_precision prec, void* workspace, size_t workspace_bytes,
                                void* stream);

/* ===================================================================================== */
/* A6. Multi-way cyclic joins: DHN closed-walk pattern aggregates                        */
/* ===================================================================================== */
/* The deep homomorphism network rules (config 5), read as closed walks
 * (PAPER.md:1481; Eq. 3 of the appendix, :1500; SURVEY sec 8c reading #9):
 *
 *   C_k(n) = f0(n) (.) sum over closed walks n -> v1 -> ... -> v_{k-1} -> n of
 *                                 f1(v1) (.) f2(v2) (.) ... (.) f_{k-1}(v_{k-1})
 *   k = 2: the single atom Edge(n, v1) (no closing edge: C2(n) = f0(n) (.) sum_{n->v} f1(v))
 *   k = 3: Edge(n,v1), Edge(v1,v2), Edge(v2,n)        (triangle rule)
 *   k = 4: Edge(n,v1), Edge(v1,v2), Edge(v2,v3), Edge(v3,n)   (4-cycle)
 * with multiplicity: duplicated Edge tuples give distinct join rows (distinct walks).
 *
 * adj: the join index of Edge(n, v) |x| Node(v) |x| Node(n) grouped by n, i.e. built with
 *      e_src_key = v, e_dst_key = n and S = T = the node relation (n_src_rows == n_dst_rows),
 *      WITH the transposed CSR (not RNN_IDX_NO_TRANSPOSE).  Any other flag is accepted.
 *      Roots are its groups: out-neighbours of group g are src_row[group_ptr[g] ..], the
 *      in-neighbours of node row r are src_group[src_ptr[r] ..].
 * f:   k operands, RNN_BY_ROW over node rows, all of dim d (1 <= d <= 128), any ld.
 *      f[0].data may be NULL (all ones).
 * out: [n_groups, ld_out] fp32, C_k of every root in group order (overwritten).
 *
 * Closed walks are rotation invariant, so the backward is the same kernel with rotated
 * operands (d f_j(x) = the walk aggregate rooted at x of (f_{j+1}, ..., g, ..., f_{j-1}),
 * g = f0 (.) dOut), and d f0 = dOut (.) sum_walks prod f_i.
 * Work: k = 3 probes the sum_v deg(v)^2 candidate wedges n -> v -> w against a shared-memory
 * hash set of the root's in-neighbours (a per-CTA mark array for in-degrees > 6144).
 * k = 4 is factorised through the middle vertex w: S1(w) = sum_{n->v->w} f1(v) accumulates
 * in a hash table of the root's 2-hop keys (shared memory; values in an L2-resident per-CTA
 * slab), then every in-wedge w -> p -> n adds f3(p) (.) f2(w) (.) S1(w).  Roots with more
 * than 8192 possible 2-hop keys run in hash partitions of w (adjacency lists pre-sorted by
 * the hash, per-neighbour cursors).  k = 3 and k = 4 accumulate with fp32 atomics (shared
 * memory / L2), so their rounding order (only) is not deterministic. */
rnn_status rnn_dhn_workspace_size(const rnn_join_index* adj, int32_t k, int32_t d,
                                  size_t* bytes);   /* host-only, no device work */
rnn_status rnn_dhn_fwd(const rnn_join_index* adj, int32_t k, const rnn_operand* f, float* out,
                       int64_t ld_out, void* workspace, size_t workspace_bytes, void* stream);
/* d_out [n_groups, ld_dout]; d_f[i] [n_src_rows, ld_df] by node row, overwritten (rows that
 * are on no closed walk get 0); any d_f[i] may be NULL. */
rnn_status rnn_dhn_bwd(const rnn_join_index* adj, int32_t k, const rnn_operand* f,
                       const float* d_out, int64_t ld_dout, float* const* d_f, int64_t ld_df,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Saved walk sum (reverse-mode reuse of the forward): rnn_dhn_fwd_save also writes
 * walk_sum [n_groups, ld_ws] (group order) = sum over closed walks of prod_{i>=1} f_i, i.e.
 * C_k before the root factor f0; rnn_dhn_bwd_saved then forms d f0 = dOut (.) walk_sum
 * elementwise instead of a k-th walk launch (d f0 is linear in the walk sum, PAPER.md:943-946;
 * the other d f_j are computed as in rnn_dhn_bwd).  Same arguments, layouts and errors as
 * rnn_dhn_fwd / rnn_dhn_bwd; walk_sum is caller-owned device memory, NULL is an error when
 * n_groups > 0, ld_ws >= d. */
rnn_status rnn_dhn_fwd_save(const rnn_join_index* adj, int32_t k, const rnn_operand* f,
                            float* out, int64_t ld_out, float* walk_sum, int64_t ld_ws,
                            void* workspace, size_t workspace_bytes, void* stream);
/* flags of rnn_dhn_bwd_saved: RNN_DHN_SYMMETRIC_EDGE -- the caller asserts that Edge is
 * symmetric ((n, v) and (v, n) occur with equal multiplicity, e.g. an undirected graph stored
 * in both directions, reading 10).  Closed walks then reverse, so for k = 4 the
 * d f1 and d f3 walks share both partial sums and run as ONE walk with two middle operands
 * (d f1 | d f3), and for k = 3 the d f1 and d f2 walks share the probe work and run as one
 * walk with two first-hop operands.  Results are undefined if the assertion is false.
 * Unknown bits: error. */
#define RNN_DHN_SYMMETRIC_EDGE 1u
rnn_status rnn_dhn_bwd_saved(const rnn_join_index* adj, int32_t k, const rnn_operand* f,
                             const float* d_out, int64_t ld_dout, const float* walk_sum,
                             int64_t ld_ws, float* const* d_f, int64_t ld_df, uint32_t flags,
                             void* workspace, size_t workspace_bytes, void* stream);

/* Root subsets (multi-GPU: roots hash-partitioned over ranks, the adjacency replicated,
 * SURVEY sec 8e): the same operations restricted to the roots listed in roots[n_roots]
 * (group ids of adj, device memory; ids outside [0, n_groups) and repeats are ignored).
 * Forward: out (and walk_sum, nullable here) rows of listed roots are written, other rows
 * are left untouched.  Backward: d f_j(x) is the walk aggregate ROOTED AT x with rotated
 * operands, so the listed roots x get their complete gradient rows (every other row of d_f
 * is 0, as are rows on no walk); g = f0 (.) d_out must be valid for EVERY root (d_out rows
 * of all groups, e.g. all-gathered), and d f0 = d_out (.) walk_sum is written for every
 * group when walk_sum is given.  k = 2 ignores the subset (every root; it is one gather).
 * Otherwise the arguments, layouts and errors of rnn_dhn_fwd_save / rnn_dhn_bwd_saved. */
rnn_status rnn_dhn_fwd_roots(const rnn_join_index* adj, int32_t k, const rnn_operand* f,
                             const int32_t* roots, int64_t n_roots, float* out, int64_t ld_out,
                             float* walk_sum, int64_t ld_ws, void* workspace,
                             size_t workspace_bytes, void* stream);
rnn_status rnn_dhn_bwd_roots(const rnn_join_index* adj, int32_t k, const rnn_operand* f,
                             const int32_t* roots, int64_t n_roots, const float* d_out,
                             int64_t ld_dout, const float* walk_sum, int64_t ld_ws,
                             float* const* d_f, int64_t ld_df, uint32_t flags, void* workspace,
                             size_t workspace_bytes, void* stream);

/* Exact closed-walk (homomorphism) counts: counts[g] = number of closed k-walks rooted at
 * group g's node, with Edge multiplicity -- C_k(n) of the rule above with every operand 1,
 * i.e. (A^k)_nn of the Edge relation's (multi)adjacency matrix (Eq. 3 :1500
 * with mu = 1; k = 2: the out-degree, the single Edge atom of the C2 rule :1509).  Integer
 * arithmetic throughout (int64 totals, uint64 partial counts), so the result is exact and
 * deterministic -- unlike rnn_dhn_fwd, whose fp32 atomics are exact only below 2^24 and in
 * any rounding order.  adj: as for rnn_dhn_fwd.  counts [n_groups] int64 (device, group
 * order), overwritten.  workspace: rnn_dhn_count_workspace_size (host-only query).
 * k outside 2..4: RNN_ERR_UNSUPPORTED. */
rnn_status rnn_dhn_count_workspace_size(const rnn_join_index* adj, int32_t k, size_t* bytes);
rnn_status rnn_dhn_count(const rnn_join_index* adj, int32_t k, int64_t* counts, void* workspace,
                         size_t workspace_bytes, void* stream);

/* ===================================================================================== */
/* Program helpers                                                                       */
/* ===================================================================================== */
/* GCN normalisation as a per-join-position weight (use with RNN_BY_POSITION):
 * w[p] = deg(s_p)^-1/2 * deg(t_g)^-1/2 with deg = group size of the node (in-degree of the
 * self-looped edge relation, PyG gcn_norm reading).  S and T must be the same node relation
 * (n_src_rows == n_dst_rows). */
rnn_status rnn_gcn_norm(const rnn_join_index* idx, float* w, void* workspace,
                        size_t workspace_bytes, void* stream);

/* Sharded GCN normalisation (multi-GPU): S is the all-gathered source relation
 * of every rank, so deg(s) comes from its owner: w[p] = src_deg[src_row[p]]^-1/2 * |g|^-1/2
 * (0 where src_deg is 0).  src_deg [n_src_rows] int32 (device). */
rnn_status rnn_gcn_norm_src_deg(const rnn_join_index* idx, const int32_t* src_deg, float* w,
                                void* stream);
/* size[g] = number of join rows of group g (int32, device) -- the in-degree a rank owns. */
rnn_status rnn_group_sizes(const rnn_join_index* idx, int32_t* size, void* stream);

/* Union over relations of materialised per-relation results that share a head relation
 * (PAPER.md:451-460, e.g. HGT's H_tilda = sum over relation types, :1408-1409):
 * y[r, c] = beta * y[r, c] + x[r, c] for r < rows, c < cols (fp32, row-major, any ld). */
rnn_status rnn_accumulate(float* y, int64_t ldy, const float* x, int64_t ldx, int64_t rows,
                          int32_t cols, float beta, void* stream);

/* Row gather (multi-GPU plumbing: permuting gathered rows into group order, packing /
 * unpacking exchanged rows): y[i, c] = x[idx[i], c] for i < n, c < cols, and 0 where
 * idx[i] < 0 (fp32, row-major, any ld; idx int32, device).  Indices are not range-checked. */
rnn_status rnn_gather_rows(float* y, int64_t ldy, const float* x, int64_t ldx, const int32_t* idx,
                           int64_t n, int32_t cols, void* stream);

/* Row scatter-add (mini-batch streaming: adding one batch's source-gradient rows into the
 * full gradient): y[idx[i], c] += x[i, c] for i < n (idx[i] < 0 skipped).  The indices of one
 * call must be distinct (no two rows collide; calls on one stream apply in order, so the
 * result is deterministic). */
rnn_status rnn_scatter_add_rows(float* y, int64_t ldy, const float* x, int64_t ldx,
                                const int32_t* idx, int64_t n, int32_t cols, void* stream);

/* Multi-GPU ownership of group keys: owner[i] = splitmix64(keys[i] ^ seed) mod P. */
rnn_status rnn_hash_partition(const int64_t* keys, int64_t n, int32_t P, uint64_t seed,
                              int32_t* owner, void* stream);

/* Residency hint for the gathered embedding matrix (north_star: "keep hot rows on chip"):
 * sets `stream`'s L2 access-policy window to [base, base + bytes) with the given hit ratio
 * (hits persisting, misses streaming) and reserves min(bytes * hit_ratio, device maximum)
 * of L2 for persisting lines; bytes = 0 clears the window and resets persisting lines.
 * Kernels launched on the stream afterwards (and kernel nodes captured from it) carry the
 * window.  SYNC for the limit change (cudaDeviceSetLimit). */
rnn_status rnn_stream_l2_window(void* stream, const void* base, size_t bytes, float hit_ratio);

#ifdef __cplusplus
}
#endif
#endif /* RNN_H */
