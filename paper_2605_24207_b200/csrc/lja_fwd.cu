// lja_fwd.cu -- A3/A4: fused gather - combine - segmented reduce, forward.
//
// out[g] = alpha_{p in group g} c(z_s[src_row[p]], z_e[edge_row[p]], z_t[group_dst_row[g]])
// (the join rule's U_{alpha,t}(T_c(E |><| S |><| T))).  One warp per work
// item; each join row's embedding is gathered with 128-bit loads (LPR lanes per row, RPW rows
// side by side), combined in registers and reduced in registers + warp shuffles -- the
// [E', d] join result the paper materialises with index_select never exists,
// and no atomics are used (the paper's scatter_add).  A group-side MUL factor
// and the MEAN divisor are applied once after the reduction.
//
// SOFTMAX (HGT, Fig. 4): per group and head an online (running max / sum)
// softmax over the rows' scores scale * <K'[s], Q[t]>, weighting the gathered values M'[s];
// the log-sum-exp is saved for the backward.
#include "smsplit.cuh"

namespace rnn {
namespace {

constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// ------------------------------------------------------------------------------------------
// SUM / MEAN with SRC, MUL, ADD combines
// ------------------------------------------------------------------------------------------
template <class L>
struct FwdSum {
  LjaArgs a;
  int n4s, n4e, n4t, n4o;
  static constexpr int U = L::VEC == 1 ? 8 : 4;
  struct State { float4 acc[L::VEC]; };

  __device__ __forceinline__ void init(State& s, int64_t) const {
#pragma unroll
    for (int v = 0; v < L::VEC; ++v) s.acc[v] = f4_zero();
  }

  __device__ __forceinline__ void rows(State& s, int64_t, int64_t r0, int64_t r1) const {
    const int lane = lane_id(), slot = L::slot();
    const bool has_src = a.src.p != nullptr, has_edge = a.edge.p != nullptr;
    const bool edge_scalar = has_edge && a.edge.dim == 1;
    for (int64_t base = r0; base < r1; base += 32) {
      const int P = (int)((r1 - base) < 32 ? (r1 - base) : 32);
      int ms = 0, me = 0;
      float mw = 1.f;
      if (lane < P) {
        const int64_t p = base + lane;
        if (has_src) ms = a.src_row[p];
        if (has_edge) {
          me = a.edge.mode ? (int)p : a.edge_row[p];
          if (edge_scalar) mw = __ldg(a.edge.p + (int64_t)me * a.edge.ld);
        }
      }
      const int nk = (P + L::RPW - 1) / L::RPW;
      for (int k0 = 0; k0 < nk; k0 += U) {
        float4 sv[U][L::VEC], ev[U][L::VEC];
        float w[U], mk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int li = (k0 + u) * L::RPW + slot;
          const bool ok = li < P;
          const int s_ = __shfl_sync(FULL, ms, li & 31);
          const int e_ = __shfl_sync(FULL, me, li & 31);
          const float wu = __shfl_sync(FULL, mw, li & 31);
          mk[u] = ok ? 1.f : 0.f;
          w[u] = ok ? wu : 0.f;
#pragma unroll
          for (int v = 0; v < L::VEC; ++v) {
            const int k = L::col4(v);
            sv[u][v] = (ok && has_src) ? load4(a.src.p, s_, a.src.ld, k, n4s) : f4_zero();
            ev[u][v] = (ok && has_edge && !edge_scalar) ? load4(a.edge.p, e_, a.edge.ld, k, n4e)
                                                        : f4_zero();          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int v = 0; v < L::VEC; ++v) {
            if (a.combine == RNN_COMBINE_SRC) {
              s.acc[v] = f4_fma(w[u], sv[u][v], s.acc[v]);
            } else if (a.combine == RNN_COMBINE_MUL) {
              float4 x = has_src ? sv[u][v] : make_float4(1.f, 1.f, 1.f, 1.f);
              if (edge_scalar) x = f4_scale(w[u], x);
              else if (has_edge) x = f4_mul(x, ev[u][v]);
              s.acc[v] = f4_fma(mk[u], x, s.acc[v]);
            } else {  // ADD
              float4 x = sv[u][v];
              if (edge_scalar) x = f4_add(x, make_float4(w[u], w[u], w[u], w[u]));
              else if (has_edge) x = f4_add(x, ev[u][v]);
              s.acc[v] = f4_fma(mk[u], x, s.acc[v]);
            }
          }
        }
      }
    }
    if (L::RPW > 1) {
#pragma unroll
      for (int v = 0; v < L::VEC; ++v) s.acc[v] = L::reduce_slots(s.acc[v]);
    }
  }

  __device__ __forceinline__ void finish(State& s, int64_t g) const {
    if (L::slot() != 0) return;
    const int64_t n = a.group_ptr[g + 1] - a.group_ptr[g];
    const bool has_dst = a.dst.p != nullptr;
    const int64_t t = has_dst ? (a.dst.mode ? g : (int64_t)a.dst_row[g]) : 0;
#pragma unroll
    for (int v = 0; v < L::VEC; ++v) {
      const int k = L::col4(v);
      if (k >= n4o) continue;
      float4 x = s.acc[v];
      if (has_dst) {
        float4 z;
        if (a.dst.dim == 1) { float z0 = __ldg(a.dst.p + t * a.dst.ld); z = make_float4(z0, z0, z0, z0); }
        else z = load4(a.dst.p, t, a.dst.ld, k, n4t);
        if (a.combine == RNN_COMBINE_MUL) x = f4_mul(x, z);
        else if (a.combine == RNN_COMBINE_ADD) x = f4_add(x, f4_scale((float)n, z));
      }
      if (a.mean) x = f4_scale(n > 0 ? 1.f / (float)n : 0.f, x);
      if (n == 0) x = f4_zero();  // empty group (dense index): aggregate of {} is 0
      if (a.beta != 0.f) x = f4_add(x, f4_scale(a.beta, load4_clip(a.out, g, a.ld_out, k, a.D)));
      store4_clip(a.out, g, a.ld_out, k, a.D, x);
    }
  }

  __device__ __forceinline__ void save(const State& s, float* dst) const {
    if (L::slot() != 0) return;
#pragma unroll
    for (int v = 0; v < L::VEC; ++v) {
      const int k = L::col4(v);
      if (k < n4o) __stcg(reinterpret_cast<float4*>(dst + 4 * k), s.acc[v]);
    }
  }
  __device__ __forceinline__ void merge(State& s, const float* src) const {
#pragma unroll
    for (int v = 0; v < L::VEC; ++v) {
      const int k = L::col4(v);
      if (k < n4o) s.acc[v] = f4_add(s.acc[v], ld_f4_cg(src + 4 * k));
    }
  }
};

// ------------------------------------------------------------------------------------------
// SOFTMAX aggregation (online softmax over each group's rows, per head)
// ------------------------------------------------------------------------------------------
template <class L>
struct FwdSoftmax {
  LjaArgs a;
  int heads, LH;       // LH = lanes per head
  float scale_log2;    // scale * log2(e)
  static constexpr int U = 4;
  struct State { float4 acc; float m, l; };

  __device__ __forceinline__ void init(State& s, int64_t) const {
    s.acc = f4_zero(); s.m = -INFINITY; s.l = 0.f;
  }
  __device__ __forceinline__ float head_sum(float x) const {
    for (int m = 1; m < LH; m <<= 1) x += __shfl_xor_sync(FULL, x, m);
    return x;
  }
  __device__ __forceinline__ static void combine(State& s, float m2, float l2, float4 acc2) {
    const float mn = fmaxf(s.m, m2);
    if (mn == -INFINITY) return;
    const float c1 = exp2f(s.m - mn), c2 = exp2f(m2 - mn);
    s.l = s.l * c1 + l2 * c2;
    s.acc = f4_add(f4_scale(c1, s.acc), f4_scale(c2, acc2));
    s.m = mn;
  }

  __device__ __forceinline__ void rows(State& s, int64_t g, int64_t r0, int64_t r1) const {
    const int lane = lane_id(), slot = L::slot(), k = L::sub();
    const int64_t t = a.dst.mode ? g : (int64_t)a.dst_row[g];
    const float4 q = ld_f4(a.dst.p + t * a.dst.ld + 4 * k);
    for (int64_t base = r0; base < r1; base += 32) {
      const int P = (int)((r1 - base) < 32 ? (r1 - base) : 32);
      const int ms = lane < P ? a.src_row[base + lane] : 0;
      const int nk = (P + L::RPW - 1) / L::RPW;
      for (int k0 = 0; k0 < nk; k0 += U) {
        float4 kv[U], vv[U];
        float sc[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int li = (k0 + u) * L::RPW + slot;
          ok[u] = li < P;
          const int s_ = __shfl_sync(FULL, ms, li & 31);
          kv[u] = ok[u] ? ld_f4(a.src_key.p + (int64_t)s_ * a.src_key.ld + 4 * k) : f4_zero();
          vv[u] = ok[u] ? ld_f4(a.src.p + (int64_t)s_ * a.src.ld + 4 * k) : f4_zero();
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float d = head_sum(f4_dot(kv[u], q));
          sc[u] = ok[u] ? d * scale_log2 : -INFINITY;
        }
        float mb = sc[0];
#pragma unroll
        for (int u = 1; u < U; ++u) mb = fmaxf(mb, sc[u]);
        const float mn = fmaxf(s.m, mb);
        if (mn == -INFINITY) continue;
        const float corr = exp2f(s.m - mn);
        s.l *= corr;
        s.acc = f4_scale(corr, s.acc);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float pu = exp2f(sc[u] - mn);
          s.l += pu;
          s.acc = f4_fma(pu, vv[u], s.acc);
        }
        s.m = mn;
      }
    }
    if (L::RPW > 1) {
#pragma unroll
      for (int m = L::LPR; m < 32; m <<= 1) {
        const float m2 = __shfl_xor_sync(FULL, s.m, m), l2 = __shfl_xor_sync(FULL, s.l, m);
        const float4 a2 = f4_shfl_xor(s.acc, m);
        combine(s, m2, l2, a2);
      }
    }
  }

  __device__ __forceinline__ void finish(State& s, int64_t g) const {
    if (L::slot() != 0) return;
    const int k = L::sub();
    const bool empty = s.l == 0.f;  // empty group (dense index): out 0, lse -inf
    float4 x = empty ? f4_zero() : f4_scale(1.f / s.l, s.acc);
    if (a.beta != 0.f) x = f4_add(x, f4_scale(a.beta, ld_f4(a.out + g * a.ld_out + 4 * k)));
    st_f4(a.out + g * a.ld_out + 4 * k, x);
    if (k % LH == 0) a.lse[g * heads + k / LH] = empty ? -INFINITY : (s.m + log2f(s.l)) * LN2;
  }
  __device__ __forceinline__ void save(const State& s, float* dst) const {
    if (L::slot() != 0) return;
    const int k = L::sub();
    __stcg(reinterpret_cast<float4*>(dst + 4 * k), s.acc);
    if (k % LH == 0) {
      __stcg(dst + 4 * L::LPR + 2 * (k / LH), s.m);
      __stcg(dst + 4 * L::LPR + 2 * (k / LH) + 1, s.l);
    }
  }
  __device__ __forceinline__ void merge(State& s, const float* src) const {
    const int k = L::sub();
    const float4 a2 = ld_f4_cg(src + 4 * k);
    const float m2 = __ldcg(src + 4 * L::LPR + 2 * (k / LH));
    const float l2 = __ldcg(src + 4 * L::LPR + 2 * (k / LH) + 1);
    combine(s, m2, l2, a2);
  }
};

// ------------------------------------------------------------------------------------------
// SUM / MEAN, row-split hot loop (rows wider than 64 floats; src operand present)
// ------------------------------------------------------------------------------------------
// MODE 0: row value = c * z_s          (SRC with/without weight, MUL with a scalar or no edge)
// MODE 1: row value = c * (z_s op z_e)  (MUL / ADD with a vector edge embedding)
// MODE 2: row value = c * (z_s + w)     (ADD with a scalar edge)
// c folds the edge weight and, for MEAN, 1/|g| (so the finish never reloads group sizes).
template <int VEC, int MODE>
struct FwdRS {
  LjaArgs a;
  int n4s, n4e, n4t, n4o;
  bool has_dst;
  struct Meta { int idx, e; float c, wa; };

  __device__ __forceinline__ Meta meta(int64_t r, int g) const {
    Meta m{a.src_row[r], 0, 1.f, 0.f};
    if (a.edge.p) {
      m.e = a.edge.mode ? (int)r : a.edge_row[r];
      if (a.edge.dim == 1) {
        const float w = __ldg(a.edge.p + (int64_t)m.e * a.edge.ld);
        if (MODE == 2) m.wa = w; else m.c = w;
      }
    }
    if (a.mean) m.c *= 1.f / (float)(a.group_ptr[g + 1] - a.group_ptr[g]);
    return m;
  }
  __device__ __forceinline__ Meta shfl(const Meta& m, int src) const {
    Meta o;
    o.idx = __shfl_sync(FULL, m.idx, src);
    o.e = MODE == 1 ? __shfl_sync(FULL, m.e, src) : 0;
    o.c = __shfl_sync(FULL, m.c, src);
    o.wa = MODE == 2 ? __shfl_sync(FULL, m.wa, src) : 0.f;
    return o;
  }
  __device__ __forceinline__ float4 load(const Meta& m, bool ok, int w) const {
    const int k = lane_id() + 32 * w;
    return ld_row4(a.src.p, m.idx, a.src.ld, k, ok && k < n4s);
  }
  __device__ __forceinline__ float4 load_f(const Meta& m, bool ok, int w) const {
    if (MODE != 1) return f4_zero();
    const int k = lane_id() + 32 * w;
    return ld_row4(a.edge.p, m.e, a.edge.ld, k, ok && k < n4e);
  }
  __device__ __forceinline__ float4 add(float4 acc, const Meta& m, float4 x, float4 f) const {
    if (MODE == 1) x = a.combine == RNN_COMBINE_MUL ? f4_mul(x, f) : f4_add(x, f);
    if (MODE == 2) x = f4_add(x, make_float4(m.wa, m.wa, m.wa, m.wa));
    return f4_fma(m.c, x, acc);
  }
  __device__ __forceinline__ void finish(const float4 (&acc)[4], int64_t g) const {
    const int lane = lane_id();
    int64_t t = 0;
    float n = 1.f;
    if (has_dst) {
      t = a.dst.mode ? g : (int64_t)a.dst_row[g];
      if (a.combine == RNN_COMBINE_ADD && !a.mean) n = (float)(a.group_ptr[g + 1] - a.group_ptr[g]);
    }
#pragma unroll
    for (int w = 0; w < VEC; ++w) {
      const int k = lane + 32 * w;
      if (k >= n4o) continue;
      float4 x = acc[w];
      if (has_dst) {
        float4 z;
        if (a.dst.dim == 1) { const float z0 = __ldg(a.dst.p + t * a.dst.ld); z = make_float4(z0, z0, z0, z0); }
        else z = load4(a.dst.p, t, a.dst.ld, k, n4t);
        if (a.combine == RNN_COMBINE_MUL) x = f4_mul(x, z);
        else if (a.combine == RNN_COMBINE_ADD) x = f4_add(x, f4_scale(n, z));  // mean folded: + z
      }
      if (a.beta != 0.f) x = f4_add(x, f4_scale(a.beta, load4_clip(a.out, g, a.ld_out, k, a.D)));
      store4_clip(a.out, g, a.ld_out, k, a.D, x);
    }
  }
  __device__ __forceinline__ void zero(int64_t g) const {
    if (a.beta != 0.f) return;  // empty group: out = beta*out + 0
    const int lane = lane_id();
#pragma unroll
    for (int w = 0; w < VEC; ++w) {
      const int k = lane + 32 * w;
      if (k < n4o) store4_clip(a.out, g, a.ld_out, k, a.D, f4_zero());
    }
  }
};

template <int VEC, int MODE>
rnn_status launch_rs(const LjaArgs& a, const RSCtx& cx, cudaStream_t st) {
  FwdRS<VEC, MODE> pol;
  pol.a = a;
  pol.n4s = (a.src.dim + 3) / 4;
  pol.n4e = a.edge.p ? (a.edge.dim + 3) / 4 : 0;
  pol.n4t = a.dst.p ? (a.dst.dim + 3) / 4 : 0;
  pol.n4o = (a.D + 3) / 4;
  pol.has_dst = a.dst.p != nullptr;
  return launch_rowsplit<FwdRS<VEC, MODE>, VEC>(pol, cx, st);
}

// metadata of the lean kernel (rowsplit.cuh): idx = src_row[r], c = w_r (/|g| for MEAN)
struct LeanFwdMeta {
  const int32_t* src_row;
  const int32_t* edge_row;
  const int64_t* group_ptr;
  const float* w;  // scalar edge weight (nullptr: 1)
  int64_t ldw;
  int w_by_pos;
  int mean;
  struct Meta { int idx; float c; };
  __device__ __forceinline__ Meta meta(int64_t r, int g) const {
    Meta m{src_row[r], 1.f};
    if (w) m.c = __ldg(w + (w_by_pos ? r : (int64_t)edge_row[r]) * ldw);
    if (mean) m.c *= 1.f / (float)(group_ptr[g + 1] - group_ptr[g]);
    return m;
  }
};

template <int VEC>
rnn_status launch_rs_mode(const LjaArgs& a, const RSCtx& cx, cudaStream_t st) {
  // lean path: full-width rows, row value = c * z_s, no group-side factor
  const bool scaled = a.combine == RNN_COMBINE_SRC ||
                      (a.combine == RNN_COMBINE_MUL && (!a.edge.p || a.edge.dim == 1));
  if (scaled && !a.dst.p && a.D == 128 * VEC && a.ld_out % 4 == 0) {
    LeanFwdMeta mp{a.src_row, a.edge_row, a.group_ptr, a.edge.p, a.edge.ld, a.edge.mode, a.mean};
    LeanOut o{a.src.p, a.src.ld, a.out, a.ld_out, a.beta};
    if (a.epi.on && a.epi_done) *a.epi_done = 1;
    return launch_lean<LeanFwdMeta, VEC>(mp, cx, o, st, a.epi);
  }
  const bool ev = a.edge.p && a.edge.dim > 1;
  if (ev) return launch_rs<VEC, 1>(a, cx, st);
  if (a.combine == RNN_COMBINE_ADD && a.edge.p) return launch_rs<VEC, 2>(a, cx, st);
  return launch_rs<VEC, 0>(a, cx, st);
}

// ------------------------------------------------------------------------------------------
// CONCAT (and any width layout): one warp per group, lanes stride over output columns
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) fwd_concat_kernel(LjaArgs a, int64_t n_groups) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= n_groups) return;
  const int lane = lane_id();
  const int ds = a.src.p ? a.src.dim : 0, de = a.edge.p ? a.edge.dim : 0;
  const int64_t b = a.group_ptr[g], e = a.group_ptr[g + 1];
  const int64_t t = a.dst.p ? (a.dst.mode ? g : (int64_t)a.dst_row[g]) : 0;
  for (int c = lane; c < a.D; c += 32) {
    float acc = 0.f;
    if (c < ds) {
      for (int64_t p = b; p < e; ++p) acc += __ldg(a.src.p + (int64_t)a.src_row[p] * a.src.ld + c);
    } else if (c < ds + de) {
      for (int64_t p = b; p < e; ++p) {
        const int64_t er = a.edge.mode ? p : (int64_t)a.edge_row[p];
        acc += __ldg(a.edge.p + er * a.edge.ld + (c - ds));
      }
    } else {
      acc = (float)(e - b) * __ldg(a.dst.p + t * a.dst.ld + (c - ds - de));
    }
    if (a.mean) acc *= e > b ? 1.f / (float)(e - b) : 0.f;
    float* o = a.out + g * a.ld_out + c;
    *o = a.beta != 0.f ? acc + a.beta * *o : acc;
  }
}

// lse of groups with no join row (dense index, E' = 0): log-sum-exp of {} = -inf
__global__ void fill_neg_inf_kernel(float* __restrict__ p, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = -INFINITY;
}

template <template <class> class Pol, class L>
rnn_status launch_pol(Pol<L> pol, const SegCtx& cx, cudaStream_t st) {
  if (cx.n_work <= 0) return RNN_OK;
  const int64_t blocks = ceil_div(cx.n_work, 8);
  seg_kernel<Pol<L>><<<(unsigned)blocks, 256, 0, st>>>(pol, cx);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

template <class L>
rnn_status launch_sum(const LjaArgs& a, const SegCtx& cx, cudaStream_t st) {
  FwdSum<L> pol;
  pol.a = a;
  pol.n4s = a.src.p ? (a.src.dim + 3) / 4 : 0;
  pol.n4e = a.edge.p ? (a.edge.dim + 3) / 4 : 0;
  pol.n4t = a.dst.p ? (a.dst.dim + 3) / 4 : 0;
  pol.n4o = (a.D + 3) / 4;
  return launch_pol<FwdSum, L>(pol, cx, st);
}

template <class L>
rnn_status launch_softmax(const LjaArgs& a, int heads, float scale, const SegCtx& cx,
                          cudaStream_t st) {
  FwdSoftmax<L> pol;
  pol.a = a;
  pol.heads = heads;
  pol.LH = L::LPR / heads;
  pol.scale_log2 = scale * LOG2E;
  return launch_pol<FwdSoftmax, L>(pol, cx, st);
}

}  // namespace

struct Union2 { float* out; int64_t ld; float beta; bool done; };
rnn_status lja_fwd_core(const rnn_join_index* idx, const rnn_lifted_query* q, float* out,
                        int64_t ld_out, float beta, float* lse, void* ws, size_t ws_bytes,
                        cudaStream_t st, const EpiD* epi, int* epi_done, Union2* un = nullptr);

rnn_status lja_fwd_impl(const rnn_join_index* idx, const rnn_lifted_query* q, float* out,
                        int64_t ld_out, float beta, float* lse, void* ws, size_t ws_bytes,
                        cudaStream_t st, const EpiD* epi) {
  if (epi && epi->on) {
    // the aggregate, with the epilogue fused into the lean store where that path runs, else
    // applied in place afterwards (one extra pass over [G, D])
    int done = 0;
    EpiD e = *epi;
    RNN_TRY(lja_fwd_core(idx, q, out, ld_out, beta, lse, ws, ws_bytes, st, &e, &done));
    if (!done && idx->n_groups > 0) {
      QueryInfo qi;
      RNN_TRY(check_query(idx, q, &qi));
      RNN_TRY(epilogue_inplace(out, ld_out, idx->n_groups, qi.D, e, st));
    }
    return RNN_OK;
  }
  return lja_fwd_core(idx, q, out, ld_out, beta, lse, ws, ws_bytes, st, nullptr, nullptr);
}

rnn_status lja_fwd_core(const rnn_join_index* idx, const rnn_lifted_query* q, float* out,
                        int64_t ld_out, float beta, float* lse, void* ws, size_t ws_bytes,
                        cudaStream_t st, const EpiD* epi, int* epi_done, Union2* un) {
  QueryInfo qi;
  RNN_TRY(check_query(idx, q, &qi));
  if (idx->n_groups == 0) return RNN_OK;
  RNN_REQUIRE(out && ld_out >= qi.D, RNN_ERR_INVALID_ARGUMENT, "out NULL or ld_out < %d", qi.D);
  RNN_REQUIRE(qi.concat || (ld_out % 4 == 0 && aligned16(out)), RNN_ERR_INVALID_ARGUMENT,
              "out must be 16-byte aligned with ld_out %% 4 == 0");
  RNN_REQUIRE(beta == 0.f || beta == 1.f, RNN_ERR_INVALID_ARGUMENT, "beta must be 0 or 1");
  RNN_REQUIRE(beta == 0.f || q->agg != RNN_AGG_MEAN, RNN_ERR_UNSUPPORTED,
              "beta = 1 with MEAN is not decomposable (PAPER.md:340)");
  if (idx->n_groups == 0) return RNN_OK;
  if (idx->n_join_rows == 0 && !qi.concat) {
    // every group is empty (dense index over an empty join): the aggregate of {} is 0, so
    // out = beta * out + 0, and lse = -inf -- no work items exist for the walkers to do this
    if (beta == 0.f)
      RNN_CUDA(cudaMemset2DAsync(out, sizeof(float) * ld_out, 0, sizeof(float) * qi.D,
                                 idx->n_groups, st));
    if (q->agg == RNN_AGG_SOFTMAX && lse) {
      const int64_t n = idx->n_groups * q->heads;
      fill_neg_inf_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(lse, n);
      RNN_LAUNCH_CHECK();
    }
    return RNN_OK;
  }
  LjaArgs a = make_args(idx, q, out, ld_out, beta, lse, qi.D);
  if (epi) {
    a.epi = *epi;
    a.epi_done = epi_done;
  }
  if (qi.concat) {
    fwd_concat_kernel<<<(unsigned)ceil_div(idx->n_groups, 8), 256, 0, st>>>(a, idx->n_groups);
    RNN_LAUNCH_CHECK();
    return RNN_OK;
  }
  size_t need = 0;
  RNN_TRY(lja_fwd_ws(idx, q, &need));
  RNN_REQUIRE(ws_bytes >= need && (need == 0 || ws), RNN_ERR_WORKSPACE_TOO_SMALL,
              "forward workspace %zu < %zu bytes", ws_bytes, need);
  SegCtx cx;
  cx.ptr = idx->group_ptr; cx.n_seg = idx->n_groups;
  cx.work_ptr = idx->work_ptr; cx.n_work = idx->n_work;
  Carve c(ws);
  cx.pstride = qi.pstride;
  cx.partial = c.take<float>((size_t)idx->n_work * qi.pstride);
  cx.counter = c.take<int>((size_t)idx->n_work);
  RNN_CUDA(cudaMemsetAsync(cx.counter, 0, sizeof(int) * idx->n_work, st));
  const int lc = lane_config(qi.D);
  if (q->agg != RNN_AGG_SOFTMAX && lc >= 32 && q->src.data && idx->pos_group) {
    RSCtx rx{idx->pos_group, idx->group_ptr, idx->n_groups, idx->n_join_rows, idx->work_ptr,
             idx->n_work, cx.partial, cx.pstride, cx.counter, 1};
    if (lc == 32) return launch_rs_mode<1>(a, rx, st);
    if (lc == 64) return launch_rs_mode<2>(a, rx, st);
    return launch_rs_mode<4>(a, rx, st);
  }
  if (q->agg == RNN_AGG_SOFTMAX && sm_rowsplit_ok(idx, q, qi.D)) {
    SmFwdPol pol;
    pol.a = sm_rows(idx, q);
    pol.out = out; pol.ld_out = ld_out; pol.beta = beta; pol.lse = lse;
    if (un) {   // union store fused into the walker's finish
      pol.out2 = un->out; pol.ld_out2 = un->ld; pol.beta2 = un->beta;
      un->done = true;
    }
    RSCtx rx{idx->pos_group, idx->group_ptr, idx->n_groups, idx->n_join_rows, idx->work_ptr,
             idx->n_work, cx.partial, cx.pstride, cx.counter, 1};
    return launch_st_var(pol, rx, st, 0);
  }
  if (q->agg == RNN_AGG_SOFTMAX) {
    switch (qi.D / 4) {
      case 1: return launch_softmax<Lanes<1, 1>>(a, q->heads, q->scale, cx, st);
      case 2: return launch_softmax<Lanes<2, 1>>(a, q->heads, q->scale, cx, st);
      case 4: return launch_softmax<Lanes<4, 1>>(a, q->heads, q->scale, cx, st);
      case 8: return launch_softmax<Lanes<8, 1>>(a, q->heads, q->scale, cx, st);
      case 16: return launch_softmax<Lanes<16, 1>>(a, q->heads, q->scale, cx, st);
      case 32: return launch_softmax<Lanes<32, 1>>(a, q->heads, q->scale, cx, st);
    }
    RNN_FAIL(RNN_ERR_UNSUPPORTED, "SOFTMAX width %d", qi.D);
  }
  switch (lane_config(qi.D)) {
    case 1: return launch_sum<Lanes<1, 1>>(a, cx, st);
    case 2: return launch_sum<Lanes<2, 1>>(a, cx, st);
    case 4: return launch_sum<Lanes<4, 1>>(a, cx, st);
    case 8: return launch_sum<Lanes<8, 1>>(a, cx, st);
    case 16: return launch_sum<Lanes<16, 1>>(a, cx, st);
    case 32: return launch_sum<Lanes<32, 1>>(a, cx, st);
    case 64: return launch_sum<Lanes<32, 2>>(a, cx, st);
    case 128: return launch_sum<Lanes<32, 4>>(a, cx, st);
  }
  RNN_FAIL(RNN_ERR_UNSUPPORTED, "width %d", qi.D);
}

}  // namespace rnn

extern "C" rnn_status rnn_join_aggregate_fwd(const rnn_join_index* idx, const rnn_lifted_query* q,
                                             float* out, int64_t ld_out, float beta, float* lse,
                                             void* workspace, size_t workspace_bytes,
                                             void* stream) {
  rnn::clear_error();
  return rnn::lja_fwd_impl(idx, q, out, ld_out, beta, lse, workspace, workspace_bytes,
                           rnn::as_stream(stream));
}

extern "C" rnn_status rnn_join_aggregate_fwd_union(const rnn_join_index* idx,
                                                   const rnn_lifted_query* q, float* out,
                                                   int64_t ld_out, float* lse, float* acc,
                                                   int64_t ld_acc, float beta_acc,
                                                   void* workspace, size_t workspace_bytes,
                                                   void* stream) {
  rnn::clear_error();
  RNN_REQUIRE(beta_acc == 0.f || beta_acc == 1.f, RNN_ERR_INVALID_ARGUMENT,
              "beta_acc must be 0 or 1");
  RNN_REQUIRE(q && q->agg != RNN_AGG_MEAN, RNN_ERR_UNSUPPORTED,
              "a union over relations of MEAN is not decomposable (PAPER.md:340)");
  rnn::QueryInfo qi;
  RNN_TRY(rnn::check_query(idx, q, &qi));
  if (idx->n_groups == 0) return RNN_OK;
  RNN_REQUIRE(acc && ld_acc >= qi.D && ld_acc % 4 == 0 && rnn::aligned16(acc) && acc != out,
              RNN_ERR_INVALID_ARGUMENT, "acc NULL, aliasing out, unaligned or ld_acc < %d", qi.D);
  cudaStream_t st = rnn::as_stream(stream);
  rnn::Union2 un{acc, ld_acc, beta_acc, false};
  RNN_TRY(rnn::lja_fwd_core(idx, q, out, ld_out, 0.f, lse, workspace, workspace_bytes, st,
                            nullptr, nullptr, &un));
  if (!un.done)   // paths without the fused store: one pass acc = beta_acc acc + out
    return rnn_accumulate(acc, ld_acc, out, ld_out, idx->n_groups, qi.D, beta_acc, stream);
  return RNN_OK;
}

extern "C" rnn_status rnn_join_aggregate_fwd_epi(const rnn_join_index* idx,
                                                 const rnn_lifted_query* q,
                                                 const rnn_epilogue* epi, float* out,
                                                 int64_t ld_out, void* workspace,
                                                 size_t workspace_bytes, void* stream) {
  rnn::clear_error();
  RNN_REQUIRE(epi, RNN_ERR_INVALID_ARGUMENT, "epilogue is NULL");
  RNN_REQUIRE(q && q->agg != RNN_AGG_SOFTMAX, RNN_ERR_UNSUPPORTED,
              "the fused epilogue takes SUM / MEAN aggregates");
  RNN_REQUIRE(epi->act >= RNN_ACT_NONE && epi->act <= RNN_ACT_GELU, RNN_ERR_INVALID_ARGUMENT,
              "unknown activation");
  RNN_REQUIRE(!epi->resid || (epi->gate >= 0.f && epi->gate <= 1.f), RNN_ERR_INVALID_ARGUMENT,
              "gate outside [0, 1]");
  RNN_REQUIRE((!epi->bias || rnn::aligned16(epi->bias)) && (!epi->pre || (rnn::aligned16(epi->pre) &&
              epi->ld_pre % 4 == 0)) && (!epi->resid || (rnn::aligned16(epi->resid) &&
              epi->ld_resid % 4 == 0)), RNN_ERR_INVALID_ARGUMENT,
              "epilogue operands must be 16-byte aligned with ld %% 4 == 0");
  const rnn::EpiD e = rnn::epi_from_abi(epi);
  return rnn::lja_fwd_impl(idx, q, out, ld_out, 0.f, nullptr, workspace, workspace_bytes,
                           rnn::as_stream(stream), &e);
}
