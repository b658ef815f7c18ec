// lja_bwd.cu -- A5: backward of the lifted join-aggregate, plus the standalone grouped softmax.
//
// Gradients flow only through embeddings, never through the index (Fig. 3).
// The paper's autograd scatters source gradients with index_add_ atomics;
// here the source gradient is a GATHER over the transposed (source-major) CSR built once with
// the index: d_src[s] = sum_{q in src s} coef_q * Y[group(q)] -- no atomics, fixed order.
//   SRC : Y = dOut, coef = w_p (/|g| for MEAN)               -> d_src
//   MUL : Y = dOut (.) z_t (precomputed per group), coef = w_p or (.) z_e
//   ADD : Y = dOut, coef = 1 (/|g|)
// Group-major passes produce the per-row edge gradients and the group-side gradients.
// SOFTMAX (flash-style, two passes): pass 1 (group-major) recomputes a = exp(e - lse) and
// writes (a, de) per row and head, de = a (<dOut, M'_s> - <dOut, Out>), plus dQ; pass 2
// (source-major) gathers dM'_s = sum a dOut_t and dK'_s = scale sum de Q_t.
#include "smsplit.cuh"

namespace rnn {
namespace {

constexpr float LOG2E = 1.4426950408889634f;

// ------------------------------------------------------------------------------------------
// transposed gather for d_src (SRC / MUL / ADD / CONCAT block 0)
// ------------------------------------------------------------------------------------------
struct SrcArgs {
  const int32_t* src_group;
  const int32_t* src_pos;
  const int32_t* edge_row;
  const int64_t* group_ptr;
  const float* Y; int64_t ldy; int n4y;
  OpndD edge;        // scalar weight or vector factor (nullptr: none)
  bool mean;
  float* d; int64_t ldd; int D;
};

template <class L>
struct BwdSrc {
  SrcArgs a;
  static constexpr int U = L::VEC == 1 ? 8 : 4;
  struct State { float4 acc[L::VEC]; };
  __device__ __forceinline__ void init(State& s, int64_t) const {
#pragma unroll
    for (int v = 0; v < L::VEC; ++v) s.acc[v] = f4_zero();
  }
  __device__ __forceinline__ void rows(State& s, int64_t, int64_t r0, int64_t r1) const {
    const int lane = lane_id(), slot = L::slot();
    const bool has_edge = a.edge.p != nullptr, scalar = has_edge && a.edge.dim == 1;
    const int n4e = has_edge ? (a.edge.dim + 3) / 4 : 0;
    for (int64_t base = r0; base < r1; base += 32) {
      const int P = (int)((r1 - base) < 32 ? (r1 - base) : 32);
      int mg = 0, me = 0;
      float mc = 1.f;
      if (lane < P) {
        const int64_t q = base + lane;
        mg = a.src_group[q];
        const int p = a.src_pos[q];
        if (has_edge) {
          me = a.edge.mode ? p : a.edge_row[p];
          if (scalar) mc = __ldg(a.edge.p + (int64_t)me * a.edge.ld);
        }
        if (a.mean) mc *= 1.f / (float)(a.group_ptr[mg + 1] - a.group_ptr[mg]);
      }
      const int nk = (P + L::RPW - 1) / L::RPW;
      for (int k0 = 0; k0 < nk; k0 += U) {
        float4 yv[U][L::VEC], ev[U][L::VEC];
        float c[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int li = (k0 + u) * L::RPW + slot;
          ok[u] = li < P;
          const int g_ = __shfl_sync(FULL, mg, li & 31);
          const int e_ = __shfl_sync(FULL, me, li & 31);
          c[u] = __shfl_sync(FULL, mc, li & 31);
#pragma unroll
          for (int v = 0; v < L::VEC; ++v) {
            const int k = L::col4(v);
            yv[u][v] = ok[u] ? load4(a.Y, g_, a.ldy, k, a.n4y) : f4_zero();
            ev[u][v] = (ok[u] && has_edge && !scalar) ? load4(a.edge.p, e_, a.edge.ld, k, n4e)
                                                      : f4_zero();
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!ok[u]) continue;
#pragma unroll
          for (int v = 0; v < L::VEC; ++v) {
            float4 y = yv[u][v];
            if (has_edge && !scalar) y = f4_mul(y, ev[u][v]);
            s.acc[v] = f4_fma(c[u], y, s.acc[v]);
          }
        }
      }
    }
    if (L::RPW > 1) {
#pragma unroll
      for (int v = 0; v < L::VEC; ++v) s.acc[v] = L::reduce_slots(s.acc[v]);
    }
  }
  __device__ __forceinline__ void finish(State& s, int64_t seg) const {
    if (L::slot() != 0) return;
    const int n4 = (a.D + 3) / 4;
#pragma unroll
    for (int v = 0; v < L::VEC; ++v) {
      const int k = L::col4(v);
      if (k < n4) store4_clip(a.d, seg, a.ldd, k, a.D, s.acc[v]);
    }
  }
  __device__ __forceinline__ void save(const State& s, float* dst) const {
    if (L::slot() != 0) return;
    const int n4 = (a.D + 3) / 4;
#pragma unroll
    for (int v = 0; v < L::VEC; ++v) {
      const int k = L::col4(v);
      if (k < n4) __stcg(reinterpret_cast<float4*>(dst + 4 * k), s.acc[v]);
    }
  }
  __device__ __forceinline__ void merge(State& s, const float* src) const {
    const int n4 = (a.D + 3) / 4;
#pragma unroll
    for (int v = 0; v < L::VEC; ++v) {
      const int k = L::col4(v);
      if (k < n4) s.acc[v] = f4_add(s.acc[v], ld_f4_cg(src + 4 * k));
    }
  }
};

// row-split version of the transposed gather (rows wider than 64 floats)
template <int VEC, bool EV>  // EV: vector edge factor (MUL with an edge embedding)
struct BwdRS {
  SrcArgs a;
  int n4e;
  struct Meta { int g, e; float c; };
  __device__ __forceinline__ Meta meta(int64_t q, int) const {
    Meta m{a.src_group[q], 0, 1.f};
    const int p = a.src_pos[q];
    if (a.edge.p) {
      m.e = a.edge.mode ? p : a.edge_row[p];
      if (!EV) m.c = __ldg(a.edge.p + (int64_t)m.e * a.edge.ld);
    }
    if (a.mean) m.c *= 1.f / (float)(a.group_ptr[m.g + 1] - a.group_ptr[m.g]);
    return m;
  }
  __device__ __forceinline__ Meta shfl(const Meta& m, int src) const {
    Meta o;
    o.g = __shfl_sync(FULL, m.g, src);
    o.e = EV ? __shfl_sync(FULL, m.e, src) : 0;
    o.c = __shfl_sync(FULL, m.c, src);
    return o;
  }
  __device__ __forceinline__ float4 load(const Meta& m, bool ok, int w) const {
    const int k = lane_id() + 32 * w;
    return ld_row4(a.Y, m.g, a.ldy, k, ok && k < a.n4y);
  }
  __device__ __forceinline__ float4 load_f(const Meta& m, bool ok, int w) const {
    if (!EV) return f4_zero();
    const int k = lane_id() + 32 * w;
    return ld_row4(a.edge.p, m.e, a.edge.ld, k, ok && k < n4e);
  }
  __device__ __forceinline__ float4 add(float4 acc, const Meta& m, float4 x, float4 f) const {
    return f4_fma(m.c, EV ? f4_mul(x, f) : x, acc);
  }
  __device__ __forceinline__ void finish(const float4 (&acc)[4], int64_t seg) const {
    const int lane = lane_id();
    const int n4 = (a.D + 3) / 4;
#pragma unroll
    for (int w = 0; w < VEC; ++w) {
      const int k = lane + 32 * w;
      if (k < n4) store4_clip(a.d, seg, a.ldd, k, a.D, acc[w]);
    }
  }
  __device__ __forceinline__ void zero(int64_t seg) const {
    const int lane = lane_id();
    const int n4 = (a.D + 3) / 4;
#pragma unroll
    for (int w = 0; w < VEC; ++w) {
      const int k = lane + 32 * w;
      if (k < n4) store4_clip(a.d, seg, a.ldd, k, a.D, f4_zero());
    }
  }
};

template <int VEC, bool EV>
rnn_status launch_src_rs(const SrcArgs& a, const RSCtx& cx, cudaStream_t st) {
  BwdRS<VEC, EV> pol;
  pol.a = a;
  pol.n4e = a.edge.p ? (a.edge.dim + 3) / 4 : 0;
  return launch_rowsplit<BwdRS<VEC, EV>, VEC>(pol, cx, st);
}

// metadata of the lean kernel: idx = group of the position, c = w_p (/|g| for MEAN)
struct LeanBwdMeta {
  const int32_t* src_group;
  const int32_t* src_pos;
  const int32_t* edge_row;
  const int64_t* group_ptr;
  const float* w;  // scalar edge weight (nullptr: 1)
  int64_t ldw;
  int w_by_pos;
  int mean;
  struct Meta { int idx; float c; };
  __device__ __forceinline__ Meta meta(int64_t q, int) const {
    Meta m{src_group[q], 1.f};
    if (w) {
      const int p = src_pos[q];
      m.c = __ldg(w + (w_by_pos ? (int64_t)p : (int64_t)edge_row[p]) * ldw);
    }
    if (mean) m.c *= 1.f / (float)(group_ptr[m.idx + 1] - group_ptr[m.idx]);
    return m;
  }
};

rnn_status dispatch_src_rs(const SrcArgs& a, const RSCtx& cx, cudaStream_t st) {
  const int lc = lane_config(a.D);
  const bool ev = a.edge.p && a.edge.dim > 1;
  if (!ev && a.D == 4 * lc && a.ldd % 4 == 0 && a.ldy % 4 == 0) {
    LeanBwdMeta mp{a.src_group, a.src_pos, a.edge_row, a.group_ptr, a.edge.p, a.edge.ld,
                   a.edge.mode, a.mean};
    LeanOut o{a.Y, a.ldy, a.d, a.ldd, 0.f};
    if (lc == 32) return launch_lean<LeanBwdMeta, 1>(mp, cx, o, st);
    if (lc == 64) return launch_lean<LeanBwdMeta, 2>(mp, cx, o, st);
    return launch_lean<LeanBwdMeta, 4>(mp, cx, o, st);
  }
  if (lc == 32) return ev ? launch_src_rs<1, true>(a, cx, st) : launch_src_rs<1, false>(a, cx, st);
  if (lc == 64) return ev ? launch_src_rs<2, true>(a, cx, st) : launch_src_rs<2, false>(a, cx, st);
  return ev ? launch_src_rs<4, true>(a, cx, st) : launch_src_rs<4, false>(a, cx, st);
}

// U[g] = dOut[g] (.) z_t[g]  (MUL with a group-side factor), ld = ldu
__global__ void mul_dst_kernel(const float* __restrict__ dO, int64_t ld_do, OpndD dst,
                               const int32_t* __restrict__ dst_row, int64_t G, int D,
                               float* __restrict__ Uo, int64_t ldu) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= G * D) return;
  const int64_t g = i / D;
  const int c = (int)(i % D);
  const int64_t t = dst.mode ? g : (int64_t)dst_row[g];
  const float z = dst.dim == 1 ? dst.p[t * dst.ld] : dst.p[t * dst.ld + c];
  Uo[g * ldu + c] = dO[g * ld_do + c] * z;
}

// ------------------------------------------------------------------------------------------
// group-major per-row edge gradients (no cross-row reduction => no partial states)
// ------------------------------------------------------------------------------------------
template <class L>
__global__ void __launch_bounds__(256) bwd_edge_kernel(LjaArgs a, const float* __restrict__ dO,
                                                       int64_t ld_do, float* __restrict__ d_edge,
                                                       int64_t ld_de, const int64_t* work_ptr,
                                                       int64_t n_work, int64_t n_groups) {
  const int64_t item = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (item >= n_work) return;
  const int lane = lane_id(), slot = L::slot();
  const int64_t b = work_ptr[item], e = work_ptr[item + 1];
  const bool has_src = a.src.p, has_dst = a.dst.p, scalar = a.edge.dim == 1;
  const int n4s = has_src ? (a.src.dim + 3) / 4 : 0, n4t = has_dst ? (a.dst.dim + 3) / 4 : 0;
  const int n4o = (a.D + 3) / 4;
  int64_t g = upper_bound_dev(a.group_ptr, 0, n_groups + 1, b) - 1;
  for (int64_t r = b; r < e; ++g) {
    const int64_t gb = a.group_ptr[g], ge = a.group_ptr[g + 1];
    const int64_t r1 = ge < e ? ge : e;
    const float cg = a.mean ? 1.f / (float)(ge - gb) : 1.f;
    const int64_t t = has_dst ? (a.dst.mode ? g : (int64_t)a.dst_row[g]) : 0;
    float4 dov[L::VEC], ztv[L::VEC];
#pragma unroll
    for (int v = 0; v < L::VEC; ++v) {
      const int k = L::col4(v);
      dov[v] = f4_scale(cg, load4(dO, g, ld_do, k, n4o));
      if (has_dst && a.combine == RNN_COMBINE_MUL) {
        if (a.dst.dim == 1) { float z = a.dst.p[t * a.dst.ld]; ztv[v] = make_float4(z, z, z, z); }
        else ztv[v] = load4(a.dst.p, t, a.dst.ld, k, n4t);
      } else {
        ztv[v] = make_float4(1.f, 1.f, 1.f, 1.f);
      }
    }
    for (int64_t p0 = r; p0 < r1; p0 += L::RPW) {
      const int64_t p = p0 + slot;
      const bool ok = p < r1;
      const int64_t er = ok ? (a.edge.mode ? p : (int64_t)a.edge_row[p]) : 0;
      const int64_t sr = (ok && has_src) ? (int64_t)a.src_row[p] : 0;
      float part = 0.f;
#pragma unroll
      for (int v = 0; v < L::VEC; ++v) {
        const int k = L::col4(v);
        float4 x;
        if (a.combine == RNN_COMBINE_ADD) {
          x = dov[v];
        } else {  // SRC or MUL: dOut (.) (product of the other operands)
          float4 zs = (ok && has_src) ? load4(a.src.p, sr, a.src.ld, k, n4s)
                                      : make_float4(1.f, 1.f, 1.f, 1.f);
          x = f4_mul(f4_mul(dov[v], zs), ztv[v]);
        }
        if (k >= n4o) x = f4_zero();
        const int c0 = 4 * k;  // exclude columns >= D (row padding)
        if (c0 + 1 >= a.D) x.y = 0.f;
        if (c0 + 2 >= a.D) x.z = 0.f;
        if (c0 + 3 >= a.D) x.w = 0.f;
        if (scalar) part += x.x + x.y + x.z + x.w;
        else if (ok && k < n4o) store4_clip(d_edge, er, ld_de, k, a.D, x);
      }
      if (scalar) {
        part = L::reduce_row(part);
        if (ok && L::sub() == 0) d_edge[er * ld_de] = part;
      }
    }
    r = r1;
  }
  (void)lane;
}

// d_dst[t] = cg * dOut[g] (.) A[g]   (MUL: A = sum_p z_s (.) z_e)   or   |g| cg dOut (ADD)
__global__ void bwd_dst_kernel(const float* __restrict__ dO, int64_t ld_do,
                               const float* __restrict__ A, int64_t lda, int adim, OpndD dst,
                               const int32_t* __restrict__ dst_row, const int64_t* group_ptr,
                               int64_t G, int D, int combine, int mean, float* __restrict__ dd,
                               int64_t ldd) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= G) return;
  const int lane = lane_id();
  const float n = (float)(group_ptr[g + 1] - group_ptr[g]);
  const float cg = mean ? (n > 0.f ? 1.f / n : 0.f) : 1.f;
  const int64_t t = dst.mode ? g : (int64_t)dst_row[g];
  float sum = 0.f;
  for (int c = lane; c < D; c += 32) {
    float x = cg * dO[g * ld_do + c];
    x = combine == RNN_COMBINE_MUL ? x * A[g * lda + (adim == 1 ? 0 : c)] : x * n;
    if (dst.dim == 1) sum += x;
    else dd[t * ldd + c] = x;
  }
  if (dst.dim == 1) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) sum += __shfl_xor_sync(FULL, sum, m);
    if (lane == 0) dd[t * ldd] = sum;
  }
}

// CONCAT: d_edge / d_dst blocks (per column), warp per group
__global__ void bwd_concat_kernel(LjaArgs a, const float* __restrict__ dO, int64_t ld_do,
                                  float* d_edge, int64_t ld_de, float* d_dst, int64_t ld_dd,
                                  int64_t G) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= G) return;
  const int lane = lane_id();
  const int ds = a.src.p ? a.src.dim : 0, de = a.edge.p ? a.edge.dim : 0;
  const int dt = a.dst.p ? a.dst.dim : 0;
  const int64_t b = a.group_ptr[g], e = a.group_ptr[g + 1];
  const float cg = a.mean ? 1.f / (float)(e - b) : 1.f;
  if (d_edge && de)
    for (int64_t p = b; p < e; ++p) {
      const int64_t er = a.edge.mode ? p : (int64_t)a.edge_row[p];
      for (int c = lane; c < de; c += 32) d_edge[er * ld_de + c] = cg * dO[g * ld_do + ds + c];
    }
  if (d_dst && dt) {
    const int64_t t = a.dst.mode ? g : (int64_t)a.dst_row[g];
    for (int c = lane; c < dt; c += 32)
      d_dst[t * ld_dd + c] = (float)(e - b) * cg * dO[g * ld_do + ds + de + c];
  }
}

// ------------------------------------------------------------------------------------------
// SOFTMAX backward
// ------------------------------------------------------------------------------------------
struct SmArgs {
  const int64_t* group_ptr;
  const int32_t* src_row;
  const int32_t* dst_row;
  const int32_t* src_group;
  const int32_t* src_pos;
  OpndD key, val, q;
  const float* out; int64_t ld_out;
  const float* lse;
  const float* dO; int64_t ld_do;
  float* AD;            // [E', 2h]: a then de
  float* dq; int64_t ld_dq;
  float* dv; int64_t ld_dv;
  float* dk; int64_t ld_dk;
  int heads, LH;
  float scale;
};

template <class L>
struct BwdSm1 {
  SmArgs a;
  static constexpr int U = 4;
  struct State { float4 dq; };
  __device__ __forceinline__ float head_sum(float x) const {
    for (int m = 1; m < a.LH; m <<= 1) x += __shfl_xor_sync(FULL, x, m);
    return x;
  }
  __device__ __forceinline__ void init(State& s, int64_t) const { s.dq = f4_zero(); }
  __device__ __forceinline__ void rows(State& s, int64_t g, int64_t r0, int64_t r1) const {
    const int lane = lane_id(), slot = L::slot(), k = L::sub(), head = k / a.LH;
    const int64_t t = a.q.mode ? g : (int64_t)a.dst_row[g];
    const float4 q = ld_f4(a.q.p + t * a.q.ld + 4 * k);
    const float4 dO = ld_f4(a.dO + g * a.ld_do + 4 * k);
    const float Dh = head_sum(f4_dot(dO, ld_f4(a.out + g * a.ld_out + 4 * k)));
    const float lse2 = a.lse[g * a.heads + head] * LOG2E;
    const float sl2 = a.scale * LOG2E;
    for (int64_t base = r0; base < r1; base += 32) {
      const int P = (int)((r1 - base) < 32 ? (r1 - base) : 32);
      const int ms = lane < P ? a.src_row[base + lane] : 0;
      const int nk = (P + L::RPW - 1) / L::RPW;
      for (int k0 = 0; k0 < nk; k0 += U) {
        float4 kv[U], vv[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int li = (k0 + u) * L::RPW + slot;
          ok[u] = li < P;
          const int s_ = __shfl_sync(FULL, ms, li & 31);
          kv[u] = ok[u] ? ld_f4(a.key.p + (int64_t)s_ * a.key.ld + 4 * k) : f4_zero();
          vv[u] = ok[u] ? ld_f4(a.val.p + (int64_t)s_ * a.val.ld + 4 * k) : f4_zero();
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float sc = head_sum(f4_dot(kv[u], q));
          const float da = head_sum(f4_dot(dO, vv[u]));
          if (!ok[u]) continue;
          const float pa = exp2f(sc * sl2 - lse2);
          const float de = pa * (da - Dh);
          s.dq = f4_fma(de, kv[u], s.dq);
          if (k % a.LH == 0) {
            const int64_t p = base + (k0 + u) * L::RPW + slot;
            a.AD[p * 2 * a.heads + head] = pa;
            a.AD[p * 2 * a.heads + a.heads + head] = de;
          }
        }
      }
    }
    if (L::RPW > 1) s.dq = L::reduce_slots(s.dq);
  }
  __device__ __forceinline__ void finish(State& s, int64_t g) const {
    if (!a.dq || L::slot() != 0) return;
    const int k = L::sub();
    const int64_t t = a.q.mode ? g : (int64_t)a.dst_row[g];
    st_f4(a.dq + t * a.ld_dq + 4 * k, f4_scale(a.scale, s.dq));
  }
  __device__ __forceinline__ void save(const State& s, float* dst) const {
    if (L::slot() == 0) __stcg(reinterpret_cast<float4*>(dst + 4 * L::sub()), s.dq);
  }
  __device__ __forceinline__ void merge(State& s, const float* src) const {
    s.dq = f4_add(s.dq, ld_f4_cg(src + 4 * L::sub()));
  }
};

template <class L>
struct BwdSm2 {
  SmArgs a;
  static constexpr int U = 4;
  struct State { float4 dv, dk; };
  __device__ __forceinline__ void init(State& s, int64_t) const { s.dv = f4_zero(); s.dk = f4_zero(); }
  __device__ __forceinline__ void rows(State& s, int64_t, int64_t r0, int64_t r1) const {
    const int lane = lane_id(), slot = L::slot(), k = L::sub(), head = k / a.LH;
    for (int64_t base = r0; base < r1; base += 32) {
      const int P = (int)((r1 - base) < 32 ? (r1 - base) : 32);
      int mg = 0, mp = 0, mt = 0;
      if (lane < P) {
        mg = a.src_group[base + lane];
        mp = a.src_pos[base + lane];
        mt = a.q.mode ? mg : a.dst_row[mg];
      }
      const int nk = (P + L::RPW - 1) / L::RPW;
      for (int k0 = 0; k0 < nk; k0 += U) {
        float4 dov[U], qv[U];
        float av[U], dev[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int li = (k0 + u) * L::RPW + slot;
          ok[u] = li < P;
          const int g_ = __shfl_sync(FULL, mg, li & 31);
          const int p_ = __shfl_sync(FULL, mp, li & 31);
          const int t_ = __shfl_sync(FULL, mt, li & 31);
          dov[u] = ok[u] ? ld_f4(a.dO + (int64_t)g_ * a.ld_do + 4 * k) : f4_zero();
          qv[u] = ok[u] ? ld_f4(a.q.p + (int64_t)t_ * a.q.ld + 4 * k) : f4_zero();
          av[u] = ok[u] ? a.AD[(int64_t)p_ * 2 * a.heads + head] : 0.f;
          dev[u] = ok[u] ? a.AD[(int64_t)p_ * 2 * a.heads + a.heads + head] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          s.dv = f4_fma(av[u], dov[u], s.dv);
          s.dk = f4_fma(dev[u], qv[u], s.dk);
        }
      }
    }
    if (L::RPW > 1) { s.dv = L::reduce_slots(s.dv); s.dk = L::reduce_slots(s.dk); }
  }
  __device__ __forceinline__ void finish(State& s, int64_t seg) const {
    if (L::slot() != 0) return;
    const int k = L::sub();
    if (a.dv) st_f4(a.dv + seg * a.ld_dv + 4 * k, s.dv);
    if (a.dk) st_f4(a.dk + seg * a.ld_dk + 4 * k, f4_scale(a.scale, s.dk));
  }
  __device__ __forceinline__ void save(const State& s, float* dst) const {
    if (L::slot() != 0) return;
    __stcg(reinterpret_cast<float4*>(dst + 4 * L::sub()), s.dv);
    __stcg(reinterpret_cast<float4*>(dst + 4 * L::LPR + 4 * L::sub()), s.dk);
  }
  __device__ __forceinline__ void merge(State& s, const float* src) const {
    s.dv = f4_add(s.dv, ld_f4_cg(src + 4 * L::sub()));
    s.dk = f4_add(s.dk, ld_f4_cg(src + 4 * L::LPR + 4 * L::sub()));
  }
};

template <class Pol>
rnn_status launch_seg(const Pol& pol, const SegCtx& cx, cudaStream_t st) {
  if (cx.n_work <= 0) return RNN_OK;
  RNN_CUDA(cudaMemsetAsync(cx.counter, 0, sizeof(int) * cx.n_work, st));
  seg_kernel<Pol><<<(unsigned)ceil_div(cx.n_work, 8), 256, 0, st>>>(pol, cx);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

template <class L>
rnn_status launch_src(const SrcArgs& a, const SegCtx& cx, cudaStream_t st) {
  BwdSrc<L> pol;
  pol.a = a;
  return launch_seg(pol, cx, st);
}

rnn_status dispatch_src(const SrcArgs& a, const SegCtx& cx, cudaStream_t st) {
  switch (lane_config(a.D)) {
    case 1: return launch_src<Lanes<1, 1>>(a, cx, st);
    case 2: return launch_src<Lanes<2, 1>>(a, cx, st);
    case 4: return launch_src<Lanes<4, 1>>(a, cx, st);
    case 8: return launch_src<Lanes<8, 1>>(a, cx, st);
    case 16: return launch_src<Lanes<16, 1>>(a, cx, st);
    case 32: return launch_src<Lanes<32, 1>>(a, cx, st);
    case 64: return launch_src<Lanes<32, 2>>(a, cx, st);
    case 128: return launch_src<Lanes<32, 4>>(a, cx, st);
  }
  RNN_FAIL(RNN_ERR_UNSUPPORTED, "width %d", a.D);
}

template <class L>
rnn_status launch_edge(const LjaArgs& a, const float* dO, int64_t ld_do, float* d_edge,
                       int64_t ld_de, const rnn_join_index* idx, cudaStream_t st) {
  if (idx->n_work <= 0) return RNN_OK;
  bwd_edge_kernel<L><<<(unsigned)ceil_div(idx->n_work, 8), 256, 0, st>>>(
      a, dO, ld_do, d_edge, ld_de, idx->work_ptr, idx->n_work, idx->n_groups);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

rnn_status dispatch_edge(const LjaArgs& a, const float* dO, int64_t ld_do, float* d_edge,
                         int64_t ld_de, const rnn_join_index* idx, cudaStream_t st) {
  switch (lane_config(a.D)) {
    case 1: return launch_edge<Lanes<1, 1>>(a, dO, ld_do, d_edge, ld_de, idx, st);
    case 2: return launch_edge<Lanes<2, 1>>(a, dO, ld_do, d_edge, ld_de, idx, st);
    case 4: return launch_edge<Lanes<4, 1>>(a, dO, ld_do, d_edge, ld_de, idx, st);
    case 8: return launch_edge<Lanes<8, 1>>(a, dO, ld_do, d_edge, ld_de, idx, st);
    case 16: return launch_edge<Lanes<16, 1>>(a, dO, ld_do, d_edge, ld_de, idx, st);
    case 32: return launch_edge<Lanes<32, 1>>(a, dO, ld_do, d_edge, ld_de, idx, st);
    case 64: return launch_edge<Lanes<32, 2>>(a, dO, ld_do, d_edge, ld_de, idx, st);
    case 128: return launch_edge<Lanes<32, 4>>(a, dO, ld_do, d_edge, ld_de, idx, st);
  }
  RNN_FAIL(RNN_ERR_UNSUPPORTED, "width %d", a.D);
}

template <class L>
rnn_status launch_sm(const SmArgs& a, const rnn_join_index* idx, float* part1, int* cnt1,
                     float* part2, int* cnt2, cudaStream_t st) {
  BwdSm1<L> p1;
  p1.a = a;
  SegCtx c1{idx->group_ptr, idx->n_groups, idx->work_ptr, idx->n_work, part1, 4 * L::LPR, cnt1};
  RNN_TRY(launch_seg(p1, c1, st));
  if (a.dv || a.dk) {
    BwdSm2<L> p2;
    p2.a = a;
    SegCtx c2{idx->src_ptr, idx->n_src_rows, idx->src_work_ptr, idx->n_src_work, part2,
              8 * L::LPR, cnt2};
    RNN_TRY(launch_seg(p2, c2, st));
  }
  return RNN_OK;
}

struct BwdLayout {
  float* part_src; int* cnt_src;   // transposed pass partials  [n_src_work, pstride]
  float* Ubuf;                     // [G, ld4] (MUL with dst: U; MUL d_dst: A)
  float* part_fwd; int* cnt_fwd;   // forward recompute partials / softmax pass 1
  float* AD;                       // [E', 2h]
  size_t bytes;
};

BwdLayout bwd_layout(const rnn_join_index* idx, const rnn_lifted_query* q, const QueryInfo& qi,
                     void* ws) {
  Carve c(ws);
  BwdLayout L{};
  const int64_t ld4 = (qi.D + 3) / 4 * 4;
  const int64_t ps = q->agg == RNN_AGG_SOFTMAX ? 2 * ld4 : flat_pstride(qi.D);
  L.part_src = c.take<float>((size_t)idx->n_src_work * ps);
  L.cnt_src = c.take<int>((size_t)idx->n_src_work);
  L.Ubuf = c.take<float>((size_t)idx->n_groups * ld4);
  L.part_fwd = c.take<float>((size_t)idx->n_work * qi.pstride);
  L.cnt_fwd = c.take<int>((size_t)idx->n_work);
  if (q->agg == RNN_AGG_SOFTMAX) L.AD = c.take<float>((size_t)idx->n_join_rows * 2 * q->heads);
  L.bytes = c.used + 512;
  return L;
}

// ------------------------------------------------------------------------------------------
// standalone grouped softmax: one warp per group, lanes stride over the group's rows
// ------------------------------------------------------------------------------------------
__global__ void group_softmax_kernel(const int64_t* __restrict__ gp, int64_t G,
                                     const float* __restrict__ s, int heads, float* __restrict__ p) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= G) return;
  const int lane = lane_id();
  const int64_t b = gp[g], e = gp[g + 1];
  for (int h = 0; h < heads; ++h) {
    float m = -INFINITY;
    for (int64_t r = b + lane; r < e; r += 32) m = fmaxf(m, s[r * heads + h]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
    float z = 0.f;
    for (int64_t r = b + lane; r < e; r += 32) z += __expf(s[r * heads + h] - m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(FULL, z, o);
    const float inv = 1.f / z;
    for (int64_t r = b + lane; r < e; r += 32) p[r * heads + h] = __expf(s[r * heads + h] - m) * inv;
  }
}

__global__ void group_softmax_bwd_kernel(const int64_t* __restrict__ gp, int64_t G,
                                         const float* __restrict__ p, const float* __restrict__ dp,
                                         int heads, float* __restrict__ ds) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= G) return;
  const int lane = lane_id();
  const int64_t b = gp[g], e = gp[g + 1];
  for (int h = 0; h < heads; ++h) {
    float dot = 0.f;
    for (int64_t r = b + lane; r < e; r += 32) dot += p[r * heads + h] * dp[r * heads + h];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(FULL, dot, o);
    for (int64_t r = b + lane; r < e; r += 32)
      ds[r * heads + h] = p[r * heads + h] * (dp[r * heads + h] - dot);
  }
}

}  // namespace

rnn_status lja_bwd_ws(const rnn_join_index* idx, const rnn_lifted_query* q, size_t* b) {
  QueryInfo qi;
  RNN_TRY(check_query(idx, q, &qi));
  *b = bwd_layout(idx, q, qi, nullptr).bytes;
  return RNN_OK;
}

}  // namespace rnn

using namespace rnn;

extern "C" rnn_status rnn_lja_workspace_size(const rnn_join_index* idx, const rnn_lifted_query* q,
                                             size_t* fwd_bytes, size_t* bwd_bytes) {
  clear_error();
  RNN_REQUIRE(fwd_bytes || bwd_bytes, RNN_ERR_INVALID_ARGUMENT, "no output");
  if (fwd_bytes) RNN_TRY(lja_fwd_ws(idx, q, fwd_bytes));
  if (bwd_bytes) RNN_TRY(lja_bwd_ws(idx, q, bwd_bytes));
  return RNN_OK;
}

static rnn_status lja_bwd_impl(const rnn_join_index* idx, const rnn_lifted_query* q,
                               const float* out, int64_t ld_out, const float* lse,
                               const float* d_out, int64_t ld_dout, float* d_src,
                               float* d_src_key, float* d_edge, float* d_dst, float beta_dst,
                               void* workspace, size_t workspace_bytes, void* stream) {
  QueryInfo qi;
  RNN_TRY(check_query(idx, q, &qi));
  cudaStream_t st = as_stream(stream);
  RNN_REQUIRE(d_out && ld_dout >= qi.D, RNN_ERR_INVALID_ARGUMENT, "d_out NULL or ld_dout < width");
  const bool vec_ok = ld_dout % 4 == 0 && aligned16(d_out);
  RNN_REQUIRE(qi.concat || vec_ok, RNN_ERR_INVALID_ARGUMENT,
              "d_out must be 16-byte aligned with ld_dout %% 4 == 0");
  if (!q->src.data) d_src = nullptr;
  if (!q->src_key.data) d_src_key = nullptr;
  if (!q->edge.data) d_edge = nullptr;
  if (!q->dst.data) d_dst = nullptr;
  const bool acc_dst = d_dst && beta_dst != 0.f;   // d_dst += (rows never referenced: + 0)
  RNN_REQUIRE(!acc_dst || idx->n_join_rows == 0 ||   // (an empty join adds nothing)
                  (q->agg == RNN_AGG_SOFTMAX && sm_rowsplit_ok(idx, q, qi.D) && idx->src_seg &&
                   !getenv("RNN_SM_TWOPASS")),
              RNN_ERR_UNSUPPORTED,
              "beta_dst = 1 needs the SOFTMAX source-major backward (d = 128, dim/heads in {4..32})");
  const bool need_t = d_src || d_src_key;
  RNN_REQUIRE(!need_t || idx->n_groups == 0 ||
                  (idx->src_ptr && idx->src_pos && idx->src_group && idx->src_work_ptr),
              RNN_ERR_INVALID_ARGUMENT, "source gradients need the transposed index");
  const BwdLayout Lw = bwd_layout(idx, q, qi, workspace);
  RNN_REQUIRE(workspace_bytes >= Lw.bytes && workspace, RNN_ERR_WORKSPACE_TOO_SMALL,
              "backward workspace %zu < %zu bytes", workspace_bytes, Lw.bytes);
  // rows never referenced by a join row get zero gradient
  const int64_t n_s = idx->n_src_rows;
  RNN_REQUIRE(!d_src || vec_ok, RNN_ERR_INVALID_ARGUMENT,
              "source gradients need d_out 16-byte aligned with ld_dout %% 4 == 0");
  // (2D memsets: a gradient buffer may be a column block of a wider matrix)
  auto zero2d = [&](float* p, int64_t ld, int dim, int64_t rows) -> rnn_status {
    if (rows > 0)
      RNN_CUDA(cudaMemset2DAsync(p, sizeof(float) * ld, 0, sizeof(float) * dim, rows, st));
    return RNN_OK;
  };
  if (d_src && idx->n_join_rows == 0) RNN_TRY(zero2d(d_src, q->src.ld, q->src.dim, n_s));
  if (d_src_key && idx->n_join_rows == 0)
    RNN_TRY(zero2d(d_src_key, q->src_key.ld, q->src_key.dim, n_s));
  if (d_edge && q->edge.mode == RNN_BY_ROW)
    RNN_TRY(zero2d(d_edge, q->edge.ld, q->edge.dim, idx->n_edge_rows));
  if (d_dst && !acc_dst && q->dst.mode == RNN_BY_ROW && idx->n_groups < idx->n_dst_rows)
    RNN_TRY(zero2d(d_dst, q->dst.ld, q->dst.dim, idx->n_dst_rows));
  if (idx->n_groups == 0) return RNN_OK;
  if (idx->n_join_rows == 0) {
    // dense groups over an empty join: every group-side gradient is 0 (no work items run)
    if (d_dst && !acc_dst)
      RNN_TRY(zero2d(d_dst, q->dst.ld, q->dst.dim,
                     q->dst.mode == RNN_BY_ROW ? idx->n_dst_rows : idx->n_groups));
    return RNN_OK;
  }
  LjaArgs a = make_args(idx, q, nullptr, 0, 0.f, nullptr, qi.D);
  const int64_t ld4 = (qi.D + 3) / 4 * 4;

  if (q->agg == RNN_AGG_SOFTMAX) {
    RNN_REQUIRE(out && lse && ld_out % 4 == 0 && aligned16(out), RNN_ERR_INVALID_ARGUMENT,
                "SOFTMAX backward needs the forward's out (aligned) and lse");
    SmArgs s{};
    s.group_ptr = idx->group_ptr; s.src_row = idx->src_row; s.dst_row = idx->group_dst_row;
    s.src_group = idx->src_group; s.src_pos = idx->src_pos;
    s.key = opnd(q->src_key); s.val = opnd(q->src); s.q = opnd(q->dst);
    s.out = out; s.ld_out = ld_out; s.lse = lse; s.dO = d_out; s.ld_do = ld_dout;
    s.AD = Lw.AD;
    s.dq = d_dst; s.ld_dq = q->dst.ld;
    s.dv = d_src; s.ld_dv = q->src.ld;
    s.dk = d_src_key; s.ld_dk = q->src_key.ld;
    s.heads = q->heads; s.scale = q->scale;
    static const bool two_pass = getenv("RNN_SM_TWOPASS") != nullptr;
    if (sm_rowsplit_ok(idx, q, qi.D) && idx->src_seg && !two_pass) {
      // source-major backward: D, pass A (dM', dK', DE), pass B (dQ)
      const SmRows rows = sm_rows(idx, q);
      float* Dg = Lw.Ubuf;     // [G, h] <= [G, ld4]
      float* DE = Lw.AD;       // [E', h] <= [E', 2h]
      sm_d_kernel<<<(unsigned)ceil_div(idx->n_groups, 8), 256, 0, st>>>(
          d_out, ld_dout, out, ld_out, idx->n_groups, q->heads, rows.LH, Dg);
      RNN_LAUNCH_CHECK();
      SmBwdAPol pa;
      pa.a = rows;
      pa.dO = d_out; pa.ld_do = ld_dout; pa.lse = lse; pa.Dg = Dg; pa.DE = DE;
      pa.dv = d_src; pa.ld_dv = q->src.ld; pa.dk = d_src_key; pa.ld_dk = q->src_key.ld;
      RSCtx c2{idx->src_seg, idx->src_ptr, idx->n_src_rows, idx->n_join_rows,
               idx->src_work_ptr, idx->n_src_work, Lw.part_src, 2 * ld4, Lw.cnt_src, 1};
      RNN_TRY(launch_st_var(pa, c2, st, 1));
      if (d_dst) {
        SmBwdBPol pb;
        pb.a = rows;
        pb.DE = DE; pb.dq = d_dst; pb.ld_dq = q->dst.ld;
        pb.beta = acc_dst ? 1.f : 0.f;
        RSCtx c1{idx->pos_group, idx->group_ptr, idx->n_groups, idx->n_join_rows, idx->work_ptr,
                 idx->n_work, Lw.part_fwd, qi.pstride, Lw.cnt_fwd, 1};
        RNN_TRY(launch_st_var(pb, c1, st, 2));
      }
      return RNN_OK;
    }
    if (sm_rowsplit_ok(idx, q, qi.D) && idx->src_seg) {
      SmBwd1Pol p1;
      p1.a = sm_rows(idx, q);
      p1.out = out; p1.ld_out = ld_out; p1.lse = lse; p1.dO = d_out; p1.ld_do = ld_dout;
      p1.AD = Lw.AD; p1.dq = d_dst; p1.ld_dq = q->dst.ld;
      RSCtx c1{idx->pos_group, idx->group_ptr, idx->n_groups, idx->n_join_rows, idx->work_ptr,
               idx->n_work, Lw.part_fwd, qi.pstride, Lw.cnt_fwd, 1};
      RNN_TRY(launch_st_var(p1, c1, st, 1));
      if (d_src || d_src_key) {
        SmBwd2Pol p2;
        p2.a = p1.a;
        p2.dO = d_out; p2.ld_do = ld_dout; p2.AD = Lw.AD;
        p2.dv = d_src; p2.ld_dv = q->src.ld; p2.dk = d_src_key; p2.ld_dk = q->src_key.ld;
        RSCtx c2{idx->src_seg, idx->src_ptr, idx->n_src_rows, idx->n_join_rows,
                 idx->src_work_ptr, idx->n_src_work, Lw.part_src, 2 * ld4, Lw.cnt_src, 1};
        RNN_TRY(launch_st_var(p2, c2, st, 2));
      }
      return RNN_OK;
    }
    const int LPR = qi.D / 4;
    s.LH = LPR / q->heads;
    switch (LPR) {
      case 1: return launch_sm<Lanes<1, 1>>(s, idx, Lw.part_fwd, Lw.cnt_fwd, Lw.part_src, Lw.cnt_src, st);
      case 2: return launch_sm<Lanes<2, 1>>(s, idx, Lw.part_fwd, Lw.cnt_fwd, Lw.part_src, Lw.cnt_src, st);
      case 4: return launch_sm<Lanes<4, 1>>(s, idx, Lw.part_fwd, Lw.cnt_fwd, Lw.part_src, Lw.cnt_src, st);
      case 8: return launch_sm<Lanes<8, 1>>(s, idx, Lw.part_fwd, Lw.cnt_fwd, Lw.part_src, Lw.cnt_src, st);
      case 16: return launch_sm<Lanes<16, 1>>(s, idx, Lw.part_fwd, Lw.cnt_fwd, Lw.part_src, Lw.cnt_src, st);
      case 32: return launch_sm<Lanes<32, 1>>(s, idx, Lw.part_fwd, Lw.cnt_fwd, Lw.part_src, Lw.cnt_src, st);
    }
    RNN_FAIL(RNN_ERR_UNSUPPORTED, "SOFTMAX width %d", qi.D);
  }

  // ---- d_src: transposed gather ----
  if (d_src) {
    RNN_REQUIRE(q->src.ld % 4 == 0 && aligned16(d_src), RNN_ERR_INVALID_ARGUMENT,
                "d_src must be 16-byte aligned");
    SrcArgs s{};
    s.src_group = idx->src_group; s.src_pos = idx->src_pos; s.edge_row = idx->edge_row;
    s.group_ptr = idx->group_ptr;
    s.Y = d_out; s.ldy = ld_dout;
    s.edge = OpndD{nullptr, 0, 0, 0};
    s.mean = q->agg == RNN_AGG_MEAN;
    s.d = d_src; s.ldd = q->src.ld; s.D = q->src.dim;
    s.n4y = (s.D + 3) / 4;
    if (q->combine == RNN_COMBINE_SRC || q->combine == RNN_COMBINE_MUL) s.edge = opnd(q->edge);
    if (q->combine == RNN_COMBINE_MUL && q->dst.data) {
      const int64_t G = idx->n_groups;
      mul_dst_kernel<<<(unsigned)ceil_div(G * qi.D, 256), 256, 0, st>>>(
          d_out, ld_dout, opnd(q->dst), idx->group_dst_row, G, qi.D, Lw.Ubuf, ld4);
      RNN_LAUNCH_CHECK();
      s.Y = Lw.Ubuf; s.ldy = ld4;
    }
    if (q->combine == RNN_COMBINE_CONCAT) s.edge = OpndD{nullptr, 0, 0, 0};
    SegCtx cx{idx->src_ptr, n_s, idx->src_work_ptr, idx->n_src_work, Lw.part_src,
              flat_pstride(s.D), Lw.cnt_src};
    if (lane_config(s.D) >= 32 && idx->src_seg) {
      RSCtx rx{idx->src_seg, idx->src_ptr, n_s, idx->n_join_rows, idx->src_work_ptr,
               idx->n_src_work, Lw.part_src, flat_pstride(s.D), Lw.cnt_src, 1};
      RNN_TRY(dispatch_src_rs(s, rx, st));
    } else {
      RNN_TRY(dispatch_src(s, cx, st));
    }
  }
  if (q->combine == RNN_COMBINE_CONCAT) {
    if (d_edge || d_dst) {
      bwd_concat_kernel<<<(unsigned)ceil_div(idx->n_groups, 8), 256, 0, st>>>(
          a, d_out, ld_dout, d_edge, q->edge.ld, d_dst, q->dst.ld, idx->n_groups);
      RNN_LAUNCH_CHECK();
    }
    return RNN_OK;
  }
  // ---- d_edge: group-major per row ----
  if (d_edge) {
    if (q->edge.dim != 1)
      RNN_REQUIRE(q->edge.ld % 4 == 0 && aligned16(d_edge), RNN_ERR_INVALID_ARGUMENT,
                  "d_edge must be 16-byte aligned");
    RNN_TRY(dispatch_edge(a, d_out, ld_dout, d_edge, q->edge.ld, idx, st));
  }
  // ---- d_dst ----
  if (d_dst) {
    const float* A = nullptr;
    int a_dim = qi.D;
    if (q->combine == RNN_COMBINE_MUL) {
      // A[g] = sum_p z_s (.) z_e : the forward without the group-side factor, un-normalised
      rnn_lifted_query qa = *q;
      qa.dst = rnn_operand{nullptr, 0, 0, 0};
      qa.agg = RNN_AGG_SUM;
      if (!qa.src.data && !qa.edge.data) {
        qa.combine = RNN_COMBINE_MUL;
      }
      if (qa.src.data || qa.edge.data) {
        size_t need = 0;
        RNN_TRY(lja_fwd_ws(idx, &qa, &need));
        QueryInfo qai;
        RNN_TRY(check_query(idx, &qa, &qai));
        a_dim = qai.D;
        RNN_TRY(lja_fwd_impl(idx, &qa, Lw.Ubuf, ld4, 0.f, nullptr, Lw.part_fwd,
                             need, st));
        A = Lw.Ubuf;
      } else {
        // no src / edge: A = |g| * ones
        A = nullptr;
      }
    }
    if (q->combine == RNN_COMBINE_MUL && !A) {
      // d_dst = cg * dOut * |g|  (same as ADD)
      bwd_dst_kernel<<<(unsigned)ceil_div(idx->n_groups, 8), 256, 0, st>>>(
          d_out, ld_dout, nullptr, 0, 0, opnd(q->dst), idx->group_dst_row, idx->group_ptr,
          idx->n_groups, qi.D, RNN_COMBINE_ADD, a.mean, d_dst, q->dst.ld);
    } else {
      bwd_dst_kernel<<<(unsigned)ceil_div(idx->n_groups, 8), 256, 0, st>>>(
          d_out, ld_dout, A, ld4, a_dim, opnd(q->dst), idx->group_dst_row, idx->group_ptr,
          idx->n_groups, qi.D, q->combine, a.mean, d_dst, q->dst.ld);
    }
    RNN_LAUNCH_CHECK();
  }
  return RNN_OK;
}

extern "C" rnn_status rnn_group_softmax(const rnn_join_index* idx, const float* scores,
                                        int32_t heads, float* probs, void* stream) {
  clear_error();
  RNN_REQUIRE(idx && idx->group_ptr && scores && probs && heads >= 1, RNN_ERR_INVALID_ARGUMENT,
              "bad argument");
  if (idx->n_groups == 0) return RNN_OK;
  group_softmax_kernel<<<(unsigned)ceil_div(idx->n_groups, 8), 256, 0, as_stream(stream)>>>(
      idx->group_ptr, idx->n_groups, scores, heads, probs);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

extern "C" rnn_status rnn_group_softmax_bwd(const rnn_join_index* idx, const float* probs,
                                            const float* d_probs, int32_t heads, float* d_scores,
                                            void* stream) {
  clear_error();
  RNN_REQUIRE(idx && idx->group_ptr && probs && d_probs && d_scores && heads >= 1,
              RNN_ERR_INVALID_ARGUMENT, "bad argument");
  if (idx->n_groups == 0) return RNN_OK;
  group_softmax_bwd_kernel<<<(unsigned)ceil_div(idx->n_groups, 8), 256, 0, as_stream(stream)>>>(
      idx->group_ptr, idx->n_groups, probs, d_probs, heads, d_scores);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

extern "C" rnn_status rnn_join_aggregate_bwd(const rnn_join_index* idx, const rnn_lifted_query* q,
                                             const float* out, int64_t ld_out, const float* lse,
                                             const float* d_out, int64_t ld_dout, float* d_src,
                                             float* d_src_key, float* d_edge, float* d_dst,
                                             void* workspace, size_t workspace_bytes,
                                             void* stream) {
  rnn::clear_error();
  return lja_bwd_impl(idx, q, out, ld_out, lse, d_out, ld_dout, d_src, d_src_key, d_edge,
                           d_dst, 0.f, workspace, workspace_bytes, stream);
}

extern "C" rnn_status rnn_join_aggregate_bwd_acc(const rnn_join_index* idx,
                                                 const rnn_lifted_query* q, const float* out,
                                                 int64_t ld_out, const float* lse,
                                                 const float* d_out, int64_t ld_dout,
                                                 float* d_src, float* d_src_key, float* d_edge,
                                                 float* d_dst, float beta_dst, void* workspace,
                                                 size_t workspace_bytes, void* stream) {
  rnn::clear_error();
  RNN_REQUIRE(beta_dst == 0.f || beta_dst == 1.f, RNN_ERR_INVALID_ARGUMENT,
              "beta_dst must be 0 or 1");
  return lja_bwd_impl(idx, q, out, ld_out, lse, d_out, ld_dout, d_src, d_src_key, d_edge,
                           d_dst, beta_dst, workspace, workspace_bytes, stream);
}
