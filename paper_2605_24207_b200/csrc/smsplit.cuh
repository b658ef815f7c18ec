// smsplit.cuh -- row-split walker with an arbitrary per-segment state, and the softmax-
// weighted aggregate (HGT attention, Fig. 4) on top of it.
//
// Same schedule and metadata as rowsplit.cuh (one warp per work item of a key-grouped CSR,
// a segment id per position, segment ends as a ballot bitmask, U rows of gathers in flight),
// but the per-segment state is a policy type: the online softmax carries (running max,
// running sum, weighted accumulator) per head, the backward passes carry one or two float4
// accumulators.  Rows of one 128-float embedding map one float4 per lane; a head of dh
// floats is LH = dh / 4 consecutive lanes, so head dot products are LH-lane shuffle trees.
// Split hubs follow rowsplit.cuh: pieces save their state, the last ticket merges them in
// item order (deterministic, no float atomics).
#pragma once
#include "rowsplit.cuh"

namespace rnn {

// Pol:
//   struct Meta; struct Row; struct State;
//   Meta meta(int64_t pos, int seg) const;    Meta shfl(const Meta&, int lane) const;
//   void load(Row&, const Meta&, bool ok) const;  void prep(Row&) const  (warp-converged)
//   void row(State&, const Row&, int64_t pos) const;
//   void init(State&) const;  void finish(const State&, int64_t seg) const;
//   void zero(int64_t seg) const;  (empty segment)
//   void save(const State&, float* dst) const;  void merge(State&, const float* src) const;
template <class Pol>
__device__ __noinline__ void st_piece(const Pol& pol, const RSCtx& cx, int64_t item, int64_t g,
                                      typename Pol::State st) {
  const int lane = lane_id();
  pol.save(st, cx.partial + item * cx.pstride);
  __threadfence();
  __syncwarp();
  int64_t i0 = 0, i1 = 0;
  int last = 0;
  if (lane == 0) {
    i0 = lower_bound_dev(cx.work_ptr, 0, cx.n_work + 1, cx.ptr[g]);
    i1 = lower_bound_dev(cx.work_ptr, 0, cx.n_work + 1, cx.ptr[g + 1]);
    last = atomicAdd(&cx.counter[i0], 1) == (int)(i1 - i0 - 1);
  }
  last = __shfl_sync(FULL, last, 0);
  if (!last) return;
  i0 = __shfl_sync(FULL, i0, 0);
  i1 = __shfl_sync(FULL, i1, 0);
  __threadfence();
  pol.init(st);
  for (int64_t i = i0; i < i1; ++i) pol.merge(st, cx.partial + i * cx.pstride);
  pol.finish(st, g);
}

template <class Pol>
__device__ __noinline__ void st_zero_range(const Pol& pol, int64_t g0, int64_t g1) {
  for (int64_t g = g0; g < g1; ++g) pol.zero(g);
}

template <class Pol, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) st_kernel(Pol pol, RSCtx cx) {
  const int64_t item = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (item >= cx.n_work) return;
  const int lane = lane_id();
  const int64_t b = cx.work_ptr[item], e = cx.work_ptr[item + 1];
  bool head_piece = b > 0 && cx.seg[b - 1] == cx.seg[b];
  typename Pol::State st;
  pol.init(st);
  bool pending = false;
  int g_tail = -1;
  for (int64_t r0 = b; r0 < e; r0 += 32) {
    const int P = (int)((e - r0) < 32 ? (e - r0) : 32);
    typename Pol::Meta m{};
    int gl = -1;
    bool endf = false;
    if (lane < P) {
      const int64_t r = r0 + lane;
      gl = cx.seg[r];
      m = pol.meta(r, gl);
      endf = r + 1 >= cx.E || cx.seg[r + 1] != gl;
    }
    if (cx.zero_empty) {
      const int gprev = lane < P ? (r0 + lane > 0 ? cx.seg[r0 + lane - 1] : -1) : 0;
      unsigned gaps = __ballot_sync(FULL, lane < P && gl > gprev + 1);
      while (gaps) {
        const int j = __ffs(gaps) - 1;
        gaps &= gaps - 1;
        st_zero_range(pol, __shfl_sync(FULL, gprev, j) + 1, __shfl_sync(FULL, gl, j));
      }
    }
    const unsigned ends = __ballot_sync(FULL, endf);
    for (int j0 = 0; j0 < P; j0 += U) {
      typename Pol::Row rw[U];
#pragma unroll
      for (int u = 0; u < U; ++u) pol.load(rw[u], pol.shfl(m, (j0 + u) & 31), j0 + u < P);
#pragma unroll
      for (int u = 0; u < U; ++u) pol.prep(rw[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + u;
        if (j < P) {
          pol.row(st, rw[u], r0 + j);
          pending = true;
          if ((ends >> j) & 1u) {
            const int g = __shfl_sync(FULL, gl, j);
            if (head_piece) st_piece(pol, cx, item, g, st);
            else pol.finish(st, g);
            head_piece = false;
            pending = false;
            pol.init(st);
          }
        }
      }
    }
    g_tail = __shfl_sync(FULL, gl, P - 1);
  }
  if (pending) st_piece(pol, cx, item, g_tail, st);
  if (cx.zero_empty && item == cx.n_work - 1)
    st_zero_range(pol, cx.E > 0 ? cx.seg[cx.E - 1] + 1 : 0, cx.n_seg);
}

template <class Pol, int U, int MINB = 1>
rnn_status launch_st(const Pol& pol, RSCtx cx, cudaStream_t st) {
  if (cx.n_work <= 0) return RNN_OK;
  RNN_CUDA(cudaMemsetAsync(cx.counter, 0, sizeof(int) * cx.n_work, st));
  st_kernel<Pol, U, MINB><<<(unsigned)ceil_div(cx.n_work, 8), 256, 0, st>>>(pol, cx);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

// (rows in flight U, min CTAs per SM) of the three softmax walkers; RNN_ST_VAR="fU,fB,aU,aB,bU,bB"
// selects another instantiated variant (measurement only)
struct StVar { int u[3], b[3]; };
inline StVar st_var() {
  static StVar v = [] {
    // measured best on MAG (profiles/r01/st_var, sm_src; round 2 profiles/r02/stvar: pass B
    // at 2 rows x 6 CTAs/SM, lja_bwd 2.69 -> 2.59 ms per relation, step 20.34 -> 19.96 ms)
    StVar r{{4, 1, 2}, {3, 4, 6}};
    if (const char* e = getenv("RNN_ST_VAR"))
      sscanf(e, "%d,%d,%d,%d,%d,%d", &r.u[0], &r.b[0], &r.u[1], &r.b[1], &r.u[2], &r.b[2]);
    return r;
  }();
  return v;
}
template <class Pol>
rnn_status launch_st_var(const Pol& pol, RSCtx cx, cudaStream_t st, int which) {
  const StVar v = st_var();
  const int U = v.u[which], B = v.b[which];
  if (U == 2 && B == 3) return launch_st<Pol, 2, 3>(pol, cx, st);
  if (U == 6 && B == 2) return launch_st<Pol, 6, 2>(pol, cx, st);
  if (U == 1 && B == 4) return launch_st<Pol, 1, 4>(pol, cx, st);
  if (U == 2 && B == 4) return launch_st<Pol, 2, 4>(pol, cx, st);
  if (U == 3 && B == 4) return launch_st<Pol, 3, 4>(pol, cx, st);
  if (U == 4 && B == 4) return launch_st<Pol, 4, 4>(pol, cx, st);
  if (U == 8 && B == 4) return launch_st<Pol, 8, 4>(pol, cx, st);
  // more resident CTAs than 4 (256 threads each): fewer registers per thread
  if (U == 4 && B == 6) return launch_st<Pol, 4, 6>(pol, cx, st);
  if (U == 4 && B == 8) return launch_st<Pol, 4, 8>(pol, cx, st);
  if (U == 2 && B == 6) return launch_st<Pol, 2, 6>(pol, cx, st);
  if (U == 1 && B == 6) return launch_st<Pol, 1, 6>(pol, cx, st);
  if (U == 2 && B == 8) return launch_st<Pol, 2, 8>(pol, cx, st);
  if (U == 3 && B == 6) return launch_st<Pol, 3, 6>(pol, cx, st);
  if (U == 1 && B == 8) return launch_st<Pol, 1, 8>(pol, cx, st);
  if (U == 2 && B == 5) return launch_st<Pol, 2, 5>(pol, cx, st);
  return launch_st<Pol, 4, 3>(pol, cx, st);
}

// ------------------------------------------------------------------------------------------
// softmax-weighted aggregate over 128-float rows (lane = float4 column, LH lanes per head)
// ------------------------------------------------------------------------------------------
constexpr float SM_LOG2E = 1.4426950408889634f;
constexpr float SM_LN2 = 0.6931471805599453f;

struct SmRows {
  const int64_t* group_ptr;
  const int32_t* src_row;     // group-major gather rows
  const int32_t* dst_row;     // [G] query row of a group (unused when q_by_group)
  const int32_t* src_group;   // source-major: group of each position
  const int32_t* src_pos;     // source-major: group-major position
  const float* key; int64_t ld_key;   // K' [n_s, 128]
  const float* val; int64_t ld_val;   // M' [n_s, 128]
  const float* q;   int64_t ld_q;     // Q  [n_t, 128] (or [G, 128] by group)
  int q_by_group;
  int heads, LH;
  float scale;                        // score scale (natural units)
};

// the row-split softmax kernels take 128-float rows (HGT's d = 128, reading 12)
inline bool sm_rowsplit_ok(const rnn_join_index* idx, const rnn_lifted_query* q, int D) {
  return D == 128 && idx->pos_group && idx->n_join_rows > 0 && q->heads >= 1 && q->heads <= 32;
}

inline SmRows sm_rows(const rnn_join_index* idx, const rnn_lifted_query* q) {
  SmRows a{};
  a.group_ptr = idx->group_ptr;
  a.src_row = idx->src_row;
  a.dst_row = idx->group_dst_row;
  a.src_group = idx->src_group;
  a.src_pos = idx->src_pos;
  a.key = q->src_key.data; a.ld_key = q->src_key.ld;
  a.val = q->src.data; a.ld_val = q->src.ld;
  a.q = q->dst.data; a.ld_q = q->dst.ld;
  a.q_by_group = q->dst.mode == RNN_BY_POSITION;
  a.heads = q->heads;
  a.LH = 32 / q->heads;
  a.scale = q->scale;
  return a;
}

__device__ __forceinline__ float sm_head_sum(float x, int LH) {
  for (int m = 1; m < LH; m <<= 1) x += __shfl_xor_sync(FULL, x, m);
  return x;
}

// forward: out[g] = sum_r softmax_r(scale <K'[s_r], Q[t_g]>) M'[s_r] per head; lse saved
struct SmFwdPol {
  SmRows a;
  float* out; int64_t ld_out; float beta;
  float* lse;
  float* out2 = nullptr; int64_t ld_out2 = 0; float beta2 = 0.f;   // union: out2 = beta2 out2 + x
  struct Meta { int s, t; };
  struct Row { float4 k, v, q; float sc; };
  struct State { float4 acc; float m, l; };

  __device__ __forceinline__ Meta meta(int64_t r, int g) const {
    return Meta{a.src_row[r], a.q_by_group ? g : a.dst_row[g]};
  }
  __device__ __forceinline__ Meta shfl(const Meta& m, int j) const {
    return Meta{__shfl_sync(FULL, m.s, j), __shfl_sync(FULL, m.t, j)};
  }
  __device__ __forceinline__ void load(Row& w, const Meta& m, bool) const {
    const int k = lane_id();
    w.k = ld_f4(a.key + (int64_t)m.s * a.ld_key + 4 * k);
    w.v = ld_f4(a.val + (int64_t)m.s * a.ld_val + 4 * k);
    w.q = ld_f4(a.q + (int64_t)m.t * a.ld_q + 4 * k);
  }
  __device__ __forceinline__ void prep(Row& w) const {
    w.sc = sm_head_sum(f4_dot(w.k, w.q), a.LH) * (a.scale * SM_LOG2E);
  }
  __device__ __forceinline__ void init(State& s) const { s.acc = f4_zero(); s.m = -INFINITY; s.l = 0.f; }
  // one exp2 per row: the larger of (running max, score) is the new max
  __device__ __forceinline__ void row(State& s, const Row& w, int64_t) const {
    const float d = w.sc - s.m;
    const bool up = d > 0.f;
    const float x = exp2f(-fabsf(d));
    const float cs = up ? x : 1.f, p = up ? 1.f : x;
    s.l = fmaf(s.l, cs, p);
    s.acc = f4_fma(p, w.v, f4_scale(cs, s.acc));
    s.m = up ? w.sc : s.m;
  }
  __device__ __forceinline__ void finish(const State& s, int64_t g) const {
    const int k = lane_id();
    const bool empty = s.l == 0.f;
    float4 x = empty ? f4_zero() : f4_scale(1.f / s.l, s.acc);
    if (out2) {
      float* o2 = out2 + g * ld_out2 + 4 * k;
      st_f4(o2, beta2 != 0.f ? f4_add(x, ld_f4_cg(o2)) : x);
    }
    float* o = out + g * ld_out + 4 * k;
    if (beta != 0.f) x = f4_fma(beta, ld_f4_cg(o), x);
    st_f4(o, x);
    if (k % a.LH == 0) lse[g * a.heads + k / a.LH] = empty ? -INFINITY : (s.m + log2f(s.l)) * SM_LN2;
  }
  __device__ __forceinline__ void zero(int64_t g) const {
    State s;
    init(s);
    finish(s, g);
  }
  __device__ __forceinline__ void save(const State& s, float* dst) const {
    const int k = lane_id();
    __stcg(reinterpret_cast<float4*>(dst + 4 * k), s.acc);
    if (k % a.LH == 0) {
      __stcg(dst + 128 + 2 * (k / a.LH), s.m);
      __stcg(dst + 128 + 2 * (k / a.LH) + 1, s.l);
    }
  }
  __device__ __forceinline__ void merge(State& s, const float* src) const {
    const int k = lane_id();
    const float4 a2 = ld_f4_cg(src + 4 * k);
    const float m2 = __ldcg(src + 128 + 2 * (k / a.LH)), l2 = __ldcg(src + 128 + 2 * (k / a.LH) + 1);
    const float mn = fmaxf(s.m, m2);
    if (mn == -INFINITY) return;
    const float c1 = exp2f(s.m - mn), c2 = exp2f(m2 - mn);
    s.l = s.l * c1 + l2 * c2;
    s.acc = f4_add(f4_scale(c1, s.acc), f4_scale(c2, a2));
    s.m = mn;
  }
};

// backward pass 1 (group-major): a = softmax recomputed from lse; D = <dO, O> per head;
// de = a (<dO, M'[s]> - D); dQ[t] = scale sum_r de K'[s]; (a, de) saved per position
struct SmBwd1Pol {
  SmRows a;
  const float* out; int64_t ld_out;
  const float* lse;
  const float* dO; int64_t ld_do;
  float* AD;                       // [E', 2h]
  float* dq; int64_t ld_dq;        // nullable
  struct Meta { int s, t, g; };
  struct Row { float4 k, v, q, dO, o; float lse2, sc, da, D; };
  struct State { float4 dq; };

  __device__ __forceinline__ Meta meta(int64_t r, int g) const {
    return Meta{a.src_row[r], a.q_by_group ? g : a.dst_row[g], g};
  }
  __device__ __forceinline__ Meta shfl(const Meta& m, int j) const {
    return Meta{__shfl_sync(FULL, m.s, j), __shfl_sync(FULL, m.t, j), __shfl_sync(FULL, m.g, j)};
  }
  __device__ __forceinline__ void load(Row& w, const Meta& m, bool) const {
    const int k = lane_id();
    w.k = ld_f4(a.key + (int64_t)m.s * a.ld_key + 4 * k);
    w.v = ld_f4(a.val + (int64_t)m.s * a.ld_val + 4 * k);
    w.q = ld_f4(a.q + (int64_t)m.t * a.ld_q + 4 * k);
    w.dO = ld_f4(dO + (int64_t)m.g * ld_do + 4 * k);
    w.o = ld_f4(out + (int64_t)m.g * ld_out + 4 * k);
    w.lse2 = __ldg(lse + (int64_t)m.g * a.heads + k / a.LH) * SM_LOG2E;
  }
  __device__ __forceinline__ void prep(Row& w) const {
    w.sc = sm_head_sum(f4_dot(w.k, w.q), a.LH);
    w.da = sm_head_sum(f4_dot(w.dO, w.v), a.LH);
    w.D = sm_head_sum(f4_dot(w.dO, w.o), a.LH);
  }
  __device__ __forceinline__ void init(State& s) const { s.dq = f4_zero(); }
  __device__ __forceinline__ void row(State& s, const Row& w, int64_t p) const {
    const int k = lane_id();
    const float pa = exp2f(w.sc * (a.scale * SM_LOG2E) - w.lse2);
    const float de = pa * (w.da - w.D);
    s.dq = f4_fma(de, w.k, s.dq);
    if (k % a.LH == 0) {
      float* ad = AD + p * 2 * a.heads + k / a.LH;
      ad[0] = pa;
      ad[a.heads] = de;
    }
  }
  __device__ __forceinline__ int64_t qrow(int64_t g) const {
    return a.q_by_group ? g : (int64_t)a.dst_row[g];
  }
  __device__ __forceinline__ void finish(const State& s, int64_t g) const {
    if (dq) st_f4(dq + qrow(g) * ld_dq + 4 * lane_id(), f4_scale(a.scale, s.dq));
  }
  __device__ __forceinline__ void zero(int64_t g) const {
    if (dq) st_f4(dq + qrow(g) * ld_dq + 4 * lane_id(), f4_zero());
  }
  __device__ __forceinline__ void save(const State& s, float* dst) const {
    __stcg(reinterpret_cast<float4*>(dst + 4 * lane_id()), s.dq);
  }
  __device__ __forceinline__ void merge(State& s, const float* src) const {
    s.dq = f4_add(s.dq, ld_f4_cg(src + 4 * lane_id()));
  }
};

// backward pass 2 (source-major): dM'[s] = sum_r a_r dO[g_r];  dK'[s] = scale sum_r de_r Q[t_r]
struct SmBwd2Pol {
  SmRows a;
  const float* dO; int64_t ld_do;
  const float* AD;
  float* dv; int64_t ld_dv;        // nullable
  float* dk; int64_t ld_dk;        // nullable
  struct Meta { int g, t, p; };
  struct Row { float4 dO, q; float pa, de; };
  struct State { float4 dv, dk; };

  __device__ __forceinline__ Meta meta(int64_t r, int) const {
    const int g = a.src_group[r];
    return Meta{g, a.q_by_group ? g : a.dst_row[g], a.src_pos[r]};
  }
  __device__ __forceinline__ Meta shfl(const Meta& m, int j) const {
    return Meta{__shfl_sync(FULL, m.g, j), __shfl_sync(FULL, m.t, j), __shfl_sync(FULL, m.p, j)};
  }
  __device__ __forceinline__ void load(Row& w, const Meta& m, bool) const {
    const int k = lane_id();
    w.dO = ld_f4(dO + (int64_t)m.g * ld_do + 4 * k);
    w.q = ld_f4(a.q + (int64_t)m.t * a.ld_q + 4 * k);
    const float* ad = AD + (int64_t)m.p * 2 * a.heads + k / a.LH;
    w.pa = __ldg(ad);
    w.de = __ldg(ad + a.heads);
  }
  __device__ __forceinline__ void prep(Row&) const {}
  __device__ __forceinline__ void init(State& s) const { s.dv = f4_zero(); s.dk = f4_zero(); }
  __device__ __forceinline__ void row(State& s, const Row& w, int64_t) const {
    s.dv = f4_fma(w.pa, w.dO, s.dv);
    s.dk = f4_fma(w.de, w.q, s.dk);
  }
  __device__ __forceinline__ void finish(const State& s, int64_t src) const {
    const int k = lane_id();
    if (dv) st_f4(dv + src * ld_dv + 4 * k, s.dv);
    if (dk) st_f4(dk + src * ld_dk + 4 * k, f4_scale(a.scale, s.dk));
  }
  __device__ __forceinline__ void zero(int64_t src) const {
    State s;
    init(s);
    finish(s, src);
  }
  __device__ __forceinline__ void save(const State& s, float* dst) const {
    const int k = lane_id();
    __stcg(reinterpret_cast<float4*>(dst + 4 * k), s.dv);
    __stcg(reinterpret_cast<float4*>(dst + 128 + 4 * k), s.dk);
  }
  __device__ __forceinline__ void merge(State& s, const float* src) const {
    const int k = lane_id();
    s.dv = f4_add(s.dv, ld_f4_cg(src + 4 * k));
    s.dk = f4_add(s.dk, ld_f4_cg(src + 128 + 4 * k));
  }
};


// ------------------------------------------------------------------------------------------
// Source-major softmax backward (default): the probabilities are recomputed where the source
// rows are resident, so M' is never gathered again and no (a, de) pair makes a round trip.
//   D[g, h]  = <dO[g], O[g]> per head                          (sm_d_kernel, warp per group)
//   pass A (source-major, segment = source s; K'[s], M'[s] stay in L1 across the segment):
//     a = exp(<K'[s], Q[t]> - lse[g]),  de = a (<dO[g], M'[s]> - D[g])
//     dM'[s] = sum a dO[g],  dK'[s] = scale sum de Q[t],  DE[p] = de   (p = group-major pos)
//   pass B (group-major): dQ[t] = scale sum_p DE[p] K'[s_p]
// Per join row: pass A gathers Q[t] and dO[g] (8d bytes) + 8h, writes 4h; pass B gathers K'
// (4d) + 4h -- against 16d + 16h for the two-pass (a, de) scheme above.
// ------------------------------------------------------------------------------------------
static __global__ void sm_d_kernel(const float* __restrict__ dO, int64_t ld_do, const float* __restrict__ O,
                            int64_t ld_o, int64_t G, int heads, int LH, float* __restrict__ D) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= G) return;
  const int k = lane_id();
  const float x = sm_head_sum(f4_dot(ld_f4(dO + g * ld_do + 4 * k), ld_f4(O + g * ld_o + 4 * k)), LH);
  if (k % LH == 0) D[g * heads + k / LH] = x;
}

struct SmBwdAPol {
  SmRows a;
  const float* dO; int64_t ld_do;
  const float* lse;
  const float* Dg;                 // [G, h]
  float* DE;                       // [E', h] by group-major position
  float* dv; int64_t ld_dv;        // nullable
  float* dk; int64_t ld_dk;        // nullable
  struct Meta { int g, t, p, s; };
  struct Row { float4 k, v, q, dO; float lse2, D, sc, da; int p; };
  struct State { float4 dv, dk; };

  __device__ __forceinline__ Meta meta(int64_t r, int seg) const {
    const int g = a.src_group[r];
    return Meta{g, a.q_by_group ? g : a.dst_row[g], a.src_pos[r], seg};
  }
  __device__ __forceinline__ Meta shfl(const Meta& m, int j) const {
    return Meta{__shfl_sync(FULL, m.g, j), __shfl_sync(FULL, m.t, j), __shfl_sync(FULL, m.p, j),
                __shfl_sync(FULL, m.s, j)};
  }
  __device__ __forceinline__ void load(Row& w, const Meta& m, bool) const {
    const int k = lane_id();
    w.k = ld_f4(a.key + (int64_t)m.s * a.ld_key + 4 * k);
    w.v = ld_f4(a.val + (int64_t)m.s * a.ld_val + 4 * k);
    w.q = ld_f4(a.q + (int64_t)m.t * a.ld_q + 4 * k);
    w.dO = ld_f4(dO + (int64_t)m.g * ld_do + 4 * k);
    const int64_t gh = (int64_t)m.g * a.heads + k / a.LH;
    w.lse2 = __ldg(lse + gh) * SM_LOG2E;
    w.D = __ldg(Dg + gh);
    w.p = m.p;
  }
  __device__ __forceinline__ void prep(Row& w) const {
    w.sc = sm_head_sum(f4_dot(w.k, w.q), a.LH);
    w.da = sm_head_sum(f4_dot(w.dO, w.v), a.LH);
  }
  __device__ __forceinline__ void init(State& s) const { s.dv = f4_zero(); s.dk = f4_zero(); }
  __device__ __forceinline__ void row(State& s, const Row& w, int64_t) const {
    const int k = lane_id();
    const float pa = exp2f(w.sc * (a.scale * SM_LOG2E) - w.lse2);
    const float de = pa * (w.da - w.D);
    s.dv = f4_fma(pa, w.dO, s.dv);
    s.dk = f4_fma(de, w.q, s.dk);
    if (k % a.LH == 0) DE[(int64_t)w.p * a.heads + k / a.LH] = de;
  }
  __device__ __forceinline__ void finish(const State& s, int64_t src) const {
    const int k = lane_id();
    if (dv) st_f4(dv + src * ld_dv + 4 * k, s.dv);
    if (dk) st_f4(dk + src * ld_dk + 4 * k, f4_scale(a.scale, s.dk));
  }
  __device__ __forceinline__ void zero(int64_t src) const {
    State s;
    init(s);
    finish(s, src);
  }
  __device__ __forceinline__ void save(const State& s, float* dst) const {
    const int k = lane_id();
    __stcg(reinterpret_cast<float4*>(dst + 4 * k), s.dv);
    __stcg(reinterpret_cast<float4*>(dst + 128 + 4 * k), s.dk);
  }
  __device__ __forceinline__ void merge(State& s, const float* src) const {
    const int k = lane_id();
    s.dv = f4_add(s.dv, ld_f4_cg(src + 4 * k));
    s.dk = f4_add(s.dk, ld_f4_cg(src + 128 + 4 * k));
  }
};

struct SmBwdBPol {
  SmRows a;
  const float* DE;                 // [E', h]
  float* dq; int64_t ld_dq;
  float beta = 0.f;                // 1: dq accumulates (a query shared by several relations)
  struct Meta { int s; };
  struct Row { float4 k; float de; };
  struct State { float4 dq; };
  __device__ __forceinline__ Meta meta(int64_t r, int) const { return Meta{a.src_row[r]}; }
  __device__ __forceinline__ Meta shfl(const Meta& m, int j) const {
    return Meta{__shfl_sync(FULL, m.s, j)};
  }
  __device__ __forceinline__ void load(Row& w, const Meta& m, bool) const {
    const int k = lane_id();
    w.k = ld_f4(a.key + (int64_t)m.s * a.ld_key + 4 * k);
  }
  __device__ __forceinline__ void prep(Row&) const {}
  __device__ __forceinline__ void init(State& s) const { s.dq = f4_zero(); }
  __device__ __forceinline__ void row(State& s, const Row& w, int64_t p) const {
    const float de = __ldg(DE + p * a.heads + lane_id() / a.LH);
    s.dq = f4_fma(de, w.k, s.dq);
  }
  __device__ __forceinline__ int64_t qrow(int64_t g) const {
    return a.q_by_group ? g : (int64_t)a.dst_row[g];
  }
  __device__ __forceinline__ void finish(const State& s, int64_t g) const {
    float* o = dq + qrow(g) * ld_dq + 4 * lane_id();
    const float4 x = f4_scale(a.scale, s.dq);
    st_f4(o, beta != 0.f ? f4_add(x, ld_f4_cg(o)) : x);
  }
  __device__ __forceinline__ void zero(int64_t g) const {
    if (beta == 0.f) st_f4(dq + qrow(g) * ld_dq + 4 * lane_id(), f4_zero());
  }
  __device__ __forceinline__ void save(const State& s, float* dst) const {
    __stcg(reinterpret_cast<float4*>(dst + 4 * lane_id()), s.dq);
  }
  __device__ __forceinline__ void merge(State& s, const float* src) const {
    s.dq = f4_add(s.dq, ld_f4_cg(src + 4 * lane_id()));
  }
};
}  // namespace rnn
