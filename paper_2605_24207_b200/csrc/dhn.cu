// dhn.cu -- A6: DHN closed-walk pattern aggregates C2 / C3 / C4 (multi-way cyclic joins).
//
// PAPER.md:938-950 (the DHN rule, C3 written out at :943-946), closed walks :1481, Eq. 3
// :1500 (t_mu(F, G, u) = sum over homomorphisms rooted at u of prod_v mu_v(h(phi(v)))),
// SURVEY sec 8a A6.  rnn.h documents the operation; this file is the B200 realisation:
//
//  * every operand is first gathered into GROUP order (root space) so the walk only touches
//    int32 group ids: nbr[p] = group of the neighbour at join position p (-1 if it has no
//    out-edges and so cannot continue a walk), in-neighbours of group n = src_group[] over
//    the transposed CSR of n's row;
//  * one CTA (32 warps) per root, roots taken heaviest-first from an atomic counter;
//  * C3: the root's in-neighbours go into a shared-memory hash set (count = multiplicity of
//    the closing Edge rows), then the warps walk the wedges n->v->w with lanes over w and
//    probe the set; the hits gather f1(v) (.) f2(w) with lane = channel;
//  * C4: factorised through the middle vertex w (see dhn4_kernel): S1(w) accumulates over
//    out-wedges in a shared-memory hash of 2-hop keys with compact ids (values: a dense,
//    L2-resident per-CTA slab), the in-wedges w->p->n then add f3(p) (.) f2(w) (.) S1(w);
//    big roots run in hash partitions of w over hash-sorted adjacency lists;
//  * the backward is the same kernels with rotated operands (rnn.h).
#include <algorithm>

#include "common.cuh"

namespace rnn {
namespace {

// C3 CTA shape (compile-time; -D overrides for measurement builds, profiles/build_variant.py)
// (4 CTAs of 8 warps per SM: one CTA's per-root barriers overlap the others' walks;
// 0.1-scale products C3 fwd 25.1 -> 15.8 ms against 1 x 1024, profiles/r02/c3lb)
#ifndef DHN_THREADS_CFG
#define DHN_THREADS_CFG 256
#endif
#ifndef DHN_CTAS_CFG
#define DHN_CTAS_CFG 4
#endif
#ifndef H3_CAP_CFG
#define H3_CAP_CFG 4096
#endif
constexpr int DHN_THREADS = DHN_THREADS_CFG;
constexpr int DHN_WARPS = DHN_THREADS / 32;
constexpr int DHN_CTAS_PER_SM = DHN_CTAS_CFG;

struct DhnArgs {
  int64_t G;
  int d;
  const int64_t* gp;      // group_ptr [G+1]
  const int32_t* nbr;     // [E'] group id of the neighbour at each position (or -1)
  const int64_t* sp;      // src_ptr [n_rows+1]
  const int32_t* sg;      // src_group [E']
  const int32_t* row_of;  // group_dst_row [G]
  const float* F1;        // walk operands in group order [G, d] (ld d)
  const float* F2;
  const float* F3;
  const float* rm;        // root multiplier (nullable = 1)
  int64_t ld_rm;
  int rm_by_group;        // rm rows: group id (1) or node row (0)
  float* out;
  int64_t ld_out;
  int out_by_row;         // write out[row_of[n]] instead of out[n]
  const int32_t* order;   // roots, heaviest first (active roots first)
  int* counter;
  const int* n_active;    // number of active roots at the head of order[] (device)
  int* mark;              // k=3: per-CTA [G] int32
  const uint32_t* wout;   // k=4: out-wedges per root (bound on distinct 2-hop w)
  float* slab;            // k=4: per-CTA S1 values [H4_CAP][32]
  const int32_t* nbrh;    // k=4: nbr[] with every group's list sorted by hash partition
  const int32_t* sgh;     // k=4: src_group[] with every row's list sorted likewise
  int64_t cta_stride;     // elements between consecutive CTAs' mark
  float* sum_out;         // optional: the walk sum before the root multiplier [G, ld_sum]
  int64_t ld_sum;
  const float* F2b;       // k=4, optional second middle operand (symmetric Edge)
  const float* F1b;       // k=3, optional second first-hop operand (symmetric Edge)
  float* out_b;           // its result (same layout as out, no root multiplier)
  int part_keys;          // k=4 slot-indexed walk: target distinct keys per partition (0: H4_PART)
};

__device__ __forceinline__ void dhn_store(const DhnArgs& a, int64_t n, int c, float v) {
  if (a.sum_out) a.sum_out[n * a.ld_sum + c] = v;
  if (a.rm) {
    const int64_t rr = a.rm_by_group ? n : (int64_t)a.row_of[n];
    v *= a.rm[rr * a.ld_rm + c];
  }
  const int64_t orow = a.out_by_row ? (int64_t)a.row_of[n] : n;
  a.out[orow * a.ld_out + c] = v;
}

__device__ __forceinline__ int64_t dhn_next_root(const DhnArgs& a, int* s_root) {
  __syncthreads();
  if (threadIdx.x == 0) *s_root = atomicAdd(a.counter, 1);
  __syncthreads();
  const int i = *s_root;
  return i < *a.n_active ? (int64_t)a.order[i] : -1;
}

// Path counters of the walk kernels (which code paths a launch took), read by the internal
// hook rnn_internal_dhn_stats so the tests can prove the big-root paths ran:
//   [0] C3 roots, [1] C3 roots on the global mark array (in-degree > H3_MAX_INDEG),
//   [2] C4 roots, [3] C4 (root, partition) passes, [4] of them in chunked mode,
//   [5] C4 long runs queued for phase B, [6] long runs past the queue (walked inline),
//   [7] C4 roots with hash partitions (P > 1), [8] C4 keys refused by a full value table
//   (shared-memory variant; must stay 0).
// Counted per CTA (registers / shared memory) and added once per CTA at exit.
__device__ unsigned long long g_dhn_paths[16];

// -------------------------------------------------------------------------------------
// shared-memory open-addressing hash sets keyed by group id (linear probing, key -1 = empty)
// -------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t dhn_hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7FEB352Du; x ^= x >> 15; x *= 0x846CA68Bu; x ^= x >> 16;
  return x;
}
// slot of key w (inserted if absent); -1 if the table is full
__device__ __forceinline__ int hs_insert(int* keys, int cap_mask, int w) {
  uint32_t s = dhn_hash((uint32_t)w) & (uint32_t)cap_mask;
  for (int t = 0; t <= cap_mask; ++t) {
    const int prev = atomicCAS(&keys[s], -1, w);
    if (prev == -1 || prev == w) return (int)s;
    s = (s + 1) & (uint32_t)cap_mask;
  }
  return -1;
}
__device__ __forceinline__ int hs_find(const int* keys, int cap_mask, int w) {
  uint32_t s = dhn_hash((uint32_t)w) & (uint32_t)cap_mask;
  for (int t = 0; t <= cap_mask; ++t) {
    const int k = keys[s];
    if (k == w) return (int)s;
    if (k == -1) return -1;
    s = (s + 1) & (uint32_t)cap_mask;
  }
  return -1;
}

// -------------------------------------------------------------------------------------
// C3: triangles n -> v -> w -> n.  The root's in-neighbours w (with multiplicity = number of
// closing Edge rows w -> n) go into a shared-memory hash set; the CTA's warps walk the wedges
// n -> v -> w with lanes over w, probe the set, and the hits gather f1(v) (.) f2(w) with
// lane = channel.  Roots whose in-degree exceeds the set use a per-CTA global mark array.
// -------------------------------------------------------------------------------------
constexpr int H3_CAP = H3_CAP_CFG;           // slots (keys + counts: 64 KB at 8,192)
constexpr int H3_MAX_INDEG = H3_CAP / 4 * 3; // load factor <= 0.75
constexpr int H3_LONG = 256;                 // N(v) longer than this: split over all warps
constexpr int H3_QMAX = 256;                 // long lists queued per root (overflow: inline)

template <int DPL, bool DUAL = false>
__global__ void __launch_bounds__(DHN_THREADS, DHN_CTAS_PER_SM) dhn3_kernel(DhnArgs a) {
  extern __shared__ int h3[];
  int* keys = h3;
  int* cnt = h3 + H3_CAP;
  int* used = cnt + H3_CAP;                                  // [H3_MAX_INDEG] slots taken
  float* s_acc = reinterpret_cast<float*>(used + H3_MAX_INDEG);   // [DHN_WARPS][DPL * 32]
  int64_t* q_b = reinterpret_cast<int64_t*>(s_acc + DHN_WARPS * DPL * 32);   // [H3_QMAX]
  int64_t* q_e = q_b + H3_QMAX;
  int32_t* q_v = reinterpret_cast<int32_t*>(q_e + H3_QMAX);
  int32_t* q_i = q_v + H3_QMAX;     // neighbour index of each queued list
  int32_t* q_ord = q_i + H3_QMAX;   // queue slots in neighbour order
  __shared__ int s_root, s_qn;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int* mark = a.mark + (int64_t)blockIdx.x * a.cta_stride;
  const int d = a.d;
  for (int i = threadIdx.x; i < H3_CAP; i += DHN_THREADS) { keys[i] = -1; cnt[i] = 0; }
  if (threadIdx.x == 0) s_qn = 0;
  unsigned long long c_roots = 0, c_mark = 0;   // path counters (thread 0)
  for (;;) {
    const int64_t n = dhn_next_root(a, &s_root);
    if (n < 0) break;
    const int32_t r = a.row_of[n];
    const int64_t ib = a.sp[r], ie = a.sp[r + 1];
    const bool hashed = ie - ib <= H3_MAX_INDEG;
    ++c_roots;
    c_mark += !hashed;
    if (hashed) {
      for (int64_t q = ib + threadIdx.x; q < ie; q += DHN_THREADS) {
        const int sl = hs_insert(keys, H3_CAP - 1, a.sg[q]);
        atomicAdd(&cnt[sl], 1);
        used[q - ib] = sl;
      }
    } else {
      for (int64_t q = ib + threadIdx.x; q < ie; q += DHN_THREADS) atomicAdd(&mark[a.sg[q]], 1);
    }
    __syncthreads();
    float acc[DPL], acc_b[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) acc[j] = acc_b[j] = 0.f;
    const int64_t pb = a.gp[n], pe = a.gp[n + 1];
    // the wedges n -> v -> w, w in [i_beg, i_end) of N(v): two 32-entry chunks per step (both
    // loads in flight before either probe); hits gather f1(v) (.) f2(w), 4 per round
    auto walk_range = [&](int32_t v, int64_t i_beg, int64_t i_end) {
      float f1v[DPL], f1bv[DPL];
#pragma unroll
      for (int j = 0; j < DPL; ++j) {
        const int c = lane + 32 * j;
        f1v[j] = c < d ? a.F1[(int64_t)v * d + c] : 0.f;
        f1bv[j] = DUAL && c < d ? a.F1b[(int64_t)v * d + c] : 0.f;
      }
      for (int64_t i0 = i_beg; i0 < i_end; i0 += 64) {
        const int32_t w2[2] = {i0 + lane < i_end ? a.nbr[i0 + lane] : -1,
                               i0 + 32 + lane < i_end ? a.nbr[i0 + 32 + lane] : -1};
        int m2[2] = {0, 0};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (w2[h] >= 0) {
            if (hashed) {
              const int sl = hs_find(keys, H3_CAP - 1, w2[h]);
              m2[h] = sl >= 0 ? cnt[sl] : 0;
            } else {
              m2[h] = __ldcg(&mark[w2[h]]);
            }
          }
        }
#pragma unroll
        for (int hc = 0; hc < 2; ++hc) {
          const int32_t w = w2[hc];
          const int m = m2[hc];
          unsigned bal = __ballot_sync(FULL, m != 0);
          while (bal) {
            int ww[4], mm[4], nh = 0;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              ww[h] = 0; mm[h] = 0;
              if (bal) {
                const int b = __ffs(bal) - 1;
                bal &= bal - 1;
                ww[h] = __shfl_sync(FULL, w, b);
                mm[h] = __shfl_sync(FULL, m, b);
                ++nh;
              }
            }
#pragma unroll
            for (int j = 0; j < DPL; ++j) {
              const int c = lane + 32 * j;
              if (c < d) {
                float x[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) x[h] = h < nh ? a.F2[(int64_t)ww[h] * d + c] : 0.f;
                float t = 0.f;
#pragma unroll
                for (int h = 0; h < 4; ++h) t += (float)mm[h] * x[h];
                acc[j] += f1v[j] * t;
                if (DUAL) acc_b[j] += f1bv[j] * t;
              }
            }
          }
        }
      }
    };
    // phase A: neighbour i goes to warp i % WARPS (a fixed order per warp: the walk is
    // deterministic); lists longer than H3_LONG are queued instead
    for (int64_t i = warp; pb + i < pe; i += DHN_WARPS) {
      const int32_t v = a.nbr[pb + i];
      if (v < 0) continue;
      const int64_t vb = a.gp[v], ve = a.gp[v + 1];
      if (ve - vb > H3_LONG) {
        int slot = 0;
        if (lane == 0) slot = atomicAdd(&s_qn, 1);
        slot = __shfl_sync(FULL, slot, 0);
        if (slot < H3_QMAX) {
          if (lane == 0) { q_v[slot] = v; q_b[slot] = vb; q_e[slot] = ve; q_i[slot] = (int)i; }
          continue;
        }
      }
      walk_range(v, vb, ve);
    }
    __syncthreads();
    // phase B: the queued lists in neighbour order (rank of q_i: the queue's slot order
    // depends on timing), cut into 128-entry pieces; piece g goes to warp g % WARPS
    const int nq = s_qn < H3_QMAX ? s_qn : H3_QMAX;
    if (nq > 0) {
      for (int t = threadIdx.x; t < nq; t += DHN_THREADS) {
        int rk = 0;
        for (int j = 0; j < nq; ++j) rk += q_i[j] < q_i[t];
        q_ord[rk] = t;
      }
      __syncthreads();
      int k = 0;
      int64_t k_beg = 0, k_end = 0;
      for (int g = warp;; g += DHN_WARPS) {
        while (g >= k_end && k < nq) {
          const int it = q_ord[k];
          k_beg = k_end;
          k_end += (q_e[it] - q_b[it] + 127) / 128;
          ++k;
        }
        if (g >= k_end) break;
        const int it = q_ord[k - 1];
        const int64_t b0 = q_b[it] + (int64_t)(g - k_beg) * 128;
        const int64_t e0 = b0 + 128 < q_e[it] ? b0 + 128 : q_e[it];
        walk_range(q_v[it], b0, e0);
      }
    }
#pragma unroll
    for (int j = 0; j < DPL; ++j) s_acc[warp * DPL * 32 + lane + 32 * j] = acc[j];
    __syncthreads();
    if (threadIdx.x == 0) s_qn = 0;   // every warp is past phase B
    for (int c = threadIdx.x; c < d; c += DHN_THREADS) {
      float s = 0.f;
      for (int w = 0; w < DHN_WARPS; ++w) s += s_acc[w * DPL * 32 + c];
      dhn_store(a, n, c, s);
    }
    if (DUAL) {   // the second first-hop operand's result (no root multiplier)
      __syncthreads();
#pragma unroll
      for (int j = 0; j < DPL; ++j) s_acc[warp * DPL * 32 + lane + 32 * j] = acc_b[j];
      __syncthreads();
      const int64_t orow = a.out_by_row ? (int64_t)a.row_of[n] : n;
      for (int c = threadIdx.x; c < d; c += DHN_THREADS) {
        float s = 0.f;
        for (int w = 0; w < DHN_WARPS; ++w) s += s_acc[w * DPL * 32 + c];
        a.out_b[orow * a.ld_out + c] = s;
      }
    }
    if (hashed) {   // exactly the slots the inserts took (a repeated key clears twice)
      for (int64_t q = threadIdx.x; q < ie - ib; q += DHN_THREADS) {
        keys[used[q]] = -1;
        cnt[used[q]] = 0;
      }
    } else {
      for (int64_t q = ib + threadIdx.x; q < ie; q += DHN_THREADS) mark[a.sg[q]] = 0;
    }
  }
  if (threadIdx.x == 0) {
    atomicAdd(&g_dhn_paths[0], c_roots);
    atomicAdd(&g_dhn_paths[1], c_mark);
  }
}

// -------------------------------------------------------------------------------------
// C4: closed 4-walks n -> v -> w -> p -> n, factorised through w:
//   C4(n) = f0(n) (.) sum_{in-wedges w -> p -> n} f3(p) (.) G(w),
//   G(w)  = f2(w) (.) S1(w),  S1(w) = sum_{out-wedges n -> v -> w} f1(v).
// S1 lives in a shared-memory hash table keyed by w holding a 32-channel lane slice per entry
// (lane = channel: every wedge is ONE conflict-free 128-byte smem atomic).  A root whose
// out-wedges could name more distinct w than the table holds is processed in P = 2^b
// partitions of w by the top b bits of hash(w).  Every adjacency list is pre-sorted by that
// hash (prepare: segmented radix sort), so partition k of a list is a contiguous run that
// starts where partition k-1 ended: per-neighbour cursors in shared memory make each pass
// touch only its own entries (no re-scan), lanes test 32 neighbours' cursors at a time.
// -------------------------------------------------------------------------------------
// measurement builds only (-DRNN_PROBES): thread 0's clock between the C4 phases
// [0] root setup, [1] out sweep, [3] in sweep, [4] clear, [5] reduce/store
__device__ unsigned long long g_dhn4_clock[16];
#ifdef RNN_PROBES
#define H4_T(slot)                                                                  \
  do {                                                                              \
    if (threadIdx.x == 0) {                                                         \
      const long long t_ = clock64();                                               \
      atomicAdd(&g_dhn4_clock[slot], (unsigned long long)(t_ - t_last));            \
      t_last = t_;                                                                  \
    }                                                                               \
  } while (0)
#else
#define H4_T(slot) \
  do {             \
  } while (0)
#endif

// C4 CTA shape (compile-time; -D overrides for measurement builds)
#ifndef H4_THREADS_CFG
#define H4_THREADS_CFG 1024
#endif
#ifndef H4_CTAS_CFG
#define H4_CTAS_CFG 1
#endif
#ifndef H4_CAP_CFG
#define H4_CAP_CFG 16384
#endif
#ifndef H4_DEG_CAP_CFG
#define H4_DEG_CAP_CFG 8192
#endif
constexpr int H4_THREADS = H4_THREADS_CFG;   // threads per C4 CTA (one root at a time)
constexpr int H4_WARPS = H4_THREADS / 32;
constexpr int H4_CTAS = H4_CTAS_CFG;         // C4 CTAs per SM
constexpr int H4_CAP = H4_CAP_CFG;           // key slots in shared memory
constexpr int H4_PART = H4_CAP / 2;          // target distinct w per partition (load <= 0.5)
constexpr int H4_DEG_CAP = H4_DEG_CAP_CFG;   // neighbours with smem cursors (per side)
constexpr int H4_HBITS = 16;                 // hash bits the lists are sorted by

__device__ __forceinline__ uint32_t h4_top(int32_t w) {   // sort key / partition source
  return dhn_hash((uint32_t)w ^ 0x5bd1e995u) >> (32 - H4_HBITS);
}

// first position in [b, e) of list L whose partition (top `bits` of the 16-bit hash) >= k
__device__ __forceinline__ int64_t h4_lower(const int32_t* L, int64_t b, int64_t e, uint32_t k,
                                           int sh) {
  while (b < e) {
    const int64_t m = b + ((e - b) >> 1);
    if ((h4_top(L[m]) >> sh) < k) b = m + 1; else e = m;
  }
  return b;
}

#ifndef H4_LONG_CFG
#define H4_LONG_CFG 96
#endif
constexpr int H4_LONG = H4_LONG_CFG;        // runs longer than this are split over all warps
constexpr int H4_LONG_MAX = 512;             // long runs queued per sweep (overflow: inline)

// One 32-entry chunk of a run: OUT inserts w and adds f1(v) to S1(w) (one 128-byte red per
// entry); IN finds w and sums G(w) into t (8 slab rows in flight per round).
// compact id of key w in the C4 table (inserted if absent): the CAS winner draws the next id
// (so a root's S1 rows are a dense prefix of the CTA's slab and stay L2-resident); a lane
// that finds w already present waits for the winner to publish the id.
// CAP: hash slots; MAXID: value rows (ids >= MAXID are refused: -2 is published so waiting
// lanes give up too, and the overflow is counted -- the shared-memory variant sizes its
// partitions so this does not happen, tests assert it)
template <int CAP = H4_CAP, int MAXID = (1 << 30)>
__device__ __forceinline__ int h4_insert(int* keys, int* ids, int* n_ids, int w) {
  uint32_t s = dhn_hash((uint32_t)w) & (uint32_t)(CAP - 1);
  for (int t = 0; t < CAP; ++t) {
    const int prev = atomicCAS(&keys[s], -1, w);
    if (prev == -1) {
      int id = atomicAdd(n_ids, 1);
      if (id >= MAXID) {
        id = -2;
        atomicAdd(&g_dhn_paths[8], 1ull);
      }
      atomicExch(&ids[s], id);
      return id < 0 ? -1 : id;
    }
    if (prev == w) {
      int id;
      do { id = *((volatile int*)&ids[s]); } while (id == -1);
      return id < 0 ? -1 : id;
    }
    s = (s + 1) & (uint32_t)(CAP - 1);
  }
  return -1;
}

// One 32-entry chunk of a run: OUT inserts w and adds f1(v) to S1(w) (one 128-byte red per
// entry); IN finds w and sums G(w) into t (8 slab rows in flight per round).
template <bool OUT, int CAP = H4_CAP, int MAXID = (1 << 30), bool DUAL = false>
__device__ __forceinline__ void h4_chunk(int* keys, int* ids, int* n_ids, float* S, int32_t w,
                                         bool in, float fv, float& t, int lane,
                                         const float* F2c, int d, float* tb = nullptr,
                                         const float* F2bc = nullptr) {
  if (OUT) {
    const int sl = (in && w >= 0) ? h4_insert<CAP, MAXID>(keys, ids, n_ids, w) : -1;
    unsigned bal = __ballot_sync(FULL, sl >= 0);
    while (bal) {
      const int q = __ffs(bal) - 1;
      bal &= bal - 1;
      atomicAdd(&S[__shfl_sync(FULL, sl, q) * 32 + lane], fv);
    }
  } else {
    int sl = (in && w >= 0) ? hs_find(keys, CAP - 1, w) : -1;
    if (sl >= 0) sl = ids[sl];
    unsigned bal = __ballot_sync(FULL, sl >= 0);
    while (bal) {   // G(w) = f2(w) (.) S1(w) formed on the fly, 8 hits in flight
      float x[8], y[8], yb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        int q = -1;
        if (bal) { q = __ffs(bal) - 1; bal &= bal - 1; }
        const int slq = __shfl_sync(FULL, sl, q < 0 ? 0 : q);
        const int wq = __shfl_sync(FULL, w, q < 0 ? 0 : q);
        x[u] = q >= 0 ? S[slq * 32 + lane] : 0.f;
        y[u] = q >= 0 ? F2c[(int64_t)wq * d] : 0.f;
        if (DUAL) yb[u] = q >= 0 ? F2bc[(int64_t)wq * d] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        t = fmaf(x[u], y[u], t);
        if (DUAL) *tb = fmaf(x[u], yb[u], *tb);
      }
    }
  }
}

// V4 variant of h4_chunk: lane = (hit slot sub = lane / 8, channel quad cq = lane % 8), so
// one instruction moves FOUR hits' 32-channel rows -- OUT: one red.global.add.v4.f32 per lane
// (4x fewer L2 reduction requests than one 4-byte red per lane per hit); IN: float4 loads of
// S1(w) and f2(w).  fv4 / t4: channels 4 cq .. 4 cq + 3 of this 32-channel block.
__device__ __forceinline__ int h4_take4(unsigned& bal, int sub) {
  int mine = -1;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int q = bal ? __ffs(bal) - 1 : -1;
    if (q >= 0) bal &= bal - 1;
    if (k == sub) mine = q;
  }
  return mine;
}
template <bool OUT, bool DUAL = false>
__device__ __forceinline__ void h4_chunk4(int* keys, int* ids, int* n_ids, float* S, int32_t w,
                                          bool in, float4 fv4, float4& t4, int lane,
                                          const float* F2q, int d, float4* t4b = nullptr,
                                          const float* F2bq = nullptr) {
  const int sub = lane >> 3, cq = lane & 7;
  if (OUT) {
    const int sl = (in && w >= 0) ? h4_insert(keys, ids, n_ids, w) : -1;
    unsigned bal = __ballot_sync(FULL, sl >= 0);
    while (bal) {
      const int mine = h4_take4(bal, sub);
      const int slq = __shfl_sync(FULL, sl, mine < 0 ? 0 : mine);
      if (mine >= 0)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(S + slq * 32 + 4 * cq),
                     "f"(fv4.x), "f"(fv4.y), "f"(fv4.z), "f"(fv4.w)
                     : "memory");
    }
  } else {
    int sl = (in && w >= 0) ? hs_find(keys, H4_CAP - 1, w) : -1;
    if (sl >= 0) sl = ids[sl];
    unsigned bal = __ballot_sync(FULL, sl >= 0);
    while (bal) {   // G(w) = f2(w) (.) S1(w) formed on the fly, 8 hits in flight (2 per slot)
      float4 x[2], y[2], yb[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int mine = h4_take4(bal, sub);
        const int slq = __shfl_sync(FULL, sl, mine < 0 ? 0 : mine);
        const int wq = __shfl_sync(FULL, w, mine < 0 ? 0 : mine);
        x[u] = mine >= 0 ? __ldcg(reinterpret_cast<const float4*>(S + slq * 32 + 4 * cq))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        y[u] = mine >= 0 ? __ldg(reinterpret_cast<const float4*>(F2q + (int64_t)wq * d))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        if (DUAL)
          yb[u] = mine >= 0 ? __ldg(reinterpret_cast<const float4*>(F2bq + (int64_t)wq * d))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        t4.x = fmaf(x[u].x, y[u].x, t4.x);
        t4.y = fmaf(x[u].y, y[u].y, t4.y);
        t4.z = fmaf(x[u].z, y[u].z, t4.z);
        t4.w = fmaf(x[u].w, y[u].w, t4.w);
        if (DUAL) {
          t4b->x = fmaf(x[u].x, yb[u].x, t4b->x);
          t4b->y = fmaf(x[u].y, yb[u].y, t4b->y);
          t4b->z = fmaf(x[u].z, yb[u].z, t4b->z);
          t4b->w = fmaf(x[u].w, yb[u].w, t4b->w);
        }
      }
    }
  }
}

struct H4Root {
  int64_t n, ib, pb;
  int deg;               // neighbours on this side
  uint32_t P, part;
  int sh;
  bool cur_ok, chunked;
};

// One side of one partition.  OUT: neighbours v = nbr[pb + i] with lists nbrh over the group
// CSR; IN: neighbours p = sg[ib + i] with lists sgh over the row CSR.  Phase A: each warp
// serves neighbours (one per warp, or 32 per step in chunked mode) and walks their runs of
// this partition; runs longer than H4_LONG are queued.  Phase B: every queued run is split
// over all warps.  Returns this thread's contribution to the root's accumulator (IN).
template <bool OUT, bool V4, bool DUAL = false, int CAP = H4_CAP, int MAXID = (1 << 30)>
__device__ float4 h4_sweep(const DhnArgs& a, const H4Root& R, int* keys, int* ids, int* n_ids,
                          float* S, int* cur, int* q_i, int64_t* q_b, int64_t* q_e, int* q_n,
                          int* grab, int c, bool cok, int* s_cnt, float4* acc_b = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t* L = OUT ? a.nbrh : a.sgh;
  const float* Fv = OUT ? a.F1 : a.F3;
  const int d = a.d;
  const float* F2c = a.F2 + (cok ? c : 0);   // f2 column of this lane (rows gathered by w)
  const float* F2bc = DUAL ? a.F2b + (cok ? c : 0) : nullptr;
  // V4: this lane's channel quad c0 + 4 (lane % 8) .. + 3
  const int cq4 = (c - lane) + 4 * (lane & 7);
  const bool cok4 = cq4 < d;
  const float* F2q = a.F2 + (cok4 ? cq4 : 0);
  const float* F2bq = DUAL ? a.F2b + (cok4 ? cq4 : 0) : nullptr;   // second middle operand
  float acc = 0.f;
  float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
  auto ld_fv4 = [&](int32_t u) {
    return cok4 ? __ldg(reinterpret_cast<const float4*>(Fv + (int64_t)u * d + cq4))
                : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto fma4 = [](float4& acc_, const float4& f, const float4& t_) {
    acc_.x = fmaf(f.x, t_.x, acc_.x); acc_.y = fmaf(f.y, t_.y, acc_.y);
    acc_.z = fmaf(f.z, t_.z, acc_.z); acc_.w = fmaf(f.w, t_.w, acc_.w);
  };
  // phase A: warps grab neighbours dynamically (chunked mode: 32 at a time, lanes in parallel)
  const int step = R.chunked ? 32 : 1;
  for (;;) {
    int base = 0;
    if (lane == 0) base = atomicAdd(grab, step);
    base = __shfl_sync(FULL, base, 0);
    if (base >= R.deg) break;
    const int i = R.chunked ? base + lane : base;
    int32_t u = -1;
    int64_t b0 = 0, e0 = 0, s0 = 0;
    bool has = false;
    if (i < R.deg && (R.chunked || lane == 0)) {
      if (OUT) {
        u = a.nbr[R.pb + i];
        if (u >= 0) { s0 = a.gp[u]; e0 = a.gp[u + 1]; }
      } else {
        u = a.sg[R.ib + i];
        const int32_t ru = a.row_of[u];
        s0 = a.sp[ru];
        e0 = a.sp[ru + 1];
      }
      if (u >= 0) {
        b0 = R.cur_ok ? s0 + cur[i] : h4_lower(L, s0, e0, R.part, R.sh);
        has = b0 < e0 && (h4_top(L[b0]) >> R.sh) == R.part;
      }
    }
    unsigned hb = __ballot_sync(FULL, has);
    while (hb) {
      const int j = __ffs(hb) - 1;
      hb &= hb - 1;
      const int32_t uj = __shfl_sync(FULL, u, j);
      const int64_t bj = __shfl_sync(FULL, b0, j), ej = __shfl_sync(FULL, e0, j);
      const int64_t sj = __shfl_sync(FULL, s0, j);
      const int ij = __shfl_sync(FULL, i, j);
      int64_t re = -1;   // run end when the run is long
      if (ej - bj > H4_LONG) {
        re = R.P == 1 ? ej : h4_lower(L, bj, ej, R.part + 1, R.sh);
        if (re - bj <= H4_LONG) re = -1;
      }
      if (re >= 0) {
        int slot = 0;
        if (lane == 0) slot = atomicAdd(q_n, 1);
        slot = __shfl_sync(FULL, slot, 0);
        if (slot < H4_LONG_MAX) {
          if (lane == 0) { q_i[slot] = uj; q_b[slot] = bj; q_e[slot] = re; atomicAdd(&s_cnt[0], 1); }
          if (R.cur_ok && lane == 0) cur[ij] = (int)(re - sj);
          continue;
        }
        if (lane == 0) atomicAdd(&s_cnt[1], 1);   // queue full: walk this long run inline
      }
      float fv = 0.f, t = 0.f, tb = 0.f;
      float4 fv4 = make_float4(0.f, 0.f, 0.f, 0.f), t4 = fv4, t4b = fv4;
      if (V4) fv4 = ld_fv4(uj);
      else fv = cok ? Fv[(int64_t)uj * d + c] : 0.f;
      int64_t t0 = bj;
      for (;;) {
        const int64_t tt = t0 + lane;
        const int32_t w = tt < ej ? L[tt] : -1;
        const bool in = tt < ej && (h4_top(w) >> R.sh) == R.part;
        const unsigned im = __ballot_sync(FULL, in);
        if (V4) h4_chunk4<OUT, DUAL>(keys, ids, n_ids, S, w, in, fv4, t4, lane, F2q, d, &t4b, F2bq);
        else h4_chunk<OUT, CAP, MAXID, DUAL>(keys, ids, n_ids, S, w, in, fv, t, lane, F2c, d, &tb, F2bc);
        t0 += __popc(im);
        if (im != FULL) break;
      }
      if (!OUT) {
        if (V4) fma4(acc4, fv4, t4);
        else acc += fv * t;
        if (DUAL) {
          if (V4) fma4(*acc_b, fv4, t4b);
          else acc_b->x += fv * tb;
        }
      }
      if (R.cur_ok && lane == 0) cur[ij] = (int)(t0 - sj);
    }
  }
  __syncthreads();
  // phase B: the 32-entry chunks of all queued long runs, grabbed dynamically by the warps
  const int nq = *q_n < H4_LONG_MAX ? *q_n : H4_LONG_MAX;
  if (nq > 0) {
    if (threadIdx.x == 0) *grab = 0;
    __syncthreads();
    int k = 0;            // current item (items are walked in order; chunk ids are global)
    int64_t k_end = 0;    // first global chunk id after item k
    int64_t k_beg = 0;
    float fv = 0.f, t = 0.f, tb = 0.f;
    float4 fv4 = make_float4(0.f, 0.f, 0.f, 0.f), t4 = fv4, t4b = fv4;
    int32_t uk = -1;
    for (;;) {
      int g = 0;
      if (lane == 0) g = atomicAdd(grab, 1);
      g = __shfl_sync(FULL, g, 0);
      // advance to the item holding chunk g (grabs are increasing per warp)
      bool done = false;
      while (g >= k_end) {
        if (uk >= 0 && !OUT) {
          if (V4) fma4(acc4, fv4, t4);
          else acc += fv * t;
          if (DUAL) {
            if (V4) fma4(*acc_b, fv4, t4b);
            else acc_b->x += fv * tb;
          }
        }
        t = 0.f;
        tb = 0.f;
        t4 = make_float4(0.f, 0.f, 0.f, 0.f);
        t4b = t4;
        uk = -1;
        if (k >= nq) { done = true; break; }
        k_beg = k_end;
        k_end += (q_e[k] - q_b[k] + 31) / 32;
        uk = q_i[k];
        if (V4) fv4 = ld_fv4(uk);
        else fv = cok ? Fv[(int64_t)uk * d + c] : 0.f;
        ++k;
      }
      if (done) break;
      const int64_t qb = q_b[k - 1], qe = q_e[k - 1];
      const int64_t tt = qb + (g - k_beg) * 32 + lane;
      const int32_t w = tt < qe ? L[tt] : -1;
      if (V4) h4_chunk4<OUT, DUAL>(keys, ids, n_ids, S, w, tt < qe, fv4, t4, lane, F2q, d, &t4b, F2bq);
      else h4_chunk<OUT, CAP, MAXID, DUAL>(keys, ids, n_ids, S, w, tt < qe, fv, t, lane, F2c, d, &tb, F2bc);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) { *q_n = 0; *grab = 0; }
  __syncthreads();
  if (!V4) acc4.x = acc;
  return acc4;
}

// SMEMS: the S1 values live in SHARED memory (H4S_KEYS rows of 32 floats, one conflict-free
// warp-wide smem atomic per wedge) with partitions sized for H4S_PART distinct keys, instead
// of the per-CTA L2 slab (one 128-byte L2 reduction per wedge)
constexpr int H4S_CAP = 2048;    // hash slots
constexpr int H4S_KEYS = 1024;   // value rows (32 floats each: 128 KB)
constexpr int H4S_PART = 384;    // expected distinct keys per partition (bound-based)
constexpr int H4S_DEG_CAP = 4096;

template <bool V4, bool DUAL = false, bool SMEMS = false>
__global__ void __launch_bounds__(H4_THREADS, H4_CTAS) dhn4_kernel(DhnArgs a) {
  constexpr int CAP = SMEMS ? H4S_CAP : H4_CAP;
  constexpr int MAXID = SMEMS ? H4S_KEYS : (1 << 30);
  constexpr int PART = SMEMS ? H4S_PART : H4_PART;
  constexpr int DEGCAP = SMEMS ? H4S_DEG_CAP : H4_DEG_CAP;
  extern __shared__ int h4[];
  int* keys = h4;
  int* ids = h4 + CAP;                                     // compact id of each slot
  float* s_red = reinterpret_cast<float*>(ids + CAP);      // [H4_WARPS][32]
  int* cur_out = reinterpret_cast<int*>(s_red + H4_WARPS * 32);   // [DEGCAP]
  int* cur_in = cur_out + DEGCAP;                                   // [DEGCAP]
  int64_t* q_b = reinterpret_cast<int64_t*>(cur_in + DEGCAP);      // [H4_LONG_MAX]
  int64_t* q_e = q_b + H4_LONG_MAX;
  int* q_i = reinterpret_cast<int*>(q_e + H4_LONG_MAX);
  // S1 values by compact id: shared (SMEMS, after the queue) or the CTA's L2 slab
  float* S = SMEMS ? reinterpret_cast<float*>(
                         (reinterpret_cast<uintptr_t>(q_i + H4_LONG_MAX) + 15) & ~uintptr_t(15))
                   : a.slab + (int64_t)blockIdx.x * a.cta_stride;
  __shared__ int s_root, q_n, n_ids, grab;
  __shared__ int s_cnt[2];   // long runs queued / walked inline (queue full)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = a.d;
  for (int i = threadIdx.x; i < CAP; i += H4_THREADS) { keys[i] = -1; ids[i] = -1; }
  if (SMEMS)
    for (int i = threadIdx.x; i < H4S_KEYS * 8; i += H4_THREADS)
      reinterpret_cast<float4*>(S)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x == 0) { q_n = 0; n_ids = 0; grab = 0; s_cnt[0] = 0; s_cnt[1] = 0; }
  RNN_PROBE(long long t_last = clock64();)
  unsigned long long c_roots = 0, c_parts = 0, c_chunked = 0, c_multi = 0;   // thread 0
  for (;;) {
    const int64_t n = dhn_next_root(a, &s_root);
    if (n < 0) break;
    ++c_roots;
    const int32_t r = a.row_of[n];
    const int64_t ib = a.sp[r], ie = a.sp[r + 1];
    const int64_t pb = a.gp[n], pe = a.gp[n + 1];
    const int deg_out = (int)(pe - pb), deg_in = (int)(ie - ib);
    const bool cur_ok = deg_out <= DEGCAP && deg_in <= DEGCAP;
    const int64_t bound = a.wout[n] < (uint32_t)a.G ? (int64_t)a.wout[n] : a.G;
    int bits = 0;
    while (bits < H4_HBITS && ((int64_t)PART << bits) < bound) ++bits;
    H4Root R{n, ib, pb, 0, 1u << bits, 0, H4_HBITS - bits, cur_ok, false};
    // lanes test 32 neighbours per step only when a neighbour's list has under one entry
    // per partition on average (hubs); otherwise one neighbour per warp
    R.chunked = (int64_t)R.P * deg_out > (int64_t)a.wout[n];
    c_multi += R.P > 1;
    for (int c0 = 0; c0 < d; c0 += 32) {
      const int c = c0 + lane;
      const bool cok = c < d;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f), acc_b = acc;
      if (cur_ok) {
        for (int i = threadIdx.x; i < deg_out; i += H4_THREADS) cur_out[i] = 0;
        for (int i = threadIdx.x; i < deg_in; i += H4_THREADS) cur_in[i] = 0;
      }
      __syncthreads();
      H4_T(0);
      for (uint32_t part = 0; part < R.P; ++part) {
        R.part = part;
        ++c_parts;
        c_chunked += R.chunked;
        // (1) S1(w) += f1(v) over out-wedges n -> v -> w of this partition
        R.deg = deg_out;
        h4_sweep<true, V4, false, CAP, MAXID>(a, R, keys, ids, &n_ids, S, cur_out, q_i, q_b, q_e,
                                              &q_n, &grab, c, cok, s_cnt);
        H4_T(1);
        // (3) acc += f3(p) (.) G(w) over in-wedges w -> p -> n of this partition
        R.deg = deg_in;
        {
          const float4 r4 = h4_sweep<false, V4, DUAL, CAP, MAXID>(a, R, keys, ids, &n_ids, S, cur_in,
                                                                  q_i, q_b, q_e, &q_n, &grab, c,
                                                                  cok, s_cnt, &acc_b);
          acc.x += r4.x; acc.y += r4.y; acc.z += r4.z; acc.w += r4.w;
        }
        H4_T(3);
        // (4) clear the table for the next partition / root
        {
          const int nz = (n_ids < MAXID ? n_ids : MAXID) * 8;
          for (int i = threadIdx.x; i < nz; i += H4_THREADS) {   // dense prefix, float4
            if (SMEMS) reinterpret_cast<float4*>(S)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            else __stcg(reinterpret_cast<float4*>(S) + i, make_float4(0.f, 0.f, 0.f, 0.f));
          }
        }
        for (int i = threadIdx.x; i < CAP; i += H4_THREADS) { keys[i] = -1; ids[i] = -1; }
        __syncthreads();
        if (threadIdx.x == 0) n_ids = 0;
        __syncthreads();
        H4_T(4);
      }
      if (V4) {
        // sum the four hit slots (lanes cq, cq + 8, cq + 16, cq + 24), then lane cq < 8 holds
        // channels 4 cq .. 4 cq + 3
#pragma unroll
        for (int m = 8; m < 32; m <<= 1) {
          acc.x += __shfl_xor_sync(FULL, acc.x, m); acc.y += __shfl_xor_sync(FULL, acc.y, m);
          acc.z += __shfl_xor_sync(FULL, acc.z, m); acc.w += __shfl_xor_sync(FULL, acc.w, m);
        }
        if (lane < 8) *reinterpret_cast<float4*>(&s_red[warp * 32 + 4 * lane]) = acc;
      } else {
        s_red[warp * 32 + lane] = acc.x;
      }
      __syncthreads();
      if (warp == 0) {
        float s = 0.f;
        for (int w = 0; w < H4_WARPS; ++w) s += s_red[w * 32 + lane];
        if (cok) dhn_store(a, n, c, s);
      }
      __syncthreads();
      if (DUAL) {   // the second middle operand's result (no root multiplier)
        if (V4) {
#pragma unroll
          for (int m = 8; m < 32; m <<= 1) {
            acc_b.x += __shfl_xor_sync(FULL, acc_b.x, m); acc_b.y += __shfl_xor_sync(FULL, acc_b.y, m);
            acc_b.z += __shfl_xor_sync(FULL, acc_b.z, m); acc_b.w += __shfl_xor_sync(FULL, acc_b.w, m);
          }
          if (lane < 8) *reinterpret_cast<float4*>(&s_red[warp * 32 + 4 * lane]) = acc_b;
        } else {
          s_red[warp * 32 + lane] = acc_b.x;
        }
        __syncthreads();
        if (warp == 0) {
          float s = 0.f;
          for (int w = 0; w < H4_WARPS; ++w) s += s_red[w * 32 + lane];
          const int64_t orow = a.out_by_row ? (int64_t)a.row_of[n] : n;
          if (cok) a.out_b[orow * a.ld_out + c] = s;
        }
        __syncthreads();
      }
      H4_T(5);
    }
  }
  if (threadIdx.x == 0) {
    atomicAdd(&g_dhn_paths[2], c_roots);
    atomicAdd(&g_dhn_paths[3], c_parts);
    atomicAdd(&g_dhn_paths[4], c_chunked);
    atomicAdd(&g_dhn_paths[5], (unsigned long long)s_cnt[0]);
    atomicAdd(&g_dhn_paths[6], (unsigned long long)s_cnt[1]);
    atomicAdd(&g_dhn_paths[7], c_multi);
  }
}

// -------------------------------------------------------------------------------------
// C4, slot-indexed (the default when rows are whole float4s): the partitioned walk of
// dhn4_kernel with three changes that remove its serialised per-hit work (ncu, 0.03-scale
// products graph: the walk issued ~35 warp instructions per wedge, half of them in the
// ballot / ffs hit selection and the id-publication spin of h4_insert):
//  * the S1 value row of key w IS its hash slot (rows [CAP][32] per CTA): an insert is one
//    shared-memory CAS, with no compact id to draw and publish;
//  * ONE hash of w gives both the partition (top bits; the lists are sorted by them) and the
//    slot (low bits);
//  * a run sorted by partition enters the current partition as a lane PREFIX of every
//    32-entry chunk, so round r's lane group sub = lane / 8 serves hit 4 r + sub directly.
// Two chunks of a run are loaded per step.  The table is cleared row by row (occupied slots).
// -------------------------------------------------------------------------------------
#ifndef H4S_INFLIGHT
#define H4S_INFLIGHT 4   // IN sweep: hits per lane group in flight per round (x4 per warp)
#endif
__device__ __forceinline__ uint32_t h4s_hash(int32_t w) { return dhn_hash((uint32_t)w ^ 0x5bd1e995u); }
__device__ __forceinline__ int h4s_insert(int* keys, uint32_t H, int w) {
  uint32_t s = H & (uint32_t)(H4_CAP - 1);
  for (int t = 0; t < H4_CAP; ++t) {
    const int prev = atomicCAS(&keys[s], -1, w);
    if (prev == -1 || prev == w) return (int)s;
    s = (s + 1) & (uint32_t)(H4_CAP - 1);
  }
  return -1;
}
__device__ __forceinline__ int h4s_find(const int* keys, uint32_t H, int w) {
  uint32_t s = H & (uint32_t)(H4_CAP - 1);
  for (int t = 0; t < H4_CAP; ++t) {
    const int k = keys[s];
    if (k == w) return (int)s;
    if (k == -1) return -1;
    s = (s + 1) & (uint32_t)(H4_CAP - 1);
  }
  return -1;
}

// one 32-entry chunk whose first cnt lanes are in the partition.  OUT: insert w, add f1(v) to
// row slot(w) (one red.global.add.v4.f32 per lane: lane group sub carries hit 4 r + sub,
// lane % 8 its channel quad).  IN: find w, t += S1(w) (.) f2(w) (8 hits in flight).
template <bool OUT, bool DUAL>
__device__ __forceinline__ void h4s_chunk(int* keys, float* S, int32_t w, uint32_t H, bool in,
                                          int cnt, const float4& fv4, float4& t4, float4& t4b,
                                          int lane, const float* F2q, const float* F2bq, int d) {
  const int sub = lane >> 3, cq = lane & 7;
  if (OUT) {
    const int sl = (in && w >= 0) ? h4s_insert(keys, H, w) : -1;
    if (in && w >= 0 && sl < 0) atomicAdd(&g_dhn_paths[8], 1ull);   // table full (tests: 0)
    for (int q0 = 0; q0 < cnt; q0 += 4) {
      const int q = q0 + sub;
      const int slq = __shfl_sync(FULL, sl, q & 31);
      if (q < cnt && slq >= 0)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(S + slq * 32 + 4 * cq),
                     "f"(fv4.x), "f"(fv4.y), "f"(fv4.z), "f"(fv4.w)
                     : "memory");
    }
  } else {
    const int sl = (in && w >= 0) ? h4s_find(keys, H, w) : -1;
    // (the dual-middle walk keeps 2 in flight: a third operand row per hit spills at 4)
    constexpr int NF = DUAL ? 2 : H4S_INFLIGHT;
    for (int q0 = 0; q0 < cnt; q0 += 4 * NF) {
      float4 x[NF], y[NF], yb[NF];
#pragma unroll
      for (int u = 0; u < NF; ++u) {
        const int q = q0 + 4 * u + sub;
        const int slq = __shfl_sync(FULL, sl, q & 31);
        const int wq = __shfl_sync(FULL, w, q & 31);
        const bool ok = q < cnt && slq >= 0;
        x[u] = ok ? __ldcg(reinterpret_cast<const float4*>(S + slq * 32 + 4 * cq)) : f4_zero();
        y[u] = ok ? __ldg(reinterpret_cast<const float4*>(F2q + (int64_t)wq * d)) : f4_zero();
        if (DUAL)
          yb[u] = ok ? __ldg(reinterpret_cast<const float4*>(F2bq + (int64_t)wq * d)) : f4_zero();
      }
#pragma unroll
      for (int u = 0; u < NF; ++u) {
        t4.x = fmaf(x[u].x, y[u].x, t4.x); t4.y = fmaf(x[u].y, y[u].y, t4.y);
        t4.z = fmaf(x[u].z, y[u].z, t4.z); t4.w = fmaf(x[u].w, y[u].w, t4.w);
        if (DUAL) {
          t4b.x = fmaf(x[u].x, yb[u].x, t4b.x); t4b.y = fmaf(x[u].y, yb[u].y, t4b.y);
          t4b.z = fmaf(x[u].z, yb[u].z, t4b.z); t4b.w = fmaf(x[u].w, yb[u].w, t4b.w);
        }
      }
    }
  }
}

// One side of one partition (as h4_sweep): phase A walks the runs of the neighbours the warps
// grab, queueing runs longer than H4_LONG; phase B splits the queued runs over all warps.
template <bool OUT, bool DUAL>
__device__ float4 h4s_sweep(const DhnArgs& a, const H4Root& R, int* keys, float* S, int* cur,
                            int* q_i, int64_t* q_b, int64_t* q_e, int* q_n, int* grab, int c0,
                            int* s_cnt, float4* acc_b) {
  const int lane = threadIdx.x & 31;
  const int32_t* L = OUT ? a.nbrh : a.sgh;
  const float* Fv = OUT ? a.F1 : a.F3;
  const int d = a.d;
  const int cq4 = c0 + 4 * (lane & 7);   // this lane's channel quad
  const bool cok4 = cq4 < d;
  const float* F2q = a.F2 + (cok4 ? cq4 : 0);
  const float* F2bq = DUAL ? a.F2b + (cok4 ? cq4 : 0) : nullptr;
  float4 acc4 = f4_zero();
  auto ld_fv4 = [&](int32_t u) {
    return cok4 ? __ldg(reinterpret_cast<const float4*>(Fv + (int64_t)u * d + cq4)) : f4_zero();
  };
  auto fma4 = [](float4& acc_, const float4& f, const float4& t_) {
    acc_.x = fmaf(f.x, t_.x, acc_.x); acc_.y = fmaf(f.y, t_.y, acc_.y);
    acc_.z = fmaf(f.z, t_.z, acc_.z); acc_.w = fmaf(f.w, t_.w, acc_.w);
  };
  auto in_part = [&](uint32_t H) { return ((H >> 16) >> R.sh) == R.part; };
  const int step = R.chunked ? 32 : 1;
  for (;;) {
    int base = 0;
    if (lane == 0) base = atomicAdd(grab, step);
    base = __shfl_sync(FULL, base, 0);
    if (base >= R.deg) break;
    const int i = R.chunked ? base + lane : base;
    int32_t u = -1;
    int64_t b0 = 0, e0 = 0, s0 = 0;
    bool has = false;
    if (i < R.deg && (R.chunked || lane == 0)) {
      if (OUT) {
        u = a.nbr[R.pb + i];
        if (u >= 0) { s0 = a.gp[u]; e0 = a.gp[u + 1]; }
      } else {
        u = a.sg[R.ib + i];
        const int32_t ru = a.row_of[u];
        s0 = a.sp[ru];
        e0 = a.sp[ru + 1];
      }
      if (u >= 0) {
        b0 = R.cur_ok ? s0 + cur[i] : h4_lower(L, s0, e0, R.part, R.sh);
        has = b0 < e0 && (h4_top(L[b0]) >> R.sh) == R.part;
      }
    }
    unsigned hb = __ballot_sync(FULL, has);
    while (hb) {
      const int j = __ffs(hb) - 1;
      hb &= hb - 1;
      const int32_t uj = __shfl_sync(FULL, u, j);
      const int64_t bj = __shfl_sync(FULL, b0, j), ej = __shfl_sync(FULL, e0, j);
      const int64_t sj = __shfl_sync(FULL, s0, j);
      const int ij = __shfl_sync(FULL, i, j);
      int64_t re = -1;
      if (ej - bj > H4_LONG) {
        re = R.P == 1 ? ej : h4_lower(L, bj, ej, R.part + 1, R.sh);
        if (re - bj <= H4_LONG) re = -1;
      }
      if (re >= 0) {
        int slot = 0;
        if (lane == 0) slot = atomicAdd(q_n, 1);
        slot = __shfl_sync(FULL, slot, 0);
        if (slot < H4_LONG_MAX) {
          if (lane == 0) { q_i[slot] = uj; q_b[slot] = bj; q_e[slot] = re; atomicAdd(&s_cnt[0], 1); }
          if (R.cur_ok && lane == 0) cur[ij] = (int)(re - sj);
          continue;
        }
        if (lane == 0) atomicAdd(&s_cnt[1], 1);
      }
      const float4 fv4 = ld_fv4(uj);
      float4 t4 = f4_zero(), t4b = f4_zero();
      int64_t t0 = bj;
      for (;;) {
        const int64_t ta = t0 + lane, tb = ta + 32;
        const int32_t wa = ta < ej ? L[ta] : -1;
        const int32_t wb = tb < ej ? L[tb] : -1;
        const uint32_t Ha = h4s_hash(wa), Hb = h4s_hash(wb);
        const bool ina = ta < ej && in_part(Ha);
        const bool inb = tb < ej && in_part(Hb);
        const unsigned ma = __ballot_sync(FULL, ina), mb = __ballot_sync(FULL, inb);
        const int ca = __popc(ma), cb = __popc(mb);
        h4s_chunk<OUT, DUAL>(keys, S, wa, Ha, ina, ca, fv4, t4, t4b, lane, F2q, F2bq, d);
        if (cb) h4s_chunk<OUT, DUAL>(keys, S, wb, Hb, inb, cb, fv4, t4, t4b, lane, F2q, F2bq, d);
        t0 += ca + cb;
        if (mb != FULL) break;
      }
      if (!OUT) {
        fma4(acc4, fv4, t4);
        if (DUAL) fma4(*acc_b, fv4, t4b);
      }
      if (R.cur_ok && lane == 0) cur[ij] = (int)(t0 - sj);
    }
  }
  __syncthreads();
  // phase B: the 32-entry chunks of all queued long runs (every entry in the partition)
  const int nq = *q_n < H4_LONG_MAX ? *q_n : H4_LONG_MAX;
  if (nq > 0) {
    if (threadIdx.x == 0) *grab = 0;
    __syncthreads();
    int k = 0;
    int64_t k_end = 0, k_beg = 0;
    float4 fv4 = f4_zero(), t4 = f4_zero(), t4b = f4_zero();
    int32_t uk = -1;
    for (;;) {
      int g = 0;
      if (lane == 0) g = atomicAdd(grab, 1);
      g = __shfl_sync(FULL, g, 0);
      bool done = false;
      while (g >= k_end) {
        if (uk >= 0 && !OUT) {
          fma4(acc4, fv4, t4);
          if (DUAL) fma4(*acc_b, fv4, t4b);
        }
        t4 = f4_zero();
        t4b = f4_zero();
        uk = -1;
        if (k >= nq) { done = true; break; }
        k_beg = k_end;
        k_end += (q_e[k] - q_b[k] + 31) / 32;
        uk = q_i[k];
        fv4 = ld_fv4(uk);
        ++k;
      }
      if (done) break;
      const int64_t qb = q_b[k - 1], qe = q_e[k - 1];
      const int64_t tt = qb + (g - k_beg) * 32 + lane;
      const int32_t w = tt < qe ? L[tt] : -1;
      const bool in = tt < qe;
      const int cnt = __popc(__ballot_sync(FULL, in));
      h4s_chunk<OUT, DUAL>(keys, S, w, h4s_hash(w), in, cnt, fv4, t4, t4b, lane, F2q, F2bq, d);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) { *q_n = 0; *grab = 0; }
  __syncthreads();
  return acc4;
}

template <bool DUAL>
__global__ void __launch_bounds__(H4_THREADS, H4_CTAS) dhn4s_kernel(DhnArgs a) {
  extern __shared__ int h4[];
  int* keys = h4;
  float* s_red = reinterpret_cast<float*>(keys + H4_CAP);          // [H4_WARPS][32]
  int* cur_out = reinterpret_cast<int*>(s_red + H4_WARPS * 32);     // [H4_DEG_CAP]
  int* cur_in = cur_out + H4_DEG_CAP;                               // [H4_DEG_CAP]
  int64_t* q_b = reinterpret_cast<int64_t*>(cur_in + H4_DEG_CAP);  // [H4_LONG_MAX]
  int64_t* q_e = q_b + H4_LONG_MAX;
  int* q_i = reinterpret_cast<int*>(q_e + H4_LONG_MAX);
  float* S = a.slab + (int64_t)blockIdx.x * a.cta_stride;          // [H4_CAP][32], zero
  __shared__ int s_root, q_n, grab;
  __shared__ int s_cnt[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = a.d;
  const int64_t part_keys = a.part_keys > 0 ? a.part_keys : H4_PART;
  for (int i = threadIdx.x; i < H4_CAP; i += H4_THREADS) keys[i] = -1;
  if (threadIdx.x == 0) { q_n = 0; grab = 0; s_cnt[0] = 0; s_cnt[1] = 0; }
  unsigned long long c_roots = 0, c_parts = 0, c_chunked = 0, c_multi = 0;   // thread 0
  for (;;) {
    const int64_t n = dhn_next_root(a, &s_root);
    if (n < 0) break;
    ++c_roots;
    const int32_t r = a.row_of[n];
    const int64_t ib = a.sp[r], ie = a.sp[r + 1];
    const int64_t pb = a.gp[n], pe = a.gp[n + 1];
    const int deg_out = (int)(pe - pb), deg_in = (int)(ie - ib);
    const bool cur_ok = deg_out <= H4_DEG_CAP && deg_in <= H4_DEG_CAP;
    const int64_t bound = a.wout[n] < (uint32_t)a.G ? (int64_t)a.wout[n] : a.G;
    int bits = 0;
    while (bits < H4_HBITS && (part_keys << bits) < bound) ++bits;
    H4Root R{n, ib, pb, 0, 1u << bits, 0, H4_HBITS - bits, cur_ok, false};
    R.chunked = (int64_t)R.P * deg_out > (int64_t)a.wout[n];
    c_multi += R.P > 1;
    for (int c0 = 0; c0 < d; c0 += 32) {
      float4 acc = f4_zero(), acc_b = f4_zero();
      if (cur_ok) {
        for (int i = threadIdx.x; i < deg_out; i += H4_THREADS) cur_out[i] = 0;
        for (int i = threadIdx.x; i < deg_in; i += H4_THREADS) cur_in[i] = 0;
      }
      __syncthreads();
      for (uint32_t part = 0; part < R.P; ++part) {
        R.part = part;
        ++c_parts;
        c_chunked += R.chunked;
        R.deg = deg_out;
        h4s_sweep<true, false>(a, R, keys, S, cur_out, q_i, q_b, q_e, &q_n, &grab, c0, s_cnt,
                               nullptr);
        R.deg = deg_in;
        acc = f4_add(acc, h4s_sweep<false, DUAL>(a, R, keys, S, cur_in, q_i, q_b, q_e, &q_n,
                                                 &grab, c0, s_cnt, &acc_b));
        // clear the occupied rows and slots for the next partition / root (the sweeps ended
        // with a barrier, so no lane still reads the table)
        for (int i = threadIdx.x; i < H4_CAP; i += H4_THREADS) {
          if (keys[i] != -1) {
            float4* row = reinterpret_cast<float4*>(S + (int64_t)i * 32);
#pragma unroll
            for (int j = 0; j < 8; ++j) __stcg(row + j, f4_zero());
            keys[i] = -1;
          }
        }
        __syncthreads();
      }
      // sum the four hit slots (lanes cq, cq + 8, cq + 16, cq + 24): lane cq < 8 then holds
      // channels c0 + 4 cq .. + 3
#pragma unroll
      for (int m = 8; m < 32; m <<= 1) acc = f4_add(acc, f4_shfl_xor(acc, m));
      if (lane < 8) *reinterpret_cast<float4*>(&s_red[warp * 32 + 4 * lane]) = acc;
      __syncthreads();
      if (warp == 0) {
        float s = 0.f;
        for (int w = 0; w < H4_WARPS; ++w) s += s_red[w * 32 + lane];
        if (c0 + lane < d) dhn_store(a, n, c0 + lane, s);
      }
      __syncthreads();
      if (DUAL) {
#pragma unroll
        for (int m = 8; m < 32; m <<= 1) acc_b = f4_add(acc_b, f4_shfl_xor(acc_b, m));
        if (lane < 8) *reinterpret_cast<float4*>(&s_red[warp * 32 + 4 * lane]) = acc_b;
        __syncthreads();
        if (warp == 0) {
          float s = 0.f;
          for (int w = 0; w < H4_WARPS; ++w) s += s_red[w * 32 + lane];
          const int64_t orow = a.out_by_row ? (int64_t)a.row_of[n] : n;
          if (c0 + lane < d) a.out_b[orow * a.ld_out + c0 + lane] = s;
        }
        __syncthreads();
      }
    }
  }
  if (threadIdx.x == 0) {
    atomicAdd(&g_dhn_paths[2], c_roots);
    atomicAdd(&g_dhn_paths[3], c_parts);
    atomicAdd(&g_dhn_paths[4], c_chunked);
    atomicAdd(&g_dhn_paths[5], (unsigned long long)s_cnt[0]);
    atomicAdd(&g_dhn_paths[6], (unsigned long long)s_cnt[1]);
    atomicAdd(&g_dhn_paths[7], c_multi);
  }
}

// sort keys of the hash-ordered adjacency lists: (segment << 16) | top 16 bits of hash(w)
__global__ void h4_keys_kernel(const int32_t* __restrict__ seg, const int32_t* __restrict__ val,
                               int64_t E, uint64_t* __restrict__ key, int32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= E) return;
  const int32_t w = val[i];
  key[i] = ((uint64_t)(uint32_t)seg[i] << H4_HBITS) | h4_top(w);
  out[i] = w;
}

// -------------------------------------------------------------------------------------
// C2 and helpers
// -------------------------------------------------------------------------------------
// out(n) = rm(n) (.) sum_{p in group n} f1[src_row[p]]   -- warp per root, lane = channel
__global__ void dhn2_kernel(DhnArgs a, const int32_t* __restrict__ src_row,
                            const float* __restrict__ f1, int64_t ld1) {
  const int64_t n = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (n >= a.G) return;
  const int lane = threadIdx.x & 31;
  const int64_t pb = a.gp[n], pe = a.gp[n + 1];
  for (int c = lane; c < a.d; c += 32) {
    float s = 0.f;
    for (int64_t p = pb; p < pe; ++p) s += f1[(int64_t)src_row[p] * ld1 + c];
    dhn_store(a, n, c, s);
  }
}

// d f1(x) = sum_{n -> x} g(n)  over the transposed CSR of row x (g in group order)
__global__ void dhn2_bwd_kernel(int64_t n_rows, int d, const int64_t* __restrict__ sp,
                                const int32_t* __restrict__ sg, const float* __restrict__ g,
                                float* __restrict__ out, int64_t ld_out) {
  const int64_t x = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (x >= n_rows) return;
  const int lane = threadIdx.x & 31;
  const int64_t b = sp[x], e = sp[x + 1];
  for (int c = lane; c < d; c += 32) {
    float s = 0.f;
    for (int64_t q = b; q < e; ++q) s += g[(int64_t)sg[q] * d + c];
    out[x * ld_out + c] = s;
  }
}

__global__ void grp_of_row_kernel(const int32_t* __restrict__ row_of, int64_t G,
                                  int32_t* __restrict__ gor) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g < G) gor[row_of[g]] = (int32_t)g;
}

__global__ void nbr_kernel(const int32_t* __restrict__ src_row, int64_t E,
                           const int32_t* __restrict__ gor, int32_t* __restrict__ nbr) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < E) nbr[p] = gor[src_row[p]];
}

// F[g, c] = f[row_of[g], c] (* m[g, c] if m: the rotated operand g = f0 (.) dOut)
__global__ void to_group_kernel(const float* __restrict__ f, int64_t ldf,
                                const int32_t* __restrict__ row_of, int64_t G, int d,
                                const float* __restrict__ m, int64_t ldm, float* __restrict__ F) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= G * d) return;
  const int64_t g = i / d;
  const int c = (int)(i % d);
  float v = f ? f[(int64_t)row_of[g] * ldf + c] : 1.f;
  if (m) v *= m[g * ldm + c];
  F[i] = v;
}

// heaviest-first root order: key = 2^24-1 - min(work, 2^24-1)
__global__ void work_kernel(int k, int64_t G, const int64_t* __restrict__ gp,
                            const int32_t* __restrict__ nbr, const int64_t* __restrict__ sp,
                            const int32_t* __restrict__ sg, const int32_t* __restrict__ row_of,
                            uint32_t* __restrict__ key, int32_t* __restrict__ order,
                            uint32_t* __restrict__ wout) {
  const int64_t n = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (n >= G) return;
  const int lane = threadIdx.x & 31;
  int64_t w = 0;
  for (int64_t p = gp[n] + lane; p < gp[n + 1]; p += 32) {
    const int32_t v = nbr[p];
    if (v >= 0) w += gp[v + 1] - gp[v];
  }
  if (k == 4) {
    int64_t o = w;   // out-wedges n -> v -> w: bound on the distinct w of the S1 table
#pragma unroll
    for (int s = 16; s; s >>= 1) o += __shfl_xor_sync(FULL, o, s);
    if (lane == 0) wout[n] = (uint32_t)(o < (int64_t)UINT32_MAX ? o : UINT32_MAX);
    const int32_t r = row_of[n];
    for (int64_t q = sp[r] + lane; q < sp[r + 1]; q += 32) {
      const int32_t rp = row_of[sg[q]];
      w += 2 * (sp[rp + 1] - sp[rp]);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(FULL, w, o);
  if (lane == 0) {
    const uint32_t cap = (1u << 24) - 1;
    key[n] = cap - (uint32_t)(w < (int64_t)cap ? w : cap);
    order[n] = (int32_t)n;
  }
}

// -------------------------------------------------------------------------------------
// Exact closed-walk counts (rnn_dhn_count): C_k(n) with every operand 1, in int64.
// The float kernels above accumulate with fp32 atomics (exact only below 2^24 and in any
// rounding order); this integer path is the homomorphism count itself (PAPER.md:1481,
// Eq. 3 :1500 with mu = 1): (A^k)_nn for k = 3, 4.  One CTA per root (heaviest first), a
// shared-memory hash of group id -> uint64 count, and P = 2^b passes over hash partitions
// of the keyed vertex when the root could name more keys than the table holds:
//   k = 3: key = in-neighbour w of n (count = closing Edge rows w -> n); every out-wedge
//          n -> v -> w of the pass adds count(w);
//   k = 4: key = middle vertex w, count = S1(n, w) = #(n -> v -> w); every in-wedge
//          w -> p -> n of the pass adds S1(n, w)   (= sum_w S1(n, w) S3(n, w)).
// -------------------------------------------------------------------------------------
constexpr int HC_THREADS = 512;
constexpr int HC_CAP = 8192;      // slots: int32 key + uint64 count = 96 KB
constexpr int HC_PART = HC_CAP / 2;

struct CountArgs {
  int k;
  int64_t G;
  const int64_t* gp; const int32_t* nbr; const int64_t* sp; const int32_t* sg;
  const int32_t* row_of; const int32_t* order; int* counter; const uint32_t* wout;
  int64_t* out;
};

__device__ __forceinline__ uint32_t hc_part(int32_t w, int bits) {
  return bits ? dhn_hash((uint32_t)w ^ 0x2545F491u) >> (32 - bits) : 0u;
}

// count one occurrence of key w.  The table never fills: a pass holds at most
// max(bound, 2 * HC_PART / 2^bits ...) keys -- cap >= 2 (bound / P + 1) -- so a failed insert
// (slot -1) cannot happen; it is still guarded (no out-of-range shared store).
__device__ __forceinline__ void hc_add(unsigned long long* cnt, int* keys, int mask, int32_t w) {
  const int sl = hs_insert(keys, mask, w);
  if (sl >= 0) atomicAdd(&cnt[sl], 1ull);
}

__global__ void __launch_bounds__(HC_THREADS) dhn_count_kernel(CountArgs a) {
  extern __shared__ unsigned long long hc_raw[];
  unsigned long long* cnt = hc_raw;                       // [HC_CAP]
  int* keys = reinterpret_cast<int*>(cnt + HC_CAP);        // [HC_CAP]
  __shared__ int s_root;
  __shared__ long long s_tot[HC_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = HC_THREADS / 32;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_root = atomicAdd(a.counter, 1);
    __syncthreads();
    if (s_root >= a.G) break;
    const int64_t n = a.order[s_root];
    const int32_t r = a.row_of[n];
    const int64_t pb = a.gp[n], pe = a.gp[n + 1], ib = a.sp[r], ie = a.sp[r + 1];
    // bound on the distinct keys of the table: k = 3 the in-degree, k = 4 the out-wedges
    int64_t bound = a.k == 3 ? ie - ib : (int64_t)a.wout[n];
    if (bound > a.G) bound = a.G;
    int bits = 0;
    while (((int64_t)HC_PART << bits) < bound) ++bits;
    int cap = 32;
    while (cap < HC_CAP && (int64_t)cap < 2 * ((bound >> bits) + 1)) cap <<= 1;
    const int mask = cap - 1;
    long long tot = 0;
    for (uint32_t part = 0; part < (1u << bits); ++part) {
      for (int i = threadIdx.x; i < cap; i += HC_THREADS) { keys[i] = -1; cnt[i] = 0; }
      __syncthreads();
      if (a.k == 3) {
        // keys: in-neighbours of this partition, with multiplicity
        for (int64_t q = ib + threadIdx.x; q < ie; q += HC_THREADS) {
          const int32_t w = a.sg[q];
          if (hc_part(w, bits) == part) hc_add(cnt, keys, mask, w);
        }
      } else {
        // S1(n, w): out-wedges n -> v -> w (w must have out-edges to continue the walk)
        for (int64_t pos = pb + warp; pos < pe; pos += NW) {
          const int32_t v = a.nbr[pos];
          if (v < 0) continue;
          for (int64_t i = a.gp[v] + lane; i < a.gp[v + 1]; i += 32) {
            const int32_t w = a.nbr[i];
            if (w >= 0 && hc_part(w, bits) == part) hc_add(cnt, keys, mask, w);
          }
        }
      }
      __syncthreads();
      if (a.k == 3) {
        // out-wedges n -> v -> w closing on a keyed in-neighbour w
        for (int64_t pos = pb + warp; pos < pe; pos += NW) {
          const int32_t v = a.nbr[pos];
          if (v < 0) continue;
          for (int64_t i = a.gp[v] + lane; i < a.gp[v + 1]; i += 32) {
            const int32_t w = a.nbr[i];
            if (w >= 0 && hc_part(w, bits) == part) {
              const int sl = hs_find(keys, mask, w);
              if (sl >= 0) tot += (long long)cnt[sl];
            }
          }
        }
      } else {
        // in-wedges w -> p -> n: p = in-neighbour of n, w = in-neighbour of p
        for (int64_t q = ib + warp; q < ie; q += NW) {
          const int32_t pg = a.sg[q];
          const int32_t rp = a.row_of[pg];
          for (int64_t i = a.sp[rp] + lane; i < a.sp[rp + 1]; i += 32) {
            const int32_t w = a.sg[i];
            if (hc_part(w, bits) == part) {
              const int sl = hs_find(keys, mask, w);
              if (sl >= 0) tot += (long long)cnt[sl];
            }
          }
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
    if (lane == 0) s_tot[warp] = tot;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0;
      for (int w = 0; w < NW; ++w) t += s_tot[w];
      a.out[n] = t;
    }
  }
}

__global__ void dhn_count2_kernel(int64_t G, const int64_t* __restrict__ gp, int64_t* __restrict__ out) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g < G) out[g] = gp[g + 1] - gp[g];
}

// active roots: every key gets bit 24 (sorted after all real keys); listed roots clear it
// and count themselves once (duplicates and out-of-range ids are ignored)
__global__ void root_exclude_kernel(uint32_t* __restrict__ key, int64_t G) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g < G) key[g] |= 1u << 24;
}
__global__ void root_include_kernel(const int32_t* __restrict__ roots, int64_t n, int64_t G,
                                    uint32_t* __restrict__ key, int* __restrict__ n_active) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t g = roots[i];
  if (g < 0 || g >= G) return;
  const uint32_t old = atomicAnd(&key[g], ~(1u << 24));
  if (old & (1u << 24)) atomicAdd(n_active, 1);
}
__global__ void set_int_kernel(int* p, int v) { *p = v; }

// ---------------------------------------------------------------------------------------
// plan: workspace layout
// ---------------------------------------------------------------------------------------
struct Plan {
  int k, d, n_cta;
  int64_t G, E, R;
  size_t fixed, per_cta;
  const int32_t* roots = nullptr;   // active root subset (group ids); NULL = every group
  int64_t n_roots = 0;
};
constexpr int ACTIVE_SLOT = 63;     // counter[63]: number of active roots (device)

struct Bufs {
  int32_t* gor; int32_t* nbr; float* F[4]; uint32_t* key; int32_t* order; int* counter;
  uint32_t* wout; void* sort_ws; char* cta;
  uint64_t* hkey; int32_t* nbrh; int32_t* sgh;   // k = 4: hash-ordered adjacency lists
};

Bufs carve(const Plan& P, void* base, size_t* used = nullptr) {
  Carve c(base);
  Bufs b;
  b.gor = c.take<int32_t>(P.R);
  b.nbr = c.take<int32_t>(P.E);
  for (int i = 0; i < 4; ++i) b.F[i] = i < P.k ? c.take<float>((size_t)P.G * P.d) : nullptr;
  b.key = c.take<uint32_t>(P.G);
  b.order = c.take<int32_t>(P.G);
  b.counter = c.take<int>(64);
  b.wout = c.take<uint32_t>(P.G);
  b.hkey = P.k == 4 ? c.take<uint64_t>(P.E) : nullptr;
  b.nbrh = P.k == 4 ? c.take<int32_t>(P.E) : nullptr;
  b.sgh = P.k == 4 ? c.take<int32_t>(P.E) : nullptr;
  b.sort_ws = c.take<char>(radix_sort_workspace_bytes(P.k == 4 ? std::max(P.G, P.E) : P.G));
  b.cta = c.take<char>(0);
  if (used) *used = c.used;
  return b;
}

Plan make_plan(const rnn_join_index* adj, int k, int d) {
  Plan P;
  P.k = k; P.d = d;
  P.G = adj->n_groups; P.E = adj->n_join_rows; P.R = adj->n_src_rows;
  P.n_cta = (int)std::min<int64_t>((int64_t)num_sms() * (k == 4 ? H4_CTAS : DHN_CTAS_PER_SM),
                                    std::max<int64_t>(P.G, 1));
  // k = 3: per-CTA global mark array for roots whose in-degree exceeds the smem hash set;
  // k = 4: per-CTA value slab of the S1 hash table (H4_CAP x 32 floats, zero between roots)
  P.per_cta = k == 3 ? ((size_t)P.G * sizeof(int32_t) + 255) & ~size_t(255)
            : k == 4 ? (size_t)H4_CAP * 32 * sizeof(float) : 0;
  carve(P, nullptr, &P.fixed);
  P.fixed = (P.fixed + 255) & ~size_t(255);
  return P;
}

rnn_status check_adj(const rnn_join_index* adj, int k, int d) {
  RNN_REQUIRE(adj, RNN_ERR_INVALID_ARGUMENT, "adj is NULL");
  RNN_REQUIRE(k >= 2 && k <= 4, RNN_ERR_UNSUPPORTED, "DHN pattern length k=%d (2..4 supported)", k);
  RNN_REQUIRE(d >= 1 && d <= 128, RNN_ERR_UNSUPPORTED, "DHN operand width d=%d (1..128)", d);
  RNN_REQUIRE(adj->n_src_rows == adj->n_dst_rows, RNN_ERR_SHAPE_MISMATCH,
              "DHN adjacency must join Edge with one node relation (n_src_rows %lld != n_dst_rows %lld)",
              (long long)adj->n_src_rows, (long long)adj->n_dst_rows);
  RNN_REQUIRE(adj->n_groups == 0 || (adj->group_ptr && adj->src_row && adj->group_dst_row),
              RNN_ERR_INVALID_ARGUMENT, "index arrays missing");
  RNN_REQUIRE(adj->n_groups == 0 || (adj->src_ptr && adj->src_group), RNN_ERR_INVALID_ARGUMENT,
              "DHN needs the transposed CSR (index built without RNN_IDX_NO_TRANSPOSE)");
  RNN_REQUIRE(adj->n_groups <= INT32_MAX && adj->n_src_rows < INT32_MAX, RNN_ERR_UNSUPPORTED,
              "DHN group / row ids are int32");
  RNN_REQUIRE(k != 4 || adj->n_groups == 0 || (adj->pos_group && adj->src_seg),
              RNN_ERR_INVALID_ARGUMENT, "DHN k = 4 needs pos_group and src_seg in the index");
  return RNN_OK;
}

rnn_status check_ops(const rnn_operand* f, int k, int d, int64_t R) {
  RNN_REQUIRE(f, RNN_ERR_INVALID_ARGUMENT, "operands NULL");
  for (int i = 0; i < k; ++i) {
    RNN_REQUIRE(f[i].mode == RNN_BY_ROW, RNN_ERR_UNSUPPORTED, "DHN operands are RNN_BY_ROW");
    if (i == 0 && !f[i].data) continue;
    RNN_REQUIRE(f[i].data || R == 0, RNN_ERR_INVALID_ARGUMENT, "operand f[%d] missing", i);
    RNN_REQUIRE(f[i].dim == d, RNN_ERR_SHAPE_MISMATCH, "operand f[%d] dim %d != f[1] dim %d", i,
                f[i].dim, d);
    RNN_REQUIRE(f[i].ld >= d, RNN_ERR_SHAPE_MISMATCH, "operand f[%d] ld %lld < dim", i,
                (long long)f[i].ld);
  }
  return RNN_OK;
}

// one walk-aggregate launch (k >= 3) with operands W[0..k-2] in group order
rnn_status walk(const Plan& P, const Bufs& b, const rnn_join_index* adj, const float* const* W,
                const float* rm, int64_t ld_rm, int rm_by_group, float* out, int64_t ld_out,
                int out_by_row, int launch_id, cudaStream_t st, float* sum_out = nullptr,
                int64_t ld_sum = 0, const float* Fb = nullptr, float* out_b = nullptr) {
  // Fb (symmetric Edge): k = 3 second first-hop operand, k = 4 second middle operand
  DhnArgs a{};
  a.sum_out = sum_out; a.ld_sum = ld_sum;
  a.F2b = P.k == 4 ? Fb : nullptr;
  a.F1b = P.k == 3 ? Fb : nullptr;
  a.out_b = out_b;
  const float* F2b = a.F2b;
  a.G = P.G; a.d = P.d;
  a.gp = adj->group_ptr; a.nbr = b.nbr; a.sp = adj->src_ptr; a.sg = adj->src_group;
  a.row_of = adj->group_dst_row;
  a.F1 = W[0]; a.F2 = W[1]; a.F3 = P.k == 4 ? W[2] : nullptr;
  a.rm = rm; a.ld_rm = ld_rm; a.rm_by_group = rm_by_group;
  a.out = out; a.ld_out = ld_out; a.out_by_row = out_by_row;
  a.order = b.order; a.counter = b.counter + launch_id;
  a.n_active = b.counter + ACTIVE_SLOT;
  a.cta_stride = (int64_t)(P.per_cta / (P.k == 3 ? sizeof(int32_t) : sizeof(float)));
  // the kernels leave their per-CTA scratch zeroed, so only the first launch clears it
  if (launch_id == 0) RNN_CUDA(cudaMemsetAsync(b.cta, 0, P.per_cta * P.n_cta, st));
  if (P.k == 3) {
    a.mark = reinterpret_cast<int*>(b.cta);
    const int dpl = (P.d + 31) / 32;
    const size_t smem = (2 * H3_CAP + H3_MAX_INDEG) * sizeof(int) +
                        (size_t)DHN_WARPS * dpl * 32 * sizeof(float) +
                        H3_QMAX * (2 * sizeof(int64_t) + 3 * sizeof(int32_t));
    auto kern = a.F1b ? (dpl == 1 ? dhn3_kernel<1, true> : dpl == 2 ? dhn3_kernel<2, true>
                         : dpl == 3 ? dhn3_kernel<3, true> : dhn3_kernel<4, true>)
                      : (dpl == 1 ? dhn3_kernel<1> : dpl == 2 ? dhn3_kernel<2>
                         : dpl == 3 ? dhn3_kernel<3> : dhn3_kernel<4>);
    RNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<P.n_cta, DHN_THREADS, smem, st>>>(a);
  } else {
    a.wout = b.wout; a.nbrh = b.nbrh; a.sgh = b.sgh;
    a.slab = reinterpret_cast<float*>(b.cta);
    // the L2 slab (default) or shared-memory S1 values (RNN_DHN_SMEM_S1=1; measured 5.8x
    // slower on the products graph, profiles/r02/dhn: the 384-key partitions multiply the
    // passes over every adjacency list and the 128 KB value table leaves one CTA per SM)
    const bool smem_s1 = getenv("RNN_DHN_SMEM_S1") != nullptr;
    if (smem_s1) {
      const size_t smem_s = 2 * H4S_CAP * sizeof(int) + (size_t)H4_WARPS * 32 * sizeof(float) +
                            2 * H4S_DEG_CAP * sizeof(int) +
                            H4_LONG_MAX * (2 * sizeof(int64_t) + sizeof(int)) + 16 +
                            (size_t)H4S_KEYS * 32 * sizeof(float);
      auto kern = a.F2b ? dhn4_kernel<false, true, true> : dhn4_kernel<false, false, true>;
      RNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s));
      kern<<<P.n_cta, H4_THREADS, smem_s, st>>>(a);
      RNN_LAUNCH_CHECK();
      return RNN_OK;
    }
    const size_t smem = 2 * H4_CAP * sizeof(int) + (size_t)H4_WARPS * 32 * sizeof(float) +
                        2 * H4_DEG_CAP * sizeof(int) + H4_LONG_MAX * (2 * sizeof(int64_t) + sizeof(int));
    // four hits per instruction (float4 per lane) when rows are whole float4s
    static const bool scalar = getenv("RNN_DHN_SCALAR") != nullptr;
    const bool v4 = !scalar && P.d % 4 == 0 && aligned16(a.F1) && aligned16(a.F2) &&
                    aligned16(a.F3) && aligned16(a.slab);
    RNN_REQUIRE(!F2b || (v4 && aligned16(F2b)), RNN_ERR_UNSUPPORTED,
                "dual-middle C4 walk needs the float4 path");
    // slot-indexed walk (default); RNN_DHN_COMPACT_IDS=1 selects the compact-id walk it
    // replaced (kept for measurement, profiles/r02/dhn)
    const bool compact = getenv("RNN_DHN_COMPACT_IDS") != nullptr;   // read per launch (tests)
    if (v4 && !compact) {
      static const int part_keys = getenv("RNN_DHN_PART_KEYS") ? atoi(getenv("RNN_DHN_PART_KEYS")) : 0;
      a.part_keys = std::min(part_keys, H4_PART);
      const size_t smem_s = H4_CAP * sizeof(int) + (size_t)H4_WARPS * 32 * sizeof(float) +
                            2 * H4_DEG_CAP * sizeof(int) +
                            H4_LONG_MAX * (2 * sizeof(int64_t) + sizeof(int));
      auto kern = F2b ? dhn4s_kernel<true> : dhn4s_kernel<false>;
      RNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s));
      kern<<<P.n_cta, H4_THREADS, smem_s, st>>>(a);
      RNN_LAUNCH_CHECK();
      return RNN_OK;
    }
    auto kern = F2b ? dhn4_kernel<true, true> : v4 ? dhn4_kernel<true> : dhn4_kernel<false>;
    RNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<P.n_cta, H4_THREADS, smem, st>>>(a);
  }
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

// shared preparation: group map, neighbour groups, root order, group-ordered operands
rnn_status prepare(const Plan& P, const Bufs& b, const rnn_join_index* adj, cudaStream_t st) {
  RNN_CUDA(cudaMemsetAsync(b.gor, 0xff, sizeof(int32_t) * std::max<int64_t>(P.R, 1), st));
  RNN_CUDA(cudaMemsetAsync(b.counter, 0, sizeof(int) * 64, st));
  if (P.G == 0) return RNN_OK;
  grp_of_row_kernel<<<(unsigned)ceil_div(P.G, 256), 256, 0, st>>>(adj->group_dst_row, P.G, b.gor);
  if (P.E > 0)
    nbr_kernel<<<(unsigned)ceil_div(P.E, 256), 256, 0, st>>>(adj->src_row, P.E, b.gor, b.nbr);
  RNN_LAUNCH_CHECK();
  if (P.k >= 3) {
    work_kernel<<<(unsigned)ceil_div(P.G, 8), 256, 0, st>>>(P.k, P.G, adj->group_ptr, b.nbr,
                                                            adj->src_ptr, adj->src_group,
                                                            adj->group_dst_row, b.key, b.order,
                                                            b.wout);
    RNN_LAUNCH_CHECK();
    int* n_active = b.counter + ACTIVE_SLOT;
    if (P.roots) {
      root_exclude_kernel<<<(unsigned)ceil_div(P.G, 256), 256, 0, st>>>(b.key, P.G);
      if (P.n_roots > 0)
        root_include_kernel<<<(unsigned)ceil_div(P.n_roots, 256), 256, 0, st>>>(
            P.roots, P.n_roots, P.G, b.key, n_active);
      RNN_LAUNCH_CHECK();
    } else {
      set_int_kernel<<<1, 1, 0, st>>>(n_active, (int)P.G);
      RNN_LAUNCH_CHECK();
    }
    RNN_TRY(radix_sort_u32(b.key, b.order, P.G, P.roots ? 25 : 24, b.sort_ws, st));
  }
  if (P.k == 4 && P.E > 0) {
    // every out-list (group segment) and in-list (row segment) sorted by hash partition
    auto bitlen = [](int64_t x) { int b = 1; while ((int64_t(1) << b) <= x) ++b; return b; };
    const unsigned g = (unsigned)ceil_div(P.E, 256);
    h4_keys_kernel<<<g, 256, 0, st>>>(adj->pos_group, b.nbr, P.E, b.hkey, b.nbrh);
    RNN_LAUNCH_CHECK();
    RNN_TRY(radix_sort_u64(b.hkey, b.nbrh, P.E, H4_HBITS + bitlen(P.G), b.sort_ws, st));
    h4_keys_kernel<<<g, 256, 0, st>>>(adj->src_seg, adj->src_group, P.E, b.hkey, b.sgh);
    RNN_LAUNCH_CHECK();
    RNN_TRY(radix_sort_u64(b.hkey, b.sgh, P.E, H4_HBITS + bitlen(P.R), b.sort_ws, st));
  }
  return RNN_OK;
}

rnn_status to_group(const Plan& P, const rnn_join_index* adj, const float* f, int64_t ldf,
                    const float* m, int64_t ldm, float* F, cudaStream_t st) {
  const int64_t n = P.G * P.d;
  if (n == 0) return RNN_OK;
  to_group_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(f, ldf, adj->group_dst_row, P.G,
                                                              P.d, m, ldm, F);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

rnn_status ws_check(const Plan& P, void* ws, size_t bytes, int* n_cta) {
  const size_t need_min = P.fixed + P.per_cta + 256;
  if (!ws) RNN_REQUIRE(bytes == 0, RNN_ERR_INVALID_ARGUMENT, "workspace NULL");
  RNN_REQUIRE(ws && bytes >= need_min, RNN_ERR_WORKSPACE_TOO_SMALL,
              "DHN workspace needs at least %zu bytes (rnn_dhn_workspace_size)", need_min);
  int64_t fit = P.per_cta ? (int64_t)((bytes - P.fixed - 256) / P.per_cta) : P.n_cta;
  *n_cta = (int)std::max<int64_t>(1, std::min<int64_t>(fit, P.n_cta));
  return RNN_OK;
}

}  // namespace
}  // namespace rnn

using namespace rnn;

extern "C" rnn_status rnn_dhn_workspace_size(const rnn_join_index* adj, int32_t k, int32_t d,
                                             size_t* bytes) {
  clear_error();
  RNN_TRY(check_adj(adj, k, d));
  RNN_REQUIRE(bytes, RNN_ERR_INVALID_ARGUMENT, "bytes is NULL");
  const Plan P = make_plan(adj, k, d);
  *bytes = P.fixed + P.per_cta * (size_t)P.n_cta + 256;
  return RNN_OK;
}

// d f0 (row of n) = dOut(n) (.) S(n), S = the forward's walk sum (group order)
static __global__ void dhn_df0_kernel(int64_t G, int d, const int32_t* __restrict__ row_of,
                               const float* __restrict__ dout, int64_t ld_dout,
                               const float* __restrict__ S, int64_t ld_s, float* __restrict__ df0,
                               int64_t ld_df) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= G * d) return;
  const int64_t n = i / d;
  const int c = (int)(i % d);
  df0[(int64_t)row_of[n] * ld_df + c] = dout[n * ld_dout + c] * S[n * ld_s + c];
}

static __global__ void dhn_df0_roots_kernel(const int32_t* __restrict__ roots, int64_t n_roots,
                                            int64_t G, int d, const int32_t* __restrict__ row_of,
                                            const float* __restrict__ dout, int64_t ld_dout,
                                            const float* __restrict__ S, int64_t ld_s,
                                            float* __restrict__ df0, int64_t ld_df) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_roots * d) return;
  const int64_t n = roots[i / d];
  const int c = (int)(i % d);
  if (n < 0 || n >= G) return;
  df0[(int64_t)row_of[n] * ld_df + c] = dout[n * ld_dout + c] * S[n * ld_s + c];
}

static rnn_status dhn_fwd_impl(const rnn_join_index* adj, int32_t k, const rnn_operand* f, float* out,
                        int64_t ld_out, float* walk_sum, int64_t ld_ws, void* workspace,
                        size_t workspace_bytes, void* stream, const int32_t* roots = nullptr,
                        int64_t n_roots = 0);
static rnn_status dhn_bwd_impl(const rnn_join_index* adj, int32_t k, const rnn_operand* f,
                        const float* d_out, int64_t ld_dout, const float* walk_sum, int64_t ld_ws,
                        float* const* d_f, int64_t ld_df, void* workspace, size_t workspace_bytes,
                        void* stream, uint32_t flags = 0, const int32_t* roots = nullptr,
                        int64_t n_roots = 0);

extern "C" rnn_status rnn_dhn_fwd(const rnn_join_index* adj, int32_t k, const rnn_operand* f,
                                  float* out, int64_t ld_out, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  clear_error();
  return dhn_fwd_impl(adj, k, f, out, ld_out, nullptr, 0, workspace, workspace_bytes, stream);
}

extern "C" rnn_status rnn_dhn_fwd_save(const rnn_join_index* adj, int32_t k,
                                       const rnn_operand* f, float* out, int64_t ld_out,
                                       float* walk_sum, int64_t ld_ws, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  clear_error();
  RNN_REQUIRE(walk_sum || !adj || adj->n_groups == 0, RNN_ERR_INVALID_ARGUMENT,
              "walk_sum is NULL");
  return dhn_fwd_impl(adj, k, f, out, ld_out, walk_sum, ld_ws, workspace, workspace_bytes,
                      stream);
}

extern "C" rnn_status rnn_dhn_bwd_saved(const rnn_join_index* adj, int32_t k,
                                        const rnn_operand* f, const float* d_out,
                                        int64_t ld_dout, const float* walk_sum, int64_t ld_ws,
                                        float* const* d_f, int64_t ld_df, uint32_t flags,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  clear_error();
  RNN_REQUIRE(walk_sum || !adj || adj->n_groups == 0, RNN_ERR_INVALID_ARGUMENT,
              "walk_sum is NULL");
  RNN_REQUIRE((flags & ~(uint32_t)RNN_DHN_SYMMETRIC_EDGE) == 0, RNN_ERR_INVALID_ARGUMENT,
              "unknown DHN flags 0x%x", flags);
  return dhn_bwd_impl(adj, k, f, d_out, ld_dout, walk_sum, ld_ws, d_f, ld_df, workspace,
                      workspace_bytes, stream, flags);
}

static rnn_status dhn_fwd_impl(const rnn_join_index* adj, int32_t k, const rnn_operand* f, float* out,
                        int64_t ld_out, float* walk_sum, int64_t ld_ws, void* workspace,
                        size_t workspace_bytes, void* stream, const int32_t* roots,
                        int64_t n_roots) {
  RNN_TRY(check_adj(adj, k, f ? f[1].dim : 0));
  const int d = f[1].dim;
  RNN_TRY(check_ops(f, k, d, adj->n_src_rows));
  RNN_REQUIRE(out || adj->n_groups == 0, RNN_ERR_INVALID_ARGUMENT, "out is NULL");
  RNN_REQUIRE(ld_out >= d, RNN_ERR_SHAPE_MISMATCH, "ld_out %lld < d %d", (long long)ld_out, d);
  RNN_REQUIRE(!walk_sum || ld_ws >= d, RNN_ERR_SHAPE_MISMATCH, "ld_ws %lld < d %d",
              (long long)ld_ws, d);
  RNN_REQUIRE(n_roots >= 0 && (n_roots == 0 || roots), RNN_ERR_INVALID_ARGUMENT,
              "roots NULL with n_roots %lld", (long long)n_roots);
  Plan P = make_plan(adj, k, d);
  P.roots = roots;
  P.n_roots = n_roots;
  RNN_TRY(ws_check(P, workspace, workspace_bytes, &P.n_cta));
  if (P.G == 0) return RNN_OK;
  cudaStream_t st = as_stream(stream);
  Bufs b = carve(P, workspace);
  RNN_TRY(prepare(P, b, adj, st));
  if (k == 2) {
    DhnArgs a{};
    a.G = P.G; a.d = d; a.gp = adj->group_ptr; a.row_of = adj->group_dst_row;
    a.rm = f[0].data; a.ld_rm = f[0].ld; a.rm_by_group = 0; a.out = out; a.ld_out = ld_out;
    a.sum_out = walk_sum; a.ld_sum = ld_ws;
    dhn2_kernel<<<(unsigned)ceil_div(P.G, 8), 256, 0, st>>>(a, adj->src_row, f[1].data, f[1].ld);
    RNN_LAUNCH_CHECK();
    return RNN_OK;
  }
  for (int i = 1; i < k; ++i)
    RNN_TRY(to_group(P, adj, f[i].data, f[i].ld, nullptr, 0, b.F[i - 1], st));
  const float* W[3] = {b.F[0], b.F[1], b.F[2]};
  return walk(P, b, adj, W, f[0].data, f[0].ld, 0, out, ld_out, 0, 0, st, walk_sum, ld_ws);
}

extern "C" rnn_status rnn_dhn_bwd(const rnn_join_index* adj, int32_t k, const rnn_operand* f,
                                  const float* d_out, int64_t ld_dout, float* const* d_f,
                                  int64_t ld_df, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  clear_error();
  return dhn_bwd_impl(adj, k, f, d_out, ld_dout, nullptr, 0, d_f, ld_df, workspace,
                      workspace_bytes, stream);
}

static rnn_status dhn_bwd_impl(const rnn_join_index* adj, int32_t k, const rnn_operand* f,
                        const float* d_out, int64_t ld_dout, const float* walk_sum, int64_t ld_ws,
                        float* const* d_f, int64_t ld_df, void* workspace, size_t workspace_bytes,
                        void* stream, uint32_t flags, const int32_t* roots, int64_t n_roots) {
  RNN_TRY(check_adj(adj, k, f ? f[1].dim : 0));
  const int d = f[1].dim;
  RNN_TRY(check_ops(f, k, d, adj->n_src_rows));
  RNN_REQUIRE(d_f, RNN_ERR_INVALID_ARGUMENT, "d_f is NULL");
  RNN_REQUIRE(d_out || adj->n_groups == 0, RNN_ERR_INVALID_ARGUMENT, "d_out is NULL");
  RNN_REQUIRE(ld_dout >= d && ld_df >= d, RNN_ERR_SHAPE_MISMATCH, "ld < d");
  RNN_REQUIRE(!walk_sum || ld_ws >= d, RNN_ERR_SHAPE_MISMATCH, "ld_ws < d");
  RNN_REQUIRE(n_roots >= 0 && (n_roots == 0 || roots), RNN_ERR_INVALID_ARGUMENT,
              "roots NULL with n_roots %lld", (long long)n_roots);
  Plan P = make_plan(adj, k, d);
  P.roots = roots;
  P.n_roots = n_roots;
  RNN_TRY(ws_check(P, workspace, workspace_bytes, &P.n_cta));
  cudaStream_t st = as_stream(stream);
  for (int i = 0; i < k; ++i)
    if (d_f[i] && P.R > 0)
      RNN_CUDA(cudaMemset2DAsync(d_f[i], sizeof(float) * ld_df, 0, sizeof(float) * d, P.R, st));
  if (P.G == 0) return RNN_OK;
  Bufs b = carve(P, workspace);
  RNN_TRY(prepare(P, b, adj, st));
  // g = f0 (.) dOut in group order (slot k-1)
  float* g = b.F[k - 1];
  RNN_TRY(to_group(P, adj, f[0].data, f[0].ld, d_out, ld_dout, g, st));
  if (d_f[0] && walk_sum) {   // d f0 = dOut (.) the forward's walk sum: no walk needed
    if (P.roots && k > 2) {    // listed roots only (the walk sum exists for those)
      if (P.n_roots > 0) {
        const int64_t n = P.n_roots * d;
        dhn_df0_roots_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
            P.roots, P.n_roots, P.G, d, adj->group_dst_row, d_out, ld_dout, walk_sum, ld_ws,
            d_f[0], ld_df);
      }
    } else {
      const int64_t n = P.G * d;
      dhn_df0_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(P.G, d, adj->group_dst_row,
                                                                 d_out, ld_dout, walk_sum, ld_ws,
                                                                 d_f[0], ld_df);
    }
    RNN_LAUNCH_CHECK();
  }
  if (k == 2) {
    if (d_f[0] && !walk_sum) {   // d f0(n) = dOut(n) (.) sum f1
      DhnArgs a{};
      a.G = P.G; a.d = d; a.gp = adj->group_ptr; a.row_of = adj->group_dst_row;
      a.rm = d_out; a.ld_rm = ld_dout; a.rm_by_group = 1; a.out = d_f[0]; a.ld_out = ld_df;
      a.out_by_row = 1;
      dhn2_kernel<<<(unsigned)ceil_div(P.G, 8), 256, 0, st>>>(a, adj->src_row, f[1].data, f[1].ld);
      RNN_LAUNCH_CHECK();
    }
    if (d_f[1] && P.R > 0) {
      dhn2_bwd_kernel<<<(unsigned)ceil_div(P.R, 8), 256, 0, st>>>(P.R, d, adj->src_ptr,
                                                                 adj->src_group, g, d_f[1], ld_df);
      RNN_LAUNCH_CHECK();
    }
    return RNN_OK;
  }
  for (int i = 1; i < k; ++i)
    RNN_TRY(to_group(P, adj, f[i].data, f[i].ld, nullptr, 0, b.F[i - 1], st));
  // operand sequence around the cycle: position 0 = g, positions 1..k-1 = f_i
  const float* cyc[4] = {g, b.F[0], b.F[1], b.F[2]};
  int launch = 0;
  if (d_f[0] && !walk_sum) {
    const float* W[3] = {cyc[1], cyc[2], cyc[3]};
    RNN_TRY(walk(P, b, adj, W, d_out, ld_dout, 1, d_f[0], ld_df, 1, launch++, st));
  }
  // symmetric Edge, k = 4: the d f1 walk (f2, f3, g) and the d f3 walk (g, f1, f2) -- reversed,
  // (f2, f1, g) -- share both partial sums S_f2 and S_g and differ only in the middle operand,
  // so one walk with two middle operands yields both
  // k = 3 likewise: the d f1 walk (f2, g) and the d f2 walk (g, f1) -- reversed, (f1, g) --
  // share the probe and the g gathers; one walk with two first-hop operands yields both
  bool dual = false;
  const bool sym = (flags & RNN_DHN_SYMMETRIC_EDGE) && !getenv("RNN_DHN_NO_DUAL");
  if (sym && k == 4 && d_f[1] && d_f[3] && d % 4 == 0 && !getenv("RNN_DHN_SCALAR")) {
    const float* W[3] = {cyc[2], cyc[3], cyc[0]};
    RNN_TRY(walk(P, b, adj, W, nullptr, 0, 0, d_f[1], ld_df, 1, launch++, st, nullptr, 0, cyc[1],
                 d_f[3]));
    dual = true;
  }
  if (sym && k == 3 && d_f[1] && d_f[2]) {
    const float* W[3] = {cyc[2], cyc[0], nullptr};
    RNN_TRY(walk(P, b, adj, W, nullptr, 0, 0, d_f[1], ld_df, 1, launch++, st, nullptr, 0, cyc[1],
                 d_f[2]));
    dual = true;
  }
  for (int j = 1; j < k; ++j) {
    if (!d_f[j] || (dual && (k == 3 || j == 1 || j == 3))) continue;
    const float* W[3] = {nullptr, nullptr, nullptr};
    for (int i = 1; i < k; ++i) W[i - 1] = cyc[(j + i) % k];
    RNN_TRY(walk(P, b, adj, W, nullptr, 0, 0, d_f[j], ld_df, 1, launch++, st));
  }
  return RNN_OK;
}

extern "C" rnn_status rnn_dhn_fwd_roots(const rnn_join_index* adj, int32_t k,
                                        const rnn_operand* f, const int32_t* roots,
                                        int64_t n_roots, float* out, int64_t ld_out,
                                        float* walk_sum, int64_t ld_ws, void* workspace,
                                        size_t workspace_bytes, void* stream) {
  clear_error();
  RNN_REQUIRE(roots || n_roots == 0, RNN_ERR_INVALID_ARGUMENT, "roots is NULL");
  static const int32_t none = 0;
  return dhn_fwd_impl(adj, k, f, out, ld_out, walk_sum, ld_ws, workspace, workspace_bytes,
                      stream, roots ? roots : &none, n_roots);
}

extern "C" rnn_status rnn_dhn_bwd_roots(const rnn_join_index* adj, int32_t k,
                                        const rnn_operand* f, const int32_t* roots,
                                        int64_t n_roots, const float* d_out, int64_t ld_dout,
                                        const float* walk_sum, int64_t ld_ws, float* const* d_f,
                                        int64_t ld_df, uint32_t flags, void* workspace,
                                        size_t workspace_bytes, void* stream) {
  clear_error();
  RNN_REQUIRE(roots || n_roots == 0, RNN_ERR_INVALID_ARGUMENT, "roots is NULL");
  RNN_REQUIRE((flags & ~(uint32_t)RNN_DHN_SYMMETRIC_EDGE) == 0, RNN_ERR_INVALID_ARGUMENT,
              "unknown DHN flags 0x%x", flags);
  static const int32_t none = 0;
  return dhn_bwd_impl(adj, k, f, d_out, ld_dout, walk_sum, ld_ws, d_f, ld_df, workspace,
                      workspace_bytes, stream, flags, roots ? roots : &none, n_roots);
}

// ---- exact counts ----
namespace {
struct CountBufs {
  int32_t* gor; int32_t* nbr; uint32_t* key; int32_t* order; int* counter; uint32_t* wout;
  void* sort_ws;
};
CountBufs carve_count(const rnn_join_index* adj, void* base, size_t* used) {
  Carve c(base);
  CountBufs b;
  const int64_t G = adj->n_groups, E = adj->n_join_rows, R = adj->n_src_rows;
  b.gor = c.take<int32_t>(R);
  b.nbr = c.take<int32_t>(E);
  b.key = c.take<uint32_t>(G);
  b.order = c.take<int32_t>(G);
  b.counter = c.take<int>(64);
  b.wout = c.take<uint32_t>(G);
  b.sort_ws = c.take<char>(radix_sort_workspace_bytes(G));
  if (used) *used = (c.used + 255) & ~size_t(255);
  return b;
}
}  // namespace

extern "C" rnn_status rnn_dhn_count_workspace_size(const rnn_join_index* adj, int32_t k,
                                                   size_t* bytes) {
  clear_error();
  RNN_TRY(check_adj(adj, k, 1));
  RNN_REQUIRE(bytes, RNN_ERR_INVALID_ARGUMENT, "bytes is NULL");
  carve_count(adj, nullptr, bytes);
  return RNN_OK;
}

extern "C" rnn_status rnn_dhn_count(const rnn_join_index* adj, int32_t k, int64_t* counts,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  clear_error();
  RNN_TRY(check_adj(adj, k, 1));
  const int64_t G = adj->n_groups;
  RNN_REQUIRE(counts || G == 0, RNN_ERR_INVALID_ARGUMENT, "counts is NULL");
  size_t need = 0;
  CountBufs b = carve_count(adj, workspace, &need);
  RNN_REQUIRE(workspace && workspace_bytes >= need, RNN_ERR_WORKSPACE_TOO_SMALL,
              "DHN count workspace needs %zu bytes (rnn_dhn_count_workspace_size)", need);
  if (G == 0) return RNN_OK;
  cudaStream_t st = as_stream(stream);
  if (k == 2) {
    dhn_count2_kernel<<<(unsigned)ceil_div(G, 256), 256, 0, st>>>(G, adj->group_ptr, counts);
    RNN_LAUNCH_CHECK();
    return RNN_OK;
  }
  const int64_t E = adj->n_join_rows, R = adj->n_src_rows;
  RNN_CUDA(cudaMemsetAsync(b.gor, 0xff, sizeof(int32_t) * std::max<int64_t>(R, 1), st));
  RNN_CUDA(cudaMemsetAsync(b.counter, 0, sizeof(int) * 64, st));
  grp_of_row_kernel<<<(unsigned)ceil_div(G, 256), 256, 0, st>>>(adj->group_dst_row, G, b.gor);
  if (E > 0) nbr_kernel<<<(unsigned)ceil_div(E, 256), 256, 0, st>>>(adj->src_row, E, b.gor, b.nbr);
  // heaviest roots first; k = 4 also yields the out-wedge bound wout
  work_kernel<<<(unsigned)ceil_div(G, 8), 256, 0, st>>>(4, G, adj->group_ptr, b.nbr, adj->src_ptr,
                                                        adj->src_group, adj->group_dst_row, b.key,
                                                        b.order, b.wout);
  RNN_LAUNCH_CHECK();
  RNN_TRY(radix_sort_u32(b.key, b.order, G, 24, b.sort_ws, st));
  CountArgs a{k, G, adj->group_ptr, b.nbr, adj->src_ptr, adj->src_group, adj->group_dst_row,
              b.order, b.counter, b.wout, counts};
  const size_t smem = (size_t)HC_CAP * (sizeof(unsigned long long) + sizeof(int));
  RNN_CUDA(cudaFuncSetAttribute(dhn_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  const int n_cta = (int)std::min<int64_t>((int64_t)num_sms() * 2, G);
  dhn_count_kernel<<<n_cta, HC_THREADS, smem, st>>>(a);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

// internal hook (not part of rnn.h): which = 0 -> the path counters g_dhn_paths,
// 1 -> the C4 phase clocks (measurement builds only; zeros otherwise).  SYNC.
extern "C" int rnn_internal_dhn_stats(unsigned long long* out, int reset, int which) {
  const void* sym = which ? (const void*)&rnn::g_dhn4_clock : (const void*)&rnn::g_dhn_paths;
  if (cudaMemcpyFromSymbol(out, sym, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
  if (reset) {
    unsigned long long z[16] = {0};
    if (cudaMemcpyToSymbol(sym, z, sizeof(z)) != cudaSuccess) return 1;
  }
  return 0;
}
