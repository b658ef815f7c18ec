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
//  * one CTA per root, roots taken heaviest-first from an atomic counter (persistent grid);
//  * C3: the root's in-neighbours are counted into a per-CTA mark array (multiplicity =
//    number of closing Edge rows), then the CTA's warps walk the wedges n->v->w with lanes
//    over w and ballot the marked ones; the hits gather f1(v) (.) f2(w) with lane = channel;
//  * C4: factorised through the middle vertex w: S3(w) = sum_{w->p->n} f3(p) is scattered
//    (fp32 red) into a per-CTA dense slab indexed by group, then every 2-path n->v->w reads
//    it: C4(n) = f0(n) (.) sum_{n->v->w} f1(v) (.) f2(w) (.) S3(w).  The slab holds a DS-wide
//    channel slice (DS chosen so the slabs of all resident CTAs fit the workspace budget);
//    the walk is repeated per slice, and the touched slab entries are re-zeroed by walking
//    the same lists again (no full clears);
//  * the backward is the same kernels with rotated operands (rnn.h).
#include <algorithm>

#include "common.cuh"

namespace rnn {
namespace {

constexpr int DHN_THREADS = 512;
constexpr int DHN_WARPS = DHN_THREADS / 32;
constexpr int DHN_CTAS_PER_SM = 2;
constexpr size_t DHN_SLAB_BUDGET = size_t(16) << 30;   // bytes of k=4 slabs across all CTAs

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
  const int32_t* order;   // roots, heaviest first
  int* counter;
  int* mark;              // k=3: per-CTA [G] int32
  float* slab;            // k=4: per-CTA [G * ds]
  int64_t cta_stride;     // elements between consecutive CTAs' mark / slab
};

__device__ __forceinline__ void dhn_store(const DhnArgs& a, int64_t n, int c, float v) {
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
  return i < a.G ? (int64_t)a.order[i] : -1;
}

// -------------------------------------------------------------------------------------
// C3: triangles n -> v -> w -> n
// -------------------------------------------------------------------------------------
template <int DPL>
__global__ void __launch_bounds__(DHN_THREADS, DHN_CTAS_PER_SM) dhn3_kernel(DhnArgs a) {
  __shared__ int s_root;
  __shared__ float s_acc[DHN_WARPS][DPL * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int* mark = a.mark + (int64_t)blockIdx.x * a.cta_stride;
  const int d = a.d;
  for (;;) {
    const int64_t n = dhn_next_root(a, &s_root);
    if (n < 0) break;
    const int32_t r = a.row_of[n];
    const int64_t ib = a.sp[r], ie = a.sp[r + 1];
    for (int64_t q = ib + threadIdx.x; q < ie; q += DHN_THREADS) atomicAdd(&mark[a.sg[q]], 1);
    __syncthreads();
    float acc[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) acc[j] = 0.f;
    const int64_t pe = a.gp[n + 1];
    for (int64_t pos = a.gp[n] + warp; pos < pe; pos += DHN_WARPS) {
      const int32_t v = a.nbr[pos];
      if (v < 0) continue;
      float f1v[DPL];
#pragma unroll
      for (int j = 0; j < DPL; ++j) {
        const int c = lane + 32 * j;
        f1v[j] = c < d ? a.F1[(int64_t)v * d + c] : 0.f;
      }
      const int64_t we = a.gp[v + 1];
      for (int64_t i0 = a.gp[v]; i0 < we; i0 += 32) {
        const int64_t i = i0 + lane;
        const int32_t w = i < we ? a.nbr[i] : -1;
        const int m = w >= 0 ? __ldcg(&mark[w]) : 0;
        unsigned bal = __ballot_sync(FULL, m != 0);
        while (bal) {
          // up to 4 hits per round so their row loads are in flight together
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
            }
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < DPL; ++j) s_acc[warp][lane + 32 * j] = acc[j];
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += DHN_THREADS) {
      float s = 0.f;
#pragma unroll 4
      for (int w = 0; w < DHN_WARPS; ++w) s += s_acc[w][c];
      dhn_store(a, n, c, s);
    }
    for (int64_t q = ib + threadIdx.x; q < ie; q += DHN_THREADS) mark[a.sg[q]] = 0;
  }
}

// -------------------------------------------------------------------------------------
// C4: 4-cycles n -> v -> w -> p -> n, factorised through w
// -------------------------------------------------------------------------------------
template <int DS>
__global__ void __launch_bounds__(DHN_THREADS, DHN_CTAS_PER_SM) dhn4_kernel(DhnArgs a) {
  constexpr int S = 32 / DS;   // 2-paths processed side by side per warp
  __shared__ int s_root;
  __shared__ float s_out[128];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % DS, sub = lane / DS;
  float* slab = a.slab + (int64_t)blockIdx.x * a.cta_stride;
  const int d = a.d;
  for (;;) {
    const int64_t n = dhn_next_root(a, &s_root);
    if (n < 0) break;
    const int32_t r = a.row_of[n];
    const int64_t ib = a.sp[r], ie = a.sp[r + 1];
    const int64_t pb = a.gp[n], pe = a.gp[n + 1];
    for (int i = threadIdx.x; i < d; i += DHN_THREADS) s_out[i] = 0.f;
    for (int c0 = 0; c0 < d; c0 += DS) {
      const int ch = c0 + c;
      // (A) S3(w) += f3(p) for w -> p -> n
      for (int64_t q = ib + warp; q < ie; q += DHN_WARPS) {
        const int32_t p = a.sg[q];
        const int32_t rp = a.row_of[p];
        const float f3p = a.F3[(int64_t)p * d + ch];
        const int64_t e2 = a.sp[rp + 1];
        for (int64_t q2 = a.sp[rp] + sub; q2 < e2; q2 += S)
          atomicAdd(&slab[(int64_t)a.sg[q2] * DS + c], f3p);
      }
      __syncthreads();
      // (B) acc += f1(v) f2(w) S3(w) over n -> v -> w
      float acc = 0.f;
      for (int64_t pos = pb + warp; pos < pe; pos += DHN_WARPS) {
        const int32_t v = a.nbr[pos];
        if (v < 0) continue;
        const float f1v = a.F1[(int64_t)v * d + ch];
        const int64_t we = a.gp[v + 1];
        float t = 0.f;
        for (int64_t i = a.gp[v] + sub; i < we; i += S) {
          const int32_t w = a.nbr[i];
          if (w >= 0) t += a.F2[(int64_t)w * d + ch] * __ldcg(&slab[(int64_t)w * DS + c]);
        }
        acc += f1v * t;
      }
#pragma unroll
      for (int o = DS; o < 32; o <<= 1) acc += __shfl_xor_sync(FULL, acc, o);
      if (sub == 0) atomicAdd(&s_out[ch], acc);
      __syncthreads();
      // (C) re-zero the touched slab entries
      for (int64_t q = ib + warp; q < ie; q += DHN_WARPS) {
        const int32_t rp = a.row_of[a.sg[q]];
        const int64_t e2 = a.sp[rp + 1];
        for (int64_t q2 = a.sp[rp] + sub; q2 < e2; q2 += S)
          slab[(int64_t)a.sg[q2] * DS + c] = 0.f;
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < d; i += DHN_THREADS) dhn_store(a, n, i, s_out[i]);
  }
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
                            uint32_t* __restrict__ key, int32_t* __restrict__ order) {
  const int64_t n = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (n >= G) return;
  const int lane = threadIdx.x & 31;
  int64_t w = 0;
  for (int64_t p = gp[n] + lane; p < gp[n + 1]; p += 32) {
    const int32_t v = nbr[p];
    if (v >= 0) w += gp[v + 1] - gp[v];
  }
  if (k == 4) {
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

// ---------------------------------------------------------------------------------------
// plan: workspace layout
// ---------------------------------------------------------------------------------------
struct Plan {
  int k, d, ds, n_cta;
  int64_t G, E, R;
  size_t fixed, per_cta;
};

int pick_ds(int64_t G, int d, int n_cta) {
  for (int ds : {32, 16, 8, 4, 2, 1}) {
    if (ds > d || d % ds) continue;
    if ((size_t)n_cta * (size_t)G * ds * sizeof(float) <= DHN_SLAB_BUDGET) return ds;
  }
  return 1;
}

struct Bufs {
  int32_t* gor; int32_t* nbr; float* F[4]; uint32_t* key; int32_t* order; int* counter;
  void* sort_ws; char* cta;
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
  b.sort_ws = c.take<char>(radix_sort_workspace_bytes(P.G));
  b.cta = c.take<char>(0);
  if (used) *used = c.used;
  return b;
}

Plan make_plan(const rnn_join_index* adj, int k, int d) {
  Plan P;
  P.k = k; P.d = d;
  P.G = adj->n_groups; P.E = adj->n_join_rows; P.R = adj->n_src_rows;
  P.n_cta = (int)std::min<int64_t>((int64_t)num_sms() * DHN_CTAS_PER_SM, std::max<int64_t>(P.G, 1));
  P.ds = k == 4 ? pick_ds(P.G, d, P.n_cta) : 0;
  P.per_cta = k == 3 ? ((size_t)P.G * sizeof(int32_t) + 255) & ~size_t(255)
            : k == 4 ? ((size_t)P.G * P.ds * sizeof(float) + 255) & ~size_t(255) : 0;
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
                int out_by_row, int launch_id, cudaStream_t st) {
  DhnArgs a{};
  a.G = P.G; a.d = P.d;
  a.gp = adj->group_ptr; a.nbr = b.nbr; a.sp = adj->src_ptr; a.sg = adj->src_group;
  a.row_of = adj->group_dst_row;
  a.F1 = W[0]; a.F2 = W[1]; a.F3 = P.k == 4 ? W[2] : nullptr;
  a.rm = rm; a.ld_rm = ld_rm; a.rm_by_group = rm_by_group;
  a.out = out; a.ld_out = ld_out; a.out_by_row = out_by_row;
  a.order = b.order; a.counter = b.counter + launch_id;
  a.cta_stride = (int64_t)(P.per_cta / (P.k == 3 ? sizeof(int32_t) : sizeof(float)));
  // the kernels leave their per-CTA scratch zeroed, so only the first launch clears it
  if (launch_id == 0) RNN_CUDA(cudaMemsetAsync(b.cta, 0, P.per_cta * P.n_cta, st));
  if (P.k == 3) {
    a.mark = reinterpret_cast<int*>(b.cta);
    const int dpl = (P.d + 31) / 32;
    switch (dpl) {
      case 1: dhn3_kernel<1><<<P.n_cta, DHN_THREADS, 0, st>>>(a); break;
      case 2: dhn3_kernel<2><<<P.n_cta, DHN_THREADS, 0, st>>>(a); break;
      case 3: dhn3_kernel<3><<<P.n_cta, DHN_THREADS, 0, st>>>(a); break;
      default: dhn3_kernel<4><<<P.n_cta, DHN_THREADS, 0, st>>>(a); break;
    }
  } else {
    a.slab = reinterpret_cast<float*>(b.cta);
    switch (P.ds) {
      case 32: dhn4_kernel<32><<<P.n_cta, DHN_THREADS, 0, st>>>(a); break;
      case 16: dhn4_kernel<16><<<P.n_cta, DHN_THREADS, 0, st>>>(a); break;
      case 8: dhn4_kernel<8><<<P.n_cta, DHN_THREADS, 0, st>>>(a); break;
      case 4: dhn4_kernel<4><<<P.n_cta, DHN_THREADS, 0, st>>>(a); break;
      case 2: dhn4_kernel<2><<<P.n_cta, DHN_THREADS, 0, st>>>(a); break;
      default: dhn4_kernel<1><<<P.n_cta, DHN_THREADS, 0, st>>>(a); break;
    }
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
                                                            adj->group_dst_row, b.key, b.order);
    RNN_LAUNCH_CHECK();
    RNN_TRY(radix_sort_u32(b.key, b.order, P.G, 24, b.sort_ws, st));
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

extern "C" rnn_status rnn_dhn_fwd(const rnn_join_index* adj, int32_t k, const rnn_operand* f,
                                  float* out, int64_t ld_out, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  clear_error();
  RNN_TRY(check_adj(adj, k, f ? f[1].dim : 0));
  const int d = f[1].dim;
  RNN_TRY(check_ops(f, k, d, adj->n_src_rows));
  RNN_REQUIRE(out || adj->n_groups == 0, RNN_ERR_INVALID_ARGUMENT, "out is NULL");
  RNN_REQUIRE(ld_out >= d, RNN_ERR_SHAPE_MISMATCH, "ld_out %lld < d %d", (long long)ld_out, d);
  Plan P = make_plan(adj, k, d);
  RNN_TRY(ws_check(P, workspace, workspace_bytes, &P.n_cta));
  if (P.G == 0) return RNN_OK;
  cudaStream_t st = as_stream(stream);
  Bufs b = carve(P, workspace);
  RNN_TRY(prepare(P, b, adj, st));
  if (k == 2) {
    DhnArgs a{};
    a.G = P.G; a.d = d; a.gp = adj->group_ptr; a.row_of = adj->group_dst_row;
    a.rm = f[0].data; a.ld_rm = f[0].ld; a.rm_by_group = 0; a.out = out; a.ld_out = ld_out;
    dhn2_kernel<<<(unsigned)ceil_div(P.G, 8), 256, 0, st>>>(a, adj->src_row, f[1].data, f[1].ld);
    RNN_LAUNCH_CHECK();
    return RNN_OK;
  }
  for (int i = 1; i < k; ++i)
    RNN_TRY(to_group(P, adj, f[i].data, f[i].ld, nullptr, 0, b.F[i - 1], st));
  const float* W[3] = {b.F[0], b.F[1], b.F[2]};
  return walk(P, b, adj, W, f[0].data, f[0].ld, 0, out, ld_out, 0, 0, st);
}

extern "C" rnn_status rnn_dhn_bwd(const rnn_join_index* adj, int32_t k, const rnn_operand* f,
                                  const float* d_out, int64_t ld_dout, float* const* d_f,
                                  int64_t ld_df, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  clear_error();
  RNN_TRY(check_adj(adj, k, f ? f[1].dim : 0));
  const int d = f[1].dim;
  RNN_TRY(check_ops(f, k, d, adj->n_src_rows));
  RNN_REQUIRE(d_f, RNN_ERR_INVALID_ARGUMENT, "d_f is NULL");
  RNN_REQUIRE(d_out || adj->n_groups == 0, RNN_ERR_INVALID_ARGUMENT, "d_out is NULL");
  RNN_REQUIRE(ld_dout >= d && ld_df >= d, RNN_ERR_SHAPE_MISMATCH, "ld < d");
  Plan P = make_plan(adj, k, d);
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
  if (k == 2) {
    if (d_f[0]) {   // d f0(n) = dOut(n) (.) sum f1
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
  if (d_f[0]) {
    const float* W[3] = {cyc[1], cyc[2], cyc[3]};
    RNN_TRY(walk(P, b, adj, W, d_out, ld_dout, 1, d_f[0], ld_df, 1, launch++, st));
  }
  for (int j = 1; j < k; ++j) {
    if (!d_f[j]) continue;
    const float* W[3] = {nullptr, nullptr, nullptr};
    for (int i = 1; i < k; ++i) W[i - 1] = cyc[(j + i) % k];
    RNN_TRY(walk(P, b, adj, W, nullptr, 0, 0, d_f[j], ld_df, 1, launch++, st));
  }
  return RNN_OK;
}
