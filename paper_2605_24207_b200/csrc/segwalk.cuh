// segwalk.cuh -- warp-per-work-item traversal of a segmented CSR with a deterministic
// combine of split segments.
//
// A work schedule (built once with the join index) cuts the positions [0, E') into items:
// runs of whole short segments, or single pieces of a long segment (power-law hubs).  One
// warp owns one item.  A segment fully inside the item is reduced and finalised by that
// warp.  A piece writes its partial state to workspace; the warp that completes the LAST
// piece (atomic ticket) merges all pieces in item order and finalises -- so the summation
// order is fixed by the schedule, never by timing: results are bit-reproducible and no
// floating-point atomics are used.
#pragma once
#include "common.cuh"

namespace rnn {

struct SegCtx {
  const int64_t* ptr;       // [n_seg + 1]
  int64_t n_seg;
  const int64_t* work_ptr;  // [n_work + 1]
  int64_t n_work;
  float* partial;           // [n_work, pstride]
  int64_t pstride;          // floats per partial state
  int* counter;             // [n_work], zero on entry
};

// Pol must provide:
//   struct State;  init(State&, seg);  rows(State&, seg, r0, r1);  finish(State&, seg);
//   save(const State&, float*);  merge(State&, const float*)   (merge in call order)
template <class Pol>
__device__ __forceinline__ void run_segment(Pol& pol, const SegCtx& cx, int64_t item,
                                            int64_t seg, int64_t r0, int64_t r1, bool full) {
  typename Pol::State st;
  __syncwarp();
  pol.init(st, seg);
  pol.rows(st, seg, r0, r1);
  if (full) {
    pol.finish(st, seg);
    __syncwarp();
    return;
  }
  pol.save(st, cx.partial + item * cx.pstride);
  __threadfence();
  __syncwarp();
  int64_t i0 = 0, i1 = 0;
  int last = 0;
  if (lane_id() == 0) {
    i0 = lower_bound_dev(cx.work_ptr, 0, cx.n_work + 1, cx.ptr[seg]);
    i1 = lower_bound_dev(cx.work_ptr, 0, cx.n_work + 1, cx.ptr[seg + 1]);
    last = atomicAdd(&cx.counter[i0], 1) == (int)(i1 - i0 - 1);
  }
  last = __shfl_sync(FULL, last, 0);
  if (!last) return;
  i0 = __shfl_sync(FULL, i0, 0);
  i1 = __shfl_sync(FULL, i1, 0);
  __threadfence();
  pol.init(st, seg);
  for (int64_t i = i0; i < i1; ++i) pol.merge(st, cx.partial + i * cx.pstride);
  pol.finish(st, seg);
}

// Walk every segment overlapping item `item`.  Segments starting in [b, e) belong to the item
// (the last item also owns empty segments starting at E'), plus the piece of the segment
// containing b when b is not a segment start.
template <class Pol>
__device__ __forceinline__ void walk_item(Pol& pol, const SegCtx& cx, int64_t item) {
  const int64_t b = cx.work_ptr[item], e = cx.work_ptr[item + 1];
  const bool last_item = item == cx.n_work - 1;
  int64_t s = lower_bound_dev(cx.ptr, 0, cx.n_seg + 1, b);
  if (s > cx.n_seg || cx.ptr[s] > b) {
    const int64_t seg = s - 1;
    const int64_t stop = s <= cx.n_seg ? cx.ptr[s] : e;
    const int64_t r1 = stop < e ? stop : e;
    run_segment(pol, cx, item, seg, b, r1, false);
  }
  for (; s < cx.n_seg; ++s) {
    const int64_t a = cx.ptr[s];
    if (a > e || (a == e && !last_item)) break;
    const int64_t z = cx.ptr[s + 1];
    run_segment(pol, cx, item, s, a, z < e ? z : e, z <= e);
  }
}

template <class Pol>
__global__ void __launch_bounds__(256) seg_kernel(Pol pol, SegCtx cx) {
  const int64_t item = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (item >= cx.n_work) return;
  walk_item(pol, cx, item);
}

// ------------------------------------------------------------------------------------------
// lane layout for a row of D floats: LPR lanes per row (power of two), VEC float4 per lane,
// RPW = 32 / LPR rows processed side by side by one warp.
// ------------------------------------------------------------------------------------------
template <int LPR_, int VEC_>
struct Lanes {
  static constexpr int LPR = LPR_, VEC = VEC_, RPW = 32 / LPR_;
  __device__ __forceinline__ static int slot() { return lane_id() / LPR; }
  __device__ __forceinline__ static int sub() { return lane_id() % LPR; }
  // float4 column index of vector v of this lane
  __device__ __forceinline__ static int col4(int v) { return sub() + LPR * v; }
  // sum a float4 across the RPW row slots (all slots end with the total)
  __device__ __forceinline__ static float4 reduce_slots(float4 a) {
#pragma unroll
    for (int m = LPR; m < 32; m <<= 1) a = f4_add(a, f4_shfl_xor(a, m));
    return a;
  }
  // sum a scalar across the LPR lanes of one row
  __device__ __forceinline__ static float reduce_row(float x) {
#pragma unroll
    for (int m = 1; m < LPR; m <<= 1) x += __shfl_xor_sync(FULL, x, m);
    return x;
  }
};

// masked float4 load of columns [4k, 4k+4) of row `row` (columns >= n4*4 read as zero)
__device__ __forceinline__ float4 load4(const float* base, int64_t row, int64_t ld, int k, int n4) {
  return k < n4 ? ld_f4(base + row * ld + 4 * (int64_t)k) : f4_zero();
}

// store columns [4k, 4k+4) of a row clipped to D columns
__device__ __forceinline__ void store4_clip(float* base, int64_t row, int64_t ld, int k, int D,
                                            float4 v) {
  float* p = base + row * ld + 4 * (int64_t)k;
  const int c = 4 * k;
  if (c + 3 < D) { st_f4(p, v); return; }
  if (c < D) p[0] = v.x;
  if (c + 1 < D) p[1] = v.y;
  if (c + 2 < D) p[2] = v.z;
}

__device__ __forceinline__ float4 load4_clip(const float* base, int64_t row, int64_t ld, int k,
                                             int D) {
  const float* p = base + row * ld + 4 * (int64_t)k;
  const int c = 4 * k;
  if (c + 3 < D) return *reinterpret_cast<const float4*>(p);
  float4 v = f4_zero();
  if (c < D) v.x = p[0];
  if (c + 1 < D) v.y = p[1];
  if (c + 2 < D) v.z = p[2];
  return v;
}

}  // namespace rnn
