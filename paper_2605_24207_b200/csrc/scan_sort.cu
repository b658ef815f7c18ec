// scan_sort.cu -- device-wide exclusive scan and stable LSD radix sort used by the join-index
// builder (A1).  Deterministic: counts are exact integers and every scatter position is a
// function of the input order (stable in-tile ranking with warp match + sequential steps).
#include "common.cuh"

namespace rnn {

namespace {

constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int64_t SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ int64_t warp_inclusive_scan(int64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t u = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// exclusive scan of one value per thread across the block; returns the prefix, writes total
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
  __shared__ int64_t warp_tot[SCAN_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t inc = warp_inclusive_scan(v);
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < SCAN_THREADS / 32 ? warp_tot[lane] : 0;
    int64_t wi = warp_inclusive_scan(w);
    if (lane < SCAN_THREADS / 32) warp_tot[lane] = wi - w;
    if (lane == SCAN_THREADS / 32 - 1) *total = wi;
  }
  __syncthreads();
  int64_t r = warp_tot[warp] + inc - v;
  return r;
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_tile_sums(const int64_t* __restrict__ in,
                                                               int64_t n, int64_t* sums) {
  __shared__ int64_t tot;
  const int64_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k)
    if (base + k < n) s += in[base + k];
  block_exclusive_scan(s, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_tiles(const int64_t* in, int64_t* out,
                                                           int64_t n, const int64_t* offs) {
  __shared__ int64_t tot;
  const int64_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    s += v[k];
  }
  int64_t run = block_exclusive_scan(s, &tot) + (offs ? offs[blockIdx.x] : 0);
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (base + k < n) {
      out[base + k] = run;
      if (base + k == n - 1) out[n] = run + v[k];
    }
    run += v[k];
  }
}

// ------------------------------------------------------------------------------------------
// radix sort (8-bit digits)
// ------------------------------------------------------------------------------------------
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_STEPS = 16;                       // 32-item steps per warp
constexpr int64_t RS_TILE = RS_THREADS * RS_STEPS; // 4096 items per tile

template <class K>
__global__ void __launch_bounds__(RS_THREADS) radix_hist(const K* __restrict__ keys, int64_t n,
                                                         int shift, int64_t n_tiles,
                                                         int64_t* __restrict__ hist) {
  __shared__ int cnt[256];
  for (int i = threadIdx.x; i < 256; i += RS_THREADS) cnt[i] = 0;
  __syncthreads();
  const int64_t base = blockIdx.x * RS_TILE;
  for (int k = threadIdx.x; k < RS_TILE; k += RS_THREADS) {
    int64_t i = base + k;
    if (i < n) atomicAdd(&cnt[(int)((keys[i] >> shift) & 255)], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += RS_THREADS) hist[(int64_t)d * n_tiles + blockIdx.x] = cnt[d];
}

template <class K>
__global__ void __launch_bounds__(RS_THREADS)
    radix_scatter(const K* __restrict__ keys_in, const int32_t* __restrict__ vals_in,
                  K* __restrict__ keys_out, int32_t* __restrict__ vals_out, int64_t n, int shift,
                  const int64_t* __restrict__ offs, int64_t n_tiles) {
  __shared__ int cnt[RS_WARPS][256];
  __shared__ int wofs[RS_WARPS][256];
  for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t base = blockIdx.x * RS_TILE + (int64_t)warp * (RS_STEPS * 32);
  int dig[RS_STEPS], pos[RS_STEPS];
#pragma unroll
  for (int s = 0; s < RS_STEPS; ++s) {
    const int64_t i = base + s * 32 + lane;
    const bool valid = i < n;
    const int d = valid ? (int)((keys_in[i] >> shift) & 255) : -1;
    const unsigned peers = __match_any_sync(FULL, d);
    const int rank = __popc(peers & lt_mask);
    const int leader = __ffs(peers) - 1;
    int old = valid ? cnt[warp][d] : 0;
    __syncwarp();
    if (valid && lane == leader) cnt[warp][d] = old + __popc(peers);
    __syncwarp();
    dig[s] = d;
    pos[s] = old + rank;
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += RS_THREADS) {
    int run = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) { wofs[w][d] = run; run += cnt[w][d]; }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < RS_STEPS; ++s) {
    const int64_t i = base + s * 32 + lane;
    if (i < n) {
      const int d = dig[s];
      const int64_t dst = offs[(int64_t)d * n_tiles + blockIdx.x] + wofs[warp][d] + pos[s];
      keys_out[dst] = keys_in[i];
      vals_out[dst] = vals_in[i];
    }
  }
}

size_t scan_ws_rec(int64_t n) {
  if (n <= SCAN_TILE) return 0;
  int64_t tiles = ceil_div(n, SCAN_TILE);
  size_t here = ((size_t)(tiles + 1) * sizeof(int64_t) + 255) & ~size_t(255);
  return here + scan_ws_rec(tiles);
}

template <class K>
rnn_status radix_sort_impl(K* keys, int32_t* vals, int64_t n, int bits, void* ws,
                           cudaStream_t st) {
  if (n <= 1 || bits <= 0) return RNN_OK;
  const int64_t n_tiles = ceil_div(n, RS_TILE);
  Carve c(ws);
  K* kalt = c.take<K>(n);
  int32_t* valt = c.take<int32_t>(n);
  int64_t* hist = c.take<int64_t>((size_t)256 * n_tiles + 1);
  void* sws = c.take<char>(scan_workspace_bytes(256 * n_tiles));
  K* kin = keys; int32_t* vin = vals; K* kout = kalt; int32_t* vout = valt;
  const int passes = (bits + 7) / 8;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    radix_hist<K><<<(unsigned)n_tiles, RS_THREADS, 0, st>>>(kin, n, shift, n_tiles, hist);
    RNN_LAUNCH_CHECK();
    RNN_TRY(exclusive_scan_i64(hist, hist, 256 * n_tiles, sws, st));
    radix_scatter<K><<<(unsigned)n_tiles, RS_THREADS, 0, st>>>(kin, vin, kout, vout, n, shift,
                                                               hist, n_tiles);
    RNN_LAUNCH_CHECK();
    K* tk = kin; kin = kout; kout = tk;
    int32_t* tv = vin; vin = vout; vout = tv;
  }
  if (kin != keys) {
    RNN_CUDA(cudaMemcpyAsync(keys, kin, sizeof(K) * n, cudaMemcpyDeviceToDevice, st));
    RNN_CUDA(cudaMemcpyAsync(vals, vin, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  }
  return RNN_OK;
}

}  // namespace

size_t scan_workspace_bytes(int64_t n) { return scan_ws_rec(n) + 256; }

rnn_status exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* ws,
                              cudaStream_t st) {
  if (n <= 0) {
    RNN_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
    return RNN_OK;
  }
  const int64_t tiles = ceil_div(n, SCAN_TILE);
  if (tiles == 1) {
    scan_tiles<<<1, SCAN_THREADS, 0, st>>>(in, out, n, nullptr);
    RNN_LAUNCH_CHECK();
    return RNN_OK;
  }
  Carve c(ws);
  int64_t* sums = c.take<int64_t>(tiles + 1);
  void* rest = c.base + ((c.used + 255) & ~size_t(255));
  scan_tile_sums<<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(in, n, sums);
  RNN_LAUNCH_CHECK();
  RNN_TRY(exclusive_scan_i64(sums, sums, tiles, rest, st));
  scan_tiles<<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(in, out, n, sums);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

size_t radix_sort_workspace_bytes(int64_t n) {
  const int64_t n_tiles = ceil_div(n > 0 ? n : 1, RS_TILE);
  size_t b = 0;
  auto add = [&](size_t x) { b = ((b + 255) & ~size_t(255)) + x; };
  add(sizeof(uint64_t) * n);
  add(sizeof(int32_t) * n);
  add(sizeof(int64_t) * (256 * n_tiles + 1));
  add(scan_workspace_bytes(256 * n_tiles));
  return b + 256;
}

rnn_status radix_sort_u64(uint64_t* keys, int32_t* vals, int64_t n, int bits, void* ws,
                          cudaStream_t st) {
  return radix_sort_impl<uint64_t>(keys, vals, n, bits, ws, st);
}
rnn_status radix_sort_u32(uint32_t* keys, int32_t* vals, int64_t n, int bits, void* ws,
                          cudaStream_t st) {
  return radix_sort_impl<uint32_t>(keys, vals, n, bits, ws, st);
}

}  // namespace rnn
