// misc.cu -- program helpers: GCN normalisation weights and the multi-GPU hash partition.
#include "common.cuh"
#include <algorithm>

namespace rnn {
namespace {

__global__ void deg_kernel(const int64_t* __restrict__ gp, const int32_t* __restrict__ dst_row,
                           int64_t G, int32_t* deg, int* bad) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= G) return;
  const int32_t r = dst_row[g];
  if (r < 0) { *bad = 1; return; }
  deg[r] = (int32_t)(gp[g + 1] - gp[g]);
}

// w[p] = deg(s_p)^-1/2 deg(t_g)^-1/2 ; warp per group
__global__ void norm_kernel(const int64_t* __restrict__ gp, const int32_t* __restrict__ src_row,
                            int64_t G, const int32_t* __restrict__ deg, float* __restrict__ w) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= G) return;
  const int64_t b = gp[g], e = gp[g + 1];
  const float rt = 1.f / sqrtf((float)(e - b));
  for (int64_t p = b + (threadIdx.x & 31); p < e; p += 32) {
    const int32_t ds = deg[src_row[p]];
    w[p] = ds > 0 ? rt * (1.f / sqrtf((float)ds)) : 0.f;
  }
}

// w[p] = src_deg[s_p]^-1/2 |g|^-1/2 ; warp per group (sharded GCN: S spans every rank's rows)
__global__ void norm_deg_kernel(const int64_t* __restrict__ gp, const int32_t* __restrict__ src_row,
                                int64_t G, const int32_t* __restrict__ sdeg, float* __restrict__ w) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= G) return;
  const int64_t b = gp[g], e = gp[g + 1];
  const float rt = 1.f / sqrtf((float)(e - b));
  for (int64_t p = b + (threadIdx.x & 31); p < e; p += 32) {
    const int32_t ds = sdeg[src_row[p]];
    w[p] = ds > 0 ? rt * (1.f / sqrtf((float)ds)) : 0.f;
  }
}

__global__ void group_size_kernel(const int64_t* __restrict__ gp, int64_t G, int32_t* __restrict__ sz) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g < G) sz[g] = (int32_t)(gp[g + 1] - gp[g]);
}

__global__ void partition_kernel(const int64_t* __restrict__ keys, int64_t n, uint32_t P,
                                 uint64_t seed, int32_t* __restrict__ owner) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) owner[i] = (int32_t)(splitmix64((uint64_t)keys[i] ^ seed) % P);
}

}  // namespace
}  // namespace rnn

using namespace rnn;

extern "C" rnn_status rnn_gcn_norm(const rnn_join_index* idx, float* w, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  clear_error();
  RNN_REQUIRE(idx && idx->group_ptr, RNN_ERR_INVALID_ARGUMENT, "index required");
  RNN_REQUIRE(idx->n_src_rows == idx->n_dst_rows && idx->n_src_rows > 0, RNN_ERR_INVALID_ARGUMENT,
              "GCN normalisation needs S and T to be the same node relation");
  const size_t need = sizeof(int32_t) * (size_t)idx->n_dst_rows + 256;
  if (!workspace) {
    RNN_REQUIRE(workspace_bytes == 0, RNN_ERR_INVALID_ARGUMENT, "workspace NULL");
  }
  RNN_REQUIRE(workspace && workspace_bytes >= need, RNN_ERR_WORKSPACE_TOO_SMALL,
              "workspace needs %zu bytes", need);
  RNN_REQUIRE(w || idx->n_join_rows == 0, RNN_ERR_INVALID_ARGUMENT, "w required");
  cudaStream_t st = as_stream(stream);
  int32_t* deg = static_cast<int32_t*>(workspace);
  int* bad = reinterpret_cast<int*>(static_cast<char*>(workspace) + need - 256);
  RNN_CUDA(cudaMemsetAsync(workspace, 0, need, st));
  const int64_t G = idx->n_groups;
  if (G == 0) return RNN_OK;
  deg_kernel<<<(unsigned)ceil_div(G, 256), 256, 0, st>>>(idx->group_ptr, idx->group_dst_row, G,
                                                          deg, bad);
  norm_kernel<<<(unsigned)ceil_div(G, 8), 256, 0, st>>>(idx->group_ptr, idx->src_row, G, deg, w);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

extern "C" rnn_status rnn_group_sizes(const rnn_join_index* idx, int32_t* size, void* stream) {
  clear_error();
  RNN_REQUIRE(idx && (idx->n_groups == 0 || (idx->group_ptr && size)), RNN_ERR_INVALID_ARGUMENT,
              "index / size required");
  if (idx->n_groups == 0) return RNN_OK;
  group_size_kernel<<<(unsigned)ceil_div(idx->n_groups, 256), 256, 0, as_stream(stream)>>>(
      idx->group_ptr, idx->n_groups, size);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

extern "C" rnn_status rnn_gcn_norm_src_deg(const rnn_join_index* idx, const int32_t* src_deg,
                                           float* w, void* stream) {
  clear_error();
  RNN_REQUIRE(idx && (idx->n_groups == 0 || (idx->group_ptr && idx->src_row)),
              RNN_ERR_INVALID_ARGUMENT, "index required");
  RNN_REQUIRE(idx->n_join_rows == 0 || (src_deg && w), RNN_ERR_INVALID_ARGUMENT,
              "src_deg and w required");
  if (idx->n_groups == 0) return RNN_OK;
  norm_deg_kernel<<<(unsigned)ceil_div(idx->n_groups, 8), 256, 0, as_stream(stream)>>>(
      idx->group_ptr, idx->src_row, idx->n_groups, src_deg, w);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

extern "C" rnn_status rnn_hash_partition(const int64_t* keys, int64_t n, int32_t P, uint64_t seed,
                                         int32_t* owner, void* stream) {
  clear_error();
  RNN_REQUIRE(P >= 1 && n >= 0 && (n == 0 || (keys && owner)), RNN_ERR_INVALID_ARGUMENT,
              "bad argument");
  if (n == 0) return RNN_OK;
  partition_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(keys, n, (uint32_t)P,
                                                                              seed, owner);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

namespace rnn {
namespace {
__global__ void accumulate_kernel(float* __restrict__ y, int64_t ldy, const float* __restrict__ x,
                                  int64_t ldx, int64_t rows, int cols, float beta) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  const int64_t r = i / cols;
  const int c = (int)(i % cols);
  float v = x[r * ldx + c];
  if (beta != 0.f) v += beta * y[r * ldy + c];
  y[r * ldy + c] = v;
}
}  // namespace
}  // namespace rnn

extern "C" rnn_status rnn_accumulate(float* y, int64_t ldy, const float* x, int64_t ldx,
                                     int64_t rows, int32_t cols, float beta, void* stream) {
  clear_error();
  RNN_REQUIRE(rows >= 0 && cols >= 0 && (rows == 0 || cols == 0 || (x && y)) && ldy >= cols &&
                  ldx >= cols,
              RNN_ERR_INVALID_ARGUMENT, "bad argument");
  if (rows == 0 || cols == 0) return RNN_OK;
  accumulate_kernel<<<(unsigned)ceil_div(rows * cols, 256), 256, 0, as_stream(stream)>>>(
      y, ldy, x, ldx, rows, cols, beta);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

namespace rnn {
namespace {
// y[i, :] = x[idx[i], :] (0 where idx[i] < 0): one warp per row, lanes over columns
__global__ void gather_rows_kernel(float* __restrict__ y, int64_t ldy, const float* __restrict__ x,
                                   int64_t ldx, const int32_t* __restrict__ idx, int64_t n,
                                   int cols) {
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int lane = threadIdx.x & 31;
  const int32_t r = idx[i];
  for (int c = lane; c < cols; c += 32) y[i * ldy + c] = r >= 0 ? x[(int64_t)r * ldx + c] : 0.f;
}
}  // namespace
}  // namespace rnn

extern "C" rnn_status rnn_gather_rows(float* y, int64_t ldy, const float* x, int64_t ldx,
                                      const int32_t* idx, int64_t n, int32_t cols, void* stream) {
  clear_error();
  RNN_REQUIRE(n >= 0 && cols >= 0 && (n == 0 || cols == 0 || (x && y && idx)) && ldy >= cols &&
                  ldx >= cols,
              RNN_ERR_INVALID_ARGUMENT, "bad argument");
  if (n == 0 || cols == 0) return RNN_OK;
  gather_rows_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, as_stream(stream)>>>(y, ldy, x, ldx, idx,
                                                                             n, cols);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

namespace rnn {
namespace {
// y[idx[i], :] += x[i, :] (idx distinct within one call: no two rows collide)
__global__ void scatter_add_rows_kernel(float* __restrict__ y, int64_t ldy,
                                        const float* __restrict__ x, int64_t ldx,
                                        const int32_t* __restrict__ idx, int64_t n, int cols) {
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int lane = threadIdx.x & 31;
  const int32_t r = idx[i];
  if (r < 0) return;
  for (int c = lane; c < cols; c += 32) y[(int64_t)r * ldy + c] += x[i * ldx + c];
}
}  // namespace
}  // namespace rnn

extern "C" rnn_status rnn_scatter_add_rows(float* y, int64_t ldy, const float* x, int64_t ldx,
                                           const int32_t* idx, int64_t n, int32_t cols,
                                           void* stream) {
  clear_error();
  RNN_REQUIRE(n >= 0 && cols >= 0 && (n == 0 || cols == 0 || (x && y && idx)) && ldy >= cols &&
                  ldx >= cols,
              RNN_ERR_INVALID_ARGUMENT, "bad argument");
  if (n == 0 || cols == 0) return RNN_OK;
  scatter_add_rows_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, as_stream(stream)>>>(y, ldy, x, ldx,
                                                                                  idx, n, cols);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

extern "C" rnn_status rnn_stream_l2_window(void* stream, const void* base, size_t bytes,
                                           float hit_ratio) {
  clear_error();
  RNN_REQUIRE((bytes == 0 || base) && hit_ratio >= 0.f && hit_ratio <= 1.f,
              RNN_ERR_INVALID_ARGUMENT, "bad argument");
  cudaStream_t st = as_stream(stream);
  int dev = 0, max_persist = 0, max_window = 0;
  RNN_CUDA(cudaGetDevice(&dev));
  RNN_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
  RNN_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev));
  cudaStreamAttrValue v{};
  if (bytes == 0) {
    v.accessPolicyWindow.base_ptr = nullptr;
    v.accessPolicyWindow.num_bytes = 0;
    v.accessPolicyWindow.hitRatio = 0.f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyNormal;
    v.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
    RNN_CUDA(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v));
    RNN_CUDA(cudaCtxResetPersistingL2Cache());
    RNN_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
    return RNN_OK;
  }
  const size_t win = std::min(bytes, (size_t)max_window);
  const size_t want = (size_t)((double)win * hit_ratio);
  RNN_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(want, (size_t)max_persist)));
  v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  v.accessPolicyWindow.num_bytes = win;
  v.accessPolicyWindow.hitRatio = hit_ratio;
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  RNN_CUDA(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v));
  return RNN_OK;
}
