// lja_max.cu -- the MAX aggregate of the projected union ("sum, mean, or max",
// :755 scatter aggregates), forward and backward.
//
//   out[g, c] = max over join rows p of group g of  w_p * z_s[src_row[p], c]     (SRC combine)
//   arg[g, c] = the LOWEST join position attaining it (deterministic tie-break; -1 and out = 0
//               for an empty group -- the scatter_max convention)
//   d z_s[s, c] = sum over (g, c) with src_row[arg[g, c]] = s of w_p d_out[g, c]
//   d w_p       = sum over c with arg[g, c] = p of d_out[g, c] z_s[s_p, c]
//
// Forward: one warp per group, lanes over float4 column quads, 4 rows in flight (values and
// the strict > comparison keep the first position on ties).  Backward: the transposed CSR
// (source-major, no atomics): for every join row of source s the warp gathers the group's
// arg-max row and adds w_p d_out[g] where it points at p.
#include "lja.cuh"

namespace rnn {
namespace {

__global__ void __launch_bounds__(256) max_fwd_kernel(const int64_t* __restrict__ gp, int64_t G,
                                                      const int32_t* __restrict__ src_row,
                                                      const int32_t* __restrict__ edge_row,
                                                      const float* __restrict__ z, int64_t ldz,
                                                      int D, const float* __restrict__ w,
                                                      int64_t ldw, int w_by_pos,
                                                      float* __restrict__ out, int64_t ldo,
                                                      int32_t* __restrict__ arg, int64_t lda) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= G) return;
  const int lane = threadIdx.x & 31;
  const int64_t b = gp[g], e = gp[g + 1];
  for (int c0 = 4 * lane; c0 < D; c0 += 128) {
    float best[4];
    int32_t ap[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) { best[j] = 0.f; ap[j] = -1; }
    for (int64_t p0 = b; p0 < e; p0 += 4) {
      float4 v[4];
      float wp[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t p = p0 + u < e ? p0 + u : b;
        const int32_t s = src_row[p];
        v[u] = *reinterpret_cast<const float4*>(z + (int64_t)s * ldz + c0);
        wp[u] = w ? __ldg(w + (w_by_pos ? p : (int64_t)edge_row[p]) * ldw) : 1.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (p0 + u >= e) break;
        const float x[4] = {wp[u] * v[u].x, wp[u] * v[u].y, wp[u] * v[u].z, wp[u] * v[u].w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (ap[j] < 0 || x[j] > best[j]) { best[j] = x[j]; ap[j] = (int32_t)(p0 + u); }
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (c0 + j < D) {
        out[g * ldo + c0 + j] = ap[j] < 0 ? 0.f : best[j];
        arg[g * lda + c0 + j] = ap[j];
      }
  }
}

// one warp per source row s: lanes over columns; d z[s] and (optionally) d w per join row
__global__ void __launch_bounds__(256) max_bwd_kernel(const int64_t* __restrict__ sp, int64_t n_s,
                                                      const int32_t* __restrict__ src_pos,
                                                      const int32_t* __restrict__ src_group,
                                                      const int32_t* __restrict__ edge_row,
                                                      const float* __restrict__ z, int64_t ldz,
                                                      int D, const float* __restrict__ w,
                                                      int64_t ldw, int w_by_pos,
                                                      const int32_t* __restrict__ arg, int64_t lda,
                                                      const float* __restrict__ dO, int64_t lddo,
                                                      float* __restrict__ dz, int64_t lddz,
                                                      float* __restrict__ dw, int64_t lddw) {
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= n_s) return;
  const int lane = threadIdx.x & 31;
  const int64_t qb = sp[s], qe = sp[s + 1];
  for (int c0 = 0; c0 < D; c0 += 32) {
    const int c = c0 + lane;
    const bool ok = c < D;
    const float zc = ok && dw ? z[s * ldz + c] : 0.f;
    float acc = 0.f;
    for (int64_t q = qb; q < qe; ++q) {
      const int32_t p = src_pos[q];
      const int64_t g = src_group[q];
      const int64_t wi = w_by_pos ? (int64_t)p : (int64_t)edge_row[p];
      const bool hit = ok && arg[g * lda + c] == p;
      const float d = hit ? dO[g * lddo + c] : 0.f;
      acc += (w ? __ldg(w + wi * ldw) : 1.f) * d;
      if (dw) {
        float t = d * zc;
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
        if (lane == 0) dw[wi * lddw] = c0 == 0 ? t : dw[wi * lddw] + t;
      }
    }
    if (ok && dz) dz[s * lddz + c] = acc;
  }
}

rnn_status check_max(const rnn_join_index* idx, const rnn_lifted_query* q) {
  RNN_REQUIRE(idx && q, RNN_ERR_INVALID_ARGUMENT, "idx and q are required");
  RNN_REQUIRE(q->agg == RNN_AGG_MAX && q->combine == RNN_COMBINE_SRC, RNN_ERR_UNSUPPORTED,
              "MAX takes combine SRC (w * z_s)");
  RNN_REQUIRE(q->src.data && q->src.mode == RNN_BY_ROW && !q->dst.data && !q->src_key.data,
              RNN_ERR_INVALID_ARGUMENT, "MAX needs src (by row) and no dst / src_key");
  RNN_REQUIRE(!q->edge.data || q->edge.dim == 1, RNN_ERR_SHAPE_MISMATCH,
              "MAX takes a scalar (dim 1) edge weight");
  RNN_REQUIRE(q->src.dim >= 1 && q->src.dim <= 512 && q->src.ld % 4 == 0 &&
                  aligned16(q->src.data),
              RNN_ERR_UNSUPPORTED, "src: 1 <= dim <= 512, ld %% 4 == 0, 16-byte aligned");
  return RNN_OK;
}

}  // namespace
}  // namespace rnn

using namespace rnn;

extern "C" rnn_status rnn_join_aggregate_max_fwd(const rnn_join_index* idx,
                                                 const rnn_lifted_query* q, float* out,
                                                 int64_t ld_out, int32_t* argmax, int64_t ld_arg,
                                                 void* stream) {
  clear_error();
  RNN_TRY(check_max(idx, q));
  const int D = q->src.dim;
  RNN_REQUIRE(ld_out >= D && ld_arg >= D, RNN_ERR_INVALID_ARGUMENT, "ld_out / ld_arg < dim");
  if (idx->n_groups == 0) return RNN_OK;
  RNN_REQUIRE(out && argmax, RNN_ERR_INVALID_ARGUMENT, "out and argmax are required");
  max_fwd_kernel<<<(unsigned)ceil_div(idx->n_groups, 8), 256, 0, as_stream(stream)>>>(
      idx->group_ptr, idx->n_groups, idx->src_row, idx->edge_row, q->src.data, q->src.ld, D,
      q->edge.data, q->edge.ld, q->edge.mode == RNN_BY_POSITION, out, ld_out, argmax, ld_arg);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

extern "C" rnn_status rnn_join_aggregate_max_bwd(const rnn_join_index* idx,
                                                 const rnn_lifted_query* q, const int32_t* argmax,
                                                 int64_t ld_arg, const float* d_out,
                                                 int64_t ld_dout, float* d_src, float* d_edge,
                                                 void* stream) {
  clear_error();
  RNN_TRY(check_max(idx, q));
  const int D = q->src.dim;
  RNN_REQUIRE(ld_arg >= D && ld_dout >= D, RNN_ERR_INVALID_ARGUMENT, "ld_arg / ld_dout < dim");
  RNN_REQUIRE(!d_edge || q->edge.data, RNN_ERR_INVALID_ARGUMENT, "d_edge needs an edge weight");
  cudaStream_t st = as_stream(stream);
  const int64_t n_s = idx->n_src_rows;
  if (d_edge && q->edge.mode == RNN_BY_ROW && idx->n_edge_rows > 0)   // rows on no join row
    RNN_CUDA(cudaMemset2DAsync(d_edge, sizeof(float) * q->edge.ld, 0, sizeof(float),
                               idx->n_edge_rows, st));
  if (idx->n_join_rows == 0) {
    if (d_src && n_s > 0)
      RNN_CUDA(cudaMemset2DAsync(d_src, sizeof(float) * q->src.ld, 0, sizeof(float) * D, n_s, st));
    return RNN_OK;
  }
  RNN_REQUIRE(argmax && d_out, RNN_ERR_INVALID_ARGUMENT, "argmax and d_out are required");
  RNN_REQUIRE(idx->src_ptr && idx->src_pos && idx->src_group, RNN_ERR_INVALID_ARGUMENT,
              "the MAX backward needs the transposed index");
  if (n_s == 0) return RNN_OK;
  max_bwd_kernel<<<(unsigned)ceil_div(n_s, 8), 256, 0, st>>>(
      idx->src_ptr, n_s, idx->src_pos, idx->src_group, idx->edge_row, q->src.data, q->src.ld, D,
      q->edge.data, q->edge.ld, q->edge.mode == RNN_BY_POSITION, argmax, ld_arg, d_out, ld_dout,
      d_src, q->src.ld, d_edge, q->edge.ld);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}
