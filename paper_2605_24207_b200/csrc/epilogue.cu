// epilogue.cu -- node epilogues: y = gate * act(x + bias) + (1 - gate) * resid
//
// The per-node transformation of a rule after its aggregate or projection: GCN's bias and ReLU
// (PyG GCNConv, O7), the HGT skip gate sigmoid(skip) over the previous layer's
// H (PAPER.md:1392-1394 [src-only]), GELU.  The forward is normally fused into the LJA's final
// store (rowsplit.cuh lean_store); this file holds the standalone forward (other LJA paths, a
// projection output, a union accumulated first) and the backward: dx, d_bias (fixed-order
// two-stage column sums, deterministic), d_resid and d_gate.
#include "lja.cuh"

namespace rnn {
namespace {

constexpr int EPI_CHUNK = 256;    // rows per partial of the column / gate sums (2,048 left one
                                  // block per 2,048 rows walking 256 rows per thread: 125 us on
                                  // Cora's 7-wide layer)

EpiD epi_dev(const rnn_epilogue* e) {
  EpiD d{};
  if (!e) return d;
  d.on = 1;
  d.bias = e->bias;
  d.act = e->act;
  d.gate = e->resid ? e->gate : 1.f;
  d.resid = e->resid;
  d.ld_resid = e->ld_resid;
  d.pre = e->pre;
  d.ld_pre = e->ld_pre;
  return d;
}

__global__ void epi_fwd_kernel(const float* __restrict__ x, int64_t ldx, int64_t rows, int dim,
                               EpiD e, float* y, int64_t ldy) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * dim) return;
  const int64_t r = i / dim;
  const int c = (int)(i % dim);
  float v = x[r * ldx + c];
  if (e.bias) v += e.bias[c];
  if (e.pre) e.pre[r * e.ld_pre + c] = v;
  v = epi_act(e.act, v);
  if (e.resid) v = e.gate * v + (1.f - e.gate) * e.resid[r * e.ld_resid + c];
  y[r * ldy + c] = v;
}

// one block per (32-column slab, row chunk): thread (tx, ty) walks rows ty, ty + 8, ... of the
// chunk for column c0 + tx; per-chunk column partials of dx and per-chunk gate partials
__global__ void __launch_bounds__(256) epi_bwd_kernel(const float* __restrict__ dy, int64_t lddy,
                                                      const float* __restrict__ y, int64_t ldy,
                                                      int64_t rows, int dim, EpiD e,
                                                      float* dx, int64_t lddx,
                                                      float* __restrict__ dres, int64_t ldres,
                                                      float* __restrict__ part_b,
                                                      float* __restrict__ part_g) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  const int64_t r0 = (int64_t)blockIdx.y * EPI_CHUNK;
  const int64_t r1 = r0 + EPI_CHUNK < rows ? r0 + EPI_CHUNK : rows;
  float sb = 0.f, sg = 0.f;
  if (c < dim) {
#pragma unroll 4
    for (int64_t r = r0 + ty; r < r1; r += 8) {
      const float g = dy[r * lddy + c];
      float xb;          // x + bias (pre-activation)
      if (e.pre) xb = e.pre[r * e.ld_pre + c];
      else xb = y[r * ldy + c];   // act none / ReLU without resid: y decides act'
      const float d = g * e.gate * epi_dact(e.act, xb);
      if (dx) dx[r * lddx + c] = d;
      if (dres) dres[r * ldres + c] = (1.f - e.gate) * g;
      if (part_g) sg += g * (epi_act(e.act, xb) - e.resid[r * e.ld_resid + c]);
      sb += d;
    }
  }
  __shared__ float sh_b[8][33];
  __shared__ float sh_g[256];
  sh_b[ty][tx] = sb;
  sh_g[threadIdx.x] = sg;
  __syncthreads();
  if (ty == 0 && c < dim && part_b) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += sh_b[k][tx];
    part_b[(int64_t)blockIdx.y * dim + c] = t;
  }
  if (part_g) {   // fixed tree over the block, one partial per block
    for (int s = 128; s > 0; s >>= 1) {
      if (threadIdx.x < s) sh_g[threadIdx.x] += sh_g[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) part_g[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = sh_g[0];
  }
}

// vectorised variant (dim % 4 == 0, 16-byte aligned rows): block = 8 warps x EPI_VROWS rows,
// lane = one float4 column quad of a 128-column slab; per-block column partials of dx
constexpr int EPI_VROWS = 256;
__global__ void __launch_bounds__(256) epi_bwd4_kernel(const float* __restrict__ dy, int64_t lddy,
                                                       const float* __restrict__ y, int64_t ldy,
                                                       int64_t rows, int dim, EpiD e,
                                                       float* dx, int64_t lddx,
                                                       float* __restrict__ dres, int64_t ldres,
                                                       float* __restrict__ part_b,
                                                       float* __restrict__ part_g) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int c = blockIdx.x * 128 + 4 * lane;
  const int64_t r0 = (int64_t)blockIdx.y * EPI_VROWS;
  const int64_t r1 = r0 + EPI_VROWS < rows ? r0 + EPI_VROWS : rows;
  float4 sb = make_float4(0.f, 0.f, 0.f, 0.f);
  float sg = 0.f;
  if (c < dim) {
    const float4 bias = e.bias ? *reinterpret_cast<const float4*>(e.bias + c) : sb;
    for (int64_t r = r0 + wp; r < r1; r += 8) {
      const float4 g = *reinterpret_cast<const float4*>(dy + r * lddy + c);
      // act none without the gate's sum: act' = 1, the forward output is not read
      float4 xb = (e.act == 0 && !part_g) ? make_float4(0.f, 0.f, 0.f, 0.f)
                  : e.pre ? *reinterpret_cast<const float4*>(e.pre + r * e.ld_pre + c)
                          : *reinterpret_cast<const float4*>(y + r * ldy + c);
      float4 d;
      d.x = g.x * e.gate * epi_dact(e.act, xb.x);
      d.y = g.y * e.gate * epi_dact(e.act, xb.y);
      d.z = g.z * e.gate * epi_dact(e.act, xb.z);
      d.w = g.w * e.gate * epi_dact(e.act, xb.w);
      if (dx) *reinterpret_cast<float4*>(dx + r * lddx + c) = d;
      if (dres)
        *reinterpret_cast<float4*>(dres + r * ldres + c) = f4_scale(1.f - e.gate, g);
      if (part_g) {
        const float4 rr = *reinterpret_cast<const float4*>(e.resid + r * e.ld_resid + c);
        sg += g.x * (epi_act(e.act, xb.x) - rr.x) + g.y * (epi_act(e.act, xb.y) - rr.y) +
              g.z * (epi_act(e.act, xb.z) - rr.z) + g.w * (epi_act(e.act, xb.w) - rr.w);
      }
      sb = f4_add(sb, d);
      (void)bias;
    }
  }
  __shared__ float4 sh_b[8][32];
  __shared__ float sh_g[256];
  sh_b[wp][lane] = sb;
  sh_g[threadIdx.x] = sg;
  __syncthreads();
  if (wp == 0 && c < dim && part_b) {
    float4 t = sh_b[0][lane];
    for (int k = 1; k < 8; ++k) t = f4_add(t, sh_b[k][lane]);
    *reinterpret_cast<float4*>(part_b + (int64_t)blockIdx.y * dim + c) = t;
  }
  if (part_g) {
    for (int s = 128; s > 0; s >>= 1) {
      if (threadIdx.x < s) sh_g[threadIdx.x] += sh_g[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) part_g[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = sh_g[0];
  }
}

// bias-only backward (act none, no dx / d_resid / d_gate: the GCN's last layer): per-chunk
// column partials of gate * dy -- lane = float4 column quad, warp w takes rows w, w + 8, ... of
// the chunk four at a time (independent loads in flight), warps summed in a fixed order
__global__ void __launch_bounds__(256) epi_colsum4_kernel(const float* __restrict__ dy,
                                                          int64_t lddy, int64_t rows, int dim,
                                                          float gate, float* __restrict__ part_b) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int c = blockIdx.x * 128 + 4 * lane;
  const int64_t r0 = (int64_t)blockIdx.y * EPI_VROWS;
  const int64_t r1 = r0 + EPI_VROWS < rows ? r0 + EPI_VROWS : rows;
  float4 a0 = f4_zero(), a1 = f4_zero(), a2 = f4_zero(), a3 = f4_zero();
  if (c < dim) {
    int64_t r = r0 + wp;
    for (; r + 24 < r1; r += 32) {
      a0 = f4_add(a0, *reinterpret_cast<const float4*>(dy + r * lddy + c));
      a1 = f4_add(a1, *reinterpret_cast<const float4*>(dy + (r + 8) * lddy + c));
      a2 = f4_add(a2, *reinterpret_cast<const float4*>(dy + (r + 16) * lddy + c));
      a3 = f4_add(a3, *reinterpret_cast<const float4*>(dy + (r + 24) * lddy + c));
    }
    for (; r < r1; r += 8) a0 = f4_add(a0, *reinterpret_cast<const float4*>(dy + r * lddy + c));
  }
  __shared__ float4 sh[8][32];
  sh[wp][lane] = f4_add(f4_add(a0, a1), f4_add(a2, a3));
  __syncthreads();
  if (wp == 0 && c < dim) {
    float4 t = sh[0][lane];
    for (int k = 1; k < 8; ++k) t = f4_add(t, sh[k][lane]);
    *reinterpret_cast<float4*>(part_b + (int64_t)blockIdx.y * dim + c) = f4_scale(gate, t);
  }
}

// out[c] = sum over the chunks' partial rows, fixed order: block = 32 columns x 8 chunk lanes,
// lane j sums chunks j, j + 8, ... with four loads in flight, then the 8 sums in order (one
// thread per column summing 662 rows serially took 41 us at arxiv size)
__global__ void __launch_bounds__(256) epi_colsum_final(const float* __restrict__ part,
                                                        int64_t chunks, int dim,
                                                        float* __restrict__ out) {
  __shared__ float sh[8][33];
  const int lane = threadIdx.x & 31, j = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
  if (c < dim) {
    int64_t k = j;
    for (; k + 24 < chunks; k += 32) {
      t0 += part[k * dim + c];
      t1 += part[(k + 8) * dim + c];
      t2 += part[(k + 16) * dim + c];
      t3 += part[(k + 24) * dim + c];
    }
    for (; k < chunks; k += 8) t0 += part[k * dim + c];
  }
  sh[j][lane] = (t0 + t1) + (t2 + t3);
  __syncthreads();
  if (j == 0 && c < dim) {
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += sh[q][lane];
    out[c] = s;
  }
}

__global__ void epi_sum_final(const float* __restrict__ part, int64_t n, float* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  float t = 0.f;
  for (int64_t k = 0; k < n; ++k) t += part[k];
  *out = t;
}

rnn_status check_epi(const rnn_epilogue* e, int dim, bool need_pre_for_bwd) {
  RNN_REQUIRE(e, RNN_ERR_INVALID_ARGUMENT, "epilogue is NULL");
  RNN_REQUIRE(e->act >= RNN_ACT_NONE && e->act <= RNN_ACT_GELU, RNN_ERR_INVALID_ARGUMENT,
              "unknown activation %d", (int)e->act);
  RNN_REQUIRE(!e->resid || (e->gate >= 0.f && e->gate <= 1.f && e->ld_resid >= dim),
              RNN_ERR_INVALID_ARGUMENT, "resid needs gate in [0, 1] and ld_resid >= dim");
  RNN_REQUIRE(!e->pre || e->ld_pre >= dim, RNN_ERR_INVALID_ARGUMENT, "ld_pre < dim");
  if (need_pre_for_bwd)
    RNN_REQUIRE(e->pre || (e->act != RNN_ACT_GELU && !(e->act == RNN_ACT_RELU && e->resid)),
                RNN_ERR_INVALID_ARGUMENT,
                "the backward of GELU (or ReLU with a residual) needs the saved pre-activation");
  return RNN_OK;
}

}  // namespace

rnn_status epilogue_inplace(float* y, int64_t ldy, int64_t rows, int dim, const EpiD& e,
                            cudaStream_t st) {
  if (rows == 0 || dim == 0) return RNN_OK;
  epi_fwd_kernel<<<(unsigned)ceil_div(rows * dim, 256), 256, 0, st>>>(y, ldy, rows, dim, e, y, ldy);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

EpiD epi_from_abi(const rnn_epilogue* e) { return epi_dev(e); }

}  // namespace rnn

using namespace rnn;

extern "C" rnn_status rnn_epilogue_fwd(const float* x, int64_t ldx, int64_t rows, int32_t dim,
                                       const rnn_epilogue* epi, float* y, int64_t ldy,
                                       void* stream) {
  clear_error();
  RNN_TRY(check_epi(epi, dim, false));
  RNN_REQUIRE(rows >= 0 && dim >= 1 && ldx >= dim && ldy >= dim &&
                  (rows == 0 || (x && y)),
              RNN_ERR_INVALID_ARGUMENT, "bad argument");
  if (rows == 0) return RNN_OK;
  const EpiD e = epi_dev(epi);
  epi_fwd_kernel<<<(unsigned)ceil_div(rows * dim, 256), 256, 0, as_stream(stream)>>>(
      x, ldx, rows, dim, e, y, ldy);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

extern "C" rnn_status rnn_epilogue_bwd_workspace_size(int64_t rows, int32_t dim, size_t* bytes) {
  clear_error();
  RNN_REQUIRE(bytes && rows >= 0 && dim >= 1, RNN_ERR_INVALID_ARGUMENT, "bad argument");
  const int64_t chunks = ceil_div(rows > 0 ? rows : 1, EPI_VROWS);   // >= the scalar path's
  const int64_t slabs = ceil_div(dim, 32);
  *bytes = sizeof(float) * (size_t)(chunks * dim + chunks * slabs) + 256;
  return RNN_OK;
}

extern "C" rnn_status rnn_epilogue_bwd(const float* dy, int64_t lddy, const float* y, int64_t ldy,
                                       int64_t rows, int32_t dim, const rnn_epilogue* epi,
                                       float* dx, int64_t lddx, float* d_bias, float* d_resid,
                                       int64_t ld_dresid, float* d_gate, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  clear_error();
  RNN_TRY(check_epi(epi, dim, true));
  RNN_REQUIRE(rows >= 0 && dim >= 1 && lddy >= dim && (rows == 0 || dy), RNN_ERR_INVALID_ARGUMENT,
              "bad argument");
  RNN_REQUIRE(epi->pre || y || rows == 0, RNN_ERR_INVALID_ARGUMENT,
              "the forward output y is needed without a saved pre-activation");
  RNN_REQUIRE(!dx || lddx >= dim, RNN_ERR_INVALID_ARGUMENT, "lddx < dim");
  RNN_REQUIRE(!d_resid || (epi->resid && ld_dresid >= dim), RNN_ERR_INVALID_ARGUMENT,
              "d_resid needs a residual and ld_dresid >= dim");
  RNN_REQUIRE(!d_gate || (epi->resid && epi->pre), RNN_ERR_INVALID_ARGUMENT,
              "d_gate needs the residual and the saved pre-activation");
  size_t need = 0;
  RNN_TRY(rnn_epilogue_bwd_workspace_size(rows, dim, &need));
  RNN_REQUIRE(workspace && workspace_bytes >= need, RNN_ERR_WORKSPACE_TOO_SMALL,
              "epilogue backward workspace %zu < %zu bytes", workspace_bytes, need);
  cudaStream_t st = as_stream(stream);
  if (rows == 0) {
    if (d_bias) RNN_CUDA(cudaMemsetAsync(d_bias, 0, sizeof(float) * dim, st));
    if (d_gate) RNN_CUDA(cudaMemsetAsync(d_gate, 0, sizeof(float), st));
    return RNN_OK;
  }
  const EpiD e = epi_dev(epi);
  // float4 path when every row operand is 16-byte aligned with ld % 4 == 0
  auto al = [](const void* p, int64_t ld) { return !p || (aligned16(p) && ld % 4 == 0); };
  const bool vec = dim % 4 == 0 && al(dy, lddy) && al(y, ldy) && al(dx, lddx) &&
                   al(d_resid, ld_dresid) && al(epi->pre, epi->ld_pre) &&
                   al(epi->resid, epi->ld_resid) && al(epi->bias, 4);
  const int64_t chunks = vec ? ceil_div(rows, EPI_VROWS) : ceil_div(rows, EPI_CHUNK);
  const int64_t slabs = vec ? ceil_div(dim, 128) : ceil_div(dim, 32);
  float* part_b = reinterpret_cast<float*>(workspace);
  float* part_g = part_b + chunks * dim;
  dim3 grid((unsigned)slabs, (unsigned)chunks);
  const bool bias_only = vec && d_bias && !dx && !d_resid && !d_gate && epi->act == RNN_ACT_NONE;
  if (bias_only)
    epi_colsum4_kernel<<<grid, 256, 0, st>>>(dy, lddy, rows, dim, e.gate, part_b);
  else if (vec)
    epi_bwd4_kernel<<<grid, 256, 0, st>>>(dy, lddy, y, ldy, rows, dim, e, dx, lddx, d_resid,
                                          ld_dresid, d_bias ? part_b : nullptr,
                                          d_gate ? part_g : nullptr);
  else
    epi_bwd_kernel<<<grid, 256, 0, st>>>(dy, lddy, y, ldy, rows, dim, e, dx, lddx, d_resid,
                                         ld_dresid, d_bias ? part_b : nullptr,
                                         d_gate ? part_g : nullptr);
  RNN_LAUNCH_CHECK();
  if (d_bias) {
    epi_colsum_final<<<(unsigned)ceil_div(dim, 32), 256, 0, st>>>(part_b, chunks, dim, d_bias);
    RNN_LAUNCH_CHECK();
  }
  if (d_gate) {
    epi_sum_final<<<1, 32, 0, st>>>(part_g, chunks * slabs, d_gate);
    RNN_LAUNCH_CHECK();
  }
  return RNN_OK;
}
