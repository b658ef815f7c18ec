// train.cu -- the training step around the hot path: the loss relation
// and the fit statement's optimiser.
//
//   Loss(; CrossEntropyLoss()(Cls(z_p), z_l))  -> rnn_softmax_xent
//   ?fit <epochs = 100, lr = 0.01, weight_decay = 5e-4> Loss
//       -> rnn_adam over every parameter, per-tuple embeddings included
//
// The optimiser is not named in the paper; Adam with L2 weight decay added to the gradient
// (torch.optim.Adam semantics, the PyG GCN example the GCN row is compared with, :865) is the
// reading taken.  Both reductions (label count, loss) are fixed-order two-stage
// sums (deterministic); the Adam step counter lives in device memory so a whole training step
// can be captured once as a CUDA graph and replayed epoch after epoch.
#include "common.cuh"

namespace rnn {
namespace {

constexpr int XE_ROWS = 256;   // rows per block of the loss kernels

__global__ void xent_count_kernel(const int64_t* __restrict__ label, int64_t n,
                                  int* __restrict__ part) {
  __shared__ int sh[XE_ROWS];
  const int64_t i = blockIdx.x * (int64_t)XE_ROWS + threadIdx.x;
  sh[threadIdx.x] = i < n && label[i] >= 0;
  __syncthreads();
  for (int s = XE_ROWS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void xent_total_kernel(const int* __restrict__ part, int64_t nb, int* __restrict__ m) {
  if (threadIdx.x || blockIdx.x) return;
  int t = 0;
  for (int64_t b = 0; b < nb; ++b) t += part[b];
  *m = t;
}

// one thread per row: max, sum-exp, the row's loss and d_logits = (softmax - onehot) / m
__global__ void xent_row_kernel(const float* __restrict__ x, int64_t n, int C, int64_t ld,
                                const int64_t* __restrict__ label, const int* __restrict__ m,
                                float* __restrict__ dx, int64_t lddx, float* __restrict__ part) {
  __shared__ float sh[XE_ROWS];
  const int64_t i = blockIdx.x * (int64_t)XE_ROWS + threadIdx.x;
  float li = 0.f;
  if (i < n) {
    const float* r = x + i * ld;
    const int64_t y = label[i];
    if (y < 0) {
      if (dx) for (int c = 0; c < C; ++c) dx[i * lddx + c] = 0.f;
    } else {
      float mx = r[0];
      for (int c = 1; c < C; ++c) mx = fmaxf(mx, r[c]);
      float z = 0.f;
      for (int c = 0; c < C; ++c) z += expf(r[c] - mx);
      const float lz = logf(z);
      li = -(r[y] - mx - lz);
      const float inv_m = 1.f / (float)*m;
      if (dx)
        for (int c = 0; c < C; ++c)
          dx[i * lddx + c] = (expf(r[c] - mx - lz) - (c == y ? 1.f : 0.f)) * inv_m;
    }
  }
  sh[threadIdx.x] = li;
  __syncthreads();
  for (int s = XE_ROWS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void xent_loss_kernel(const float* __restrict__ part, int64_t nb,
                                 const int* __restrict__ m, float* __restrict__ loss) {
  if (threadIdx.x || blockIdx.x) return;
  float t = 0.f;
  for (int64_t b = 0; b < nb; ++b) t += part[b];
  *loss = *m > 0 ? t / (float)*m : 0.f;
}

__global__ void adam_tick_kernel(int64_t* t) { *t += 1; }

__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                            float* __restrict__ m, float* __restrict__ v, int64_t rows, int cols,
                            int64_t ldp, int64_t ldg, rnn_adam_config c,
                            const int64_t* __restrict__ t) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  const int64_t r = i / cols;
  const int col = (int)(i % cols);
  const double tt = (double)*t;
  const float c1 = (float)(1.0 - pow((double)c.beta1, tt));
  const float c2 = (float)(1.0 - pow((double)c.beta2, tt));
  float* pp = p + r * ldp + col;
  const float gi = g[r * ldg + col] + c.weight_decay * *pp;
  const float mi = c.beta1 * m[i] + (1.f - c.beta1) * gi;
  const float vi = c.beta2 * v[i] + (1.f - c.beta2) * gi * gi;
  m[i] = mi;
  v[i] = vi;
  *pp -= c.lr * (mi / c1) / (sqrtf(vi / c2) + c.eps);
}

}  // namespace
}  // namespace rnn

using namespace rnn;

extern "C" rnn_status rnn_softmax_xent_workspace_size(int64_t n, size_t* bytes) {
  clear_error();
  RNN_REQUIRE(bytes && n >= 0, RNN_ERR_INVALID_ARGUMENT, "bad argument");
  const int64_t nb = ceil_div(n > 0 ? n : 1, XE_ROWS);
  *bytes = (size_t)nb * (sizeof(int) + sizeof(float)) + 256;
  return RNN_OK;
}

extern "C" rnn_status rnn_softmax_xent(const float* logits, int64_t n, int32_t C, int64_t ld,
                                       const int64_t* label, float* loss, float* d_logits,
                                       int64_t ld_dlogits, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  clear_error();
  RNN_REQUIRE(n >= 0 && C >= 1 && ld >= C && loss && (n == 0 || (logits && label)) &&
                  (!d_logits || ld_dlogits >= C),
              RNN_ERR_INVALID_ARGUMENT, "bad argument");
  size_t need = 0;
  RNN_TRY(rnn_softmax_xent_workspace_size(n, &need));
  RNN_REQUIRE(workspace && workspace_bytes >= need, RNN_ERR_WORKSPACE_TOO_SMALL,
              "workspace %zu < %zu bytes", workspace_bytes, need);
  cudaStream_t st = as_stream(stream);
  const int64_t nb = ceil_div(n > 0 ? n : 1, XE_ROWS);
  int* cpart = reinterpret_cast<int*>(workspace);
  int* m = cpart + nb;
  float* lpart = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(m + 1) + 15) & ~uintptr_t(15));
  if (n == 0) {
    RNN_CUDA(cudaMemsetAsync(loss, 0, sizeof(float), st));
    return RNN_OK;
  }
  xent_count_kernel<<<(unsigned)nb, XE_ROWS, 0, st>>>(label, n, cpart);
  xent_total_kernel<<<1, 32, 0, st>>>(cpart, nb, m);
  xent_row_kernel<<<(unsigned)nb, XE_ROWS, 0, st>>>(logits, n, C, ld, label, m, d_logits,
                                                     ld_dlogits, lpart);
  xent_loss_kernel<<<1, 32, 0, st>>>(lpart, nb, m, loss);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

extern "C" rnn_status rnn_adam_tick(int64_t* step, void* stream) {
  clear_error();
  RNN_REQUIRE(step, RNN_ERR_INVALID_ARGUMENT, "step is NULL");
  adam_tick_kernel<<<1, 1, 0, as_stream(stream)>>>(step);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

extern "C" rnn_status rnn_adam(float* param, int64_t rows, int32_t cols, int64_t ld_param,
                               const float* grad, int64_t ld_grad, float* m, float* v,
                               const rnn_adam_config* cfg, const int64_t* step, void* stream) {
  clear_error();
  RNN_REQUIRE(cfg && step && rows >= 0 && cols >= 1 && ld_param >= cols && ld_grad >= cols &&
                  (rows == 0 || (param && grad && m && v)),
              RNN_ERR_INVALID_ARGUMENT, "bad argument");
  RNN_REQUIRE(cfg->beta1 >= 0.f && cfg->beta1 < 1.f && cfg->beta2 >= 0.f && cfg->beta2 < 1.f &&
                  cfg->eps >= 0.f && cfg->lr >= 0.f && cfg->weight_decay >= 0.f,
              RNN_ERR_INVALID_ARGUMENT, "Adam hyperparameters out of range");
  if (rows == 0) return RNN_OK;
  adam_kernel<<<(unsigned)ceil_div(rows * cols, 256), 256, 0, as_stream(stream)>>>(
      param, grad, m, v, rows, cols, ld_param, ld_grad, *cfg, step);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}
