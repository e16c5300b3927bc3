// Training-loop kernels for the reference's synthetic long-dependency task
// (proj/include/linrec/training.hpp): batch generation from the reference's
// counter-based splitmix64 stream, the linear readout with softmax
// cross-entropy, and a fused global-norm clip + Adam over one flat parameter
// buffer.  The layers themselves are the GILR-LSTM kernels (layers.cu).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "launch.h"
#include "linrec_cuda.h"

namespace linrec_dev {
namespace train {

// Rng::next_u64 (rng.hpp:21-27) for counter value `c` (1-based, pre-increment)
__device__ __forceinline__ uint64_t splitmix(uint64_t seed, uint64_t c) {
  uint64_t z = seed + c * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// generate_batch (training.hpp:30-43): row r draws coin() then T-1 below(p),
// so draw (r, t) is counter + r*T + t + 1.  x [T][b][p] one-hot, labels [b].
__global__ void k_synthetic_batch(uint64_t seed, uint64_t counter, int64_t T, int64_t b, int64_t p,
                                  float* __restrict__ x, int32_t* __restrict__ labels) {
  const int64_t total = T * b;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / b, r = i - t * b;
    const uint64_t d = splitmix(seed, counter + (uint64_t)(r * T + t) + 1);
    float* row = x + i * p;
    if (t == 0) {
      const bool positive = (d & 1u) != 0;
      row[0] = positive ? 1.f : -1.f;
      for (int64_t j = 1; j < p; ++j) row[j] = 0.f;
      labels[r] = positive ? 1 : 0;
    } else {
      const int64_t hot = (int64_t)(d % (uint64_t)p);
      for (int64_t j = 0; j < p; ++j) row[j] = j == hot ? 1.f : 0.f;
    }
  }
}

// logits = h_last W_out^T + b_out (model_forward :182-188); softmax_loss
// (:193-222) with d_logits = (softmax - onehot) / b; loss_acc = (mean loss,
// accuracy) summed in row order by one block (deterministic).
__global__ void k_readout_loss(const float* __restrict__ h, const float* __restrict__ W, const float* __restrict__ bo,
                               const int32_t* __restrict__ labels, float* __restrict__ logits,
                               float* __restrict__ dlogits, double* __restrict__ loss_acc, int64_t b, int64_t n,
                               int64_t b_total) {
  __shared__ double s_loss[256], s_ok[256];
  double loss = 0.0, ok = 0.0;
  for (int64_t r = threadIdx.x; r < b; r += blockDim.x) {
    float z0 = 0.f, z1 = 0.f;
    for (int64_t j = 0; j < n; ++j) {
      z0 = fmaf(h[r * n + j], W[j], z0);
      z1 = fmaf(h[r * n + j], W[n + j], z1);
    }
    z0 += bo[0];
    z1 += bo[1];
    logits[r * 2] = z0;
    logits[r * 2 + 1] = z1;
    const double a = z0, c = z1, mx = a > c ? a : c;
    const double ea = exp(a - mx), ec = exp(c - mx), zs = ea + ec;
    const int y = labels[r];
    loss -= log((y == 1 ? ec : ea) / zs);
    if ((c > a ? 1 : 0) == y) ok += 1.0;
    dlogits[r * 2] = (float)((ea / zs - (y == 0 ? 1.0 : 0.0)) / (double)b_total);
    dlogits[r * 2 + 1] = (float)((ec / zs - (y == 1 ? 1.0 : 0.0)) / (double)b_total);
  }
  s_loss[threadIdx.x] = loss;
  s_ok[threadIdx.x] = ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    double L = 0.0, A = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      L += s_loss[i];
      A += s_ok[i];
    }
    loss_acc[0] = L / (double)b_total;
    loss_acc[1] = A / (double)b_total;
  }
}

// model_backward readout (:229-240): dW_out[k][j] += sum_r dl[r][k] h[r][j],
// db_out[k] += sum_r dl[r][k], d_hlast[r][j] = sum_k dl[r][k] W_out[k][j].
__global__ void k_readout_backward(const float* __restrict__ dl, const float* __restrict__ h,
                                   const float* __restrict__ W, float* __restrict__ dW, float* __restrict__ db,
                                   float* __restrict__ dh, int64_t b, int64_t n) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    float g0 = 0.f, g1 = 0.f;
    for (int64_t r = 0; r < b; ++r) {  // fixed order: deterministic
      g0 = fmaf(dl[r * 2], h[r * n + j], g0);
      g1 = fmaf(dl[r * 2 + 1], h[r * n + j], g1);
      dh[r * n + j] = dl[r * 2] * W[j] + dl[r * 2 + 1] * W[n + j];
    }
    dW[j] += g0;
    dW[n + j] += g1;
  }
  if (blockIdx.x == 0 && threadIdx.x < 2) {
    float s = 0.f;
    for (int64_t r = 0; r < b; ++r) s += dl[r * 2 + threadIdx.x];
    db[threadIdx.x] += s;
  }
}

// clip_global_norm (:275-288) + Adam (:248-273), fused over one flat buffer.
// Pass 1: per-block sum of squares (double).
__global__ void k_sumsq(const float* __restrict__ g, int64_t count, double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = g[i];
    s += v * v;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// Pass 2: every block folds the partials in the same order (identical norm
// everywhere), then clips and applies Adam to its slice.  Block 0 reports the
// pre-clip norm.
__global__ void k_clip_adam(float* __restrict__ p, float* __restrict__ g, double* __restrict__ m,
                            double* __restrict__ v, int64_t count, const double* __restrict__ part, int nparts,
                            double lr, double beta1, double beta2, double eps, double bc1, double bc2,
                            double clip_norm, double* __restrict__ norm_out) {
  __shared__ double s_scale;
  if (threadIdx.x == 0) {
    double sq = 0.0;
    for (int i = 0; i < nparts; ++i) sq += part[i];
    const double norm = sqrt(sq);
    s_scale = (norm > clip_norm && norm > 0) ? clip_norm / norm : 1.0;
    if (blockIdx.x == 0 && norm_out != nullptr) *norm_out = norm;
  }
  __syncthreads();
  const double scale = s_scale;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    float gf = g[i];
    if (scale != 1.0) {
      gf = (float)((double)gf * scale);
      g[i] = gf;
    }
    const double gj = gf;
    const double mj = beta1 * m[i] + (1.0 - beta1) * gj;
    const double vj = beta2 * v[i] + (1.0 - beta2) * gj * gj;
    m[i] = mj;
    v[i] = vj;
    p[i] = (float)((double)p[i] - lr * (mj / bc1) / (sqrt(vj / bc2) + eps));
  }
}

}  // namespace train
}  // namespace linrec_dev

namespace {
int terr(int code, const std::string& m) { return linrec_impl::set_error(code, m.c_str()); }
#define TTRY(expr)                                                                                             \
  do {                                                                                                         \
    cudaError_t e_ = (expr);                                                                                   \
    if (e_ != cudaSuccess) return terr(LINREC_ERR_CUDA, std::string("linrec: CUDA error: ") + cudaGetErrorString(e_)); \
  } while (0)
constexpr int kAdamBlocks = 1184;  // 8 per SM; partial sums in this many slots
}  // namespace

extern "C" {

int linrec_synthetic_batch_f32(uint64_t seed, uint64_t counter, int64_t T, int64_t b, int64_t p, float* x,
                               int32_t* labels, void* stream) {
  if (p < 2) return terr(LINREC_ERR_SHAPE, "generate_batch: input_dim must be >= 2");
  if (T < 1) return terr(LINREC_ERR_SHAPE, "generate_batch: seq_len must be >= 1");
  if (b < 1 || !x || !labels) return terr(LINREC_ERR_VALUE, "generate_batch: batch >= 1 and buffers required");
  const int64_t total = T * b;
  const int64_t blocks = (total + 255) / 256;
  linrec_dev::train::k_synthetic_batch<<<(unsigned)(blocks < 65536 ? blocks : 65536), 256, 0,
                                         static_cast<cudaStream_t>(stream)>>>(seed, counter, T, b, p, x, labels);
  TTRY(cudaGetLastError());
  return LINREC_OK;
}

int linrec_readout_loss_f32(const float* h_last, const float* W_out, const float* b_out, const int32_t* labels,
                            float* logits, float* d_logits, double* loss_acc, int64_t b, int64_t n, int64_t b_total,
                            void* stream) {
  if (b < 1 || n < 1) return terr(LINREC_ERR_SHAPE, "softmax_loss: b, n must be >= 1");
  if (b_total < b) return terr(LINREC_ERR_VALUE, "softmax_loss: b_total must cover the local batch");
  if (!h_last || !W_out || !b_out || !labels || !logits || !d_logits || !loss_acc)
    return terr(LINREC_ERR_VALUE, "softmax_loss: NULL buffer");
  linrec_dev::train::k_readout_loss<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(h_last, W_out, b_out, labels,
                                                                                      logits, d_logits, loss_acc, b, n,
                                                                                      b_total);
  TTRY(cudaGetLastError());
  return LINREC_OK;
}

int linrec_readout_backward_f32(const float* d_logits, const float* h_last, const float* W_out, float* dW_out,
                                float* db_out, float* d_hlast, int64_t b, int64_t n, void* stream) {
  if (b < 1 || n < 1) return terr(LINREC_ERR_SHAPE, "readout backward: b, n must be >= 1");
  if (!d_logits || !h_last || !W_out || !dW_out || !db_out || !d_hlast)
    return terr(LINREC_ERR_VALUE, "readout backward: NULL buffer");
  linrec_dev::train::k_readout_backward<<<(unsigned)((n + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      d_logits, h_last, W_out, dW_out, db_out, d_hlast, b, n);
  TTRY(cudaGetLastError());
  return LINREC_OK;
}

size_t linrec_adam_scratch_bytes(void) { return sizeof(double) * kAdamBlocks; }

int linrec_clip_adam_f32(float* params, float* grads, double* m, double* v, int64_t count, double lr, double beta1,
                         double beta2, double eps, int64_t step, double clip_norm, double* norm_out, void* scratch,
                         size_t scratch_bytes, void* stream) {
  if (count < 1 || !params || !grads || !m || !v) return terr(LINREC_ERR_VALUE, "adam: buffers and count required");
  if (step < 1) return terr(LINREC_ERR_VALUE, "adam: step is 1-based");
  if (!scratch || scratch_bytes < linrec_adam_scratch_bytes())
    return terr(LINREC_ERR_VALUE, "adam: scratch smaller than linrec_adam_scratch_bytes()");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* part = static_cast<double*>(scratch);
  linrec_dev::train::k_sumsq<<<kAdamBlocks, 256, 0, st>>>(grads, count, part);
  TTRY(cudaGetLastError());
  const double bc1 = 1.0 - std::pow(beta1, (double)step), bc2 = 1.0 - std::pow(beta2, (double)step);
  linrec_dev::train::k_clip_adam<<<kAdamBlocks, 256, 0, st>>>(params, grads, m, v, count, part, kAdamBlocks, lr, beta1,
                                                              beta2, eps, bc1, bc2, clip_norm, norm_out);
  TTRY(cudaGetLastError());
  return LINREC_OK;
}

}  // extern "C"
