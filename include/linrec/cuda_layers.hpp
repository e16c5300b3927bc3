// linrec/cuda_layers.hpp -- C++ host mirror of the reference's layer entry
// points (proj/include/linrec/layers.hpp) over the C ABI of
// include/linrec_cuda.h.  Header-only; link against liblinrec_cuda.so.
//
// Same names and call shapes as the reference -- gilr_forward /
// gilr_backward (layers.hpp:78-133), gilr_lstm_forward / gilr_lstm_backward
// (:245-375), qrnn_forward / qrnn_backward (:449-548) -- with the Tensor3 /
// Tensor2 arguments replaced by views of caller-owned DEVICE buffers
// (DeviceTensor3 / DeviceTensor2 from cuda_scan.hpp) and the ThreadPool by a
// LayerContext (CUDA stream, GEMM precision, a scratch buffer grown on
// demand).  Gradients accumulate exactly as the reference's do; outputs are
// written into caller-provided views.  Errors throw the same exception types
// as cuda_scan.hpp (ContractViolation for shape errors).
#pragma once

#include <cstddef>
#include <string>

#include "linrec/cuda_scan.hpp"
#include "linrec_cuda.h"

namespace linrec {
namespace cuda {

enum class Activation { Tanh = LINREC_ACT_TANH, Identity = LINREC_ACT_IDENTITY, Relu = LINREC_ACT_RELU };
enum class Precision { Fp32 = LINREC_PREC_FP32, Tf32 = LINREC_PREC_TF32 };

// Stream + precision + scratch (the reference's ThreadPool slot).
class LayerContext {
 public:
  explicit LayerContext(void* stream = nullptr, Precision prec = Precision::Fp32, int device = 0)
      : stream_(stream), prec_(prec), device_(device) {}
  ~LayerContext() {
    if (buf_) linrec_device_free(buf_, device_, stream_);
  }
  LayerContext(const LayerContext&) = delete;
  LayerContext& operator=(const LayerContext&) = delete;

  void* stream() const { return stream_; }
  int precision() const { return static_cast<int>(prec_); }
  // scratch of at least `bytes` (256-byte aligned, stream-ordered growth)
  void* scratch(size_t bytes) {
    if (bytes > cap_) {
      if (buf_) linrec_device_free(buf_, device_, stream_);
      buf_ = nullptr;
      throw_status(linrec_device_malloc(&buf_, bytes, device_, stream_));
      cap_ = bytes;
    }
    return buf_;
  }
  size_t capacity() const { return cap_; }

 private:
  void* stream_;
  Precision prec_;
  int device_;
  void* buf_ = nullptr;
  size_t cap_ = 0;
};

// GilrParams<float> / GilrGrads<float> (layers.hpp:30-76) as device views.
struct GilrParams {
  const float* U = nullptr;  // [n][m]
  const float* V = nullptr;  // [n][m]
  const float* b_g = nullptr;
  const float* b_z = nullptr;
  Activation act = Activation::Tanh;
  index_t m = 0, n = 0;
  index_t input() const { return m; }
  index_t hidden() const { return n; }
  linrec_gilr_params_f32 c() const { return {U, V, b_g, b_z, static_cast<int>(act)}; }
};
struct GilrGrads {
  float *U = nullptr, *V = nullptr, *b_g = nullptr, *b_z = nullptr;
  linrec_gilr_grads_f32 c() const { return {U, V, b_g, b_z}; }
};
struct GilrCache {
  DeviceTensor3<float> g, i, h;  // activated gate, candidate, output (layers.hpp:62-64)
};

// GilrLstmParams<float> (:146-160), GilrLstmGrads (:192-211), GilrLstmCache
// (:183-188; htil holds T+1 rows, row 0 = htil0; gates = 4 planes).
struct GilrLstmParams {
  GilrParams surrogate;
  const float* U = nullptr;     // [4n][n]
  const float* V = nullptr;     // [4n][m]
  const float* bias = nullptr;  // [4n]
  index_t input() const { return surrogate.m; }
  index_t hidden() const { return surrogate.n; }
  linrec_gilr_lstm_params_f32 c() const { return {surrogate.c(), U, V, bias}; }
};
struct GilrLstmGrads {
  GilrGrads surrogate;
  float *U = nullptr, *V = nullptr, *bias = nullptr;
  linrec_gilr_lstm_grads_f32 c() const { return {surrogate.c(), U, V, bias}; }
};
struct GilrLstmCache {
  float *sg = nullptr, *si = nullptr, *htil = nullptr, *gates = nullptr, *c = nullptr;
  linrec_gilr_lstm_cache_f32 view() const { return {sg, si, htil, gates, c}; }
};

// QrnnParams<float> (:390-405): k taps packed [k][3n][m]; grads alike.
struct QrnnParams {
  const float* W = nullptr;
  const float* bias = nullptr;  // [3n]
  index_t m = 0, n = 0, k = 1;
};
struct QrnnGrads {
  float *W = nullptr, *bias = nullptr;
};
struct QrnnCache {
  float *gates = nullptr, *c = nullptr;  // [3][T][b][n], [T][b][n]
};

namespace detail {
inline void require_features(index_t have, index_t want, const char* what) {
  if (have != want) throw ContractViolation(std::string(what) + ": input feature mismatch");
}
}  // namespace detail

// gilr_forward (layers.hpp:78-100): h = GILR(x); cache g, i (and h).
inline void gilr_forward(const GilrParams& p, const DeviceTensor3<float>& x, const DeviceTensor2<float>& h0,
                         ScanMode mode, LayerContext& ctx, GilrCache& cache, DeviceTensor3<float>& h) {
  detail::require_features(x.features, p.input(), "gilr_forward");
  const size_t need = linrec_gilr_scratch_bytes(x.steps, x.batch, p.m, p.n);
  void* scr = ctx.scratch(need);  // grow first: capacity() below must see it
  const auto pc = p.c();
  throw_status(linrec_gilr_forward_f32(&pc, x.data, h0.data, h.data, cache.g.data, cache.i.data, x.steps, x.batch,
                                       p.m, p.n, static_cast<int>(mode), ctx.precision(), scr, ctx.capacity(),
                                       ctx.stream()));
  cache.h = h;
}

// gilr_backward (:102-133): accumulates into grads, writes dx (and dh0).
inline void gilr_backward(const GilrParams& p, const DeviceTensor3<float>& x, const DeviceTensor2<float>& h0,
                          const GilrCache& cache, const DeviceTensor3<float>& d_h, ScanMode mode, LayerContext& ctx,
                          GilrGrads& grads, DeviceTensor3<float>& dx, DeviceTensor2<float>* d_h0 = nullptr) {
  const size_t need = linrec_gilr_scratch_bytes(x.steps, x.batch, p.m, p.n);
  void* scr = ctx.scratch(need);  // grow first: capacity() below must see it
  const auto pc = p.c();
  auto gc = grads.c();
  throw_status(linrec_gilr_backward_f32(&pc, x.data, h0.data, cache.g.data, cache.i.data, cache.h.data, d_h.data, &gc,
                                        dx.data, d_h0 ? d_h0->data : nullptr, x.steps, x.batch, p.m, p.n,
                                        static_cast<int>(mode), ctx.precision(), scr, ctx.capacity(),
                                        ctx.stream()));
}

// gilr_lstm_forward (:245-293).
inline void gilr_lstm_forward(const GilrLstmParams& p, const DeviceTensor3<float>& x,
                              const DeviceTensor2<float>& htil0, const DeviceTensor2<float>& c0, ScanMode mode,
                              LayerContext& ctx, const GilrLstmCache& cache, DeviceTensor3<float>& h) {
  detail::require_features(x.features, p.input(), "gilr_lstm_forward");
  const size_t need = linrec_gilr_lstm_scratch_bytes(x.steps, x.batch, p.input(), p.hidden());
  void* scr = ctx.scratch(need);  // grow first: capacity() below must see it
  const auto pc = p.c();
  const auto cc = cache.view();
  throw_status(linrec_gilr_lstm_forward_f32(&pc, x.data, htil0.data, c0.data, h.data, &cc, x.steps, x.batch,
                                            p.input(), p.hidden(), static_cast<int>(mode), ctx.precision(),
                                            scr, ctx.capacity(), ctx.stream()));
}

// gilr_lstm_backward (:295-375).
inline void gilr_lstm_backward(const GilrLstmParams& p, const DeviceTensor3<float>& x,
                               const DeviceTensor2<float>& htil0, const DeviceTensor2<float>& c0,
                               const GilrLstmCache& cache, const DeviceTensor3<float>& d_h, ScanMode mode,
                               LayerContext& ctx, GilrLstmGrads& grads, DeviceTensor3<float>& dx,
                               DeviceTensor2<float>* d_htil0 = nullptr, DeviceTensor2<float>* d_c0 = nullptr) {
  const size_t need = linrec_gilr_lstm_scratch_bytes(x.steps, x.batch, p.input(), p.hidden());
  void* scr = ctx.scratch(need);  // grow first: capacity() below must see it
  const auto pc = p.c();
  const auto cc = cache.view();
  auto gc = grads.c();
  throw_status(linrec_gilr_lstm_backward_f32(&pc, x.data, htil0.data, c0.data, &cc, d_h.data, &gc, dx.data,
                                             d_htil0 ? d_htil0->data : nullptr, d_c0 ? d_c0->data : nullptr,
                                             x.steps, x.batch, p.input(), p.hidden(), static_cast<int>(mode),
                                             ctx.precision(), scr, ctx.capacity(), ctx.stream()));
}

// qrnn_forward (:449-494).
inline void qrnn_forward(const QrnnParams& p, const DeviceTensor3<float>& x, const DeviceTensor2<float>& c0,
                         ScanMode mode, LayerContext& ctx, const QrnnCache& cache, DeviceTensor3<float>& h) {
  detail::require_features(x.features, p.m, "qrnn_forward");
  if (p.k > x.steps) throw ContractViolation("qrnn_forward: filter window exceeds sequence length");
  const size_t need = linrec_qrnn_scratch_bytes(x.steps, x.batch, p.m, p.n, p.k);
  void* scr = ctx.scratch(need);  // grow first: capacity() below must see it
  throw_status(linrec_qrnn_forward_f32(p.W, p.bias, x.data, c0.data, h.data, cache.gates, cache.c, x.steps, x.batch,
                                       p.m, p.n, p.k, static_cast<int>(mode), ctx.precision(), scr, ctx.capacity(),
                                       ctx.stream()));
}

// qrnn_backward (:496-548).
inline void qrnn_backward(const QrnnParams& p, const DeviceTensor3<float>& x, const DeviceTensor2<float>& c0,
                          const QrnnCache& cache, const DeviceTensor3<float>& d_h, ScanMode mode, LayerContext& ctx,
                          QrnnGrads& grads, DeviceTensor3<float>& dx, DeviceTensor2<float>* d_c0 = nullptr) {
  const size_t need = linrec_qrnn_scratch_bytes(x.steps, x.batch, p.m, p.n, p.k);
  void* scr = ctx.scratch(need);  // grow first: capacity() below must see it
  throw_status(linrec_qrnn_backward_f32(p.W, x.data, c0.data, cache.gates, cache.c, d_h.data, grads.W, grads.bias,
                                        dx.data, d_c0 ? d_c0->data : nullptr, x.steps, x.batch, p.m, p.n, p.k,
                                        static_cast<int>(mode), ctx.precision(), scr, ctx.capacity(),
                                        ctx.stream()));
}

}  // namespace cuda
}  // namespace linrec
