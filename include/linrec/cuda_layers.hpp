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
// as cuda_scan.hpp (ContractViolation for shape errors).  Templated on the
// scalar type like the reference (float: the tcgen05 path, `precision` from
// the context; double: the linrec_*_f64 entry points).
#pragma once

#include <cstddef>
#include <string>
#include <type_traits>

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

// GilrParams<S> / GilrGrads<S> (layers.hpp:30-76) as device views, S = float
// or double (the reference templates its layers on S; test_layers.cpp runs
// double).  The unsuffixed names are the float instantiations.
template <class S>
struct GilrParamsT {
  const S* U = nullptr;  // [n][m]
  const S* V = nullptr;  // [n][m]
  const S* b_g = nullptr;
  const S* b_z = nullptr;
  Activation act = Activation::Tanh;
  index_t m = 0, n = 0;
  index_t input() const { return m; }
  index_t hidden() const { return n; }
  auto c() const {
    if constexpr (std::is_same<S, double>::value)
      return linrec_gilr_params_f64{U, V, b_g, b_z, static_cast<int>(act)};
    else
      return linrec_gilr_params_f32{U, V, b_g, b_z, static_cast<int>(act)};
  }
};
template <class S>
struct GilrGradsT {
  S *U = nullptr, *V = nullptr, *b_g = nullptr, *b_z = nullptr;
  auto c() const {
    if constexpr (std::is_same<S, double>::value)
      return linrec_gilr_grads_f64{U, V, b_g, b_z};
    else
      return linrec_gilr_grads_f32{U, V, b_g, b_z};
  }
};
template <class S>
struct GilrCacheT {
  DeviceTensor3<S> g, i, h;  // activated gate, candidate, output (layers.hpp:62-64)
};

// GilrLstmParams<S> (:146-160), GilrLstmGrads (:192-211), GilrLstmCache
// (:183-188; htil holds T+1 rows, row 0 = htil0; gates = 4 planes).
template <class S>
struct GilrLstmParamsT {
  GilrParamsT<S> surrogate;
  const S* U = nullptr;     // [4n][n]
  const S* V = nullptr;     // [4n][m]
  const S* bias = nullptr;  // [4n]
  index_t input() const { return surrogate.m; }
  index_t hidden() const { return surrogate.n; }
  auto c() const {
    if constexpr (std::is_same<S, double>::value)
      return linrec_gilr_lstm_params_f64{surrogate.c(), U, V, bias};
    else
      return linrec_gilr_lstm_params_f32{surrogate.c(), U, V, bias};
  }
};
template <class S>
struct GilrLstmGradsT {
  GilrGradsT<S> surrogate;
  S *U = nullptr, *V = nullptr, *bias = nullptr;
  auto c() const {
    if constexpr (std::is_same<S, double>::value)
      return linrec_gilr_lstm_grads_f64{surrogate.c(), U, V, bias};
    else
      return linrec_gilr_lstm_grads_f32{surrogate.c(), U, V, bias};
  }
};
template <class S>
struct GilrLstmCacheT {
  S *sg = nullptr, *si = nullptr, *htil = nullptr, *gates = nullptr, *c = nullptr;
  auto view() const {
    if constexpr (std::is_same<S, double>::value)
      return linrec_gilr_lstm_cache_f64{sg, si, htil, gates, c};
    else
      return linrec_gilr_lstm_cache_f32{sg, si, htil, gates, c};
  }
};

// QrnnParams<S> (:390-405): k taps packed [k][3n][m]; grads alike.
template <class S>
struct QrnnParamsT {
  const S* W = nullptr;
  const S* bias = nullptr;  // [3n]
  index_t m = 0, n = 0, k = 1;
};
template <class S>
struct QrnnGradsT {
  S *W = nullptr, *bias = nullptr;
};
template <class S>
struct QrnnCacheT {
  S *gates = nullptr, *c = nullptr;  // [3][T][b][n], [T][b][n]
};

using GilrParams = GilrParamsT<float>;
using GilrGrads = GilrGradsT<float>;
using GilrCache = GilrCacheT<float>;
using GilrLstmParams = GilrLstmParamsT<float>;
using GilrLstmGrads = GilrLstmGradsT<float>;
using GilrLstmCache = GilrLstmCacheT<float>;
using QrnnParams = QrnnParamsT<float>;
using QrnnGrads = QrnnGradsT<float>;
using QrnnCache = QrnnCacheT<float>;

namespace detail {
inline void require_features(index_t have, index_t want, const char* what) {
  if (have != want) throw ContractViolation(std::string(what) + ": input feature mismatch");
}
template <class S>
constexpr bool is_f64() {
  static_assert(std::is_same<S, float>::value || std::is_same<S, double>::value, "layers run float or double");
  return std::is_same<S, double>::value;
}
}  // namespace detail

// gilr_forward (layers.hpp:78-100): h = GILR(x); cache g, i (and h).
template <class S>
inline void gilr_forward(const GilrParamsT<S>& p, const DeviceTensor3<S>& x, const DeviceTensor2<S>& h0,
                         ScanMode mode, LayerContext& ctx, GilrCacheT<S>& cache, DeviceTensor3<S>& h) {
  detail::require_features(x.features, p.input(), "gilr_forward");
  const auto pc = p.c();
  if constexpr (detail::is_f64<S>()) {
    void* scr = ctx.scratch(linrec_gilr_scratch_bytes_f64(x.steps, x.batch, p.m, p.n));
    throw_status(linrec_gilr_forward_f64(&pc, x.data, h0.data, h.data, cache.g.data, cache.i.data, x.steps, x.batch,
                                         p.m, p.n, static_cast<int>(mode), scr, ctx.capacity(), ctx.stream()));
  } else {
    void* scr = ctx.scratch(linrec_gilr_scratch_bytes(x.steps, x.batch, p.m, p.n));  // grow before capacity()
    throw_status(linrec_gilr_forward_f32(&pc, x.data, h0.data, h.data, cache.g.data, cache.i.data, x.steps, x.batch,
                                         p.m, p.n, static_cast<int>(mode), ctx.precision(), scr, ctx.capacity(),
                                         ctx.stream()));
  }
  cache.h = h;
}

// gilr_backward (:102-133): accumulates into grads, writes dx (and dh0).
template <class S>
inline void gilr_backward(const GilrParamsT<S>& p, const DeviceTensor3<S>& x, const DeviceTensor2<S>& h0,
                          const GilrCacheT<S>& cache, const DeviceTensor3<S>& d_h, ScanMode mode, LayerContext& ctx,
                          GilrGradsT<S>& grads, DeviceTensor3<S>& dx, DeviceTensor2<S>* d_h0 = nullptr) {
  const auto pc = p.c();
  auto gc = grads.c();
  if constexpr (detail::is_f64<S>()) {
    void* scr = ctx.scratch(linrec_gilr_scratch_bytes_f64(x.steps, x.batch, p.m, p.n));
    throw_status(linrec_gilr_backward_f64(&pc, x.data, h0.data, cache.g.data, cache.i.data, cache.h.data, d_h.data,
                                          &gc, dx.data, d_h0 ? d_h0->data : nullptr, x.steps, x.batch, p.m, p.n,
                                          static_cast<int>(mode), scr, ctx.capacity(), ctx.stream()));
  } else {
    void* scr = ctx.scratch(linrec_gilr_scratch_bytes(x.steps, x.batch, p.m, p.n));
    throw_status(linrec_gilr_backward_f32(&pc, x.data, h0.data, cache.g.data, cache.i.data, cache.h.data, d_h.data,
                                          &gc, dx.data, d_h0 ? d_h0->data : nullptr, x.steps, x.batch, p.m, p.n,
                                          static_cast<int>(mode), ctx.precision(), scr, ctx.capacity(),
                                          ctx.stream()));
  }
}

// gilr_lstm_forward (:245-293).
template <class S>
inline void gilr_lstm_forward(const GilrLstmParamsT<S>& p, const DeviceTensor3<S>& x, const DeviceTensor2<S>& htil0,
                              const DeviceTensor2<S>& c0, ScanMode mode, LayerContext& ctx,
                              const GilrLstmCacheT<S>& cache, DeviceTensor3<S>& h) {
  detail::require_features(x.features, p.input(), "gilr_lstm_forward");
  const auto pc = p.c();
  const auto cc = cache.view();
  if constexpr (detail::is_f64<S>()) {
    void* scr = ctx.scratch(linrec_gilr_lstm_scratch_bytes_f64(x.steps, x.batch, p.input(), p.hidden()));
    throw_status(linrec_gilr_lstm_forward_f64(&pc, x.data, htil0.data, c0.data, h.data, &cc, x.steps, x.batch,
                                              p.input(), p.hidden(), static_cast<int>(mode), scr, ctx.capacity(),
                                              ctx.stream()));
  } else {
    void* scr = ctx.scratch(linrec_gilr_lstm_scratch_bytes(x.steps, x.batch, p.input(), p.hidden()));
    throw_status(linrec_gilr_lstm_forward_f32(&pc, x.data, htil0.data, c0.data, h.data, &cc, x.steps, x.batch,
                                              p.input(), p.hidden(), static_cast<int>(mode), ctx.precision(), scr,
                                              ctx.capacity(), ctx.stream()));
  }
}

// gilr_lstm_backward (:295-375).
template <class S>
inline void gilr_lstm_backward(const GilrLstmParamsT<S>& p, const DeviceTensor3<S>& x, const DeviceTensor2<S>& htil0,
                               const DeviceTensor2<S>& c0, const GilrLstmCacheT<S>& cache,
                               const DeviceTensor3<S>& d_h, ScanMode mode, LayerContext& ctx,
                               GilrLstmGradsT<S>& grads, DeviceTensor3<S>& dx, DeviceTensor2<S>* d_htil0 = nullptr,
                               DeviceTensor2<S>* d_c0 = nullptr) {
  const auto pc = p.c();
  const auto cc = cache.view();
  auto gc = grads.c();
  S* dht0 = d_htil0 ? d_htil0->data : nullptr;
  S* dc0 = d_c0 ? d_c0->data : nullptr;
  if constexpr (detail::is_f64<S>()) {
    void* scr = ctx.scratch(linrec_gilr_lstm_scratch_bytes_f64(x.steps, x.batch, p.input(), p.hidden()));
    throw_status(linrec_gilr_lstm_backward_f64(&pc, x.data, htil0.data, c0.data, &cc, d_h.data, &gc, dx.data, dht0,
                                               dc0, x.steps, x.batch, p.input(), p.hidden(), static_cast<int>(mode),
                                               scr, ctx.capacity(), ctx.stream()));
  } else {
    void* scr = ctx.scratch(linrec_gilr_lstm_scratch_bytes(x.steps, x.batch, p.input(), p.hidden()));
    throw_status(linrec_gilr_lstm_backward_f32(&pc, x.data, htil0.data, c0.data, &cc, d_h.data, &gc, dx.data, dht0,
                                               dc0, x.steps, x.batch, p.input(), p.hidden(), static_cast<int>(mode),
                                               ctx.precision(), scr, ctx.capacity(), ctx.stream()));
  }
}

// qrnn_forward (:449-494).
template <class S>
inline void qrnn_forward(const QrnnParamsT<S>& p, const DeviceTensor3<S>& x, const DeviceTensor2<S>& c0,
                         ScanMode mode, LayerContext& ctx, const QrnnCacheT<S>& cache, DeviceTensor3<S>& h) {
  detail::require_features(x.features, p.m, "qrnn_forward");
  if (p.k > x.steps) throw ContractViolation("qrnn_forward: filter window exceeds sequence length");
  if constexpr (detail::is_f64<S>()) {
    void* scr = ctx.scratch(linrec_qrnn_scratch_bytes_f64(x.steps, x.batch, p.m, p.n, p.k));
    throw_status(linrec_qrnn_forward_f64(p.W, p.bias, x.data, c0.data, h.data, cache.gates, cache.c, x.steps,
                                         x.batch, p.m, p.n, p.k, static_cast<int>(mode), scr, ctx.capacity(),
                                         ctx.stream()));
  } else {
    void* scr = ctx.scratch(linrec_qrnn_scratch_bytes(x.steps, x.batch, p.m, p.n, p.k));
    throw_status(linrec_qrnn_forward_f32(p.W, p.bias, x.data, c0.data, h.data, cache.gates, cache.c, x.steps,
                                         x.batch, p.m, p.n, p.k, static_cast<int>(mode), ctx.precision(), scr,
                                         ctx.capacity(), ctx.stream()));
  }
}

// qrnn_backward (:496-548).
template <class S>
inline void qrnn_backward(const QrnnParamsT<S>& p, const DeviceTensor3<S>& x, const DeviceTensor2<S>& c0,
                          const QrnnCacheT<S>& cache, const DeviceTensor3<S>& d_h, ScanMode mode, LayerContext& ctx,
                          QrnnGradsT<S>& grads, DeviceTensor3<S>& dx, DeviceTensor2<S>* d_c0 = nullptr) {
  S* dc0 = d_c0 ? d_c0->data : nullptr;
  if constexpr (detail::is_f64<S>()) {
    void* scr = ctx.scratch(linrec_qrnn_scratch_bytes_f64(x.steps, x.batch, p.m, p.n, p.k));
    throw_status(linrec_qrnn_backward_f64(p.W, x.data, c0.data, cache.gates, cache.c, d_h.data, grads.W, grads.bias,
                                          dx.data, dc0, x.steps, x.batch, p.m, p.n, p.k, static_cast<int>(mode), scr,
                                          ctx.capacity(), ctx.stream()));
  } else {
    void* scr = ctx.scratch(linrec_qrnn_scratch_bytes(x.steps, x.batch, p.m, p.n, p.k));
    throw_status(linrec_qrnn_backward_f32(p.W, x.data, c0.data, cache.gates, cache.c, d_h.data, grads.W, grads.bias,
                                          dx.data, dc0, x.steps, x.batch, p.m, p.n, p.k, static_cast<int>(mode),
                                          ctx.precision(), scr, ctx.capacity(), ctx.stream()));
  }
}

}  // namespace cuda
}  // namespace linrec
