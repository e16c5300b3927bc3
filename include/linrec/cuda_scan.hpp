// linrec/cuda_scan.hpp -- C++ host mirror of the reference's recurrence entry
// points (proj/include/linrec/recurrence.hpp:169-377) over the C ABI of
// include/linrec_cuda.h.  Header-only; link against liblinrec_cuda.so.
//
// The reference's functions take host Tensor3/Tensor2 (std::vector storage,
// tensor.hpp:20-91) and a ThreadPool.  Here the same names take views of
// caller-owned DEVICE buffers with the same [T][b][n] time-major layout and a
// CUDA stream; results are written into caller-provided outputs (the
// reference allocates them, recurrence.hpp:174, :327-329).  Errors throw
// linrec::cuda::ContractViolation (a std::runtime_error, like the
// reference's, common.hpp:15-22) or std::invalid_argument / ::TypeError
// equivalents for the other status codes.
#pragma once

#include <algorithm>
#include <cstdint>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "linrec_cuda.h"

namespace linrec {
namespace cuda {

using index_t = std::int64_t;

enum class ScanMode { Serial = LINREC_SERIAL, Parallel = LINREC_PARALLEL };

class ContractViolation : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DtypeError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// [T, b, n] device tensor view (tensor.hpp:49-75 layout, not owned).
template <class S>
struct DeviceTensor3 {
  S* data = nullptr;
  index_t steps = 0, batch = 0, features = 0;
  index_t step_size() const { return batch * features; }
  bool same_shape(const DeviceTensor3& o) const {
    return steps == o.steps && batch == o.batch && features == o.features;
  }
};

// [b, n] device tensor view; data == nullptr means "zeros" (linrec_py.cpp:98-100).
template <class S>
struct DeviceTensor2 {
  S* data = nullptr;
  index_t rows = 0, cols = 0;
};

inline void throw_status(int rc) {
  if (rc == LINREC_OK) return;
  const std::string msg = linrec_last_error();
  switch (rc) {
    case LINREC_ERR_SHAPE:
    case LINREC_ERR_NONFINITE:
      throw ContractViolation(msg);
    case LINREC_ERR_VALUE:
      throw std::invalid_argument(msg);
    case LINREC_ERR_DTYPE:
      throw DtypeError(msg);
    default:
      throw CudaError(msg);
  }
}

// check_same_shape (tensor.hpp:168-178) with the reference's message.
template <class S, class U>
void check_same_shape(const DeviceTensor3<S>& a, const DeviceTensor3<U>& b, const char* op) {
  if (a.steps != b.steps || a.batch != b.batch || a.features != b.features) {
    std::ostringstream os;
    os << op << ": shape mismatch, [" << a.steps << "," << a.batch << "," << a.features
       << "] vs [" << b.steps << "," << b.batch << "," << b.features << "]";
    throw ContractViolation(os.str());
  }
}

// validate_recurrence_shapes (recurrence.hpp:39-51).
template <class S, class U, class V>
void validate_recurrence_shapes(const DeviceTensor3<S>& decays, const DeviceTensor3<U>& impulses,
                                const DeviceTensor2<V>& initial) {
  check_same_shape(decays, impulses, "recurrence");
  if (initial.data != nullptr && (initial.rows != decays.batch || initial.cols != decays.features)) {
    std::ostringstream os;
    os << "recurrence: initial state [" << initial.rows << "," << initial.cols
       << "] does not match [" << decays.batch << "," << decays.features << "]";
    throw ContractViolation(os.str());
  }
}

namespace detail {
inline int scan_call(const float* l, const float* x, const float* h0, float* h, index_t T,
                     index_t W, int mode, linrec_workspace_t ws, void* st) {
  return linrec_scan_f32(l, x, h0, h, T, W, mode, ws, st);
}
inline int scan_call(const double* l, const double* x, const double* h0, double* h, index_t T,
                     index_t W, int mode, linrec_workspace_t ws, void* st) {
  return linrec_scan_f64(l, x, h0, h, T, W, mode, ws, st);
}
inline int bwd_call(const float* l, const float* h0, const float* h, const float* dh, float* dl,
                    float* dx, float* dh0, index_t T, index_t W, int mode, linrec_workspace_t ws,
                    void* st) {
  return linrec_scan_backward_f32(l, h0, h, dh, dl, dx, dh0, T, W, mode, ws, st);
}
inline int bwd_call(const double* l, const double* h0, const double* h, const double* dh,
                    double* dl, double* dx, double* dh0, index_t T, index_t W, int mode,
                    linrec_workspace_t ws, void* st) {
  return linrec_scan_backward_f64(l, h0, h, dh, dl, dx, dh0, T, W, mode, ws, st);
}
inline int plan_call(const float* l, const float* x, const float* h0, float* h, index_t T, index_t W,
                     const index_t* b, index_t p, float* P, float* R, float* C, void* st) {
  return linrec_scan_plan_f32(l, x, h0, h, T, W, b, p, P, R, C, st);
}
inline int plan_call(const double* l, const double* x, const double* h0, double* h, index_t T, index_t W,
                     const index_t* b, index_t p, double* P, double* R, double* C, void* st) {
  return linrec_scan_plan_f64(l, x, h0, h, T, W, b, p, P, R, C, st);
}
inline int plan_bwd_call(const float* l, const float* h0, const float* h, const float* dh, float* dl, float* dx,
                         float* dh0, index_t T, index_t W, const index_t* b, index_t p, void* st) {
  return linrec_scan_backward_plan_f32(l, h0, h, dh, dl, dx, dh0, T, W, b, p, st);
}
inline int plan_bwd_call(const double* l, const double* h0, const double* h, const double* dh, double* dl,
                         double* dx, double* dh0, index_t T, index_t W, const index_t* b, index_t p, void* st) {
  return linrec_scan_backward_plan_f64(l, h0, h, dh, dl, dx, dh0, T, W, b, p, st);
}
inline int screen_call(const float* v, index_t T, index_t b, index_t n, const char* name, void* st) {
  return linrec_screen_finite_f32(v, T, b, n, name, st);
}
inline int screen_call(const double* v, index_t T, index_t b, index_t n, const char* name, void* st) {
  return linrec_screen_finite_f64(v, T, b, n, name, st);
}
}  // namespace detail

// screen_finite (recurrence.hpp:133-155): ContractViolation naming the first
// non-finite element, "non-finite value in <name> at [t=.., b=.., n=..]".
template <class S>
void screen_finite(const DeviceTensor3<S>& t, const char* name, void* stream = nullptr) {
  throw_status(detail::screen_call(t.data, t.steps, t.batch, t.features, name, stream));
}
template <class S>
void screen_finite(const DeviceTensor2<S>& t, const char* name, void* stream = nullptr) {
  if (t.data == nullptr) return;  // "zeros": finite
  throw_status(detail::screen_call(t.data, 0, t.rows, t.cols, name, stream));
}
// screen_recurrence (recurrence.hpp:157-163).
template <class S>
void screen_recurrence(const DeviceTensor3<S>& decays, const DeviceTensor3<S>& impulses,
                       const DeviceTensor2<S>& initial, void* stream = nullptr) {
  screen_finite(decays, "decays", stream);
  screen_finite(impulses, "impulses", stream);
  screen_finite(initial, "initial", stream);
}

// scan_serial (recurrence.hpp:169-179): bit-exact serial recurrence.
template <class S>
void scan_serial(const DeviceTensor3<S>& decays, const DeviceTensor3<S>& impulses,
                 const DeviceTensor2<S>& initial, DeviceTensor3<S>& h, void* stream = nullptr,
                 bool check_finite = false) {
  validate_recurrence_shapes(decays, impulses, initial);
  check_same_shape(decays, h, "scan_serial(h)");
  if (check_finite) screen_recurrence(decays, impulses, initial, stream);
  throw_status(detail::scan_call(decays.data, impulses.data, initial.data, h.data, decays.steps,
                                 decays.step_size(), LINREC_SERIAL, nullptr, stream));
}

// scan_parallel (recurrence.hpp:193-245): single-pass chained scan.
template <class S>
void scan_parallel(const DeviceTensor3<S>& decays, const DeviceTensor3<S>& impulses,
                   const DeviceTensor2<S>& initial, DeviceTensor3<S>& h, void* stream = nullptr,
                   linrec_workspace_t ws = nullptr, bool check_finite = false) {
  validate_recurrence_shapes(decays, impulses, initial);
  check_same_shape(decays, h, "scan_parallel(h)");
  if (check_finite) screen_recurrence(decays, impulses, initial, stream);
  throw_status(detail::scan_call(decays.data, impulses.data, initial.data, h.data, decays.steps,
                                 decays.step_size(), LINREC_PARALLEL, ws, stream));
}

// ChunkPlan / plan_chunks (recurrence.hpp:53-80): contiguous 1-indexed
// inclusive chunks of steps 1..T, remainder to the front.
struct ChunkPlan {
  std::vector<std::pair<index_t, index_t>> bounds;
  int workers = 0;
  index_t chunks() const { return index_t(bounds.size()); }
};
inline ChunkPlan plan_chunks(index_t T, int requested_workers) {
  if (T < 1) throw ContractViolation("plan_chunks: T must be >= 1");
  if (requested_workers < 1) throw ContractViolation("plan_chunks: requested_workers must be >= 1");
  const index_t p = std::min<index_t>(requested_workers, T);
  ChunkPlan plan;
  plan.workers = int(p);
  const index_t base = T / p, rem = T % p;
  index_t start = 1;
  for (index_t i = 0; i < p; ++i) {
    const index_t len = base + (i < rem ? 1 : 0);
    plan.bounds.emplace_back(start, start + len - 1);
    start += len;
  }
  return plan;
}

// validate_plan (recurrence.hpp:84-94), the reference's messages (the C ABI
// checks the same again).
inline void validate_plan(const ChunkPlan& plan, index_t T) {
  if (plan.bounds.empty()) throw ContractViolation("ChunkPlan: no chunks");
  if (plan.bounds.front().first != 1) throw ContractViolation("ChunkPlan: first chunk must start at step 1");
  if (plan.bounds.back().second != T) throw ContractViolation("ChunkPlan: last chunk must end at step T");
  for (size_t i = 0; i < plan.bounds.size(); ++i) {
    if (plan.bounds[i].first > plan.bounds[i].second) throw ContractViolation("ChunkPlan: chunk start exceeds end");
    if (i + 1 < plan.bounds.size() && plan.bounds[i].second + 1 != plan.bounds[i + 1].first)
      throw ContractViolation("ChunkPlan: chunks must be contiguous");
  }
}

// ScanSummaries (recurrence.hpp:186-191): caller-owned [chunks, b, n] device
// views of the chunk summaries P, R and stitched chunk-end states C.
template <class S>
struct ScanSummaries {
  DeviceTensor3<S> P, R, C;
};

namespace detail {
inline std::vector<index_t> flat_bounds(const ChunkPlan& plan) {
  std::vector<index_t> b;
  for (const auto& se : plan.bounds) {
    b.push_back(se.first);
    b.push_back(se.second);
  }
  return b;
}
}  // namespace detail

// scan_parallel with an explicit plan (recurrence.hpp:193-245): the
// reference's three phases on the device, bit-identical to its result (and
// summaries) for the same plan; validate_plan's errors.
template <class S>
void scan_parallel(const DeviceTensor3<S>& decays, const DeviceTensor3<S>& impulses,
                   const DeviceTensor2<S>& initial, const ChunkPlan& plan, DeviceTensor3<S>& h,
                   ScanSummaries<S>* summaries = nullptr, void* stream = nullptr, bool check_finite = false) {
  validate_recurrence_shapes(decays, impulses, initial);
  check_same_shape(decays, h, "scan_parallel(h)");
  if (check_finite) {  // after validate_plan, as the reference (recurrence.hpp:198-200)
    validate_plan(plan, decays.steps);
    screen_recurrence(decays, impulses, initial, stream);
  }
  const auto b = detail::flat_bounds(plan);
  throw_status(detail::plan_call(decays.data, impulses.data, initial.data, h.data, decays.steps, decays.step_size(),
                                 b.data(), plan.chunks(), summaries ? summaries->P.data : nullptr,
                                 summaries ? summaries->R.data : nullptr, summaries ? summaries->C.data : nullptr,
                                 stream));
}

// scan (recurrence.hpp:255-263): mode dispatch.
template <class S>
void scan(const DeviceTensor3<S>& decays, const DeviceTensor3<S>& impulses,
          const DeviceTensor2<S>& initial, DeviceTensor3<S>& h, ScanMode mode,
          void* stream = nullptr, linrec_workspace_t ws = nullptr, bool check_finite = false) {
  if (mode == ScanMode::Serial) return scan_serial(decays, impulses, initial, h, stream, check_finite);
  scan_parallel(decays, impulses, initial, h, stream, ws, check_finite);
}

// RecurrenceGradients (recurrence.hpp:265-271) as output views.
template <class S>
struct RecurrenceGradients {
  DeviceTensor3<S> d_decays;
  DeviceTensor3<S> d_impulses;
  DeviceTensor2<S> d_initial;
};

// scan_backward (recurrence.hpp:283-363).
template <class S>
void scan_backward(const DeviceTensor3<S>& decays, const DeviceTensor2<S>& initial,
                   const DeviceTensor3<S>& h, const DeviceTensor3<S>& d_h,
                   RecurrenceGradients<S>& grads, ScanMode mode, void* stream = nullptr,
                   linrec_workspace_t ws = nullptr, bool check_finite = false) {
  check_same_shape(decays, h, "scan_backward(h)");
  check_same_shape(decays, d_h, "scan_backward(d_h)");
  validate_recurrence_shapes(decays, d_h, initial);
  if (check_finite) {  // recurrence.hpp:292-296
    screen_finite(decays, "decays", stream);
    screen_finite(d_h, "d_h", stream);
  }
  check_same_shape(decays, grads.d_decays, "scan_backward(d_decays)");
  check_same_shape(decays, grads.d_impulses, "scan_backward(d_impulses)");
  throw_status(detail::bwd_call(decays.data, initial.data, h.data, d_h.data, grads.d_decays.data,
                                grads.d_impulses.data, grads.d_initial.data, decays.steps,
                                decays.step_size(), static_cast<int>(mode), ws, stream));
}

// scan_backward with the reversed scan chunked by an explicit plan
// (recurrence.hpp:365-377; ScanMode::Parallel), bit-identical to the
// reference's for the same plan.
template <class S>
void scan_backward(const DeviceTensor3<S>& decays, const DeviceTensor2<S>& initial, const DeviceTensor3<S>& h,
                   const DeviceTensor3<S>& d_h, const ChunkPlan& plan, RecurrenceGradients<S>& grads,
                   void* stream = nullptr, bool check_finite = false) {
  validate_plan(plan, decays.steps);  // recurrence.hpp:373
  check_same_shape(decays, h, "scan_backward(h)");
  check_same_shape(decays, d_h, "scan_backward(d_h)");
  validate_recurrence_shapes(decays, d_h, initial);
  if (check_finite) {
    screen_finite(decays, "decays", stream);
    screen_finite(d_h, "d_h", stream);
  }
  check_same_shape(decays, grads.d_decays, "scan_backward(d_decays)");
  check_same_shape(decays, grads.d_impulses, "scan_backward(d_impulses)");
  const auto b = detail::flat_bounds(plan);
  throw_status(detail::plan_bwd_call(decays.data, initial.data, h.data, d_h.data, grads.d_decays.data,
                                     grads.d_impulses.data, grads.d_initial.data, decays.steps, decays.step_size(),
                                     b.data(), plan.chunks(), stream));
}

}  // namespace cuda
}  // namespace linrec
