// Python module `linrec` -- drop-in for the reference's pybind11 module
// (proj/bindings/linrec_py.cpp:144-186): same function names, signatures,
// argument checks, exception types and messages, with the compute moved to
// the sm_100a kernels behind the C ABI (include/linrec_cuda.h).
//
//   scan(decays, impulses, initial=None, *, workers=0, mode="parallel")
//   scan_backward(decays, initial, h, d_h, *, workers=0, mode="parallel")
//   plan_chunks(T, workers), predicted_speedup(workers, T), hardware_workers()
//
// numpy in -> numpy out through the pipelined host path (linrec_scan_host_*).
// Objects exposing __cuda_array_interface__ (torch/cupy CUDA tensors) are
// consumed zero-copy and the results come back as linrec.DeviceArray, which
// itself exposes __cuda_array_interface__ (torch.as_tensor(..., device="cuda")
// wraps it without a copy).
//
// Mapping of the reference's (mode, workers) onto the GPU: mode="serial" and
// workers == 1 (a one-chunk plan, which the reference evaluates bit-identically
// to the serial scan, recurrence.hpp:98-100) run the per-channel serial kernel;
// any other worker count runs the single-pass chained scan.  `workers` keeps
// its validation (ValueError when < 0) and 0 still means hardware_workers().
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "linrec/cuda_scan.hpp"
#include "linrec_cuda.h"

namespace py = pybind11;
using index_t = std::int64_t;

namespace {

[[noreturn]] void raise_status(int rc) {
  const std::string msg = linrec_last_error();
  switch (rc) {
    case LINREC_ERR_DTYPE:
      throw py::type_error(msg);
    case LINREC_ERR_VALUE:
      throw std::invalid_argument(msg);
    default:
      throw std::runtime_error(msg);
  }
}

inline void check(int rc) {
  if (rc != LINREC_OK) raise_status(rc);
}

// ---- reference-compatible argument handling ---------------------------------
template <class S>
using c_array = py::array_t<S, py::array::c_style | py::array::forcecast>;

// require_dtype (linrec_py.cpp:24-29)
template <class S>
void require_dtype(const py::array& a, const char* name) {
  if (a.dtype().num() != py::dtype::of<S>().num())
    throw py::type_error(std::string(name) + ": all arrays must share the decays dtype");
}

struct Dims3 {
  index_t T = 0, b = 0, n = 0;
};

// tensor3_from (linrec_py.cpp:31-42): dtype, rank, then Tensor3's dims >= 1
// contract (tensor.hpp:58, ContractViolation -> RuntimeError).
template <class S>
c_array<S> host3(const py::array& a, const char* name, Dims3* d) {
  require_dtype<S>(a, name);
  c_array<S> c(a);
  if (c.ndim() != 3)
    throw std::invalid_argument(std::string(name) + " must have shape [T, batch, features]");
  d->T = c.shape(0);
  d->b = c.shape(1);
  d->n = c.shape(2);
  if (d->T < 1 || d->b < 1 || d->n < 1) throw std::runtime_error("Tensor3 dimensions must be >= 1");
  return c;
}

template <class S>
c_array<S> host2(const py::array& a, const char* name, index_t* r, index_t* cdim) {
  require_dtype<S>(a, name);
  c_array<S> c(a);
  if (c.ndim() != 2)
    throw std::invalid_argument(std::string(name) + " must have shape [batch, features]");
  *r = c.shape(0);
  *cdim = c.shape(1);
  if (*r < 1 || *cdim < 1) throw std::runtime_error("Tensor2 dimensions must be >= 1");
  return c;
}

void check_same3(const Dims3& a, const Dims3& b, const char* op) {
  if (a.T != b.T || a.b != b.b || a.n != b.n) {
    std::ostringstream os;
    os << op << ": shape mismatch, [" << a.T << "," << a.b << "," << a.n << "] vs [" << b.T << ","
       << b.b << "," << b.n << "]";
    throw std::runtime_error(os.str());
  }
}

void check_initial(const Dims3& d, index_t r, index_t c) {
  if (r != d.b || c != d.n) {
    std::ostringstream os;
    os << "recurrence: initial state [" << r << "," << c << "] does not match [" << d.b << ","
       << d.n << "]";
    throw std::runtime_error(os.str());
  }
}

int mode_from(const std::string& mode) {  // linrec_py.cpp:71-75
  if (mode == "parallel") return LINREC_PARALLEL;
  if (mode == "serial") return LINREC_SERIAL;
  throw std::invalid_argument("mode must be \"parallel\" or \"serial\"");
}

int hardware_workers() {  // ThreadPool::hardware_workers (thread_pool.hpp:29-32)
  const unsigned n = std::thread::hardware_concurrency();
  return n == 0 ? 1 : int(n);
}

int resolve_workers(int workers) {  // linrec_py.cpp:77-80
  if (workers < 0) throw std::invalid_argument("workers must be >= 0");
  return workers == 0 ? hardware_workers() : workers;
}

// GPU kernel choice for the reference's (mode, workers).
int gpu_mode(int mode, int workers) { return (mode == LINREC_SERIAL || workers == 1) ? LINREC_SERIAL : LINREC_PARALLEL; }

int resolve_device(const py::object& device) {
  if (linrec_device_count() < 1)
    throw std::runtime_error("linrec: no CUDA device available (this build has no CPU path)");
  if (device.is_none()) return 0;
  return device.cast<int>();
}

// ---- CUDA array interface -----------------------------------------------------
struct CudaView {
  std::uintptr_t ptr = 0;
  std::vector<index_t> shape;
  std::string typestr;
};

bool is_cuda_array(const py::handle& o) { return !o.is_none() && py::hasattr(o, "__cuda_array_interface__"); }

CudaView cuda_view(const py::handle& o, const char* name) {
  py::dict d = o.attr("__cuda_array_interface__");
  CudaView v;
  v.typestr = d["typestr"].cast<std::string>();
  for (auto s : d["shape"]) v.shape.push_back(s.cast<index_t>());
  py::tuple data = d["data"];
  v.ptr = data[0].cast<std::uintptr_t>();
  if (d.contains("strides") && !d["strides"].is_none()) {
    // accept only C-contiguous strides
    std::vector<index_t> st;
    for (auto s : d["strides"]) st.push_back(s.cast<index_t>());
    index_t expect = v.typestr == "<f8" ? 8 : 4;
    for (int i = int(v.shape.size()) - 1; i >= 0; --i) {
      if (v.shape[i] > 1 && st[i] != expect)
        throw std::invalid_argument(std::string(name) + " must be C-contiguous on the device");
      expect *= v.shape[i];
    }
  }
  return v;
}

// Owning device buffer returned for CUDA inputs.
class DeviceArray {
 public:
  DeviceArray(std::vector<index_t> shape, std::string typestr, int device)
      : shape_(std::move(shape)), typestr_(std::move(typestr)), device_(device) {
    size_t n = 1;
    for (auto s : shape_) n *= size_t(s);
    bytes_ = n * (typestr_ == "<f8" ? 8 : 4);
    check(linrec_device_malloc(&ptr_, bytes_, device_, nullptr));
  }
  ~DeviceArray() {
    if (ptr_) linrec_device_free(ptr_, device_, nullptr);
  }
  DeviceArray(const DeviceArray&) = delete;
  DeviceArray& operator=(const DeviceArray&) = delete;

  void* ptr() const { return ptr_; }
  py::dict interface() const {
    py::dict d;
    py::list sh;
    for (auto s : shape_) sh.append(s);
    d["shape"] = py::tuple(sh);
    d["typestr"] = typestr_;
    d["data"] = py::make_tuple(reinterpret_cast<std::uintptr_t>(ptr_), false);
    d["version"] = 2;
    d["strides"] = py::none();
    return d;
  }
  std::vector<index_t> shape() const { return shape_; }
  int device() const { return device_; }

 private:
  void* ptr_ = nullptr;
  size_t bytes_ = 0;
  std::vector<index_t> shape_;
  std::string typestr_;
  int device_ = 0;
};

// ---- host (numpy) path --------------------------------------------------------
// Result arrays: freshly allocated numpy arrays as in the reference
// (linrec_py.cpp:56-69), backed by page-locked memory from the library's
// caching allocator when large, so the device->host copies land in them
// directly.  Falls back to ordinary numpy memory if pinning fails.
template <class S>
py::array_t<S> result_array(const std::vector<py::ssize_t>& shape) {
  size_t n = 1;
  for (auto d : shape) n *= size_t(d);
  const size_t bytes = n * sizeof(S);
  void* p = nullptr;
  if (bytes >= (size_t(4) << 20) && linrec_host_alloc(&p, bytes) == LINREC_OK) {
    py::capsule owner(p, [](void* q) { linrec_host_free(q); });
    return py::array_t<S>(shape, static_cast<S*>(p), owner);
  }
  return py::array_t<S>(shape);
}

template <class S>
int host_scan(const S* l, const S* x, const S* h0, S* h, index_t T, index_t W, int mode, int dev) {
  if constexpr (sizeof(S) == 4) return linrec_scan_host_f32(l, x, h0, h, T, W, mode, dev);
  else return linrec_scan_host_f64(l, x, h0, h, T, W, mode, dev);
}
template <class S>
int host_bwd(const S* l, const S* h0, const S* h, const S* dh, S* dl, S* dx, S* dh0, index_t T,
             index_t W, int mode, int dev) {
  if constexpr (sizeof(S) == 4) return linrec_scan_backward_host_f32(l, h0, h, dh, dl, dx, dh0, T, W, mode, dev);
  else return linrec_scan_backward_host_f64(l, h0, h, dh, dl, dx, dh0, T, W, mode, dev);
}

template <class S>
py::object scan_numpy(const py::array& decays, const py::array& impulses, const py::object& initial,
                      int workers, const std::string& mode, const py::object& device) {
  Dims3 dl, dx;
  auto lam = host3<S>(decays, "decays", &dl);
  auto x = host3<S>(impulses, "impulses", &dx);
  c_array<S> h0;
  index_t r = 0, c = 0;
  if (!initial.is_none()) h0 = host2<S>(initial.cast<py::array>(), "initial", &r, &c);
  const int m = mode_from(mode);
  const int w = resolve_workers(workers);
  check_same3(dl, dx, "recurrence");  // validate_recurrence_shapes, recurrence.hpp:43
  if (!initial.is_none()) check_initial(dl, r, c);
  const int dev = resolve_device(device);
  py::array_t<S> out = result_array<S>({py::ssize_t(dl.T), py::ssize_t(dl.b), py::ssize_t(dl.n)});
  S* hp = out.mutable_data();
  const S* h0p = initial.is_none() ? nullptr : h0.data();
  int rc;
  {
    py::gil_scoped_release nogil;
    rc = host_scan<S>(lam.data(), x.data(), h0p, hp, dl.T, dl.b * dl.n, gpu_mode(m, w), dev);
  }
  check(rc);
  return std::move(out);
}

template <class S>
py::object scan_backward_numpy(const py::array& decays, const py::object& initial,
                               const py::array& h, const py::array& d_h, int workers,
                               const std::string& mode, const py::object& device) {
  Dims3 dl, dh_, dd;
  auto lam = host3<S>(decays, "decays", &dl);
  auto hh = host3<S>(h, "h", &dh_);
  auto dh = host3<S>(d_h, "d_h", &dd);
  c_array<S> h0;
  index_t r = 0, c = 0;
  if (!initial.is_none()) h0 = host2<S>(initial.cast<py::array>(), "initial", &r, &c);
  const int m = mode_from(mode);
  const int w = resolve_workers(workers);
  check_same3(dl, dh_, "scan_backward(h)");  // recurrence.hpp:292-294
  check_same3(dl, dd, "scan_backward(d_h)");
  check_same3(dl, dd, "recurrence");
  if (!initial.is_none()) check_initial(dl, r, c);
  const int dev = resolve_device(device);
  const auto shape3 = std::vector<py::ssize_t>{py::ssize_t(dl.T), py::ssize_t(dl.b), py::ssize_t(dl.n)};
  py::array_t<S> g_lam = result_array<S>(shape3), g_x = result_array<S>(shape3);
  py::array_t<S> g_h0({py::ssize_t(dl.b), py::ssize_t(dl.n)});
  S* p_lam = g_lam.mutable_data();
  S* p_x = g_x.mutable_data();
  S* p_h0 = g_h0.mutable_data();
  const S* h0p = initial.is_none() ? nullptr : h0.data();
  int rc;
  {
    py::gil_scoped_release nogil;
    rc = host_bwd<S>(lam.data(), h0p, hh.data(), dh.data(), p_lam, p_x, p_h0, dl.T, dl.b * dl.n,
                     gpu_mode(m, w), dev);
  }
  check(rc);
  return py::make_tuple(g_lam, g_x, g_h0);
}

// ---- device (CUDA array interface) path ------------------------------------
std::string dtype_typestr(const CudaView& v, const char* name, const std::string& want) {
  if (!want.empty() && v.typestr != want)
    throw py::type_error(std::string(name) + ": all arrays must share the decays dtype");
  if (v.typestr != "<f4" && v.typestr != "<f8") throw py::type_error("decays must be float32 or float64");
  return v.typestr;
}

Dims3 dims3(const CudaView& v, const char* name) {
  if (v.shape.size() != 3)
    throw std::invalid_argument(std::string(name) + " must have shape [T, batch, features]");
  Dims3 d{v.shape[0], v.shape[1], v.shape[2]};
  if (d.T < 1 || d.b < 1 || d.n < 1) throw std::runtime_error("Tensor3 dimensions must be >= 1");
  return d;
}

py::object scan_cuda(const py::object& decays, const py::object& impulses, const py::object& initial,
                     int workers, const std::string& mode, const py::object& device,
                     std::uintptr_t stream) {
  CudaView vl = cuda_view(decays, "decays");
  const std::string ts = dtype_typestr(vl, "decays", "");
  if (!is_cuda_array(impulses)) throw py::type_error("impulses: all arrays must be CUDA arrays like decays");
  CudaView vx = cuda_view(impulses, "impulses");
  dtype_typestr(vx, "impulses", ts);
  const Dims3 dl = dims3(vl, "decays"), dx = dims3(vx, "impulses");
  const void* h0 = nullptr;
  if (!initial.is_none()) {
    CudaView v0 = cuda_view(initial, "initial");
    dtype_typestr(v0, "initial", ts);
    if (v0.shape.size() != 2) throw std::invalid_argument("initial must have shape [batch, features]");
    check_same3(dl, dx, "recurrence");
    check_initial(dl, v0.shape[0], v0.shape[1]);
    h0 = reinterpret_cast<const void*>(v0.ptr);
  }
  const int m = gpu_mode(mode_from(mode), resolve_workers(workers));
  check_same3(dl, dx, "recurrence");
  const int dev = resolve_device(device);
  auto out = std::make_shared<DeviceArray>(std::vector<index_t>{dl.T, dl.b, dl.n}, ts, dev);
  void* st = reinterpret_cast<void*>(stream);
  const index_t W = dl.b * dl.n;
  int rc;
  if (ts == "<f4")
    rc = linrec_scan_f32(reinterpret_cast<const float*>(vl.ptr), reinterpret_cast<const float*>(vx.ptr),
                         static_cast<const float*>(h0), static_cast<float*>(out->ptr()), dl.T, W, m,
                         nullptr, st);
  else
    rc = linrec_scan_f64(reinterpret_cast<const double*>(vl.ptr), reinterpret_cast<const double*>(vx.ptr),
                         static_cast<const double*>(h0), static_cast<double*>(out->ptr()), dl.T, W, m,
                         nullptr, st);
  check(rc);
  return py::cast(out);
}

py::object scan_backward_cuda(const py::object& decays, const py::object& initial, const py::object& h,
                              const py::object& d_h, int workers, const std::string& mode,
                              const py::object& device, std::uintptr_t stream) {
  CudaView vl = cuda_view(decays, "decays");
  const std::string ts = dtype_typestr(vl, "decays", "");
  if (!is_cuda_array(h) || !is_cuda_array(d_h))
    throw py::type_error("h, d_h: all arrays must be CUDA arrays like decays");
  CudaView vh = cuda_view(h, "h"), vd = cuda_view(d_h, "d_h");
  dtype_typestr(vh, "h", ts);
  dtype_typestr(vd, "d_h", ts);
  const Dims3 dl = dims3(vl, "decays"), dh_ = dims3(vh, "h"), dd = dims3(vd, "d_h");
  const void* h0 = nullptr;
  index_t r = dl.b, c = dl.n;
  if (!initial.is_none()) {
    CudaView v0 = cuda_view(initial, "initial");
    dtype_typestr(v0, "initial", ts);
    if (v0.shape.size() != 2) throw std::invalid_argument("initial must have shape [batch, features]");
    r = v0.shape[0];
    c = v0.shape[1];
    h0 = reinterpret_cast<const void*>(v0.ptr);
  }
  const int m = gpu_mode(mode_from(mode), resolve_workers(workers));
  check_same3(dl, dh_, "scan_backward(h)");
  check_same3(dl, dd, "scan_backward(d_h)");
  check_initial(dl, r, c);
  const int dev = resolve_device(device);
  auto g_lam = std::make_shared<DeviceArray>(std::vector<index_t>{dl.T, dl.b, dl.n}, ts, dev);
  auto g_x = std::make_shared<DeviceArray>(std::vector<index_t>{dl.T, dl.b, dl.n}, ts, dev);
  auto g_h0 = std::make_shared<DeviceArray>(std::vector<index_t>{dl.b, dl.n}, ts, dev);
  void* st = reinterpret_cast<void*>(stream);
  const index_t W = dl.b * dl.n;
  int rc;
  if (ts == "<f4")
    rc = linrec_scan_backward_f32(
        reinterpret_cast<const float*>(vl.ptr), static_cast<const float*>(h0),
        reinterpret_cast<const float*>(vh.ptr), reinterpret_cast<const float*>(vd.ptr),
        static_cast<float*>(g_lam->ptr()), static_cast<float*>(g_x->ptr()),
        static_cast<float*>(g_h0->ptr()), dl.T, W, m, nullptr, st);
  else
    rc = linrec_scan_backward_f64(
        reinterpret_cast<const double*>(vl.ptr), static_cast<const double*>(h0),
        reinterpret_cast<const double*>(vh.ptr), reinterpret_cast<const double*>(vd.ptr),
        static_cast<double*>(g_lam->ptr()), static_cast<double*>(g_x->ptr()),
        static_cast<double*>(g_h0->ptr()), dl.T, W, m, nullptr, st);
  check(rc);
  return py::make_tuple(g_lam, g_x, g_h0);
}

// dispatch (linrec_py.cpp:82-89)
py::object scan(const py::object& decays, const py::object& impulses, const py::object& initial,
                int workers, const std::string& mode, const py::object& device, std::uintptr_t stream) {
  if (is_cuda_array(decays)) return scan_cuda(decays, impulses, initial, workers, mode, device, stream);
  py::array a = py::array::ensure(decays);
  if (!a) throw py::type_error("decays must be float32 or float64");
  const int num = a.dtype().num();
  py::array b = py::array::ensure(impulses);
  if (!b) throw py::type_error("impulses: all arrays must share the decays dtype");
  if (num == py::dtype::of<float>().num()) return scan_numpy<float>(a, b, initial, workers, mode, device);
  if (num == py::dtype::of<double>().num()) return scan_numpy<double>(a, b, initial, workers, mode, device);
  throw py::type_error("decays must be float32 or float64");
}

py::object scan_backward(const py::object& decays, const py::object& initial, const py::object& h,
                         const py::object& d_h, int workers, const std::string& mode,
                         const py::object& device, std::uintptr_t stream) {
  if (is_cuda_array(decays))
    return scan_backward_cuda(decays, initial, h, d_h, workers, mode, device, stream);
  py::array a = py::array::ensure(decays);
  if (!a) throw py::type_error("decays must be float32 or float64");
  py::array hh = py::array::ensure(h), dd = py::array::ensure(d_h);
  if (!hh || !dd) throw py::type_error("h, d_h: all arrays must share the decays dtype");
  const int num = a.dtype().num();
  if (num == py::dtype::of<float>().num())
    return scan_backward_numpy<float>(a, initial, hh, dd, workers, mode, device);
  if (num == py::dtype::of<double>().num())
    return scan_backward_numpy<double>(a, initial, hh, dd, workers, mode, device);
  throw py::type_error("decays must be float32 or float64");
}

// plan_chunks (recurrence.hpp:61-80): the reference's CPU chunk plan, kept for
// API compatibility (the GPU path tiles by its own plan).
std::vector<std::pair<index_t, index_t>> plan_chunks(index_t T, int workers) {
  if (T < 1) throw std::runtime_error("plan_chunks: T must be >= 1");
  if (workers < 1) throw std::runtime_error("plan_chunks: requested_workers must be >= 1");
  const index_t p = std::min<index_t>(workers, T);
  const index_t base = T / p, rem = T % p;
  std::vector<std::pair<index_t, index_t>> out;
  out.reserve(size_t(p));
  index_t start = 1;
  for (index_t i = 0; i < p; ++i) {
    const index_t len = base + (i < rem ? 1 : 0);
    out.emplace_back(start, start + len - 1);
    start += len;
  }
  return out;
}

// predicted_speedup (bench.hpp:61-65)
double predicted_speedup(int p, index_t T) {
  if (p < 1 || T < 1) throw std::runtime_error("predicted_speedup: p and T must be >= 1");
  return double(p) * double(T) / (3.0 * (double(T) + std::log2(double(p))));
}

}  // namespace

PYBIND11_MODULE(linrec, m) {
  m.doc() =
      "B200 (sm_100a) evaluation and differentiation of first-order linear "
      "recurrences h[t] = decays[t] * h[t-1] + impulses[t] over the sequence "
      "dimension; drop-in for the reference `linrec` module.  Arrays are "
      "[T, batch, features], C order, float32 or float64 (numpy, or CUDA "
      "arrays via __cuda_array_interface__).";

  py::class_<DeviceArray, std::shared_ptr<DeviceArray>>(m, "DeviceArray",
                                                        "Owning device buffer (__cuda_array_interface__).")
      .def_property_readonly("__cuda_array_interface__", &DeviceArray::interface)
      .def_property_readonly("shape", [](const DeviceArray& a) { return py::tuple(py::cast(a.shape())); })
      .def_property_readonly("device", &DeviceArray::device)
      .def_property_readonly("ptr", [](const DeviceArray& a) { return reinterpret_cast<std::uintptr_t>(a.ptr()); });

  m.def("scan", &scan, py::arg("decays"), py::arg("impulses"), py::arg("initial") = py::none(),
        py::kw_only(), py::arg("workers") = 0, py::arg("mode") = "parallel",
        py::arg("device") = py::none(), py::arg("stream") = std::uintptr_t(0),
        "Evaluate the recurrence on the GPU; returns h with the input shape. "
        "mode \"serial\" (or workers=1) runs the bit-exact per-channel kernel; "
        "otherwise the single-pass chained scan.  Deterministic.");
  m.def("scan_backward", &scan_backward, py::arg("decays"), py::arg("initial"), py::arg("h"),
        py::arg("d_h"), py::kw_only(), py::arg("workers") = 0, py::arg("mode") = "parallel",
        py::arg("device") = py::none(), py::arg("stream") = std::uintptr_t(0),
        "Gradients of a scalar loss w.r.t. every input, given the forward output h and "
        "upstream d_h. Returns (d_decays, d_impulses, d_initial).");
  m.def("plan_chunks", &plan_chunks, py::arg("T"), py::arg("workers"),
        "Contiguous partition of steps 1..T (1-indexed, inclusive bounds) of the "
        "reference's CPU chunked scan; effective worker count is min(workers, T).");
  m.def("predicted_speedup", &predicted_speedup, py::arg("workers"), py::arg("T"),
        "Cost-model speedup p*T / (3*(T + log2(p))) of the chunked scan over the serial one.");
  m.def("hardware_workers", &hardware_workers, "Worker count used when workers=0.");
  m.def("device_count", &linrec_device_count, "CUDA devices visible to the library.");
  m.def("abi_version", &linrec_abi_version);
}
