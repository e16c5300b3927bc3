// C++ caller of the drop-in headers, as a reference C++ call site would use
// them (include/linrec/cuda_scan.hpp, include/linrec/cuda_layers.hpp):
//   * scan_serial is bit-identical to a serial fmaf loop (recurrence.hpp:98-112,
//     the reference build's contraction), scan_parallel within the
//     reference's 1e-5 normwise tolerance, scan_backward likewise;
//   * shape errors throw ContractViolation with the reference's message;
//   * gilr_lstm_forward/backward and qrnn_forward/backward run through the
//     C++ mirror: parallel and serial scan modes agree within 1e-5 and the
//     gradients are finite and non-zero; the double instantiation of the
//     layer mirror agrees with itself across modes and with the fp32 path.
// Built by `make cpp-tests`; run by tests/test_gpu_cpp_api.py on a GPU.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "linrec/cuda_layers.hpp"
#include "linrec/cuda_scan.hpp"
#include "linrec/cuda_sharded.hpp"

using namespace linrec::cuda;

static int failures = 0;
#define CHECK(cond, ...)                                 \
  do {                                                   \
    if (!(cond)) {                                       \
      std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      std::fprintf(stderr, __VA_ARGS__);                 \
      std::fprintf(stderr, "\n");                        \
      ++failures;                                        \
    }                                                    \
  } while (0)

struct Dev {
  float* p = nullptr;
  size_t n = 0;
  explicit Dev(size_t count) : n(count) {
    if (cudaMalloc(&p, count * sizeof(float) + 16) != cudaSuccess) std::abort();
    cudaMemset(p, 0, count * sizeof(float) + 16);
  }
  Dev(const std::vector<float>& h) : Dev(h.size()) { cudaMemcpy(p, h.data(), h.size() * 4, cudaMemcpyHostToDevice); }
  ~Dev() { cudaFree(p); }
  std::vector<float> get() const {
    std::vector<float> h(n);
    cudaMemcpy(h.data(), p, n * 4, cudaMemcpyDeviceToHost);
    return h;
  }
};

static std::vector<float> uniform(size_t n, float lo, float hi, unsigned seed) {
  std::mt19937 g(seed);
  std::uniform_real_distribution<float> d(lo, hi);
  std::vector<float> v(n);
  for (auto& x : v) x = d(g);
  return v;
}

static double normwise(const std::vector<float>& a, const std::vector<double>& ref) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num = std::fmax(num, std::fabs((double)a[i] - ref[i]));
    den = std::fmax(den, std::fabs(ref[i]));
  }
  return den > 0 ? num / den : num;
}

static double normwise_f(const std::vector<float>& a, const std::vector<float>& b) {
  std::vector<double> r(b.begin(), b.end());
  return normwise(a, r);
}

static bool finite_nonzero(const std::vector<float>& v) {
  bool nz = false;
  for (float x : v) {
    if (!std::isfinite(x)) return false;
    nz = nz || x != 0.f;
  }
  return nz;
}

static void test_scans() {
  const index_t T = 3000, b = 2, n = 100, W = b * n;
  auto lam = uniform(T * W, 0.05f, 0.95f, 1), x = uniform(T * W, -1, 1, 2), h0 = uniform(W, -1, 1, 3);
  auto dh = uniform(T * W, -1, 1, 4);
  Dev L(lam), X(x), H0(h0), DH(dh), Hs(T * W), Hp(T * W), DL(T * W), DX(T * W), DH0(W);
  DeviceTensor3<float> l{L.p, T, b, n}, xx{X.p, T, b, n}, hs{Hs.p, T, b, n}, hp{Hp.p, T, b, n}, d_h{DH.p, T, b, n};
  DeviceTensor2<float> i0{H0.p, b, n};
  scan_serial(l, xx, i0, hs);
  scan_parallel(l, xx, i0, hp);
  // serial fmaf loop (the reference build contracts l*prev + x into an FMA)
  std::vector<float> ref(T * W);
  std::vector<double> ref64(T * W);
  for (index_t j = 0; j < W; ++j) {
    float prev = h0[j];
    double p64 = h0[j];
    for (index_t t = 0; t < T; ++t) {
      prev = std::fmaf(lam[t * W + j], prev, x[t * W + j]);
      p64 = (double)lam[t * W + j] * p64 + x[t * W + j];
      ref[t * W + j] = prev;
      ref64[t * W + j] = p64;
    }
  }
  cudaDeviceSynchronize();
  CHECK(Hs.get() == ref, "scan_serial is not bit-identical to the serial fmaf loop");
  CHECK(normwise(Hp.get(), ref64) < 1e-5, "scan_parallel error %g", normwise(Hp.get(), ref64));
  // backward (recurrence.hpp:283-348): G_t = lam_{t+1} G_{t+1} + dh_t
  RecurrenceGradients<float> g{{DL.p, T, b, n}, {DX.p, T, b, n}, {DH0.p, b, n}};
  scan_backward(l, i0, hs, d_h, g, ScanMode::Serial);
  std::vector<float> rdx(T * W), rdl(T * W), rdh0(W);
  for (index_t j = 0; j < W; ++j) {
    float G = 0.f;
    for (index_t t = T - 1; t >= 0; --t) {
      const float mu = t + 1 < T ? lam[(t + 1) * W + j] : 0.f;
      G = std::fmaf(mu, G, dh[t * W + j]);
      rdx[t * W + j] = G;
      rdl[t * W + j] = (t == 0 ? h0[j] : ref[(t - 1) * W + j]) * G;
    }
    rdh0[j] = lam[j] * G;
  }
  cudaDeviceSynchronize();
  CHECK(DX.get() == rdx && DL.get() == rdl && DH0.get() == rdh0, "serial scan_backward not bit-identical");
  scan_backward(l, i0, hs, d_h, g, ScanMode::Parallel);
  cudaDeviceSynchronize();
  CHECK(normwise_f(DX.get(), rdx) < 1e-5 && normwise_f(DL.get(), rdl) < 1e-5, "parallel scan_backward error");
  // contract errors with the reference's messages (recurrence.hpp:39-51)
  DeviceTensor3<float> bad{X.p, 4, 1, 3}, ok{L.p, 4, 1, 2};
  try {
    scan_parallel(ok, bad, DeviceTensor2<float>{}, ok);
    CHECK(false, "shape mismatch did not throw");
  } catch (const ContractViolation& e) {
    CHECK(std::string(e.what()) == "recurrence: shape mismatch, [4,1,2] vs [4,1,3]", "message: %s", e.what());
  }
}

static void test_gilr_lstm() {
  const index_t T = 257, b = 3, m = 12, n = 16, R = T * b;
  auto sU = uniform(n * m, -.3f, .3f, 5), sV = uniform(n * m, -.3f, .3f, 6), sbg = uniform(n, 0, 1, 7);
  auto sbz = uniform(n, -.1f, .1f, 8), U = uniform(4 * n * n, -.25f, .25f, 9), V = uniform(4 * n * m, -.3f, .3f, 10);
  auto bias = uniform(4 * n, -.5f, .5f, 11), x = uniform(R * m, -1, 1, 12), dh = uniform(R * n, -1, 1, 13);
  Dev dsU(sU), dsV(sV), dsbg(sbg), dsbz(sbz), dU(U), dV(V), dbias(bias), X(x), DH(dh);
  GilrLstmParams p;
  p.surrogate = GilrParams{dsU.p, dsV.p, dsbg.p, dsbz.p, Activation::Tanh, m, n};
  p.U = dU.p;
  p.V = dV.p;
  p.bias = dbias.p;
  LayerContext ctx;
  std::vector<float> h_par, dx_par, gV_par;
  for (ScanMode mode : {ScanMode::Parallel, ScanMode::Serial}) {
    Dev sg(R * n), si(R * n), htil((T + 1) * b * n), gates(4 * R * n), c(R * n), H(R * n), DX(R * m);
    Dev gsU(n * m), gsV(n * m), gsbg(n), gsbz(n), gU(4 * n * n), gV(4 * n * m), gbias(4 * n);
    GilrLstmCache cache{sg.p, si.p, htil.p, gates.p, c.p};
    DeviceTensor3<float> xx{X.p, T, b, m}, h{H.p, T, b, n}, d_h{DH.p, T, b, n}, dx{DX.p, T, b, m};
    DeviceTensor2<float> zero{};
    gilr_lstm_forward(p, xx, zero, zero, mode, ctx, cache, h);
    GilrLstmGrads g{{gsU.p, gsV.p, gsbg.p, gsbz.p}, gU.p, gV.p, gbias.p};
    gilr_lstm_backward(p, xx, zero, zero, cache, d_h, mode, ctx, g, dx);
    cudaDeviceSynchronize();
    CHECK(finite_nonzero(H.get()) && finite_nonzero(DX.get()) && finite_nonzero(gV.get()) &&
              finite_nonzero(gsU.get()) && finite_nonzero(gbias.get()),
          "gilr_lstm outputs / gradients not finite or all zero");
    if (mode == ScanMode::Parallel) {
      h_par = H.get();
      dx_par = DX.get();
      gV_par = gV.get();
    } else {
      CHECK(normwise_f(h_par, H.get()) < 1e-5, "gilr_lstm h: parallel vs serial %g", normwise_f(h_par, H.get()));
      CHECK(normwise_f(dx_par, DX.get()) < 1e-5, "gilr_lstm dx: parallel vs serial");
      CHECK(normwise_f(gV_par, gV.get()) < 1e-5, "gilr_lstm dV: parallel vs serial");
    }
  }
  try {
    DeviceTensor3<float> wrong{X.p, T, b, m + 4};
    Dev H(R * n);
    DeviceTensor3<float> h{H.p, T, b, n};
    gilr_lstm_forward(p, wrong, DeviceTensor2<float>{}, DeviceTensor2<float>{}, ScanMode::Parallel, ctx,
                      GilrLstmCache{}, h);
    CHECK(false, "feature mismatch did not throw");
  } catch (const ContractViolation& e) {
    CHECK(std::string(e.what()) == "gilr_lstm_forward: input feature mismatch", "message: %s", e.what());
  }
}

static void test_qrnn() {
  const index_t T = 100, b = 2, m = 8, n = 12, k = 3, R = T * b;
  auto W = uniform(k * 3 * n * m, -.3f, .3f, 21), bias = uniform(3 * n, -.5f, .5f, 22);
  auto x = uniform(R * m, -1, 1, 23), dh = uniform(R * n, -1, 1, 24);
  Dev dW(W), dbias(bias), X(x), DH(dh);
  QrnnParams p{dW.p, dbias.p, m, n, k};
  LayerContext ctx(nullptr, Precision::Fp32);
  std::vector<float> h_par, dx_par;
  for (ScanMode mode : {ScanMode::Parallel, ScanMode::Serial}) {
    Dev gates(3 * R * n), c(R * n), H(R * n), DX(R * m), gW(k * 3 * n * m), gb(3 * n);
    QrnnCache cache{gates.p, c.p};
    QrnnGrads g{gW.p, gb.p};
    DeviceTensor3<float> xx{X.p, T, b, m}, h{H.p, T, b, n}, d_h{DH.p, T, b, n}, dx{DX.p, T, b, m};
    qrnn_forward(p, xx, DeviceTensor2<float>{}, mode, ctx, cache, h);
    qrnn_backward(p, xx, DeviceTensor2<float>{}, cache, d_h, mode, ctx, g, dx);
    cudaDeviceSynchronize();
    CHECK(finite_nonzero(H.get()) && finite_nonzero(DX.get()) && finite_nonzero(gW.get()), "qrnn outputs");
    if (mode == ScanMode::Parallel) {
      h_par = H.get();
      dx_par = DX.get();
    } else {
      CHECK(normwise_f(h_par, H.get()) < 1e-5 && normwise_f(dx_par, DX.get()) < 1e-5, "qrnn parallel vs serial");
    }
  }
}

// The double instantiation of the layer mirror (GilrLstmParamsT<double>,
// linrec_gilr_lstm_*_f64): parallel and serial scan modes agree within
// 1e-12, and the fp64 outputs / gradients match the fp32 path (3xTF32 GEMMs)
// within its 1e-5 on the same inputs.
static void test_gilr_lstm_f64() {
  const index_t T = 129, b = 2, m = 12, n = 16, R = T * b;
  auto sU = uniform(n * m, -.3f, .3f, 5), sV = uniform(n * m, -.3f, .3f, 6), sbg = uniform(n, 0, 1, 7);
  auto sbz = uniform(n, -.1f, .1f, 8), U = uniform(4 * n * n, -.25f, .25f, 9), V = uniform(4 * n * m, -.3f, .3f, 10);
  auto bias = uniform(4 * n, -.5f, .5f, 11), x = uniform(R * m, -1, 1, 12), dh = uniform(R * n, -1, 1, 13);
  struct DevD {
    double* p = nullptr;
    size_t n;
    explicit DevD(size_t c) : n(c) {
      if (cudaMalloc(&p, c * 8 + 16) != cudaSuccess) std::abort();
      cudaMemset(p, 0, c * 8 + 16);
    }
    explicit DevD(const std::vector<float>& h) : DevD(h.size()) {
      std::vector<double> d(h.begin(), h.end());
      cudaMemcpy(p, d.data(), d.size() * 8, cudaMemcpyHostToDevice);
    }
    ~DevD() { cudaFree(p); }
    std::vector<double> get() const {
      std::vector<double> h(n);
      cudaMemcpy(h.data(), p, n * 8, cudaMemcpyDeviceToHost);
      return h;
    }
  };
  auto nw = [](const std::vector<double>& a, const std::vector<double>& r) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
      num = std::fmax(num, std::fabs(a[i] - r[i]));
      den = std::fmax(den, std::fabs(r[i]));
    }
    return den > 0 ? num / den : num;
  };
  DevD dsU(sU), dsV(sV), dsbg(sbg), dsbz(sbz), dU(U), dV(V), dbias(bias), X(x), DH(dh);
  GilrLstmParamsT<double> p;
  p.surrogate = GilrParamsT<double>{dsU.p, dsV.p, dsbg.p, dsbz.p, Activation::Tanh, m, n};
  p.U = dU.p;
  p.V = dV.p;
  p.bias = dbias.p;
  LayerContext ctx;
  std::vector<double> h_par, dx_par, gV_par;
  for (ScanMode mode : {ScanMode::Parallel, ScanMode::Serial}) {
    DevD sg(R * n), si(R * n), htil((T + 1) * b * n), gates(4 * R * n), c(R * n), H(R * n), DX(R * m);
    DevD gsU(n * m), gsV(n * m), gsbg(n), gsbz(n), gU(4 * n * n), gV(4 * n * m), gbias(4 * n);
    GilrLstmCacheT<double> cache{sg.p, si.p, htil.p, gates.p, c.p};
    DeviceTensor3<double> xx{X.p, T, b, m}, h{H.p, T, b, n}, d_h{DH.p, T, b, n}, dx{DX.p, T, b, m};
    DeviceTensor2<double> zero{};
    gilr_lstm_forward(p, xx, zero, zero, mode, ctx, cache, h);
    GilrLstmGradsT<double> g{{gsU.p, gsV.p, gsbg.p, gsbz.p}, gU.p, gV.p, gbias.p};
    gilr_lstm_backward(p, xx, zero, zero, cache, d_h, mode, ctx, g, dx);
    cudaDeviceSynchronize();
    if (mode == ScanMode::Parallel) {
      h_par = H.get();
      dx_par = DX.get();
      gV_par = gV.get();
    } else {
      CHECK(nw(h_par, H.get()) < 1e-12 && nw(dx_par, DX.get()) < 1e-12 && nw(gV_par, gV.get()) < 1e-12,
            "gilr_lstm f64: parallel vs serial %g", nw(h_par, H.get()));
    }
  }
  // the fp32 path on the same inputs
  Dev fsU(sU), fsV(sV), fsbg(sbg), fsbz(sbz), fU(U), fV(V), fbias(bias), FX(x), FDH(dh);
  GilrLstmParams q;
  q.surrogate = GilrParams{fsU.p, fsV.p, fsbg.p, fsbz.p, Activation::Tanh, m, n};
  q.U = fU.p;
  q.V = fV.p;
  q.bias = fbias.p;
  Dev sg(R * n), si(R * n), htil((T + 1) * b * n), gates(4 * R * n), c(R * n), H(R * n), DX(R * m);
  Dev gsU(n * m), gsV(n * m), gsbg(n), gsbz(n), gU(4 * n * n), gV(4 * n * m), gbias(4 * n);
  GilrLstmCache cache{sg.p, si.p, htil.p, gates.p, c.p};
  DeviceTensor3<float> xx{FX.p, T, b, m}, h{H.p, T, b, n}, d_h{FDH.p, T, b, n}, dx{DX.p, T, b, m};
  gilr_lstm_forward(q, xx, DeviceTensor2<float>{}, DeviceTensor2<float>{}, ScanMode::Parallel, ctx, cache, h);
  GilrLstmGrads g{{gsU.p, gsV.p, gsbg.p, gsbz.p}, gU.p, gV.p, gbias.p};
  gilr_lstm_backward(q, xx, DeviceTensor2<float>{}, DeviceTensor2<float>{}, cache, d_h, ScanMode::Parallel, ctx, g,
                     dx);
  cudaDeviceSynchronize();
  CHECK(normwise(H.get(), h_par) < 1e-5 && normwise(DX.get(), dx_par) < 1e-5 && normwise(gV.get(), gV_par) < 1e-5,
        "gilr_lstm fp32 vs fp64: h %g dx %g dV %g", normwise(H.get(), h_par), normwise(DX.get(), dx_par),
        normwise(gV.get(), gV_par));
}

// scan_parallel with an explicit plan and ScanSummaries: the reference's
// hand-executed two-chunk example (test_recurrence.cpp:75-99), and the
// plan-chunked forward against the fmaf restatement of its three phases.
static void test_plan_scan() {
  {
    Dev L(std::vector<float>{1, 1, 1, 1}), X(std::vector<float>{1, 1, 1, 1}), H0(std::vector<float>{0});
    Dev H(4), P(2), R(2), C(2);
    DeviceTensor3<float> l{L.p, 4, 1, 1}, x{X.p, 4, 1, 1}, h{H.p, 4, 1, 1};
    DeviceTensor2<float> i0{H0.p, 1, 1};
    ScanSummaries<float> s{{P.p, 2, 1, 1}, {R.p, 2, 1, 1}, {C.p, 2, 1, 1}};
    const ChunkPlan plan = plan_chunks(4, 2);
    scan_parallel(l, x, i0, plan, h, &s);
    cudaDeviceSynchronize();
    CHECK(P.get() == (std::vector<float>{1, 1}) && R.get() == (std::vector<float>{2, 2}) &&
              C.get() == (std::vector<float>{2, 4}) && H.get() == (std::vector<float>{1, 2, 3, 4}),
          "two-chunk example: P, R, C or h differ");
  }
  const index_t T = 1001, W = 37;
  auto lam = uniform(T * W, -1, 1, 11), x = uniform(T * W, -1, 1, 12), h0 = uniform(W, -1, 1, 13);
  Dev L(lam), X(x), H0(h0), H(T * W);
  DeviceTensor3<float> l{L.p, T, 1, W}, xx{X.p, T, 1, W}, h{H.p, T, 1, W};
  DeviceTensor2<float> i0{H0.p, 1, W};
  const ChunkPlan plan = plan_chunks(T, 6);
  scan_parallel(l, xx, i0, plan, h);
  std::vector<float> ref(T * W), C(W);
  for (index_t j = 0; j < W; ++j) C[j] = h0[j];
  for (const auto& se : plan.bounds) {  // phases 1-2 then 3, per chunk in order
    for (index_t j = 0; j < W; ++j) {
      float P = 1.f, R = 0.f;
      for (index_t t = se.first - 1; t <= se.second - 1; ++t) {
        R = std::fmaf(lam[t * W + j], R, x[t * W + j]);
        P = P * lam[t * W + j];
      }
      float c = C[j];
      for (index_t t = se.first - 1; t <= se.second - 1; ++t) ref[t * W + j] = c = std::fmaf(lam[t * W + j], c, x[t * W + j]);
      C[j] = std::fmaf(P, C[j], R);
    }
  }
  CHECK(H.get() == ref, "plan scan_parallel is not bit-identical to the three-phase fmaf restatement");
  try {
    ChunkPlan bad = plan;
    bad.bounds[0].second += 1;
    scan_parallel(l, xx, i0, bad, h);
    CHECK(false, "a gap in the plan did not throw");
  } catch (const ContractViolation& e) {
    CHECK(std::string(e.what()).find("ChunkPlan: chunks must be contiguous") != std::string::npos, "message: %s",
          e.what());
  }
}

// "finite screening pinpoints the poisoned element" (test_recurrence.cpp:328-350):
// check_finite off -> no throw; on -> ContractViolation naming the tensor and
// the 1-based step, batch and feature of the first non-finite element.
static void test_check_finite() {
  const index_t T = 9, b = 2, n = 4, W = b * n;
  std::vector<float> lam = uniform(T * W, 0.05f, 0.95f, 108), x = uniform(T * W, -1, 1, 109);
  std::vector<float> h0 = uniform(W, -1, 1, 110), dh = uniform(T * W, -1, 1, 111);
  x[(5 * b + 1) * n + 2] = std::nanf("");  // in.impulses.at(5, 1, 2)
  Dev L(lam), X(x), H0(h0), H(T * W), DH(dh), DL(T * W), DX(T * W), D0(W);
  DeviceTensor3<float> tl{L.p, T, b, n}, tx{X.p, T, b, n}, th{H.p, T, b, n}, tdh{DH.p, T, b, n};
  DeviceTensor2<float> t0{H0.p, b, n};
  bool threw = false;
  try {
    scan_serial(tl, tx, t0, th);  // screening off: garbage in, garbage out
  } catch (...) {
    threw = true;
  }
  CHECK(!threw, "check_finite=false threw");
  auto expect = [&](auto fn, const char* name, const char* where) {
    std::string msg;
    try {
      fn();
    } catch (const ContractViolation& e) {
      msg = e.what();
    }
    CHECK(msg.find(std::string("non-finite value in ") + name) != std::string::npos && msg.find(where) != std::string::npos,
          "screen message '%s' (want %s %s)", msg.c_str(), name, where);
  };
  expect([&] { scan_serial(tl, tx, t0, th, nullptr, true); }, "impulses", "[t=6, b=1, n=2]");
  expect([&] { scan_parallel(tl, tx, t0, th, nullptr, nullptr, true); }, "impulses", "[t=6, b=1, n=2]");
  expect([&] { scan_parallel(tl, tx, t0, plan_chunks(T, 2), th, (ScanSummaries<float>*)nullptr, nullptr, true); }, "impulses",
         "[t=6, b=1, n=2]");
  expect([&] { scan(tl, tx, t0, th, ScanMode::Parallel, nullptr, nullptr, true); }, "impulses", "[t=6, b=1, n=2]");
  // decays are screened first; the initial state reports [b, n]
  std::vector<float> lam2 = lam;
  lam2[(8 * b + 0) * n + 3] = INFINITY;
  Dev L2(lam2);
  DeviceTensor3<float> tl2{L2.p, T, b, n};
  expect([&] { scan_serial(tl2, tx, t0, th, nullptr, true); }, "decays", "[t=9, b=0, n=3]");
  std::vector<float> x_ok = uniform(T * W, -1, 1, 112), h0b = h0;
  h0b[1 * n + 1] = -INFINITY;
  Dev X2(x_ok), H0b(h0b);
  DeviceTensor3<float> tx2{X2.p, T, b, n};
  DeviceTensor2<float> t0b{H0b.p, b, n};
  expect([&] { scan_serial(tl, tx2, t0b, th, nullptr, true); }, "initial", "[b=1, n=1]");
  // backward screens decays and d_h (recurrence.hpp:292-296)
  std::vector<float> dh2 = dh;
  dh2[(0 * b + 0) * n + 0] = std::nanf("");
  Dev DH2(dh2);
  DeviceTensor3<float> tdh2{DH2.p, T, b, n};
  RecurrenceGradients<float> g{{DL.p, T, b, n}, {DX.p, T, b, n}, {D0.p, b, n}};
  scan_serial(tl, tx2, t0, th, nullptr, true);  // finite: no throw
  expect([&] { scan_backward(tl, t0, th, tdh2, g, ScanMode::Parallel, nullptr, nullptr, true); }, "d_h",
         "[t=1, b=0, n=0]");
  expect([&] { scan_backward(tl, t0, th, tdh2, plan_chunks(T, 3), g, nullptr, true); }, "d_h", "[t=1, b=0, n=0]");
  threw = false;
  try {
    scan_backward(tl, t0, th, tdh, g, ScanMode::Serial, nullptr, nullptr, true);
  } catch (...) {
    threw = true;
  }
  CHECK(!threw, "finite backward inputs threw");
}

// Channel sharding of host tensors (cuda_sharded.hpp): the columns split over
// two "devices" (device 0 twice on a one-GPU box: two host threads, each its
// own column block) must reproduce the single-GPU serial scan bit for bit.
static void test_channel_sharded() {
  const index_t T = 2500, b = 3, n = 68, W = b * n;
  auto lam = uniform(T * W, 0.05f, 0.95f, 11), x = uniform(T * W, -1, 1, 12), h0 = uniform(W, -1, 1, 13);
  auto dh = uniform(T * W, -1, 1, 14);
  std::vector<float> h(T * W), hs(T * W), dl(T * W), dx(T * W), dh0(W);
  HostTensor3<float> L{lam.data(), T, b, n}, X{x.data(), T, b, n}, H{h.data(), T, b, n}, Hs{hs.data(), T, b, n};
  const std::vector<int> devs{0, 0};
  scan_channel_sharded(L, X, h0.data(), Hs, devs, ScanMode::Serial);
  scan_channel_sharded(L, X, h0.data(), H, devs);
  std::vector<float> ref(T * W);
  for (index_t j = 0; j < W; ++j) {
    float prev = h0[j];
    for (index_t t = 0; t < T; ++t) ref[t * W + j] = prev = std::fmaf(lam[t * W + j], prev, x[t * W + j]);
  }
  CHECK(hs == ref, "channel-sharded serial scan is not bit-identical to the serial loop");
  CHECK(normwise_f(h, ref) < 1e-5, "channel-sharded parallel scan error %g", normwise_f(h, ref));
  HostTensor3<float> DHt{dh.data(), T, b, n}, DL{dl.data(), T, b, n}, DX{dx.data(), T, b, n};
  scan_backward_channel_sharded(L, h0.data(), Hs, DHt, DL, DX, dh0.data(), devs, ScanMode::Serial);
  std::vector<float> rdx(T * W), rdl(T * W), rdh0(W);
  for (index_t j = 0; j < W; ++j) {
    float G = 0.f;
    for (index_t t = T - 1; t >= 0; --t) {
      const float mu = t + 1 < T ? lam[(t + 1) * W + j] : 0.f;
      G = std::fmaf(mu, G, dh[t * W + j]);
      rdx[t * W + j] = G;
      rdl[t * W + j] = (t == 0 ? h0[j] : ref[(t - 1) * W + j]) * G;
    }
    rdh0[j] = lam[j] * G;
  }
  CHECK(dx == rdx && dl == rdl && dh0 == rdh0, "channel-sharded serial backward is not bit-identical");
  bool threw = false;
  try {
    HostTensor3<float> bad{x.data(), T - 1, b, n};
    scan_channel_sharded(L, bad, h0.data(), H, devs);
  } catch (const ContractViolation& e) {
    threw = std::string(e.what()).find("recurrence: shape mismatch") != std::string::npos;
  }
  CHECK(threw, "shape mismatch did not throw the reference's ContractViolation");
}

int main() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    std::fprintf(stderr, "no CUDA device\n");
    return 2;
  }
  test_scans();
  test_plan_scan();
  test_check_finite();
  test_gilr_lstm();
  test_gilr_lstm_f64();
  test_qrnn();
  test_channel_sharded();
  if (failures == 0) std::printf("ALL OK\n");
  return failures == 0 ? 0 : 1;
}
