// C shim over the UNMODIFIED reference recurrence core -- TEST INFRASTRUCTURE.
//
// Compiled by oracle/Makefile against the headers where they lie under
// /root/reference/proj/include (never copied into this repo) into
// oracle/_ref/liblinrec_ref.so.  It exposes linrec::scan_serial,
// linrec::scan_parallel and linrec::scan_backward (recurrence.hpp:169-377)
// on raw [T][b][n] buffers so the tests can pin oracle/linrec_oracle.c to the
// reference bit for bit, and so bench.py can time the reference's own CPU
// path (cpu_baseline kind "reference").
#include <algorithm>
#include <chrono>
#include <vector>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "linrec/recurrence.hpp"
#include "linrec/rng.hpp"
#include "support/layer_oracles.hpp"  // proj/tests/support: per-step layer oracles

namespace {
thread_local std::string g_err;

template <class S>
linrec::Tensor3<S> t3(const S* p, int64_t T, int64_t b, int64_t n) {
  linrec::Tensor3<S> t(T, b, n);
  std::copy(p, p + t.size(), t.data.begin());
  return t;
}
template <class S>
linrec::Tensor2<S> t2(const S* p, int64_t b, int64_t n) {
  linrec::Tensor2<S> t(b, n);
  if (p) std::copy(p, p + t.size(), t.data.begin());
  return t;
}

template <class S>
int scan_impl(const S* lam, const S* x, const S* h0, S* h, int64_t T,
              int64_t b, int64_t n, int mode, int workers, S* P, S* R, S* C) {
  try {
    auto L = t3(lam, T, b, n);
    auto X = t3(x, T, b, n);
    auto H0 = t2(h0, b, n);
    linrec::Tensor3<S> out;
    if (mode == 0) {
      out = linrec::scan_serial(L, X, H0);
    } else {
      linrec::ThreadPool pool(workers);
      linrec::ScanSummaries<S> s;
      out = linrec::scan_parallel(L, X, H0, linrec::plan_chunks(T, workers),
                                  pool, false, &s);
      if (P) std::copy(s.P.data.begin(), s.P.data.end(), P);
      if (R) std::copy(s.R.data.begin(), s.R.data.end(), R);
      if (C) std::copy(s.C.data.begin(), s.C.data.end(), C);
    }
    std::copy(out.data.begin(), out.data.end(), h);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <class S>
int bwd_impl(const S* lam, const S* h0, const S* h, const S* dh, S* dlam,
             S* dx, S* dh0, int64_t T, int64_t b, int64_t n, int mode,
             int workers) {
  try {
    auto L = t3(lam, T, b, n);
    auto H = t3(h, T, b, n);
    auto DH = t3(dh, T, b, n);
    auto H0 = t2(h0, b, n);
    linrec::ThreadPool pool(workers);
    auto g = linrec::scan_backward(
        L, H0, H, DH,
        mode == 0 ? linrec::ScanMode::Serial : linrec::ScanMode::Parallel,
        pool);
    std::copy(g.d_decays.data.begin(), g.d_decays.data.end(), dlam);
    std::copy(g.d_impulses.data.begin(), g.d_impulses.data.end(), dx);
    std::copy(g.d_initial.data.begin(), g.d_initial.data.end(), dh0);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {
const char* ref_last_error() { return g_err.c_str(); }

int ref_scan_f32(const float* lam, const float* x, const float* h0, float* h,
                 int64_t T, int64_t b, int64_t n, int mode, int workers,
                 float* P, float* R, float* C) {
  return scan_impl(lam, x, h0, h, T, b, n, mode, workers, P, R, C);
}
int ref_scan_f64(const double* lam, const double* x, const double* h0,
                 double* h, int64_t T, int64_t b, int64_t n, int mode,
                 int workers, double* P, double* R, double* C) {
  return scan_impl(lam, x, h0, h, T, b, n, mode, workers, P, R, C);
}
int ref_scan_backward_f32(const float* lam, const float* h0, const float* h,
                          const float* dh, float* dlam, float* dx, float* dh0,
                          int64_t T, int64_t b, int64_t n, int mode,
                          int workers) {
  return bwd_impl(lam, h0, h, dh, dlam, dx, dh0, T, b, n, mode, workers);
}
int ref_scan_backward_f64(const double* lam, const double* h0,
                          const double* h, const double* dh, double* dlam,
                          double* dx, double* dh0, int64_t T, int64_t b,
                          int64_t n, int mode, int workers) {
  return bwd_impl(lam, h0, h, dh, dlam, dx, dh0, T, b, n, mode, workers);
}
// linrec::Rng(seed).split(stream) then fill_uniform (rng.hpp:15-71).
void ref_rng_fill_f32(uint64_t seed, int64_t split_stream, float* v,
                      int64_t count, double lo, double hi) {
  linrec::Rng root(seed);
  linrec::Rng rng = split_stream >= 0 ? root.split(uint64_t(split_stream))
                                      : root;
  for (int64_t i = 0; i < count; ++i) v[i] = float(rng.uniform(lo, hi));
}
uint64_t ref_rng_first(uint64_t seed, int which) {
  linrec::Rng rng(seed);
  uint64_t v = 0;
  for (int i = 0; i <= which; ++i) v = rng.next_u64();
  return v;
}
int ref_hardware_workers() { return linrec::ThreadPool::hardware_workers(); }

// The reference's own kernel-bench protocol (bench.hpp:93-107, :160-202):
// inputs built once outside the timed region, one ThreadPool(workers) and one
// plan_chunks(T, workers) reused, `warmup` untimed calls, then the median of
// `reps` steady_clock-timed calls of scan_parallel (forward) and of
// scan_backward(ScanMode::Parallel) (backward).  Output allocation inside the
// scan_* calls is timed, as in the reference.
int ref_bench_fwd_bwd_f32(const float* lam, const float* x, const float* h0,
                          const float* dh, int64_t T, int64_t b, int64_t n,
                          int workers, int warmup, int reps, double* fwd_s,
                          double* bwd_s) {
  try {
    auto L = t3(lam, T, b, n);
    auto X = t3(x, T, b, n);
    auto DH = t3(dh, T, b, n);
    auto H0 = t2(h0, b, n);
    linrec::ThreadPool pool(workers);
    const linrec::ChunkPlan plan = linrec::plan_chunks(T, workers);
    linrec::Tensor3<float> h;
    linrec::RecurrenceGradients<float> g;
    auto median = [](std::vector<double> v) {
      std::sort(v.begin(), v.end());
      const size_t m = v.size() / 2;
      return v.size() % 2 ? v[m] : 0.5 * (v[m - 1] + v[m]);
    };
    for (int i = 0; i < warmup; ++i) {
      h = linrec::scan_parallel(L, X, H0, plan, pool);
      g = linrec::scan_backward(L, H0, h, DH, linrec::ScanMode::Parallel, pool);
    }
    std::vector<double> tf, tb;
    for (int i = 0; i < reps; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      h = linrec::scan_parallel(L, X, H0, plan, pool);
      const auto t1 = std::chrono::steady_clock::now();
      g = linrec::scan_backward(L, H0, h, DH, linrec::ScanMode::Parallel, pool);
      const auto t2 = std::chrono::steady_clock::now();
      tf.push_back(std::chrono::duration<double>(t1 - t0).count());
      tb.push_back(std::chrono::duration<double>(t2 - t1).count());
    }
    *fwd_s = median(tf);
    *bwd_s = median(tb);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The same protocol for the 1-core serial path: scan_serial
// (recurrence.hpp:169-184) and scan_backward(ScanMode::Serial) -- the
// reference's single-thread baseline (SURVEY.md 8d "CPU baseline" row).
int ref_bench_serial_f32(const float* lam, const float* x, const float* h0,
                         const float* dh, int64_t T, int64_t b, int64_t n,
                         int warmup, int reps, double* fwd_s, double* bwd_s) {
  try {
    auto L = t3(lam, T, b, n);
    auto X = t3(x, T, b, n);
    auto DH = t3(dh, T, b, n);
    auto H0 = t2(h0, b, n);
    linrec::ThreadPool pool(1);
    linrec::Tensor3<float> h;
    linrec::RecurrenceGradients<float> g;
    auto median = [](std::vector<double> v) {
      std::sort(v.begin(), v.end());
      const size_t m = v.size() / 2;
      return v.size() % 2 ? v[m] : 0.5 * (v[m - 1] + v[m]);
    };
    for (int i = 0; i < warmup; ++i) {
      h = linrec::scan_serial(L, X, H0);
      g = linrec::scan_backward(L, H0, h, DH, linrec::ScanMode::Serial, pool);
    }
    std::vector<double> tf, tb;
    for (int i = 0; i < reps; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      h = linrec::scan_serial(L, X, H0);
      const auto t1 = std::chrono::steady_clock::now();
      g = linrec::scan_backward(L, H0, h, DH, linrec::ScanMode::Serial, pool);
      const auto t2 = std::chrono::steady_clock::now();
      tf.push_back(std::chrono::duration<double>(t1 - t0).count());
      tb.push_back(std::chrono::duration<double>(t2 - t1).count());
    }
    *fwd_s = median(tf);
    *bwd_s = median(tb);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The reference's per-step GILR / GILR-LSTM oracles
// (proj/tests/support/layer_oracles.hpp:28-82, fp64).  Parameters row-major
// as GilrParams / GilrLstmParams (layers.hpp:28-40, :148-165).
static linrec::Tensor2<double> t2d(const double* p, int64_t r, int64_t c) {
  linrec::Tensor2<double> t(r, c);
  std::copy(p, p + r * c, t.data.begin());
  return t;
}
int ref_gilr_lstm_oracle(const double* x, const double* sU, const double* sV, const double* sbg,
                         const double* sbz, const double* U, const double* V, const double* bias,
                         const double* htil0, const double* c0, double* h, int64_t T, int64_t b,
                         int64_t m, int64_t n) {
  try {
    linrec::GilrLstmParams<double> p;
    p.surrogate.U = t2d(sU, n, m);
    p.surrogate.V = t2d(sV, n, m);
    p.surrogate.b_g = t2d(sbg, 1, n);
    p.surrogate.b_z = t2d(sbz, 1, n);
    p.surrogate.act = linrec::Activation::Tanh;
    p.U = t2d(U, 4 * n, n);
    p.V = t2d(V, 4 * n, m);
    p.bias = t2d(bias, 1, 4 * n);
    auto X = t3(x, T, b, m);
    auto H0 = t2(htil0, b, n);
    auto C0 = t2(c0, b, n);
    auto out = oracle::gilr_lstm(p, X, H0, C0);
    std::copy(out.data.begin(), out.data.end(), h);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
int ref_gilr_oracle(const double* x, const double* U, const double* V, const double* bg, const double* bz,
                    const double* h0, double* h, int64_t T, int64_t b, int64_t m, int64_t n) {
  try {
    linrec::GilrParams<double> p;
    p.U = t2d(U, n, m);
    p.V = t2d(V, n, m);
    p.b_g = t2d(bg, 1, n);
    p.b_z = t2d(bz, 1, n);
    p.act = linrec::Activation::Tanh;
    auto X = t3(x, T, b, m);
    auto H0 = t2(h0, b, n);
    auto out = oracle::gilr(p, X, H0);
    std::copy(out.data.begin(), out.data.end(), h);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
int ref_qrnn_oracle(const double* x, const double* W, const double* bias, const double* c0, double* h,
                    int64_t T, int64_t b, int64_t m, int64_t n, int64_t k) {
  // per-step QRNN (proj/tests/support/layer_oracles.hpp:84-114); W packed [k][3n][m]
  try {
    linrec::QrnnParams<double> p;
    for (int64_t s = 0; s < k; ++s) p.W.push_back(t2d(W + s * 3 * n * m, 3 * n, m));
    p.bias = t2d(bias, 1, 3 * n);
    auto X = t3(x, T, b, m);
    auto C0 = t2(c0, b, n);
    auto out = oracle::qrnn(p, X, C0);
    std::copy(out.data.begin(), out.data.end(), h);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}
