// extern "C" implementation of include/linrec_cuda.h: argument validation
// with the reference's error classes, workspace management, dispatch to the
// sm_100a kernels, and the pipelined host-pointer path.  There is no CPU
// compute path anywhere in this library: without a CUDA device every entry
// point fails with LINREC_ERR_CUDA.
#include "linrec_cuda.h"

#include <cuda_runtime.h>
#include <immintrin.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <thread>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "launch.h"
#include "linrec_device.cuh"

using linrec_impl::BwdCall;
using linrec_impl::ChainPlan;
using linrec_impl::ChainPtrs;
using linrec_impl::FwdCall;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
namespace {
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  std::ostringstream os;
  os << "linrec: CUDA error in " << where << ": " << cudaGetErrorName(e) << " ("
     << cudaGetErrorString(e) << ")";
  return fail(LINREC_ERR_CUDA, os.str());
}

#define LINREC_CUDA_TRY(expr)                            \
  do {                                                   \
    cudaError_t e_ = (expr);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr);  \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <class S>
constexpr int vec_of() {
  return sizeof(S) == 4 ? 4 : 2;
}

// 128-bit paths need W % VEC == 0 and 16-byte aligned rows.
template <class S>
bool vec_ok(int64_t W, std::initializer_list<const void*> ptrs) {
  if (W % vec_of<S>() != 0) return false;
  for (const void* p : ptrs)
    if (p != nullptr && !aligned16(p)) return false;
  return true;
}

// Reference contract: every dimension >= 1 (tensor.hpp:58) -- a [T, b, n]
// tensor with T == 0 cannot be constructed.
int check_dims(int64_t T, int64_t W) {
  if (T < 1 || W < 1) {
    std::ostringstream os;
    os << "Tensor3 dimensions must be >= 1 (got T=" << T << ", W=" << W << ")";
    return fail(LINREC_ERR_SHAPE, os.str());
  }
  return LINREC_OK;
}

// The chained kernels index rows with 32-bit integers.
int check_rows(int64_t T) {
  if (T > (int64_t(1) << 31) - 65536)
    return fail(LINREC_ERR_SHAPE, "linrec: T >= 2^31 - 65536 rows is not supported by the parallel kernels");
  return LINREC_OK;
}

int check_mode(int mode) {
  if (mode != LINREC_SERIAL && mode != LINREC_PARALLEL)
    return fail(LINREC_ERR_VALUE, "mode must be \"parallel\" or \"serial\"");
  return LINREC_OK;
}

int check_ptr(const void* p, const char* name) {
  if (p == nullptr) return fail(LINREC_ERR_VALUE, std::string(name) + " must not be NULL");
  return LINREC_OK;
}
}  // namespace

namespace linrec_impl {
int set_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace linrec_impl

// ---------------------------------------------------------------------------
// workspace
// ---------------------------------------------------------------------------
struct linrec_workspace {
  int device = 0;
  void* base = nullptr;
  size_t cap = 0;
  std::mutex mu;
};

namespace {
constexpr size_t kCtrlBytes = 256;

// Grows `ws` to at least `bytes`, stream-ordered.  A fresh buffer is zeroed
// and its control block initialised (epoch 1) on `st`.
int ws_reserve(linrec_workspace* ws, size_t bytes, cudaStream_t st) {
  if (ws->base != nullptr && ws->cap >= bytes) return LINREC_OK;
  if (ws->base != nullptr) {
    LINREC_CUDA_TRY(cudaFreeAsync(ws->base, st));
    ws->base = nullptr;
    ws->cap = 0;
  }
  const size_t cap = std::max<size_t>(bytes, size_t(1) << 20);
  LINREC_CUDA_TRY(cudaMallocAsync(&ws->base, cap, st));
  LINREC_CUDA_TRY(cudaMemsetAsync(ws->base, 0, cap, st));
  LINREC_CUDA_TRY(linrec_impl::launch_ws_init(ws->base, st));
  ws->cap = cap;
  return LINREC_OK;
}

ChainPtrs ws_ptrs(linrec_workspace* ws, const ChainPlan& p) {
  char* b = static_cast<char*>(ws->base);
  ChainPtrs w;
  w.ctrl = b;
  w.flags = b + kCtrlBytes;
  w.agg = b + kCtrlBytes + p.flags_bytes;
  w.inc = b + kCtrlBytes + p.flags_bytes + p.rec_bytes;
  return w;
}

// Virtual-segment region, after the look-back records: vagg [nseg][2][W]
// (each segment's chain aggregate) and seg_prod [nseg*ntt][W] (the products
// entering its chain positions); the fix-up folds the carries from vagg.
template <class S>
struct VsegPtrs {
  S* vagg;
  S* seg_prod;
  S* carry;  // [nseg][W]: the carries a deep (adaptive) scan seeds its segments with
};

template <class S>
size_t vseg_region_bytes(const ChainPlan& p, int64_t W) {
  return sizeof(S) * (size_t)W * (size_t)(3 * p.nseg + p.nseg * p.ntt) + 1024;
}

template <class S>
VsegPtrs<S> vseg_ptrs(linrec_workspace* ws, const ChainPlan& p, int64_t W) {
  char* b = static_cast<char*>(ws->base) + kCtrlBytes + p.flags_bytes + 2 * p.rec_bytes;
  b = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(b) + 255) & ~uintptr_t(255));
  S* v = reinterpret_cast<S*>(b);
  VsegPtrs<S> r;
  r.vagg = v;
  r.seg_prod = v + 2 * p.nseg * W;
  r.carry = r.seg_prod + p.nseg * p.ntt * W;
  return r;
}

// ---------------------------------------------------------------------------
// Decay-adaptive stitch (fp32 TMA scans with virtual segments).  The fix-up
// that stitches virtual segments touches only the positions whose decay
// product has not underflowed: ~2 tiles per segment for the reference's bench
// decays, but the whole segment when decays are near 1 -- then it is a second
// pass (12 B/el forward, 20 B/el backward).  A probe kernel
// estimates the fix-up depth from 64 sampled rows and sets a mode word on the
// device; the launches that follow read it: in "deep" mode a reduce-only pass
// (8-12 B/el, no outputs) gives every segment's aggregate, a fold gives the
// carries entering them, the scan seeds its segments with those carries and
// the fix-up exits at once; otherwise the reduce pass and the fold exit at
// once and the stitch runs as before.  All decisions stay on the device, so
// the sequence is stream-ordered and graph-capturable.  Thresholds: the mean
// fraction of a segment the fix-up would walk, above which the reduce pass
// is cheaper (forward: 8 B/el < 12 B/el x f; backward: 8 B/el -- the reduce
// pass stages mu and dh, not h -- < 20 B/el x f / 0.76).  LINREC_ADAPTIVE=0
// disables it.
bool adaptive_stitch_on() {
  static const bool on = linrec_impl::env_int("LINREC_ADAPTIVE", 1) != 0;
  return on;
}
constexpr float kDeepFracFwd = 0.67f, kDeepFracBwd = 0.30f;

// Wide scans (many channel columns) keep enough chains without virtual
// segments: there the deep branch is not reduce pass + seeded scan (20 / 28
// B/el) but an UNSPLIT twin of the scan, one chain per column, launched
// beside the split one (each exits in the other's mode) -- one pass.  From
// LINREC_UNSPLIT_COLS columns (default 8: 1024 channels) up; measured at
// lam ~ U(0.99, 1), fwd + bwd (scripts/dev/time_shape.py): C2 1.64 -> 1.96,
// 65536 x 2048 1.17 -> 1.48, 131072 x 1024 -> 1.29 x 10^11 el/s; at 4
// columns (262144 x 512) the twin loses (1.16 -> 1.03).
int64_t unsplit_cols() {
  static const int v = linrec_impl::env_int("LINREC_UNSPLIT_COLS", 8);
  return v > 0 ? v : (int64_t(1) << 40);
}

// The plan of that twin: the same tiles and kernel configuration, one chain
// per column (its look-back state fits the split plan's workspace).
ChainPlan unsplit_plan(const ChainPlan& p, int64_t T) {
  ChainPlan u = p;
  const int64_t ntt = (T + p.rows - 1) / p.rows;
  u.nseg = 1;
  u.ntt = ntt;
  u.tseg = ntt * p.rows;
  u.ntiles = p.ncols * ntt;
  u.flags_bytes = ((size_t)u.ntiles * 4 + 255) / 256 * 256;
  u.rec_bytes = (size_t)u.ntiles * 2 * p.rec * 8;
  u.ws_bytes = 256 + u.flags_bytes + 2 * u.rec_bytes;
  u.grid = (int)(p.grid < u.ntiles ? p.grid : u.ntiles);
  return u;
}
const int* decay_mode_ptr(linrec_workspace* ws) {
  return reinterpret_cast<const int*>(static_cast<char*>(ws->base) + offsetof(linrec_dev::Ctrl, decay_mode));
}

std::atomic<int> g_kernel_policy{0};  // LINREC_KERNEL_AUTO

bool tma_allowed(int64_t T, int64_t W) {
  return g_kernel_policy.load() != LINREC_KERNEL_REGISTER && T < (int64_t(1) << 30) &&
         W < (int64_t(1) << 30);
}

std::mutex g_default_mu;
std::map<std::pair<int, cudaStream_t>, std::unique_ptr<linrec_workspace>> g_default_ws;

int current_device(int* dev) {
  LINREC_CUDA_TRY(cudaGetDevice(dev));
  return LINREC_OK;
}

linrec_workspace* default_ws(int device, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_default_mu);
  auto& slot = g_default_ws[{device, st}];
  if (!slot) {
    slot.reset(new linrec_workspace());
    slot->device = device;
  }
  return slot.get();
}

// ---------------------------------------------------------------------------
// device-pointer scans
// ---------------------------------------------------------------------------
// Parallel mode runs the per-channel kernel when the channels alone fill the
// GPU (>= 2^17 threads of VEC channels: ~900 per SM) and the sequence is short
// (T <= 2048): the time-chained scan has nothing to add there, and its
// 96-row tiles are mostly padding at small T (bench_model's T=16, b=4096:
// 112 -> 27 us per forward scan).  LINREC_CHANNEL_PARALLEL=0 disables it.
// Short sequences over many channels: the per-channel kernel's T dependent
// steps are cheaper than any split of a few rows (scripts/bench_kernel.py,
// b = 1: T = 16, W = 65536 -- 2.9 us per-channel against 40.5 us split;
// T = 64, W = 16384 -- 6.2 against 13.8; at T = 256 the split scans win
// from W = 256 to 65536).
template <class S>
bool channel_parallel_enough(int64_t T, int64_t W, bool vok) {
  static const bool on = linrec_impl::env_int("LINREC_CHANNEL_PARALLEL", 1) != 0;
  const int64_t threads = vok ? W / vec_of<S>() : W;
  return on && ((T <= 2048 && threads >= (int64_t(1) << 17)) || (T <= 32 && threads >= 1024) ||
                (T <= 128 && threads >= 4096));
}

// dx = dh * gate (the unfused gated adjoint)
template <class S>
__global__ void k_mul_rows(const S* __restrict__ a, const S* __restrict__ b, S* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] * b[i];
}
template <class S>
cudaError_t launch_mul(const S* a, const S* b, S* out, int64_t n, cudaStream_t st) {
  const int64_t blocks = (n + 255) / 256;
  k_mul_rows<S><<<(unsigned)(blocks < 8192 ? blocks : 8192), 256, 0, st>>>(a, b, out, n);
  return cudaGetLastError();
}

// The fused gated backward (k_tma_bwd<..., GATED>) exists for the default
// fp32 TMA configuration of the chained scan; other shapes / paths run
// dx = dh * gate first.
template <class S>
bool gated_fused_ok(int64_t T, int64_t W, int mode, bool vok) {
  if (sizeof(S) != 4 || mode == LINREC_SERIAL || !vok || !tma_allowed(T, W) ||
      channel_parallel_enough<S>(T, W, vok) || linrec_impl::cluster_scan_ok<S>(T, W, vok) ||
      linrec_impl::local_scan_ok<S>(T, W, vok))
    return false;
  ChainPlan p;
  return linrec_impl::plan_tma<S>(false, T, W, &p) && p.q == 32 && p.r == 12 && p.stages == 1 && p.nw == 8;
}

template <class S>
int scan_device(const S* lam, const S* x, const S* h0, S* h, int64_t T, int64_t W, int mode,
                linrec_workspace_t ws, cudaStream_t st) {
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_mode(mode)) || (rc = check_ptr(lam, "decays")) ||
      (rc = check_ptr(x, "impulses")) || (rc = check_ptr(h, "h")))
    return rc;
  const bool vok = vec_ok<S>(W, {lam, x, h0, h});
  FwdCall<S> c{lam, x, h0, h, T, W};
  if (mode == LINREC_SERIAL || channel_parallel_enough<S>(T, W, vok)) {
    LINREC_CUDA_TRY(linrec_impl::launch_serial_fwd<S>(c, vok, st));
    return LINREC_OK;
  }
  if (linrec_impl::cluster_scan_ok<S>(T, W, vok)) {  // short sequence, few channels: one cluster per column
    LINREC_CUDA_TRY(linrec_impl::launch_cluster_fwd<S>(c, st));
    return LINREC_OK;
  }
  if (linrec_impl::local_scan_ok<S>(T, W, vok)) {  // short sequence: one CTA per channel vector
    LINREC_CUDA_TRY(linrec_impl::launch_local_fwd<S>(c, vok, st));
    return LINREC_OK;
  }
  int dev;
  if ((rc = check_rows(T)) || (rc = current_device(&dev))) return rc;
  linrec_workspace* w = ws ? ws : default_ws(dev, st);
  std::lock_guard<std::mutex> lk(w->mu);
  ChainPlan p;
  const bool tma = vok && tma_allowed(T, W) && linrec_impl::plan_tma<S>(true, T, W, &p);
  if (!tma) p = linrec_impl::plan_chain<S>(true, T, W, vok);
  if (p.ntiles > 0x7fffffffLL) return fail(LINREC_ERR_SHAPE, "linrec: problem too large for one launch");
  if ((rc = ws_reserve(w, p.ws_bytes, st))) return rc;
  VsegPtrs<S> vs{};
  if (p.nseg > 1) {  // independent chains per virtual segment, stitched below
    vs = vseg_ptrs<S>(w, p, W);
    c.seg_prod = vs.seg_prod;
    c.agg_out = vs.vagg;
  }
  const bool adapt = tma && sizeof(S) == 4 && p.nseg > 1 && adaptive_stitch_on();
  const bool twin = adapt && p.ncols >= unsplit_cols();
  const int* dmode = adapt ? decay_mode_ptr(w) : nullptr;
  if (adapt) {
    LINREC_CUDA_TRY(linrec_impl::launch_decay_probe<float>(reinterpret_cast<const float*>(lam), T, W, p.cpw, p.tseg,
                                                           kDeepFracFwd, w->base, st));
    c.mode = dmode;
    if (twin) {  // deep: the unsplit twin below scans instead of the split scan
      c.role = 3;
    } else {  // deep: reduce pass + segment carries; the split scan seeds from them
      FwdCall<S> r = c;
      r.h = nullptr;
      r.seg_prod = nullptr;
      r.role = 1;
      LINREC_CUDA_TRY(linrec_impl::launch_tma_fwd<S>(p, r, ws_ptrs(w, p), st));
      LINREC_CUDA_TRY(linrec_impl::launch_vseg_finalize<S>(false, lam, vs.vagg, p.nseg, p.tseg, vs.carry, nullptr,
                                                           nullptr, nullptr, W, st, nullptr, dmode));
      c.seed_rows = vs.carry;
    }
  }
  if (tma) LINREC_CUDA_TRY(linrec_impl::launch_tma_fwd<S>(p, c, ws_ptrs(w, p), st));
  else LINREC_CUDA_TRY(linrec_impl::launch_chain_fwd<S>(p, c, ws_ptrs(w, p), st));
  if (twin) {
    const ChainPlan u = unsplit_plan(p, T);
    FwdCall<S> t{lam, x, h0, h, T, W};
    t.mode = dmode;
    t.role = 2;
    LINREC_CUDA_TRY(linrec_impl::launch_tma_fwd<S>(u, t, ws_ptrs(w, u), st));
  }
  if (p.nseg > 1)  // one stitch launch: each fix-up CTA folds its own segment's carry from vagg
    LINREC_CUDA_TRY(linrec_impl::launch_fixup<S>(false, lam, nullptr, nullptr, nullptr, vs.seg_prod, nullptr,
                                                 nullptr, nullptr, h, nullptr, T, W, p.rows, p.nseg, p.tseg, p.ntt,
                                                 vok, st, nullptr, nullptr, vs.vagg, nullptr, dmode));
  return LINREC_OK;
}

template <class S>
int scan_backward_device(const S* lam, const S* h0, const S* h, const S* dh, const S* lam_next,
                         const S* g_next, S* dlam, S* dx, S* dh0, int64_t T, int64_t W, int mode,
                         linrec_workspace_t ws, cudaStream_t st, const S* gate = nullptr) {
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_mode(mode)) || (rc = check_ptr(lam, "decays")) ||
      (rc = check_ptr(h, "h")) || (rc = check_ptr(dh, "d_h")) ||
      (rc = check_ptr(dx, "d_impulses")))
    return rc;
  const bool vok = vec_ok<S>(W, {lam, h0, h, dh, lam_next, g_next, dlam, dx, dh0, gate});
  if (gate != nullptr && !gated_fused_ok<S>(T, W, mode, vok)) {
    // gated adjoint without the fused kernel: dx = dh * gate, then the scan in
    // place (every kernel reads a row of the adjoint before writing that row)
    LINREC_CUDA_TRY(launch_mul<S>(dh, gate, dx, T * W, st));
    return scan_backward_device<S>(lam, h0, h, dx, lam_next, g_next, dlam, dx, dh0, T, W, mode, ws, st);
  }
  BwdCall<S> c{lam, h0, h, dh, lam_next, g_next, dlam, dx, dh0, T, W};
  c.gate = gate;
  if (mode == LINREC_SERIAL || channel_parallel_enough<S>(T, W, vok)) {
    LINREC_CUDA_TRY(linrec_impl::launch_serial_bwd<S>(c, vok, st));
    return LINREC_OK;
  }
  if (linrec_impl::cluster_scan_ok<S>(T, W, vok)) {
    LINREC_CUDA_TRY(linrec_impl::launch_cluster_bwd<S>(c, st));
    return LINREC_OK;
  }
  if (linrec_impl::local_scan_ok<S>(T, W, vok)) {
    LINREC_CUDA_TRY(linrec_impl::launch_local_bwd<S>(c, vok, st));
    return LINREC_OK;
  }
  int dev;
  if ((rc = check_rows(T)) || (rc = current_device(&dev))) return rc;
  linrec_workspace* w = ws ? ws : default_ws(dev, st);
  std::lock_guard<std::mutex> lk(w->mu);
  ChainPlan p;
  const bool tma = vok && tma_allowed(T, W) && linrec_impl::plan_tma<S>(false, T, W, &p);
  if (!tma) p = linrec_impl::plan_chain<S>(false, T, W, vok);
  if (p.ntiles > 0x7fffffffLL) return fail(LINREC_ERR_SHAPE, "linrec: problem too large for one launch");
  if ((rc = ws_reserve(w, p.ws_bytes, st))) return rc;
  VsegPtrs<S> vs{};
  if (p.nseg > 1) {
    vs = vseg_ptrs<S>(w, p, W);
    c.seg_prod = vs.seg_prod;
    c.agg_out = vs.vagg;
  }
  const bool adapt = tma && sizeof(S) == 4 && p.nseg > 1 && adaptive_stitch_on();
  const bool twin = adapt && p.ncols >= unsplit_cols();
  const int* dmode = adapt ? decay_mode_ptr(w) : nullptr;
  if (adapt) {  // the forward's decay-adaptive stitch in reverse time (see above)
    LINREC_CUDA_TRY(linrec_impl::launch_decay_probe<float>(reinterpret_cast<const float*>(lam), T, W, p.cpw, p.tseg,
                                                           kDeepFracBwd, w->base, st));
    c.mode = dmode;
    if (twin) {
      c.role = 3;
    } else {
      BwdCall<S> r = c;
      r.dlam = nullptr;
      r.dx = nullptr;
      r.dh0 = nullptr;
      r.seg_prod = nullptr;
      r.role = 1;
      LINREC_CUDA_TRY(linrec_impl::launch_tma_bwd<S>(p, r, ws_ptrs(w, p), st));
      LINREC_CUDA_TRY(linrec_impl::launch_vseg_finalize<S>(true, lam, vs.vagg, p.nseg, p.tseg, vs.carry, nullptr,
                                                           nullptr, nullptr, W, st, nullptr, dmode));
      c.seed_rows = vs.carry;
    }
  }
  if (tma) LINREC_CUDA_TRY(linrec_impl::launch_tma_bwd<S>(p, c, ws_ptrs(w, p), st));
  else LINREC_CUDA_TRY(linrec_impl::launch_chain_bwd<S>(p, c, ws_ptrs(w, p), st));
  if (twin) {
    const ChainPlan u = unsplit_plan(p, T);
    BwdCall<S> t{lam, h0, h, dh, lam_next, g_next, dlam, dx, dh0, T, W};
    t.gate = gate;
    t.mode = dmode;
    t.role = 2;
    LINREC_CUDA_TRY(linrec_impl::launch_tma_bwd<S>(u, t, ws_ptrs(w, u), st));
  }
  if (p.nseg > 1)  // dh0 gets its correction from the fix-up that owns row 0
    LINREC_CUDA_TRY(linrec_impl::launch_fixup<S>(true, lam, h0, h, lam_next, vs.seg_prod, nullptr, nullptr,
                                                 nullptr, dx, dlam, T, W, p.rows, p.nseg, p.tseg, p.ntt, vok, st,
                                                 nullptr, nullptr, vs.vagg, dh0, dmode));
  return LINREC_OK;
}

// ---------------------------------------------------------------------------
// host-pointer pipeline
// ---------------------------------------------------------------------------
constexpr int kSlots = 3;
constexpr size_t kChunkBytes = size_t(64) << 20;  // per array per chunk

// Parallel host memcpy for staging pageable numpy buffers through pinned
// bounce buffers: one pageable<->pinned copy per byte, split over worker
// threads (the calling thread takes a share), so the copies and the page
// faults of freshly allocated outputs run at host-memory rather than
// single-core speed while the DMA engines move the previous chunk.
// Host copy for the staging pool: non-temporal (streaming) AVX2 stores for
// large ranges, so a pageable -> pinned copy moves 2 bytes of host DRAM
// traffic per byte (read source, write destination) instead of 3 (a cached
// store first reads the destination line) -- the pageable e2e path is bound
// by host DRAM bandwidth, which the DMA engines share.  LINREC_NT_COPY=0
// falls back to memcpy.
__attribute__((target("avx2"))) void stream_copy_avx2(char* dst, const char* src, size_t n) {
  const size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
  if (head) {
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    n -= head;
  }
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
    const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
  }
  if (i < n) std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}

void stage_copy(char* dst, const char* src, size_t n) {
  static const bool nt = linrec_impl::env_int("LINREC_NT_COPY", 1) != 0 && __builtin_cpu_supports("avx2");
  if (nt && n >= (size_t(1) << 16)) stream_copy_avx2(dst, src, n);
  else std::memcpy(dst, src, n);
}

class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i + 1); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return int(th_.size()) + 1; }
  // dst[k] <- src[k] for every (dst, src, bytes) job, split across the pool.
  void copy(const std::vector<std::tuple<void*, const void*, size_t>>& jobs) {
    size_t total = 0;
    for (auto& j : jobs) total += std::get<2>(j);
    if (total == 0) return;
    const int parts = std::max(1, std::min<int>(size(), int(total >> 20)));  // >= 1 MiB each
    {
      std::unique_lock<std::mutex> lk(mu_);
      jobs_ = &jobs;
      total_ = total;
      parts_ = parts;
      pending_ = parts - 1;  // part 0 runs on the caller
      ++gen_;
    }
    cv_.notify_all();
    run_part(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    jobs_ = nullptr;
  }

 private:
  void run_part(int k) {
    const size_t lo = total_ * size_t(k) / size_t(parts_), hi = total_ * size_t(k + 1) / size_t(parts_);
    size_t off = 0;
    for (auto& j : *jobs_) {
      const size_t n = std::get<2>(j);
      const size_t a = std::max(lo, off), b = std::min(hi, off + n);
      if (a < b)
        stage_copy(static_cast<char*>(std::get<0>(j)) + (a - off), static_cast<const char*>(std::get<1>(j)) + (a - off),
                   b - a);
      off += n;
    }
  }
  void loop(int k) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (k >= parts_) continue;
      }
      run_part(k);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::vector<std::tuple<void*, const void*, size_t>>* jobs_ = nullptr;
  size_t total_ = 0;
  int parts_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct HostPipe {
  int device = -1;
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[kSlots], ev_comp[kSlots], ev_out[kSlots];
  void* buf[kSlots][3] = {};
  size_t buf_bytes = 0;
  void* small = nullptr;  // h0 / dh0 staging, 2 rows
  size_t small_bytes = 0;
  // pageable staging: pinned bounce buffers per slot (3 inputs, 2 outputs)
  void* bounce[kSlots][5] = {};
  size_t bounce_bytes = 0;
  void* small_host = nullptr;  // pinned h0 / dh0 bounce
  std::unique_ptr<CopyPool> pool;
  linrec_workspace ws;
  std::mutex mu;
};

std::mutex g_pipe_mu;
std::map<int, std::unique_ptr<HostPipe>> g_pipes;

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int pipe_for(int device, HostPipe** out) {
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  auto& p = g_pipes[device];
  if (!p) {
    std::unique_ptr<HostPipe> n(new HostPipe());
    n->device = device;
    n->ws.device = device;
    LINREC_CUDA_TRY(cudaStreamCreateWithFlags(&n->s_in, cudaStreamNonBlocking));
    LINREC_CUDA_TRY(cudaStreamCreateWithFlags(&n->s_comp, cudaStreamNonBlocking));
    LINREC_CUDA_TRY(cudaStreamCreateWithFlags(&n->s_out, cudaStreamNonBlocking));
    for (int i = 0; i < kSlots; ++i) {
      LINREC_CUDA_TRY(cudaEventCreateWithFlags(&n->ev_in[i], cudaEventDisableTiming));
      LINREC_CUDA_TRY(cudaEventCreateWithFlags(&n->ev_comp[i], cudaEventDisableTiming));
      LINREC_CUDA_TRY(cudaEventCreateWithFlags(&n->ev_out[i], cudaEventDisableTiming));
    }
    p = std::move(n);
  }
  *out = p.get();
  return LINREC_OK;
}

int pipe_reserve(HostPipe* hp, size_t bytes, size_t small_bytes) {
  if (bytes > hp->buf_bytes) {
    LINREC_CUDA_TRY(cudaDeviceSynchronize());
    for (int i = 0; i < kSlots; ++i)
      for (int j = 0; j < 3; ++j) {
        if (hp->buf[i][j]) LINREC_CUDA_TRY(cudaFree(hp->buf[i][j]));
        hp->buf[i][j] = nullptr;
      }
    hp->buf_bytes = 0;
    for (int i = 0; i < kSlots; ++i)
      for (int j = 0; j < 3; ++j) LINREC_CUDA_TRY(cudaMalloc(&hp->buf[i][j], bytes));
    hp->buf_bytes = bytes;
  }
  if (small_bytes > hp->small_bytes) {
    if (hp->small) LINREC_CUDA_TRY(cudaFree(hp->small));
    hp->small = nullptr;
    LINREC_CUDA_TRY(cudaMalloc(&hp->small, small_bytes));
    hp->small_bytes = small_bytes;
  }
  return LINREC_OK;
}

// Pinned bounce buffers + copy threads for pageable host arrays.
int pipe_reserve_bounce(HostPipe* hp, size_t bytes, size_t small_bytes) {
  if (!hp->pool) {
    const unsigned hw = std::thread::hardware_concurrency();
    hp->pool.reset(new CopyPool(int(std::max(1u, std::min(hw ? hw : 1u, 16u))) - 1));
  }
  if (bytes > hp->bounce_bytes) {
    for (int i = 0; i < kSlots; ++i)
      for (int j = 0; j < 5; ++j) {
        if (hp->bounce[i][j]) LINREC_CUDA_TRY(cudaFreeHost(hp->bounce[i][j]));
        hp->bounce[i][j] = nullptr;
      }
    hp->bounce_bytes = 0;
    for (int i = 0; i < kSlots; ++i)
      for (int j = 0; j < 5; ++j) LINREC_CUDA_TRY(cudaHostAlloc(&hp->bounce[i][j], bytes, cudaHostAllocDefault));
    hp->bounce_bytes = bytes;
  }
  if (!hp->small_host) LINREC_CUDA_TRY(cudaHostAlloc(&hp->small_host, std::max<size_t>(small_bytes, 1 << 20), 0));
  return LINREC_OK;
}

// Page-locked (or device-mapped) host buffers DMA straight from / into the
// caller's memory; pageable ones (ordinary numpy arrays) are staged through
// the pinned bounce buffers.  Decided per array.
bool pageable(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

int64_t chunk_rows(int64_t T, int64_t W, size_t elem) {
  const int64_t rows = (int64_t)(kChunkBytes / (size_t(W) * elem));
  return std::max<int64_t>(1, std::min<int64_t>(T, rows));
}

using CopyJobs = std::vector<std::tuple<void*, const void*, size_t>>;

// Host arrays may be a column block of a wider [T][ld] array (channel
// sharding, linrec_scan_host_columns_*): rows of `width` bytes at a host
// stride of ld_bytes.  Contiguous blocks stay one job / one copy.
void add_rows(CopyJobs& jobs, void* dst, size_t dst_ld, const void* src, size_t src_ld, size_t width, int64_t rows) {
  if (rows <= 0) return;
  if (dst_ld == width && src_ld == width) {
    jobs.emplace_back(dst, src, width * size_t(rows));
    return;
  }
  for (int64_t r = 0; r < rows; ++r)
    jobs.emplace_back(static_cast<char*>(dst) + size_t(r) * dst_ld, static_cast<const char*>(src) + size_t(r) * src_ld,
                      width);
}
cudaError_t copy_rows_async(void* dst, size_t dst_ld, const void* src, size_t src_ld, size_t width, int64_t rows,
                            cudaMemcpyKind kind, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (dst_ld == width && src_ld == width) return cudaMemcpyAsync(dst, src, width * size_t(rows), kind, st);
  return cudaMemcpy2DAsync(dst, dst_ld, src, src_ld, width, size_t(rows), kind, st);
}

// Caching allocator of page-locked host memory (linrec_host_alloc/free): the
// Python module allocates its numpy RESULTS here, so device->host copies land
// straight in the caller's array at full link speed (no bounce, no first-touch
// page faults) and repeated calls of one shape recycle the same blocks.
struct PinnedCache {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;  // rounded size -> block
  std::map<void*, size_t> live;
  size_t cached = 0, cap = 0;
};
PinnedCache& pinned_cache() {
  static PinnedCache* c = [] {
    auto* pc = new PinnedCache();  // leaked on purpose: outlives static destructors that free arrays
    const long pages = sysconf(_SC_PHYS_PAGES), psize = sysconf(_SC_PAGE_SIZE);
    const size_t phys = pages > 0 && psize > 0 ? size_t(pages) * size_t(psize) : (size_t(16) << 30);
    pc->cap = phys / 4;  // keep at most a quarter of RAM pinned while unused
    return pc;
  }();
  return *c;
}

template <class S>
int scan_host(const S* lam, const S* x, const S* h0, S* h, int64_t T, int64_t W, int mode,
              int device, int64_t ld = -1) {
  if (ld < 0) ld = W;  // host row stride (elements): > W for a column block
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_mode(mode)) || (rc = check_ptr(lam, "decays")) ||
      (rc = check_ptr(x, "impulses")) || (rc = check_ptr(h, "h")))
    return rc;
  DeviceGuard dg(device);
  HostPipe* hp;
  if ((rc = pipe_for(device, &hp))) return rc;
  std::lock_guard<std::mutex> lk(hp->mu);
  const int64_t Tc = chunk_rows(T, W, sizeof(S));
  const size_t row = size_t(W) * sizeof(S);
  if ((rc = pipe_reserve(hp, size_t(Tc) * row, 2 * row))) return rc;
  // pageable arrays (numpy) go through pinned bounce buffers; pinned ones DMA directly
  const bool st_l = pageable(lam), st_x = pageable(x), st_h = pageable(h);
  const bool staged = st_l || st_x || st_h || pageable(h0);
  if (staged && (rc = pipe_reserve_bounce(hp, size_t(Tc) * row, 2 * row))) return rc;
  S* d_h0 = nullptr;
  if (h0) {
    d_h0 = static_cast<S*>(hp->small);
    const S* src = h0;
    if (pageable(h0)) {
      std::memcpy(hp->small_host, h0, row);
      src = static_cast<const S*>(hp->small_host);
    }
    LINREC_CUDA_TRY(cudaMemcpyAsync(d_h0, src, row, cudaMemcpyHostToDevice, hp->s_comp));
  }
  const int64_t nchunks = (T + Tc - 1) / Tc;
  const size_t hrow = size_t(ld) * sizeof(S);  // host row stride in bytes
  auto drain = [&](int64_t k) -> int {  // chunk k's h: pinned bounce -> caller
    const int s = int(k % kSlots);
    const int64_t t0 = k * Tc, rows = std::min<int64_t>(Tc, T - t0);
    LINREC_CUDA_TRY(cudaEventSynchronize(hp->ev_out[s]));
    CopyJobs jobs;
    add_rows(jobs, h + t0 * ld, hrow, hp->bounce[s][3], row, row, rows);
    hp->pool->copy(jobs);
    return LINREC_OK;
  };
  const S* seed = d_h0;
  for (int64_t k = 0; k < nchunks; ++k) {
    const int s = int(k % kSlots);
    const int64_t t0 = k * Tc, rows = std::min<int64_t>(Tc, T - t0);
    S* dl = static_cast<S*>(hp->buf[s][0]);
    S* dxv = static_cast<S*>(hp->buf[s][1]);
    S* dhv = static_cast<S*>(hp->buf[s][2]);
    const S* src_l = lam + t0 * ld;
    const S* src_x = x + t0 * ld;
    size_t ld_l = hrow, ld_x = hrow;
    if (st_l || st_x) {  // bounce slot s is free once chunk k - kSlots's H2D finished
      if (k >= kSlots) LINREC_CUDA_TRY(cudaEventSynchronize(hp->ev_in[s]));
      CopyJobs jobs;
      if (st_l) add_rows(jobs, hp->bounce[s][0], row, src_l, hrow, row, rows);
      if (st_x) add_rows(jobs, hp->bounce[s][1], row, src_x, hrow, row, rows);
      hp->pool->copy(jobs);
      if (st_l) { src_l = static_cast<const S*>(hp->bounce[s][0]); ld_l = row; }
      if (st_x) { src_x = static_cast<const S*>(hp->bounce[s][1]); ld_x = row; }
    }
    if (k >= kSlots) LINREC_CUDA_TRY(cudaStreamWaitEvent(hp->s_in, hp->ev_comp[s], 0));
    LINREC_CUDA_TRY(copy_rows_async(dl, row, src_l, ld_l, row, rows, cudaMemcpyHostToDevice, hp->s_in));
    LINREC_CUDA_TRY(copy_rows_async(dxv, row, src_x, ld_x, row, rows, cudaMemcpyHostToDevice, hp->s_in));
    LINREC_CUDA_TRY(cudaEventRecord(hp->ev_in[s], hp->s_in));
    LINREC_CUDA_TRY(cudaStreamWaitEvent(hp->s_comp, hp->ev_in[s], 0));
    if (k >= kSlots) LINREC_CUDA_TRY(cudaStreamWaitEvent(hp->s_comp, hp->ev_out[s], 0));
    if ((rc = scan_device<S>(dl, dxv, seed, dhv, rows, W, mode, &hp->ws, hp->s_comp))) return rc;
    LINREC_CUDA_TRY(cudaEventRecord(hp->ev_comp[s], hp->s_comp));
    LINREC_CUDA_TRY(cudaStreamWaitEvent(hp->s_out, hp->ev_comp[s], 0));
    if (st_h)
      LINREC_CUDA_TRY(copy_rows_async(hp->bounce[s][3], row, dhv, row, row, rows, cudaMemcpyDeviceToHost, hp->s_out));
    else
      LINREC_CUDA_TRY(copy_rows_async(h + t0 * ld, hrow, dhv, row, row, rows, cudaMemcpyDeviceToHost, hp->s_out));
    LINREC_CUDA_TRY(cudaEventRecord(hp->ev_out[s], hp->s_out));
    seed = dhv + (rows - 1) * W;  // carry into the next chunk
    // the previous chunk's result leaves the bounce buffer while this one runs
    if (st_h && k >= 1 && (rc = drain(k - 1))) return rc;
  }
  if (st_h && (rc = drain(nchunks - 1))) return rc;
  LINREC_CUDA_TRY(cudaStreamSynchronize(hp->s_out));
  LINREC_CUDA_TRY(cudaStreamSynchronize(hp->s_comp));
  return LINREC_OK;
}

template <class S>
int scan_backward_host(const S* lam, const S* h0, const S* h, const S* dh, S* dlam, S* dx, S* dh0,
                       int64_t T, int64_t W, int mode, int device, int64_t ld = -1) {
  if (ld < 0) ld = W;  // host row stride (elements): > W for a column block
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_mode(mode)) || (rc = check_ptr(lam, "decays")) ||
      (rc = check_ptr(h, "h")) || (rc = check_ptr(dh, "d_h")) || (rc = check_ptr(dlam, "d_decays")) ||
      (rc = check_ptr(dx, "d_impulses")) || (rc = check_ptr(dh0, "d_initial")))
    return rc;
  DeviceGuard dg(device);
  HostPipe* hp;
  if ((rc = pipe_for(device, &hp))) return rc;
  std::lock_guard<std::mutex> lk(hp->mu);
  const int64_t Tc = chunk_rows(T, W, sizeof(S));
  const size_t row = size_t(W) * sizeof(S);
  // per slot: buf0 = [lam | dlam], buf1 = [h shifted by one row | dx],
  // buf2 = [dh]; each half holds Tc rows.
  if ((rc = pipe_reserve(hp, size_t(2) * size_t(Tc) * row, 3 * row))) return rc;
  const bool st_l = pageable(lam), st_h = pageable(h), st_dh = pageable(dh);
  const bool st_dl = pageable(dlam), st_dx = pageable(dx), st_h0 = pageable(h0), st_d0 = pageable(dh0);
  const bool staged = st_l || st_h || st_dh || st_dl || st_dx || st_h0 || st_d0;
  if (staged && (rc = pipe_reserve_bounce(hp, size_t(Tc) * row, 3 * row))) return rc;
  S* d_h0 = static_cast<S*>(hp->small);
  S* d_dh0 = d_h0 + W;
  S* h_dh0 = st_d0 ? static_cast<S*>(hp->small_host) + W : dh0;  // where dh0 lands on the host
  if (h0) {
    const S* src = h0;
    if (st_h0) {
      std::memcpy(hp->small_host, h0, row);
      src = static_cast<const S*>(hp->small_host);
    }
    LINREC_CUDA_TRY(cudaMemcpyAsync(d_h0, src, row, cudaMemcpyHostToDevice, hp->s_comp));
  } else {
    LINREC_CUDA_TRY(cudaMemsetAsync(d_h0, 0, row, hp->s_comp));
  }
  const int64_t nchunks = (T + Tc - 1) / Tc;
  const size_t hrow = size_t(ld) * sizeof(S);  // host row stride in bytes
  auto drain = [&](int64_t i) -> int {  // chunk i's dlam, dx: pinned bounce -> caller
    const int s = int(i % kSlots);
    const int64_t k = nchunks - 1 - i;
    const int64_t t0 = k * Tc, rows = std::min<int64_t>(Tc, T - t0);
    LINREC_CUDA_TRY(cudaEventSynchronize(hp->ev_out[s]));
    CopyJobs jobs;
    if (st_dl) add_rows(jobs, dlam + t0 * ld, hrow, hp->bounce[s][3], row, row, rows);
    if (st_dx) add_rows(jobs, dx + t0 * ld, hrow, hp->bounce[s][4], row, row, rows);
    hp->pool->copy(jobs);
    return LINREC_OK;
  };
  const bool drains = st_dl || st_dx;
  const S* lam_next = nullptr;
  const S* g_next = nullptr;
  for (int64_t i = 0; i < nchunks; ++i) {
    const int64_t k = nchunks - 1 - i;  // reverse time
    const int s = int(i % kSlots);
    const int64_t t0 = k * Tc, rows = std::min<int64_t>(Tc, T - t0);
    S* b0 = static_cast<S*>(hp->buf[s][0]);
    S* b1 = static_cast<S*>(hp->buf[s][1]);
    S* b2 = static_cast<S*>(hp->buf[s][2]);
    S* d_lam = b0;
    S* d_dlam = b0 + Tc * W;
    S* d_h = b1;  // rows t0-1 .. t0+rows-2 (or 0 .. rows-2 for t0 == 0)
    S* d_dx = b1 + Tc * W;
    S* d_dh = b2;
    // host sources of this chunk: lam and dh rows, and h shifted by one row
    const S* src_l = lam + t0 * ld;
    const S* src_dh = dh + t0 * ld;
    const S* src_h = t0 > 0 ? h + (t0 - 1) * ld : h;
    const int64_t h_rows = t0 > 0 ? rows : rows - 1;
    size_t ld_l = hrow, ld_h = hrow, ld_dh = hrow;
    if (st_l || st_h || st_dh) {
      if (i >= kSlots) LINREC_CUDA_TRY(cudaEventSynchronize(hp->ev_in[s]));
      CopyJobs jobs;
      if (st_l) add_rows(jobs, hp->bounce[s][0], row, src_l, hrow, row, rows);
      if (st_h) add_rows(jobs, hp->bounce[s][1], row, src_h, hrow, row, h_rows);
      if (st_dh) add_rows(jobs, hp->bounce[s][2], row, src_dh, hrow, row, rows);
      hp->pool->copy(jobs);
      if (st_l) { src_l = static_cast<const S*>(hp->bounce[s][0]); ld_l = row; }
      if (st_h) { src_h = static_cast<const S*>(hp->bounce[s][1]); ld_h = row; }
      if (st_dh) { src_dh = static_cast<const S*>(hp->bounce[s][2]); ld_dh = row; }
    }
    // slot s was last filled at chunk i-3, whose lam row 0 and G row 0 are
    // also read by chunk i-2 (lam_next / g_next): wait for that compute.
    if (i >= kSlots)
      LINREC_CUDA_TRY(cudaStreamWaitEvent(hp->s_in, hp->ev_comp[(i - 2) % kSlots], 0));
    LINREC_CUDA_TRY(copy_rows_async(d_lam, row, src_l, ld_l, row, rows, cudaMemcpyHostToDevice, hp->s_in));
    LINREC_CUDA_TRY(copy_rows_async(d_dh, row, src_dh, ld_dh, row, rows, cudaMemcpyHostToDevice, hp->s_in));
    const S* hprev_row;
    const S* hrows;
    LINREC_CUDA_TRY(copy_rows_async(d_h, row, src_h, ld_h, row, h_rows, cudaMemcpyHostToDevice, hp->s_in));
    if (t0 > 0) {
      hprev_row = d_h;
      hrows = d_h + W;
    } else {
      hprev_row = d_h0;
      hrows = d_h;
    }
    LINREC_CUDA_TRY(cudaEventRecord(hp->ev_in[s], hp->s_in));
    LINREC_CUDA_TRY(cudaStreamWaitEvent(hp->s_comp, hp->ev_in[s], 0));
    if (i >= kSlots) LINREC_CUDA_TRY(cudaStreamWaitEvent(hp->s_comp, hp->ev_out[s], 0));
    if ((rc = scan_backward_device<S>(d_lam, hprev_row, hrows, d_dh, lam_next, g_next, d_dlam, d_dx,
                                      k == 0 ? d_dh0 : nullptr, rows, W, mode, &hp->ws, hp->s_comp)))
      return rc;
    LINREC_CUDA_TRY(cudaEventRecord(hp->ev_comp[s], hp->s_comp));
    LINREC_CUDA_TRY(cudaStreamWaitEvent(hp->s_out, hp->ev_comp[s], 0));
    if (st_dl)
      LINREC_CUDA_TRY(copy_rows_async(hp->bounce[s][3], row, d_dlam, row, row, rows, cudaMemcpyDeviceToHost, hp->s_out));
    else
      LINREC_CUDA_TRY(copy_rows_async(dlam + t0 * ld, hrow, d_dlam, row, row, rows, cudaMemcpyDeviceToHost, hp->s_out));
    if (st_dx)
      LINREC_CUDA_TRY(copy_rows_async(hp->bounce[s][4], row, d_dx, row, row, rows, cudaMemcpyDeviceToHost, hp->s_out));
    else
      LINREC_CUDA_TRY(copy_rows_async(dx + t0 * ld, hrow, d_dx, row, row, rows, cudaMemcpyDeviceToHost, hp->s_out));
    if (k == 0) LINREC_CUDA_TRY(cudaMemcpyAsync(h_dh0, d_dh0, row, cudaMemcpyDeviceToHost, hp->s_out));
    LINREC_CUDA_TRY(cudaEventRecord(hp->ev_out[s], hp->s_out));
    lam_next = d_lam;  // lam at row t0 and G at row t0 feed the previous chunk
    g_next = d_dx;
    if (drains && i >= 1 && (rc = drain(i - 1))) return rc;
  }
  if (drains && (rc = drain(nchunks - 1))) return rc;
  LINREC_CUDA_TRY(cudaStreamSynchronize(hp->s_out));
  LINREC_CUDA_TRY(cudaStreamSynchronize(hp->s_comp));
  if (st_d0) std::memcpy(dh0, h_dh0, row);
  return LINREC_OK;
}

// ---------------------------------------------------------------------------
// sequence sharding (segment.cu): deterministic plan per (T, W, dtype, dir)
// ---------------------------------------------------------------------------
template <class S>
ChainPlan plan_segment(bool forward, int64_t T, int64_t W) {
  ChainPlan p;
  const bool v = W % vec_of<S>() == 0;
  if (!(v && tma_allowed(T, W) && linrec_impl::plan_tma<S>(forward, T, W, &p)))
    p = linrec_impl::plan_chain<S>(forward, T, W, v);
  return p;
}

// seg_prod layout: [nseg*ntt] position rows, then the virtual segments'
// aggregates [nseg][2][W] (vagg: the fix-up folds every segment's carry and
// scale from them, so they travel with seg_prod from the scan to the fix-up)
template <class P>
P seg_vagg_rows(P seg_prod, const ChainPlan& p, int64_t W) {
  return seg_prod + p.nseg * p.ntt * W;
}

// linrec_exchange_t -> the internal descriptor of one direction (p2p_impl.cuh)
int to_exchange(const linrec_exchange_t* e, int64_t W, int dir, bool publish, bool compose,
                linrec_impl::Exchange* out) {
  if (!e || !e->mboxes || e->world < 1 || e->rank < 0 || e->rank >= e->world || e->epoch < 1)
    return fail(LINREC_ERR_VALUE, "exchange: mboxes, world, rank and epoch >= 1 required");
  const int f = e->sources_first, l = e->sources_last, s = e->sources_step;
  if (e->consumers_first < 0 || e->consumers_last > e->world || (s != 1 && s != -1) ||
      (f != l && (s == 1 ? f > l : f < l)) || l < -1 || l > e->world)
    return fail(LINREC_ERR_VALUE, "exchange: consumer / source ranges out of [0, world) or step not +-1");
  for (int q = e->sources_first; q != e->sources_last; q += e->sources_step)
    if (q < 0 || q >= e->world || q == e->rank)
      return fail(LINREC_ERR_VALUE, "exchange: sources must be other ranks in [0, world)");
  linrec_impl::Exchange x;
  x.mboxes = e->mboxes;
  x.W = W;
  x.world = e->world;
  x.rank = e->rank;
  x.dir = dir;
  x.epoch = (unsigned long long)e->epoch;
  if (publish) {
    x.q0 = e->consumers_first;
    x.q1 = e->consumers_last;
    x.zero_a = e->zero_a;
  }
  if (compose) {
    x.first = e->sources_first;
    x.last = e->sources_last;
    x.step = e->sources_step;
  }
  *out = x;
  return LINREC_OK;
}

// The rank aggregate is folded in the TMA scan's tail (one CTA, 128-channel
// float4 blocks) for W <= 256 fp32; wider or register-kernel plans keep the
// fold kernel.  LINREC_TAIL_FOLD=0 forces the kernel (comparison runs).
template <class S>
bool tail_fold_ok(const ChainPlan& p, int64_t W) {
  static const bool on = linrec_impl::env_int("LINREC_TAIL_FOLD", 1) != 0;
  return on && sizeof(S) == 4 && p.kind == 1 && W <= 256 && W % 4 == 0;
}

template <class S>
int segment_scan(const S* lam, const S* x, const S* h0, S* h, S* seg_prod, S* agg, int64_t T, int64_t W,
                 linrec_workspace_t ws, cudaStream_t st, const linrec_impl::Exchange* ex = nullptr) {
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_ptr(lam, "decays")) || (rc = check_ptr(x, "impulses")) ||
      (rc = check_ptr(h, "h")) || (rc = check_ptr(seg_prod, "seg_prod")) || (rc = check_ptr(agg, "agg")))
    return rc;
  if ((rc = check_rows(T))) return rc;
  const ChainPlan p = plan_segment<S>(true, T, W);
  if (p.vec > 1 && !vec_ok<S>(W, {lam, x, h0, h, seg_prod, agg}))
    return fail(LINREC_ERR_VALUE, "segment scans need 16-byte aligned buffers");
  int dev;
  if ((rc = current_device(&dev))) return rc;
  linrec_workspace* w = ws ? ws : default_ws(dev, st);
  std::lock_guard<std::mutex> lk(w->mu);
  if ((rc = ws_reserve(w, p.ws_bytes, st))) return rc;
  FwdCall<S> c{lam, x, h0, h, T, W, seg_prod, seg_vagg_rows(seg_prod, p, W)};
  const bool tail = tail_fold_ok<S>(p, W);
  if (tail) {  // the scan's last CTA folds (and publishes) the rank aggregate
    c.rank_agg = agg;
    if (ex) c.ex = *ex;
  }
  if (p.kind == 1) LINREC_CUDA_TRY(linrec_impl::launch_tma_fwd<S>(p, c, ws_ptrs(w, p), st));
  else LINREC_CUDA_TRY(linrec_impl::launch_chain_fwd<S>(p, c, ws_ptrs(w, p), st));
  // otherwise a fold kernel makes the segment-level aggregate for the exchange
  // (with a peer exchange also stored straight into the consumers'
  // mailboxes); the fix-up folds the virtual segments' carries itself
  if (!tail)
    LINREC_CUDA_TRY(linrec_impl::launch_vseg_finalize<S>(false, lam, c.agg_out, p.nseg, p.tseg, nullptr, nullptr,
                                                         agg, nullptr, W, st, ex));
  return LINREC_OK;
}

template <class S>
int segment_scan_backward(const S* lam, const S* hprev, const S* h, const S* dh, const S* lam_next, S* dlam,
                          S* dx, S* dh0, S* seg_prod, S* agg, int64_t T, int64_t W, linrec_workspace_t ws,
                          cudaStream_t st, const linrec_impl::Exchange* ex = nullptr) {
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_ptr(lam, "decays")) || (rc = check_ptr(h, "h")) ||
      (rc = check_ptr(dh, "d_h")) || (rc = check_ptr(dlam, "d_decays")) || (rc = check_ptr(dx, "d_impulses")) ||
      (rc = check_ptr(dh0, "d_initial")) || (rc = check_ptr(seg_prod, "seg_prod")) || (rc = check_ptr(agg, "agg")))
    return rc;
  if ((rc = check_rows(T))) return rc;
  const ChainPlan p = plan_segment<S>(false, T, W);
  if (p.vec > 1 && !vec_ok<S>(W, {lam, hprev, h, dh, lam_next, dlam, dx, dh0, seg_prod, agg}))
    return fail(LINREC_ERR_VALUE, "segment scans need 16-byte aligned buffers");
  int dev;
  if ((rc = current_device(&dev))) return rc;
  linrec_workspace* w = ws ? ws : default_ws(dev, st);
  std::lock_guard<std::mutex> lk(w->mu);
  if ((rc = ws_reserve(w, p.ws_bytes, st))) return rc;
  BwdCall<S> c{lam, hprev, h, dh, lam_next, nullptr, dlam, dx, dh0, T, W, seg_prod, seg_vagg_rows(seg_prod, p, W)};
  const bool tail = tail_fold_ok<S>(p, W);
  if (tail) {
    c.rank_agg = agg;
    if (ex) c.ex = *ex;
  }
  if (p.kind == 1) LINREC_CUDA_TRY(linrec_impl::launch_tma_bwd<S>(p, c, ws_ptrs(w, p), st));
  else LINREC_CUDA_TRY(linrec_impl::launch_chain_bwd<S>(p, c, ws_ptrs(w, p), st));
  // (A', B') of the segment for the exchange, dh0 = lam_S * G_S, fix-up
  if (!tail)
    LINREC_CUDA_TRY(linrec_impl::launch_vseg_finalize<S>(true, lam, c.agg_out, p.nseg, p.tseg, nullptr, nullptr, agg,
                                                         dh0, W, st, ex));
  return LINREC_OK;
}

template <class S>
int segment_fixup(bool reverse, const S* lam, const S* hprev, const S* h, const S* lam_next, const S* seg_prod,
                  const S* carry, S* out0, S* out1, int64_t T, int64_t W, int64_t rows, cudaStream_t st,
                  const linrec_impl::Exchange* ex = nullptr, S* c_out = nullptr) {
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_ptr(lam, "decays")) || (rc = check_ptr(seg_prod, "seg_prod")) ||
      (rc = check_ptr(out0, "out")))
    return rc;  // carry may be NULL: the first rank (forward) / the last (backward)
  if (reverse && ((rc = check_ptr(h, "h")) || (rc = check_ptr(out1, "d_decays")))) return rc;
  if (rows < 1) return fail(LINREC_ERR_VALUE, "tile_rows must be >= 1");
  const bool v = vec_ok<S>(W, {lam, hprev, h, lam_next, seg_prod, carry, out0, out1});
  // the same (nseg, ntt) decomposition the segment scan used
  const ChainPlan p = plan_segment<S>(!reverse, T, W);
  if (p.rows != rows) return fail(LINREC_ERR_VALUE, "tile_rows does not match the segment scan's plan");
  LINREC_CUDA_TRY(linrec_impl::launch_fixup<S>(reverse, lam, hprev, h, lam_next, seg_prod, nullptr, nullptr, carry,
                                               out0, out1, T, W, rows, p.nseg, p.tseg, p.ntt, v, st, ex, c_out,
                                               seg_vagg_rows(seg_prod, p, W)));
  return LINREC_OK;
}

// ChunkPlan checks of validate_plan (recurrence.hpp:84-94), same messages
// (contract violations: LINREC_ERR_SHAPE, like a shape mismatch).
int check_plan(const int64_t* bounds, int64_t p, int64_t T) {
  if (!bounds || p < 1) return fail(LINREC_ERR_SHAPE, "ChunkPlan: no chunks");
  if (bounds[0] != 1) return fail(LINREC_ERR_SHAPE, "ChunkPlan: first chunk must start at step 1");
  if (bounds[2 * p - 1] != T) return fail(LINREC_ERR_SHAPE, "ChunkPlan: last chunk must end at step T");
  for (int64_t i = 0; i < p; ++i) {
    if (bounds[2 * i] > bounds[2 * i + 1]) return fail(LINREC_ERR_SHAPE, "ChunkPlan: chunk start exceeds end");
    if (i + 1 < p && bounds[2 * i + 1] + 1 != bounds[2 * i + 2])
      return fail(LINREC_ERR_SHAPE, "ChunkPlan: chunks must be contiguous");
  }
  return LINREC_OK;
}

// Stream-ordered scratch for the plan scans: the bounds on the device and
// the summaries the caller did not ask for.
template <class S>
int plan_scan(bool reverse, const S* lam, const S* x_or_dh, const S* h0, const S* h, S* out, S* dlam, S* dh0,
              int64_t T, int64_t W, const int64_t* bounds, int64_t p, S* P, S* R, S* C, cudaStream_t st) {
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_plan(bounds, p, T))) return rc;
  const size_t bb = sizeof(int64_t) * 2 * (size_t)p, sb = sizeof(S) * (size_t)(p * W);
  char* tmp = nullptr;
  const size_t need = bb + (P ? 0 : sb) + (R ? 0 : sb) + (C ? 0 : sb) + 64;
  LINREC_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tmp), need, st));
  int64_t* bd = reinterpret_cast<int64_t*>(tmp);
  char* q = tmp + (bb + 15) / 16 * 16;
  if (!P) { P = reinterpret_cast<S*>(q); q += sb; }
  if (!R) { R = reinterpret_cast<S*>(q); q += sb; }
  if (!C) { C = reinterpret_cast<S*>(q); q += sb; }
  cudaError_t e = cudaMemcpyAsync(bd, bounds, bb, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = linrec_impl::launch_plan_scan<S>(reverse, lam, x_or_dh, h0, h, out, dlam, dh0, T, W, bd, p, P, R, C, st);
  const cudaError_t ef = cudaFreeAsync(tmp, st);
  LINREC_CUDA_TRY(e);
  LINREC_CUDA_TRY(ef);
  return LINREC_OK;
}

template <class S>
int first_nonfinite(const S* v, int64_t n, int64_t* index, cudaStream_t st) {
  int rc;
  if ((rc = check_ptr(index, "index"))) return rc;
  if (n > 0 && (rc = check_ptr(v, "v"))) return rc;
  LINREC_CUDA_TRY(linrec_impl::first_nonfinite<S>(v, n, index, st));
  return LINREC_OK;
}
// screen_finite (recurrence.hpp:133-155): the first non-finite element of a
// [T][batch][features] tensor (T == 0: a [batch][features] one), reported
// with the reference's message -- steps 1-based, batch / feature 0-based.
template <class S>
int screen_finite(const S* v, int64_t T, int64_t batch, int64_t features, const char* name, cudaStream_t st) {
  int rc;
  if (batch < 1 || features < 1 || T < 0) return fail(LINREC_ERR_SHAPE, "Tensor3 dimensions must be >= 1");
  if ((rc = check_ptr(v, "v"))) return rc;
  const int64_t W = batch * features;
  int64_t bad = -1;
  LINREC_CUDA_TRY(linrec_impl::first_nonfinite<S>(v, (T > 0 ? T : 1) * W, &bad, st));
  if (bad < 0) return LINREC_OK;
  std::ostringstream os;
  os << "non-finite value in " << (name ? name : "tensor") << " at [";
  if (T > 0) os << "t=" << bad / W + 1 << ", ";
  const int64_t rest = bad % W;
  os << "b=" << rest / features << ", n=" << rest % features << "]";
  return fail(LINREC_ERR_NONFINITE, os.str());
}
}  // namespace

// ---------------------------------------------------------------------------
// exported symbols
// ---------------------------------------------------------------------------
namespace {
// ---- channel sharding of host arrays -------------------------
// Columns [c0, c1) of host [T][W] arrays: staged with strided (2-D) copies,
// scanned on one device as a contiguous [T][c1-c0] block, written back into
// the same columns.  Channels are independent (recurrence.hpp:109), so the
// block's results are exactly the full scan's columns.
int check_columns(int64_t W, int64_t c0, int64_t c1) {
  if (c0 < 0 || c1 > W || c0 >= c1) return fail(LINREC_ERR_VALUE, "columns: need 0 <= c0 < c1 <= W");
  return LINREC_OK;
}

template <class S>
int scan_host_columns(const S* lam, const S* x, const S* h0, S* h, int64_t T, int64_t W, int64_t c0, int64_t c1,
                      int mode, int device) {
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_columns(W, c0, c1)) || (rc = check_ptr(lam, "decays")) ||
      (rc = check_ptr(x, "impulses")) || (rc = check_ptr(h, "h")))
    return rc;
  return scan_host<S>(lam + c0, x + c0, h0 ? h0 + c0 : nullptr, h + c0, T, c1 - c0, mode, device, W);
}

template <class S>
int scan_backward_host_columns(const S* lam, const S* h0, const S* h, const S* dh, S* dlam, S* dx, S* dh0,
                               int64_t T, int64_t W, int64_t c0, int64_t c1, int mode, int device) {
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_columns(W, c0, c1)) || (rc = check_ptr(lam, "decays")) ||
      (rc = check_ptr(h, "h")) || (rc = check_ptr(dh, "d_h")) || (rc = check_ptr(dlam, "d_decays")) ||
      (rc = check_ptr(dx, "d_impulses")) || (rc = check_ptr(dh0, "d_initial")))
    return rc;
  return scan_backward_host<S>(lam + c0, h0 ? h0 + c0 : nullptr, h + c0, dh + c0, dlam + c0, dx + c0, dh0 + c0,
                               T, c1 - c0, mode, device, W);
}

// Column block of device d of n: contiguous, sizes in multiples of 4 channels
// where W allows (16-byte rows for the vector kernels), longer blocks first.
void column_block(int64_t W, int n, int d, int64_t* c0, int64_t* c1) {
  const int64_t unit = W % 4 == 0 ? 4 : 1, units = W / unit;
  const int64_t base = units / n, rem = units % n;
  *c0 = unit * (d * base + std::min<int64_t>(d, rem));
  *c1 = *c0 + unit * (base + (d < rem ? 1 : 0));
}

// One host thread per device, each running the host pipeline on its column
// block (its own streams, bounce buffers and copy threads); the first error
// (code and message) is returned on the calling thread.
template <class F>
int run_on_devices(int64_t W, const int* devices, int ndev, F&& per_device) {
  if (!devices || ndev < 1) return fail(LINREC_ERR_VALUE, "devices: need ndev >= 1 device ids");
  int count = 0;
  LINREC_CUDA_TRY(cudaGetDeviceCount(&count));
  for (int i = 0; i < ndev; ++i)
    if (devices[i] < 0 || devices[i] >= count) return fail(LINREC_ERR_VALUE, "devices: id out of range");
  const int n = int(std::min<int64_t>(ndev, W));
  std::vector<int> rcs(n, LINREC_OK);
  std::vector<std::string> msgs(n);
  std::vector<std::thread> th;
  for (int d = 0; d < n; ++d)
    th.emplace_back([&, d] {
      int64_t c0, c1;
      column_block(W, n, d, &c0, &c1);
      if (c0 < c1) rcs[d] = per_device(devices[d], c0, c1);
      if (rcs[d] != LINREC_OK) msgs[d] = g_last_error;
    });
  for (auto& t : th) t.join();
  for (int d = 0; d < n; ++d)
    if (rcs[d] != LINREC_OK) return fail(rcs[d], msgs[d]);
  return LINREC_OK;
}

template <class S>
int scan_host_multi(const S* lam, const S* x, const S* h0, S* h, int64_t T, int64_t W, int mode,
                    const int* devices, int ndev) {
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_mode(mode))) return rc;
  return run_on_devices(W, devices, ndev, [&](int dev, int64_t c0, int64_t c1) {
    return scan_host_columns<S>(lam, x, h0, h, T, W, c0, c1, mode, dev);
  });
}

template <class S>
int scan_backward_host_multi(const S* lam, const S* h0, const S* h, const S* dh, S* dlam, S* dx, S* dh0,
                             int64_t T, int64_t W, int mode, const int* devices, int ndev) {
  int rc;
  if ((rc = check_dims(T, W)) || (rc = check_mode(mode))) return rc;
  return run_on_devices(W, devices, ndev, [&](int dev, int64_t c0, int64_t c1) {
    return scan_backward_host_columns<S>(lam, h0, h, dh, dlam, dx, dh0, T, W, c0, c1, mode, dev);
  });
}

}  // namespace

extern "C" {

int linrec_abi_version(void) { return LINREC_ABI_VERSION; }
const char* linrec_last_error(void) { return g_last_error.c_str(); }

int linrec_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int linrec_set_kernel_policy(int policy) {
  if (policy != LINREC_KERNEL_AUTO && policy != LINREC_KERNEL_REGISTER)
    return fail(LINREC_ERR_VALUE, "kernel policy must be LINREC_KERNEL_AUTO or LINREC_KERNEL_REGISTER");
  g_kernel_policy.store(policy);
  return LINREC_OK;
}

int linrec_device_malloc(void** ptr, size_t bytes, int device, void* stream) {
  int rc;
  if ((rc = check_ptr(ptr, "ptr"))) return rc;
  DeviceGuard dg(device);
  LINREC_CUDA_TRY(cudaMallocAsync(ptr, bytes == 0 ? 16 : bytes, static_cast<cudaStream_t>(stream)));
  return LINREC_OK;
}

int linrec_device_free(void* ptr, int device, void* stream) {
  if (!ptr) return LINREC_OK;
  DeviceGuard dg(device);
  LINREC_CUDA_TRY(cudaFreeAsync(ptr, static_cast<cudaStream_t>(stream)));
  return LINREC_OK;
}

int linrec_workspace_create(linrec_workspace_t* ws, int device) {
  int rc;
  if ((rc = check_ptr(ws, "ws"))) return rc;
  *ws = new linrec_workspace();
  (*ws)->device = device;
  return LINREC_OK;
}

int linrec_workspace_destroy(linrec_workspace_t ws) {
  if (!ws) return LINREC_OK;
  if (ws->base) {
    DeviceGuard dg(ws->device);
    cudaDeviceSynchronize();
    cudaFree(ws->base);
  }
  delete ws;
  return LINREC_OK;
}

size_t linrec_workspace_bytes(int64_t T, int64_t W, int dtype_bytes) {
  if (T < 1 || W < 1) return 0;
  // the register kernels use the smallest tiles, so they bound both kinds
  if (dtype_bytes == 8) {
    const size_t a = linrec_impl::plan_chain<double>(true, T, W, W % 2 == 0).ws_bytes;
    const size_t b = linrec_impl::plan_chain<double>(false, T, W, W % 2 == 0).ws_bytes;
    return std::max(a, b);
  }
  const size_t a = linrec_impl::plan_chain<float>(true, T, W, W % 4 == 0).ws_bytes;
  const size_t b = linrec_impl::plan_chain<float>(false, T, W, W % 4 == 0).ws_bytes;
  return std::max(a, b);
}

int linrec_scan_f32(const float* lam, const float* x, const float* h0, float* h, int64_t T,
                    int64_t W, int mode, linrec_workspace_t ws, void* stream) {
  return scan_device<float>(lam, x, h0, h, T, W, mode, ws, static_cast<cudaStream_t>(stream));
}
int linrec_scan_f64(const double* lam, const double* x, const double* h0, double* h, int64_t T,
                    int64_t W, int mode, linrec_workspace_t ws, void* stream) {
  return scan_device<double>(lam, x, h0, h, T, W, mode, ws, static_cast<cudaStream_t>(stream));
}

int linrec_scan_backward_f32(const float* lam, const float* h0, const float* h, const float* dh,
                             float* dlam, float* dx, float* dh0, int64_t T, int64_t W, int mode,
                             linrec_workspace_t ws, void* stream) {
  int rc;
  if ((rc = check_ptr(dh0, "d_initial"))) return rc;
  return scan_backward_device<float>(lam, h0, h, dh, nullptr, nullptr, dlam, dx, dh0, T, W, mode,
                                     ws, static_cast<cudaStream_t>(stream));
}
int linrec_scan_backward_f64(const double* lam, const double* h0, const double* h,
                             const double* dh, double* dlam, double* dx, double* dh0, int64_t T,
                             int64_t W, int mode, linrec_workspace_t ws, void* stream) {
  int rc;
  if ((rc = check_ptr(dh0, "d_initial"))) return rc;
  return scan_backward_device<double>(lam, h0, h, dh, nullptr, nullptr, dlam, dx, dh0, T, W, mode,
                                      ws, static_cast<cudaStream_t>(stream));
}

int linrec_scan_backward_gated_f32(const float* lam, const float* h0, const float* h, const float* dh,
                                   const float* gate, float* dlam, float* dx, float* dh0, int64_t T, int64_t W,
                                   int mode, linrec_workspace_t ws, void* stream) {
  int rc;
  if ((rc = check_ptr(gate, "gate"))) return rc;
  return scan_backward_device<float>(lam, h0, h, dh, nullptr, nullptr, dlam, dx, dh0, T, W, mode, ws,
                                     static_cast<cudaStream_t>(stream), gate);
}

int linrec_scan_backward_segment_f32(const float* lam, const float* h0, const float* h,
                                     const float* dh, const float* lam_next, const float* g_next,
                                     float* dlam, float* dx, float* dh0, int64_t T, int64_t W,
                                     int mode, linrec_workspace_t ws, void* stream) {
  return scan_backward_device<float>(lam, h0, h, dh, lam_next, g_next, dlam, dx, dh0, T, W, mode,
                                     ws, static_cast<cudaStream_t>(stream));
}
int linrec_scan_backward_segment_f64(const double* lam, const double* h0, const double* h,
                                     const double* dh, const double* lam_next,
                                     const double* g_next, double* dlam, double* dx, double* dh0,
                                     int64_t T, int64_t W, int mode, linrec_workspace_t ws,
                                     void* stream) {
  return scan_backward_device<double>(lam, h0, h, dh, lam_next, g_next, dlam, dx, dh0, T, W, mode,
                                      ws, static_cast<cudaStream_t>(stream));
}

int linrec_scan_host_f32(const float* lam, const float* x, const float* h0, float* h, int64_t T,
                         int64_t W, int mode, int device) {
  return scan_host<float>(lam, x, h0, h, T, W, mode, device);
}
int linrec_scan_host_f64(const double* lam, const double* x, const double* h0, double* h,
                         int64_t T, int64_t W, int mode, int device) {
  return scan_host<double>(lam, x, h0, h, T, W, mode, device);
}
int linrec_scan_backward_host_f32(const float* lam, const float* h0, const float* h,
                                  const float* dh, float* dlam, float* dx, float* dh0, int64_t T,
                                  int64_t W, int mode, int device) {
  return scan_backward_host<float>(lam, h0, h, dh, dlam, dx, dh0, T, W, mode, device);
}
int linrec_scan_backward_host_f64(const double* lam, const double* h0, const double* h,
                                  const double* dh, double* dlam, double* dx, double* dh0,
                                  int64_t T, int64_t W, int mode, int device) {
  return scan_backward_host<double>(lam, h0, h, dh, dlam, dx, dh0, T, W, mode, device);
}

int linrec_scan_host_columns_f32(const float* lam, const float* x, const float* h0, float* h, int64_t T,
                                 int64_t W, int64_t c0, int64_t c1, int mode, int device) {
  return scan_host_columns<float>(lam, x, h0, h, T, W, c0, c1, mode, device);
}
int linrec_scan_host_columns_f64(const double* lam, const double* x, const double* h0, double* h, int64_t T,
                                 int64_t W, int64_t c0, int64_t c1, int mode, int device) {
  return scan_host_columns<double>(lam, x, h0, h, T, W, c0, c1, mode, device);
}
int linrec_scan_backward_host_columns_f32(const float* lam, const float* h0, const float* h, const float* dh,
                                          float* dlam, float* dx, float* dh0, int64_t T, int64_t W, int64_t c0,
                                          int64_t c1, int mode, int device) {
  return scan_backward_host_columns<float>(lam, h0, h, dh, dlam, dx, dh0, T, W, c0, c1, mode, device);
}
int linrec_scan_backward_host_columns_f64(const double* lam, const double* h0, const double* h, const double* dh,
                                          double* dlam, double* dx, double* dh0, int64_t T, int64_t W, int64_t c0,
                                          int64_t c1, int mode, int device) {
  return scan_backward_host_columns<double>(lam, h0, h, dh, dlam, dx, dh0, T, W, c0, c1, mode, device);
}
int linrec_scan_host_multi_f32(const float* lam, const float* x, const float* h0, float* h, int64_t T, int64_t W,
                               int mode, const int* devices, int ndev) {
  return scan_host_multi<float>(lam, x, h0, h, T, W, mode, devices, ndev);
}
int linrec_scan_host_multi_f64(const double* lam, const double* x, const double* h0, double* h, int64_t T,
                               int64_t W, int mode, const int* devices, int ndev) {
  return scan_host_multi<double>(lam, x, h0, h, T, W, mode, devices, ndev);
}
int linrec_scan_backward_host_multi_f32(const float* lam, const float* h0, const float* h, const float* dh,
                                        float* dlam, float* dx, float* dh0, int64_t T, int64_t W, int mode,
                                        const int* devices, int ndev) {
  return scan_backward_host_multi<float>(lam, h0, h, dh, dlam, dx, dh0, T, W, mode, devices, ndev);
}
int linrec_scan_backward_host_multi_f64(const double* lam, const double* h0, const double* h, const double* dh,
                                        double* dlam, double* dx, double* dh0, int64_t T, int64_t W, int mode,
                                        const int* devices, int ndev) {
  return scan_backward_host_multi<double>(lam, h0, h, dh, dlam, dx, dh0, T, W, mode, devices, ndev);
}
int linrec_column_block(int64_t W, int n, int d, int64_t* c0, int64_t* c1) {
  if (n < 1 || d < 0 || d >= n || !c0 || !c1) return fail(LINREC_ERR_VALUE, "column_block: need 0 <= d < n");
  column_block(W, n, d, c0, c1);
  return LINREC_OK;
}

uint64_t linrec_fnv1a64(const void* data, size_t len, uint64_t h) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

int linrec_host_alloc(void** ptr, size_t bytes) {
  if (!ptr) return fail(LINREC_ERR_VALUE, "host_alloc: ptr required");
  *ptr = nullptr;
  const size_t rounded = (std::max<size_t>(bytes, 1) + (size_t(2) << 20) - 1) / (size_t(2) << 20) * (size_t(2) << 20);
  PinnedCache& c = pinned_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.free_blocks.find(rounded);
    if (it != c.free_blocks.end()) {
      *ptr = it->second;
      c.free_blocks.erase(it);
      c.cached -= rounded;
      c.live[*ptr] = rounded;
      return LINREC_OK;
    }
  }
  void* p = nullptr;
  LINREC_CUDA_TRY(cudaHostAlloc(&p, rounded, cudaHostAllocPortable));
  std::lock_guard<std::mutex> lk(c.mu);
  c.live[p] = rounded;
  *ptr = p;
  return LINREC_OK;
}

int linrec_host_free(void* ptr) {
  if (!ptr) return LINREC_OK;
  PinnedCache& c = pinned_cache();
  std::vector<void*> release;
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.live.find(ptr);
    if (it == c.live.end()) return fail(LINREC_ERR_VALUE, "host_free: not a linrec_host_alloc block");
    const size_t n = it->second;
    c.live.erase(it);
    c.free_blocks.emplace(n, ptr);
    c.cached += n;
    while (c.cached > c.cap && !c.free_blocks.empty()) {  // trim the largest idle blocks
      auto big = std::prev(c.free_blocks.end());
      c.cached -= big->first;
      release.push_back(big->second);
      c.free_blocks.erase(big);
    }
  }
  for (void* q : release) LINREC_CUDA_TRY(cudaFreeHost(q));
  return LINREC_OK;
}

int linrec_first_nonfinite_f32(const float* v, int64_t n, int64_t* index, void* stream) {
  return first_nonfinite<float>(v, n, index, static_cast<cudaStream_t>(stream));
}
int linrec_first_nonfinite_f64(const double* v, int64_t n, int64_t* index, void* stream) {
  return first_nonfinite<double>(v, n, index, static_cast<cudaStream_t>(stream));
}

int linrec_screen_finite_f32(const float* v, int64_t T, int64_t batch, int64_t features, const char* name,
                             void* stream) {
  return screen_finite<float>(v, T, batch, features, name, static_cast<cudaStream_t>(stream));
}
int linrec_screen_finite_f64(const double* v, int64_t T, int64_t batch, int64_t features, const char* name,
                             void* stream) {
  return screen_finite<double>(v, T, batch, features, name, static_cast<cudaStream_t>(stream));
}

int64_t linrec_segment_prod_rows(int64_t T, int64_t W, int dtype_bytes, int backward) {
  if (T < 1 || W < 1) return 0;
  const ChainPlan p = dtype_bytes == 8 ? plan_segment<double>(!backward, T, W) : plan_segment<float>(!backward, T, W);
  return p.nseg * (p.ntt + 2);  // position rows, then the virtual segments' aggregates [nseg][2]
}

int64_t linrec_segment_tile_rows(int64_t T, int64_t W, int dtype_bytes, int backward) {
  if (T < 1 || W < 1) return 0;
  return dtype_bytes == 8 ? plan_segment<double>(!backward, T, W).rows : plan_segment<float>(!backward, T, W).rows;
}

int linrec_segment_scan_f32(const float* lam, const float* x, const float* h0, float* h, float* seg_prod,
                            float* agg, int64_t T, int64_t W, linrec_workspace_t ws, void* stream) {
  return segment_scan<float>(lam, x, h0, h, seg_prod, agg, T, W, ws, static_cast<cudaStream_t>(stream));
}
int linrec_segment_scan_f64(const double* lam, const double* x, const double* h0, double* h, double* seg_prod,
                            double* agg, int64_t T, int64_t W, linrec_workspace_t ws, void* stream) {
  return segment_scan<double>(lam, x, h0, h, seg_prod, agg, T, W, ws, static_cast<cudaStream_t>(stream));
}
int linrec_segment_scan_backward_f32(const float* lam, const float* hprev, const float* h, const float* dh,
                                     const float* lam_next, float* dlam, float* dx, float* dh0,
                                     float* seg_prod, float* agg, int64_t T, int64_t W, linrec_workspace_t ws,
                                     void* stream) {
  return segment_scan_backward<float>(lam, hprev, h, dh, lam_next, dlam, dx, dh0, seg_prod, agg, T, W, ws,
                                      static_cast<cudaStream_t>(stream));
}
int linrec_segment_scan_backward_f64(const double* lam, const double* hprev, const double* h, const double* dh,
                                     const double* lam_next, double* dlam, double* dx, double* dh0,
                                     double* seg_prod, double* agg, int64_t T, int64_t W,
                                     linrec_workspace_t ws, void* stream) {
  return segment_scan_backward<double>(lam, hprev, h, dh, lam_next, dlam, dx, dh0, seg_prod, agg, T, W, ws,
                                       static_cast<cudaStream_t>(stream));
}
int linrec_segment_fixup_f32(const float* lam, float* h, const float* seg_prod, const float* c_in, int64_t T,
                             int64_t W, int64_t tile_rows, void* stream) {
  return segment_fixup<float>(false, lam, nullptr, nullptr, nullptr, seg_prod, c_in, h, nullptr, T, W, tile_rows,
                              static_cast<cudaStream_t>(stream));
}
int linrec_segment_fixup_f64(const double* lam, double* h, const double* seg_prod, const double* c_in,
                             int64_t T, int64_t W, int64_t tile_rows, void* stream) {
  return segment_fixup<double>(false, lam, nullptr, nullptr, nullptr, seg_prod, c_in, h, nullptr, T, W, tile_rows,
                               static_cast<cudaStream_t>(stream));
}
int linrec_segment_fixup_backward_f32(const float* lam, const float* hprev, const float* h, const float* lam_next,
                                      const float* seg_prod, const float* y_in, float* dlam, float* dx, int64_t T,
                                      int64_t W, int64_t tile_rows, void* stream) {
  return segment_fixup<float>(true, lam, hprev, h, lam_next, seg_prod, y_in, dx, dlam, T, W, tile_rows,
                              static_cast<cudaStream_t>(stream));
}
int linrec_segment_fixup_backward_f64(const double* lam, const double* hprev, const double* h,
                                      const double* lam_next, const double* seg_prod, const double* y_in,
                                      double* dlam, double* dx, int64_t T, int64_t W, int64_t tile_rows,
                                      void* stream) {
  return segment_fixup<double>(true, lam, hprev, h, lam_next, seg_prod, y_in, dx, dlam, T, W, tile_rows,
                               static_cast<cudaStream_t>(stream));
}

int linrec_scan_kernel_count(int64_t T, int64_t W, int dtype_bytes, int backward, int mode) {
  if (T < 1 || W < 1 || (dtype_bytes != 4 && dtype_bytes != 8)) return -1;
  const bool f64 = dtype_bytes == 8;
  const bool vok = W % (f64 ? vec_of<double>() : vec_of<float>()) == 0;  // aligned buffers assumed
  if (mode == LINREC_SERIAL ||
      (f64 ? channel_parallel_enough<double>(T, W, vok) : channel_parallel_enough<float>(T, W, vok)) ||
      (f64 ? linrec_impl::local_scan_ok<double>(T, W, vok) : linrec_impl::local_scan_ok<float>(T, W, vok)) ||
      (!f64 && linrec_impl::cluster_scan_ok<float>(T, W, vok)))
    return 1;
  ChainPlan p;
  const bool fwd = backward == 0;
  const bool tma = vok && tma_allowed(T, W) &&
                   (f64 ? linrec_impl::plan_tma<double>(fwd, T, W, &p) : linrec_impl::plan_tma<float>(fwd, T, W, &p));
  if (!tma) p = f64 ? linrec_impl::plan_chain<double>(fwd, T, W, vok) : linrec_impl::plan_chain<float>(fwd, T, W, vok);
  if (p.nseg <= 1) return 1;
  // the scan and the fix-up that stitches the virtual segments; with the
  // decay-adaptive stitch also the probe and either the reduce pass and the
  // carry fold or, on wide scans, the unsplit twin (launched always, the
  // unused ones exit at once)
  if (tma && !f64 && adaptive_stitch_on()) return p.ncols >= unsplit_cols() ? 4 : 5;
  return 2;
}

const char* linrec_scan_kernel_name(int64_t T, int64_t W, int dtype_bytes, int backward, int mode) {
  if (T < 1 || W < 1 || (dtype_bytes != 4 && dtype_bytes != 8)) return nullptr;
  const bool f64 = dtype_bytes == 8;
  const bool vok = W % (f64 ? vec_of<double>() : vec_of<float>()) == 0;
  if (mode == LINREC_SERIAL ||
      (f64 ? channel_parallel_enough<double>(T, W, vok) : channel_parallel_enough<float>(T, W, vok)))
    return "serial";
  if (!f64 && linrec_impl::cluster_scan_ok<float>(T, W, vok)) return "cluster";
  if (f64 ? linrec_impl::local_scan_ok<double>(T, W, vok) : linrec_impl::local_scan_ok<float>(T, W, vok))
    return "local";
  ChainPlan p;
  const bool fwd = backward == 0;
  const bool tma = vok && tma_allowed(T, W) &&
                   (f64 ? linrec_impl::plan_tma<double>(fwd, T, W, &p) : linrec_impl::plan_tma<float>(fwd, T, W, &p));
  return tma ? "tma" : "chained";
}

int linrec_scan_plan_f32(const float* lam, const float* x, const float* h0, float* h, int64_t T, int64_t W,
                         const int64_t* bounds, int64_t chunks, float* P, float* R, float* C, void* stream) {
  int rc;
  if ((rc = check_ptr(lam, "decays")) || (rc = check_ptr(x, "impulses")) || (rc = check_ptr(h, "h"))) return rc;
  return plan_scan<float>(false, lam, x, h0, nullptr, h, nullptr, nullptr, T, W, bounds, chunks, P, R, C,
                          static_cast<cudaStream_t>(stream));
}
int linrec_scan_plan_f64(const double* lam, const double* x, const double* h0, double* h, int64_t T, int64_t W,
                         const int64_t* bounds, int64_t chunks, double* P, double* R, double* C, void* stream) {
  int rc;
  if ((rc = check_ptr(lam, "decays")) || (rc = check_ptr(x, "impulses")) || (rc = check_ptr(h, "h"))) return rc;
  return plan_scan<double>(false, lam, x, h0, nullptr, h, nullptr, nullptr, T, W, bounds, chunks, P, R, C,
                           static_cast<cudaStream_t>(stream));
}
int linrec_scan_backward_plan_f32(const float* lam, const float* h0, const float* h, const float* dh, float* dlam,
                                  float* dx, float* dh0, int64_t T, int64_t W, const int64_t* bounds,
                                  int64_t chunks, void* stream) {
  int rc;
  if ((rc = check_ptr(lam, "decays")) || (rc = check_ptr(h, "h")) || (rc = check_ptr(dh, "d_h")) ||
      (rc = check_ptr(dlam, "d_decays")) || (rc = check_ptr(dx, "d_impulses")) || (rc = check_ptr(dh0, "d_initial")))
    return rc;
  return plan_scan<float>(true, lam, dh, h0, h, dx, dlam, dh0, T, W, bounds, chunks, nullptr, nullptr, nullptr,
                          static_cast<cudaStream_t>(stream));
}
int linrec_scan_backward_plan_f64(const double* lam, const double* h0, const double* h, const double* dh,
                                  double* dlam, double* dx, double* dh0, int64_t T, int64_t W,
                                  const int64_t* bounds, int64_t chunks, void* stream) {
  int rc;
  if ((rc = check_ptr(lam, "decays")) || (rc = check_ptr(h, "h")) || (rc = check_ptr(dh, "d_h")) ||
      (rc = check_ptr(dlam, "d_decays")) || (rc = check_ptr(dx, "d_impulses")) || (rc = check_ptr(dh0, "d_initial")))
    return rc;
  return plan_scan<double>(true, lam, dh, h0, h, dx, dlam, dh0, T, W, bounds, chunks, nullptr, nullptr, nullptr,
                           static_cast<cudaStream_t>(stream));
}

int linrec_segment_scan_exchange_f32(const float* lam, const float* x, const float* h0, float* h, float* seg_prod,
                                     float* agg, int64_t T, int64_t W, const linrec_exchange_t* ex,
                                     linrec_workspace_t ws, void* stream) {
  linrec_impl::Exchange e;
  const int rc = to_exchange(ex, W, 0, true, false, &e);
  if (rc) return rc;
  return segment_scan<float>(lam, x, h0, h, seg_prod, agg, T, W, ws, static_cast<cudaStream_t>(stream), &e);
}
int linrec_segment_scan_backward_exchange_f32(const float* lam, const float* hprev, const float* h, const float* dh,
                                              const float* lam_next, float* dlam, float* dx, float* dh0,
                                              float* seg_prod, float* agg, int64_t T, int64_t W,
                                              const linrec_exchange_t* ex, linrec_workspace_t ws, void* stream) {
  linrec_impl::Exchange e;
  const int rc = to_exchange(ex, W, 1, true, false, &e);
  if (rc) return rc;
  return segment_scan_backward<float>(lam, hprev, h, dh, lam_next, dlam, dx, dh0, seg_prod, agg, T, W, ws,
                                      static_cast<cudaStream_t>(stream), &e);
}
int linrec_segment_fixup_exchange_f32(const float* lam, float* h, const float* seg_prod, float* c_in, int64_t T,
                                      int64_t W, int64_t tile_rows, const linrec_exchange_t* ex, void* stream) {
  linrec_impl::Exchange e;
  const int rc = to_exchange(ex, W, 0, false, true, &e);
  if (rc) return rc;
  return segment_fixup<float>(false, lam, nullptr, nullptr, nullptr, seg_prod, nullptr, h, nullptr, T, W, tile_rows,
                              static_cast<cudaStream_t>(stream), &e, c_in);
}
int linrec_segment_fixup_backward_exchange_f32(const float* lam, const float* hprev, const float* h,
                                               const float* lam_next, const float* seg_prod, float* y_in,
                                               float* dlam, float* dx, int64_t T, int64_t W, int64_t tile_rows,
                                               const linrec_exchange_t* ex, void* stream) {
  linrec_impl::Exchange e;
  const int rc = to_exchange(ex, W, 1, false, true, &e);
  if (rc) return rc;
  return segment_fixup<float>(true, lam, hprev, h, lam_next, seg_prod, nullptr, dx, dlam, T, W, tile_rows,
                              static_cast<cudaStream_t>(stream), &e, y_in);
}
int linrec_compose_carries_f32(const float* aggs, int64_t first, int64_t last, int64_t step, const float* seed,
                               float* out, int64_t W, void* stream) {
  int rc;
  if ((rc = check_ptr(aggs, "aggs")) || (rc = check_ptr(out, "out"))) return rc;
  if (step != 1 && step != -1) return fail(LINREC_ERR_VALUE, "step must be +1 or -1");
  LINREC_CUDA_TRY(linrec_impl::launch_compose<float>(aggs, first, last, step, seed, out, W,
                                                     static_cast<cudaStream_t>(stream)));
  return LINREC_OK;
}
int linrec_compose_carries_f64(const double* aggs, int64_t first, int64_t last, int64_t step, const double* seed,
                               double* out, int64_t W, void* stream) {
  int rc;
  if ((rc = check_ptr(aggs, "aggs")) || (rc = check_ptr(out, "out"))) return rc;
  if (step != 1 && step != -1) return fail(LINREC_ERR_VALUE, "step must be +1 or -1");
  LINREC_CUDA_TRY(linrec_impl::launch_compose<double>(aggs, first, last, step, seed, out, W,
                                                      static_cast<cudaStream_t>(stream)));
  return LINREC_OK;
}
int linrec_gemm_f32(const float* A, int a_mn, int64_t lda, const float* B, int b_mn, int64_t ldb, float* C,
                    int64_t ldc, int64_t M, int64_t N, int64_t K, int accumulate, int precision, int k_splits,
                    float* scratch, void* stream) {
  int rc;
  if ((rc = check_ptr(A, "A")) || (rc = check_ptr(B, "B")) || (rc = check_ptr(C, "C"))) return rc;
  if (M < 1 || N < 1 || K < 1) return fail(LINREC_ERR_SHAPE, "gemm: M, N, K must be >= 1");
  if (M >= (int64_t(1) << 31) || N >= (int64_t(1) << 31)) return fail(LINREC_ERR_SHAPE, "gemm: M, N must be < 2^31");
  if (precision != LINREC_PREC_FP32 && precision != LINREC_PREC_TF32)
    return fail(LINREC_ERR_VALUE, "gemm: precision must be LINREC_PREC_FP32 or LINREC_PREC_TF32");
  if ((lda * 4) % 16 || (ldb * 4) % 16 || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))
    return fail(LINREC_ERR_VALUE, "gemm: operand pitches and pointers must be 16-byte aligned");
  if ((ldc * 4) % 16 || (reinterpret_cast<uintptr_t>(C) & 15))
    return fail(LINREC_ERR_VALUE, "gemm: C pitch and pointer must be 16-byte aligned");
  linrec_impl::GemmOperands op;
  op.a1 = A;
  op.b1 = B;
  op.K1 = K;
  op.lda1 = lda;
  op.ldb1 = ldb;
  op.M = M;
  op.units = N;
  op.a_mn = a_mn != 0;
  op.b_mn = b_mn != 0;
  linrec_impl::GemmEpilogue ep;
  ep.C = C;
  ep.ldc = ldc;
  ep.accumulate = accumulate != 0;
  ep.split3 = precision == LINREC_PREC_FP32;
  ep.k_splits = k_splits < 1 ? 1 : k_splits;
  ep.scratch = scratch;
  if (ep.k_splits > 1 && scratch == nullptr) return fail(LINREC_ERR_VALUE, "gemm: split-K needs scratch");
  LINREC_CUDA_TRY(linrec_impl::gemm_tf32(op, 0, ep, static_cast<cudaStream_t>(stream)));
  return LINREC_OK;
}

int linrec_gemm_splits(int64_t M, int64_t N, int64_t K) { return linrec_impl::gemm_splits_for(M, N, K); }

size_t linrec_gemm_scratch_bytes(int64_t M, int64_t N, int k_splits) {
  if (M < 1 || N < 1) return 0;
  return (size_t)linrec_impl::gemm_partial_floats(M, N, k_splits) * sizeof(float);
}

}  // extern "C"
