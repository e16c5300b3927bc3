// Internal (C++) launch interface between capi.cpp and the kernel TUs.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include <mutex>
#include <set>
#include <tuple>

namespace linrec_impl {

// Sets the thread-local linrec_last_error() message; returns `code`.
int set_error(int code, const char* msg);

// Tile configuration chosen for one chained launch.
struct ChainPlan {
  int kind = 0;       // 0 = register kernel (scan_chained.cuh), 1 = TMA persistent (scan_tma.cuh)
  int stages = 0;     // TMA ring depth
  int box_cols = 0, box_rows = 0;
  int threads = 0, smem = 0, grid = 0;
  int vec = 1;        // channels per thread vector (4 f32 / 2 f64, or 1)
  int q = 32;         // lanes across channels
  int r = 8;          // rows per thread
  int nw = 8;         // warps per CTA
  int cpw = 0;        // channels per column
  int rows = 0;       // rows per tile (L)
  int rec = 0;        // carry-record stride in elements
  int64_t ncols = 0;  // channel columns
  int64_t ntt = 0;    // tiles along time per chain (per virtual segment)
  int64_t nseg = 1;   // virtual T-segments (independent chains, stitched by segment.cu)
  int64_t tseg = 0;   // rows per virtual segment
  int64_t ntiles = 0; // = ncols * ntt = grid size
  size_t flags_bytes = 0;
  size_t rec_bytes = 0;  // bytes of ONE of the two record arrays (agg or inc)
  size_t ws_bytes = 0;   // control block + flags + agg + inc
};

// Rows per thread / warps per CTA of each direction (tuned on B200).
template <class S>
ChainPlan plan_chain(bool forward, int64_t T, int64_t W, bool vec_ok);

struct ChainPtrs {  // host mirror of linrec_dev::ChainWs
  void* ctrl;
  void* flags;
  void* agg;
  void* inc;
};

inline int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// cudaFuncSetAttribute once per (kernel, attribute, device): function
// attributes are per device, so a process-wide "once" would leave the other
// GPUs of a multi-GPU process unconfigured.
inline cudaError_t func_attr_once(const void* kernel, cudaFuncAttribute attr, int value) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(std::make_tuple(kernel, dev, (int)attr, value))) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, attr, value);
  if (e == cudaSuccess) done.insert(std::make_tuple(kernel, dev, (int)attr, value));
  return e;
}
// CTAs per (segment, column) chain of the stitch fix-up (fixup_chain): the
// forward's many segments fit one wave of resident CTAs with one walker
// each, the backward's fewer segments gain from two (C4);
// LINREC_FIXUP_WALK overrides both.
inline int fixup_walkers(bool reverse) {
  static const int k = env_int("LINREC_FIXUP_WALK", 0);
  if (k > 0) return k > 8 ? 8 : k;
  return reverse ? 2 : 1;
}

// One direction of the peer-memory carry exchange as this rank sees it
// (p2p_impl.cuh; mboxes == nullptr: no exchange).
struct Exchange {
  void* const* mboxes = nullptr;  // device array [world]: every rank's mailbox, mapped here
  int64_t W = 0;
  int world = 1, rank = 0, dir = 0;
  unsigned long long epoch = 0;   // >= 1, one per step and direction
  int q0 = 0, q1 = 0;             // consumers of this rank's aggregate: [q0, q1)
  int first = 0, last = 0, step = 1;  // sources folded into the incoming carry: first, first+step, ... != last
  int zero_a = 0;                 // publish A = 0 (the forward's rank 0: h0 is folded into B)
  __host__ __device__ bool has_sources() const { return mboxes != nullptr && first != last; }
  __host__ __device__ bool has_consumers() const { return mboxes != nullptr && q0 < q1; }
};

template <class S>
struct FwdCall {
  const S* lam;
  const S* x;
  const S* h0;
  S* h;
  int64_t T, W;
  S* seg_prod = nullptr;  // sequence sharding outputs (see segment.cu)
  S* agg_out = nullptr;
  S* rank_agg = nullptr;  // non-null: fold agg_out into it in the scan's tail (TMA, fp32)
  Exchange ex{};          // ... and publish it
  // decay-adaptive stitch (capi.cpp::adaptive_stitch): device mode word
  // (1 = "deep": the decays do not underflow within a virtual segment), the
  // launch's role (0 = the scan, which seeds virtual segments from seed_rows
  // when deep; 1 = the reduce-only pass, skipped unless deep; 2 = the
  // unsplit twin of a wide scan, skipped unless deep; 3 = the split scan
  // with such a twin, skipped when deep)
  const int* mode = nullptr;
  int role = 0;
  const S* seed_rows = nullptr;
};

template <class S>
struct BwdCall {
  const S* lam;
  const S* h0;
  const S* h;
  const S* dh;
  const S* lam_next;
  const S* g_next;
  S* dlam;
  S* dx;
  S* dh0;
  int64_t T, W;
  S* seg_prod = nullptr;
  S* agg_out = nullptr;
  S* rank_agg = nullptr;
  Exchange ex{};
  const int* mode = nullptr;  // as FwdCall
  int role = 0;
  const S* seed_rows = nullptr;
  // gated adjoint (fused layer backward): the scan runs on dh * gate, e.g.
  // dc = dh * o for h = o * c (GILR-LSTM / QRNN); TMA fp32 default config
  const S* gate = nullptr;
};

template <class S>
cudaError_t launch_chain_fwd(const ChainPlan& p, const FwdCall<S>& c, const ChainPtrs& ws,
                             cudaStream_t st);
template <class S>
cudaError_t launch_chain_bwd(const ChainPlan& p, const BwdCall<S>& c, const ChainPtrs& ws,
                             cudaStream_t st);
template <class S>
cudaError_t launch_serial_fwd(const FwdCall<S>& c, bool vec_ok, cudaStream_t st);
template <class S>
cudaError_t launch_serial_bwd(const BwdCall<S>& c, bool vec_ok, cudaStream_t st);

// TMA persistent kernels: plan_tma returns false when the shape/alignment is
// not eligible (then the register kernels run).
template <class S>
bool plan_tma(bool forward, int64_t T, int64_t W, ChainPlan* p);
template <class S>
cudaError_t launch_tma_fwd(const ChainPlan& p, const FwdCall<S>& c, const ChainPtrs& ws, cudaStream_t st);
template <class S>
cudaError_t launch_tma_bwd(const ChainPlan& p, const BwdCall<S>& c, const ChainPtrs& ws, cudaStream_t st);

cudaError_t launch_ws_init(void* ctrl, cudaStream_t st);

// cluster_scan.cu: a thread-block cluster splits a short sequence, the CTAs
// exchanging their chunk aggregates through distributed shared memory
template <class S>
bool cluster_scan_ok(int64_t T, int64_t W, bool vec_ok);
template <class S>
cudaError_t launch_cluster_fwd(const FwdCall<S>& c, cudaStream_t st);
template <class S>
cudaError_t launch_cluster_bwd(const BwdCall<S>& c, cudaStream_t st);

// local_scan.cu: one CTA per channel vector over the whole (short) sequence
template <class S>
bool local_scan_ok(int64_t T, int64_t W, bool vec_ok);
template <class S>
cudaError_t launch_local_fwd(const FwdCall<S>& c, bool vec_ok, cudaStream_t st);
template <class S>
cudaError_t launch_local_bwd(const BwdCall<S>& c, bool vec_ok, cudaStream_t st);

// segment.cu
// Fix-up of the tiles of (nseg x ntt) chain positions: e_in = seg_prod[pos] *
// carry[seg or 0] (carry_stride W or 0); when scale != nullptr each position's
// seg_prod row is also multiplied in place by scale[seg] (virtual -> segment
// relative products).
template <class S>
cudaError_t launch_fixup(bool reverse, const S* lam, const S* hprev_row, const S* h, const S* lam_next,
                         const S* seg_prod, const S* carry_rows, const S* scale_rows, const S* cin, S* out0, S* out1,
                         int64_t T, int64_t W, int64_t rows, int64_t nseg, int64_t tseg, int64_t ntt,
                         bool vec_ok, cudaStream_t st, const Exchange* ex = nullptr, S* c_out = nullptr,
                         const S* vagg = nullptr, S* dh0 = nullptr, const int* skip_if_deep = nullptr);
template <class S>
cudaError_t launch_vseg_finalize(bool reverse, const S* lam, const S* vagg, int64_t nseg, int64_t tseg,
                                 S* carry, S* scale, S* agg_rank, S* dh0, int64_t W, cudaStream_t st,
                                 const Exchange* ex = nullptr, const int* run_if_deep = nullptr);
// decay probe of the adaptive stitch (segment.cu::k_decay_probe): sets the
// workspace's ctrl->decay_mode
template <class S>
cudaError_t launch_decay_probe(const S* lam, int64_t T, int64_t W, int cpw, int64_t tseg, float thr, void* ctrl,
                               cudaStream_t st);
template <class S>
cudaError_t launch_compose(const S* aggs, int64_t first, int64_t last, int64_t step, const S* seed, S* out,
                           int64_t W, cudaStream_t st);


template <class S>
cudaError_t first_nonfinite(const S* v, int64_t n, int64_t* index, cudaStream_t st);

// tcgen05 TF32 GEMM (gemm_tc.cu): C[M][N] = sum_k A(m,k) B(n,k) with the
// K range optionally split over two operand pairs.  K-major operands are
// [rows][K] with pitch lda (elements), MN-major ones [K][rows].
struct GemmOperands {
  const float* a1 = nullptr;
  const float* b1 = nullptr;
  int64_t K1 = 0, lda1 = 0, ldb1 = 0;
  const float* a2 = nullptr;
  const float* b2 = nullptr;
  int64_t K2 = 0, lda2 = 0, ldb2 = 0;
  int64_t M = 0;
  int64_t units = 0;      // output columns (per block when nb > 1)
  int nb = 1;             // blocked K-major B: nb row blocks of `units` rows ...
  int64_t b_bstride = 0;  // ... block q starting at row q * b_bstride
  // ntaps > 1: K = ntaps segments of K1 (each padded to whole k-blocks); tap s
  // reads A (K-major) rows shifted by s*a_tap and B rows (K-major) / K rows
  // (MN-major) offset by s*b_tap -- the QRNN causal convolution as one GEMM
  int ntaps = 1;
  int64_t a_tap = 0, b_tap = 0;
  // optional precomputed lo parts (v - tf32(v)) of b1 / b2, same layout and
  // pitch: with 3xTF32 the kernel then splits only A in shared memory
  const float* b1_lo = nullptr;
  const float* b2_lo = nullptr;
  bool a_mn = false, b_mn = false;
};
struct GemmEpilogue {
  float* C = nullptr;
  int64_t ldc = 0;
  bool accumulate = false;
  bool split3 = false;       // 3xTF32 (fp32-grade) instead of plain TF32
  int k_splits = 1;
  float* scratch = nullptr;  // split-K partials, gemm_partial_floats() floats
  int act = 0;               // GILR candidate activation (0 tanh, 1 identity, 2 relu)
  const float* bias[4] = {nullptr, nullptr, nullptr, nullptr};
  float* out[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  int64_t ldo = 0;
};
// epi: 0 plain (C / accumulate / split-K), 1 GILR gates (nb 2), 2 LSTM gates (nb 4),
// 3 QRNN gates (nb 3)
cudaError_t gemm_tf32(const GemmOperands& op, int epi, const GemmEpilogue& ep, cudaStream_t st);
// dst[i] = src[i] - tf32(src[i]) (the 3xTF32 lo part), count floats
cudaError_t tf32_lo(const float* src, float* dst, int64_t count, cudaStream_t st);
int gemm_splits_for(int64_t M, int64_t N, int64_t K);
// split-K partial buffer (floats) gemm_tf32 needs for `splits` splits (0 for 1)
int64_t gemm_partial_floats(int64_t M, int64_t N, int splits);
// All k taps' weight gradients dW_s[M][N] += A[. + s*shift]^T B (A, B MN-major,
// N <= 8) in one CUDA-core launch (the QRNN's first layer); cudaErrorNotSupported
// when the shape does not qualify.  scratch: wgrad_taps_partial_floats floats.
int64_t wgrad_taps_partial_floats(int64_t M, int64_t N, int64_t R, int ntaps);
cudaError_t wgrad_taps_skinny(const float* A, int64_t lda, const float* B, int64_t ldb, int64_t R, int64_t shift,
                              int ntaps, int64_t M, int64_t N, float* dW, float* scratch, cudaStream_t st);

// The reference's chunked scan with an explicit plan (plan_scan.cu): phases
// 1-3 bit-identical to recurrence.hpp's scan_parallel; reverse = the
// backward's reversed image (x_or_dh = dh, out = dx, plus dlam and dh0).
// bounds_dev: p (start, end) 1-based pairs in device memory; P, R, C [p][W].
template <class S>
cudaError_t launch_plan_scan(bool reverse, const S* lam, const S* x_or_dh, const S* h0, const S* h, S* out,
                             S* dlam, S* dh0, int64_t T, int64_t W, const int64_t* bounds_dev, int64_t p, S* P,
                             S* R, S* C, cudaStream_t st);

}  // namespace linrec_impl
