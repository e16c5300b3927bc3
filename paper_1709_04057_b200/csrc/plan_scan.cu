// The reference's chunked parallel scan with an explicit plan, on the GPU
// (recurrence.hpp:193-245 scan_parallel with a ChunkPlan and ScanSummaries,
// :365-377 scan_backward with an explicit plan): the same three phases in
// the same per-channel operation order, so results -- h and the chunk
// summaries P, R, C -- are bit-identical to the reference's for the same
// plan (and to oracle/linrec_oracle.c::oracle_scan_parallel).  Parallel over
// (chunk, channel vector); each thread walks its chunk serially.  This is
// the plan-faithful path (inspection, plan-for-plan parity); the default
// parallel mode is the single-pass chained scan (scan_tma.cuh).
#include <cuda_runtime.h>

#include <cstdint>

#include "launch.h"
#include "linrec_device.cuh"

namespace linrec_dev {
namespace plan {

// Rows of the scanned sequence.  Forward: lam, x as given.  Backward: the
// reversed image of scan_backward_impl (:305-318) without materialising it:
// row s has decay lam[T-s] (0 for s = 0) and impulse dh[T-1-s].
template <class S, bool REV>
struct Rows {
  const S* lam;
  const S* x;  // fwd: x, bwd: dh
  int64_t T, W;
  __device__ S decay(int64_t s, int64_t j) const {
    if (!REV) return lam[s * W + j];
    return s == 0 ? S(0) : lam[(T - s) * W + j];
  }
  __device__ S impulse(int64_t s, int64_t j) const { return REV ? x[(T - 1 - s) * W + j] : x[s * W + j]; }
};

// Phase 1 (chunk_summary, :114-131): P = prod decay, R = zero-seeded
// recurrence over chunk i; thread per (chunk, channel).
template <class S, bool REV>
__global__ void k_summaries(Rows<S, REV> r, const int64_t* __restrict__ bounds, int64_t p, S* __restrict__ P,
                            S* __restrict__ R) {
  const int64_t i = blockIdx.y;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < r.W; j += (int64_t)gridDim.x * blockDim.x) {
    S Pi = S(1), Ri = S(0);
    for (int64_t s = bounds[2 * i] - 1; s <= bounds[2 * i + 1] - 1; ++s) {
      const S l = r.decay(s, j);
      Ri = fma_(l, Ri, r.impulse(s, j));
      Pi = mul_(Pi, l);
    }
    P[i * r.W + j] = Pi;
    R[i * r.W + j] = Ri;
  }
}

// Phase 2 (:219-230): C_i = P_i * C_{i-1} + R_i, C_{-1} = h0; thread per
// channel, sequential over the p summaries.
template <class S>
__global__ void k_stitch(const S* __restrict__ P, const S* __restrict__ R, const S* __restrict__ h0, int64_t p,
                         int64_t W, S* __restrict__ C) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < W; j += (int64_t)gridDim.x * blockDim.x) {
    S prev = h0 != nullptr ? h0[j] : S(0);
    for (int64_t i = 0; i < p; ++i) {
      prev = fma_(P[i * W + j], prev, R[i * W + j]);
      C[i * W + j] = prev;
    }
  }
}

// Phase 3 (:232-237): chunk scans seeded with the stitched states.  Forward
// writes h; backward turns the reversed result G into dx_t = G_t,
// dlam_t = h_{t-1} G_t (h0 at t = 0) and dh0 = lam_0 G_0 (:331-346).
template <class S, bool REV>
__global__ void k_rescan(Rows<S, REV> r, const int64_t* __restrict__ bounds, const S* __restrict__ C,
                         const S* __restrict__ h0, S* __restrict__ out, const S* __restrict__ h,
                         S* __restrict__ dlam, S* __restrict__ dh0) {
  const int64_t i = blockIdx.y, W = r.W;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < W; j += (int64_t)gridDim.x * blockDim.x) {
    S c = i == 0 ? (REV ? S(0) : (h0 != nullptr ? h0[j] : S(0))) : C[(i - 1) * W + j];
    for (int64_t s = bounds[2 * i] - 1; s <= bounds[2 * i + 1] - 1; ++s) {
      c = fma_(r.decay(s, j), c, r.impulse(s, j));
      if (!REV) {
        out[s * W + j] = c;
      } else {
        const int64_t t = r.T - 1 - s;
        out[t * W + j] = c;  // dx
        const S hp = t == 0 ? (h0 != nullptr ? h0[j] : S(0)) : h[(t - 1) * W + j];
        dlam[t * W + j] = mul_(hp, c);
        if (t == 0) dh0[j] = mul_(r.lam[j], c);
      }
    }
  }
}

}  // namespace plan
}  // namespace linrec_dev

namespace linrec_impl {

template <class S>
cudaError_t launch_plan_scan(bool reverse, const S* lam, const S* x_or_dh, const S* h0, const S* h, S* out,
                             S* dlam, S* dh0, int64_t T, int64_t W, const int64_t* bounds_dev, int64_t p, S* P,
                             S* R, S* C, cudaStream_t st) {
  using namespace linrec_dev::plan;
  const int threads = 128;
  const int64_t bx = (W + threads - 1) / threads;
  const dim3 grid((unsigned)(bx < 1024 ? bx : 1024), (unsigned)p);
  const dim3 grid1((unsigned)(bx < 4096 ? bx : 4096));
  if (!reverse) {
    const Rows<S, false> r{lam, x_or_dh, T, W};
    k_summaries<S, false><<<grid, threads, 0, st>>>(r, bounds_dev, p, P, R);
    k_stitch<S><<<grid1, threads, 0, st>>>(P, R, h0, p, W, C);
    k_rescan<S, false><<<grid, threads, 0, st>>>(r, bounds_dev, C, h0, out, nullptr, nullptr, nullptr);
  } else {
    const Rows<S, true> r{lam, x_or_dh, T, W};
    k_summaries<S, true><<<grid, threads, 0, st>>>(r, bounds_dev, p, P, R);
    k_stitch<S><<<grid1, threads, 0, st>>>(P, R, nullptr, p, W, C);
    k_rescan<S, true><<<grid, threads, 0, st>>>(r, bounds_dev, C, h0, out, h, dlam, dh0);
  }
  return cudaGetLastError();
}

template cudaError_t launch_plan_scan<float>(bool, const float*, const float*, const float*, const float*, float*,
                                             float*, float*, int64_t, int64_t, const int64_t*, int64_t, float*,
                                             float*, float*, cudaStream_t);
template cudaError_t launch_plan_scan<double>(bool, const double*, const double*, const double*, const double*,
                                              double*, double*, double*, int64_t, int64_t, const int64_t*, int64_t,
                                              double*, double*, double*, cudaStream_t);

}  // namespace linrec_impl
