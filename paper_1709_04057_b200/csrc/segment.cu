// Sequence sharding support (BASELINE.json north_star: "each GPU reduces its
// segment to a per-channel (A,B) carry, the GPUs exchange that tiny carry with
// an NCCL all-gather over NVLink, and each GPU runs a local fix-up").
//
// A segment [S, E) of the sequence is first scanned with a zero carry by the
// ordinary chained kernels, which additionally emit (chain_impl/tma launch
// with ChainArgs::seg_prod / agg_out)
//   seg_prod[p][ch]  exclusive decay product entering chain position p,
//   agg[2][ch]       the segment aggregate (prod lam, zero-seeded result).
// After the aggregates are exchanged and folded (k_compose) into the carry
// c_in entering the segment, the true result differs from the zero-carry one
// by P_t * c_in (forward) -- P_t the decay product from the segment start --
// which these kernels add.  Each tile reads its entering product first and
// exits at once when P * c_in is exactly zero for all of its channels: once
// the running product underflows the correction is exactly zero, so only the
// leading tiles of a segment are touched for decays < 1 (the bench
// distribution: ~100 rows), while decays near 1 degrade to one extra pass.
#include <cstdint>

#include <type_traits>

#include "chain_impl.cuh"
#include "fixup_impl.cuh"
#include "p2p_impl.cuh"

namespace linrec_dev {

// CTA j of the J walkers of chain (virtual segment, channel column):
// fixup_chain (fixup_impl.cuh), 8 warps.  With a peer exchange (fp32) the
// CTA first composes the range's incoming carry for its column from the
// mailboxes (p2p_impl.cuh::compose_chunk; the first walker of the first
// virtual segment also stores it to c_out).
template <class S, int VEC, int Q, bool REV, int RF>
__global__ void __launch_bounds__(256, (REV && RF > 6) ? 1 : 2)  // backward at RF 12: dx, dlam, h rows in flight
k_fixup(FixupArgs<S> f, Carries<S> cr, int64_t ncols, int walkers, linrec_impl::Exchange ex,
        S* __restrict__ c_out, const int* __restrict__ skip_if_deep) {
  constexpr int CPW = Q * VEC, NWK = 8 * (32 / Q);
  if (skip_if_deep != nullptr && __ldcg(skip_if_deep) != 0) return;  // the deep scan seeded its segments
  __shared__ S s_wp[8][CPW];
  __shared__ S s_cin[CPW];
  __shared__ S s_own[CPW], s_scale[CPW];
  __shared__ S s_fa[NWK * CPW], s_fb[NWK * CPW];
  const int64_t col = blockIdx.x % ncols;
  const int j = (int)((blockIdx.x / ncols) % walkers);
  const int64_t vseg = (blockIdx.x / ncols) / walkers;
  if constexpr (std::is_same<S, float>::value) {
    if (ex.has_sources()) {
      p2p::compose_chunk(ex, col * CPW, CPW, s_cin);
      if (vseg == 0 && j == 0 && c_out != nullptr)
        for (int t = threadIdx.x; t < CPW && col * CPW + t < f.W; t += blockDim.x) c_out[col * CPW + t] = s_cin[t];
      cr.cin = s_cin - col * CPW;  // indexed by channel
    }
  }
  if (cr.vagg != nullptr) {  // the segment's own carry, folded here instead of a separate launch
    S c[VEC], sc[VEC];
    fold_carry<S, VEC, Q, REV, CtaSync>(f, cr.vagg, vseg, col, s_fa, s_fb, c, sc);
    const int q = (threadIdx.x & 31) % Q;
    if (threadIdx.x < 32 && threadIdx.x < Q)
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        s_own[q * VEC + v] = c[v];
        s_scale[q * VEC + v] = sc[v];
      }
    __syncthreads();
    cr.own = s_own - col * CPW;  // indexed by channel
    cr.own_scale = s_scale - col * CPW;
  }
  fixup_chain<S, VEC, Q, REV, CtaSync, RF>(f, vseg, col, j, walkers, cr, s_wp);
}

// out[j] = fold over q in [first, last) by `step` of c = A_q[j] * c + B_q[j],
// c starting at seed[j] (0 if seed == nullptr).  aggs: [n][2][W].
template <class S>
__global__ void k_compose(const S* __restrict__ aggs, int64_t first, int64_t last, int64_t step,
                          const S* __restrict__ seed, S* __restrict__ out, int64_t W) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < W;
       j += (int64_t)gridDim.x * blockDim.x) {
    S c = seed != nullptr ? seed[j] : S(0);
    for (int64_t q = first; q != last; q += step) c = fma_(aggs[q * 2 * W + j], c, aggs[q * 2 * W + W + j]);
    out[j] = c;
  }
}

// Virtual-segment finalisation: one CTA of 32 x G threads per 32-channel
// chunk (fixup_impl.cuh::vseg_fold): sequential depth 2*nseg/G + G instead of
// nseg (C4: 256 segments, 49 -> 8 us).
template <class S, bool REV, int G>
__global__ void __launch_bounds__(32 * G)
k_vseg_finalize(const S* __restrict__ lam, const S* __restrict__ vagg, int64_t nseg, int64_t tseg,
                S* __restrict__ carry, S* __restrict__ scale, S* __restrict__ agg_rank, S* __restrict__ dh0,
                int64_t W, linrec_impl::Exchange ex, const int* __restrict__ run_if_deep) {
  __shared__ S sA[G][32], sB[G][32];
  if (run_if_deep != nullptr && __ldcg(run_if_deep) == 0) return;  // adaptive stitch: shallow decays
  vseg_fold<S, REV, G, CtaSync>(lam, vagg, nseg, tseg, carry, scale, agg_rank, dh0, W, blockIdx.x, sA, sB);
  if constexpr (std::is_same<S, float>::value) {
    // the rank aggregate of this chunk straight into the consumers' mailboxes
    if (ex.has_consumers()) {
      const int64_t j0 = (int64_t)blockIdx.x * 32;
      p2p::publish_chunk(ex, agg_rank, j0, (int)(W - j0 < 32 ? W - j0 : 32));
    }
  }
}

// Decay probe of the adaptive stitch: is the fix-up of the virtual segments
// going to be a second pass?  CTA `col` estimates, for each channel of its
// column, how many rows the decay product takes to underflow (fp32: to
// 2^-149) from the mean log2|lam| over 64 rows sampled across T (8 blocks of
// 8 rows; a row past T counts as |lam| = 1), takes the
// column's maximum (a fix-up tile is touched while ANY of its channels is
// non-zero), and adds min(1, depth / tseg) -- the fraction of each segment
// the fix-up would walk -- to a sum; the last CTA sets ctrl->decay_mode = 1
// when the mean fraction exceeds `thr` (the fix-up would cost more than the
// reduce-only pass it replaces) and resets the sum for the next launch.
// Graph-safe (device state only), no host synchronisation.
template <class S>
__global__ void __launch_bounds__(512) k_decay_probe(const S* __restrict__ lam, int64_t T, int64_t W, int cpw,
                                                     int64_t tseg, float thr, Ctrl* ctrl) {
  // 64 sampled rows: 4 row groups x 16 rows per thread, all 16 loads in
  // flight at once (one DRAM round trip), then the groups combine
  constexpr int NS = 64, NG = 4, RPG = NS / NG;
  __shared__ float s_sum[NG][128];
  __shared__ float s_max[4];
  const int c = threadIdx.x & 127, grp = threadIdx.x >> 7;
  const int64_t ch = (int64_t)blockIdx.x * cpw + c;
  const bool ok = c < cpw && ch < W;
  float v[RPG];
#pragma unroll
  for (int k = 0; k < RPG; ++k) {
    // 8 blocks of 8 consecutive rows spread over T (few pages: the probe's one
    // DRAM round trip is not stretched by TLB misses)
    const int j = grp * RPG + k;
    const int64_t t = (T * (j >> 3)) / (NS / 8) + (j & 7);
    v[k] = ok && t < T ? (float)__ldcg(lam + t * W + ch) : 1.f;
  }
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < RPG; ++k) sum += log2f(fabsf(v[k]));  // |lam| = 0 -> -inf -> depth 0
  s_sum[grp][c] = sum;
  __syncthreads();
  float depth = 0.f;
  if (grp == 0) {
    const float mean = (s_sum[0][c] + s_sum[1][c] + s_sum[2][c] + s_sum[3][c]) / NS;
    depth = !ok ? 0.f : (mean < 0.f ? 149.f / -mean : 3.0e38f);
    for (int off = 16; off > 0; off >>= 1) depth = fmaxf(depth, __shfl_xor_sync(0xffffffffu, depth, off));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = depth;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const float d = fmaxf(fmaxf(s_max[0], s_max[1]), fmaxf(s_max[2], s_max[3]));
    const float frac = fminf(1.f, d / (float)tseg);
    atomicAdd(&ctrl->decay_sum, frac);
    __threadfence();
    if (atomicAdd(&ctrl->decay_count, 1u) == gridDim.x - 1) {
      __threadfence();
      const float mean = atomicExch(&ctrl->decay_sum, 0.f) / (float)gridDim.x;
      ctrl->decay_count = 0u;
      ctrl->decay_mode = mean > thr ? 1 : 0;
    }
  }
}

}  // namespace linrec_dev

namespace linrec_impl {

template <class S>
cudaError_t launch_fixup(bool reverse, const S* lam, const S* hprev_row, const S* h, const S* lam_next,
                         const S* seg_prod, const S* carry_rows, const S* scale_rows, const S* cin, S* out0, S* out1,
                         int64_t T, int64_t W, int64_t rows, int64_t nseg, int64_t tseg, int64_t ntt,
                         bool vec_ok, cudaStream_t st, const Exchange* ex, S* c_out, const S* vagg, S* dh0,
                         const int* skip_if_deep) {
  const Exchange exv = ex != nullptr ? *ex : Exchange{};
  constexpr int V = Tuning<S>::VEC;
  const int64_t nvec = vec_ok ? (W + V - 1) / V : W;
  const int q = pick_q(nvec);
  const int cpw = q * (vec_ok ? V : 1);
  const int64_t ncols = (W + cpw - 1) / cpw;
  const int walk = fixup_walkers(reverse);
  const dim3 grid((unsigned)(ncols * nseg * walk));
  linrec_dev::FixupArgs<S> fa{lam, hprev_row, h, lam_next, seg_prod, out0, out1, T, W, rows, nseg, tseg, ntt};
  fa.dh0 = dh0;
  linrec_dev::Carries<S> cr{carry_rows, scale_rows, cin};
  cr.vagg = vagg;
  // rows per thread of the fix-up pass (LINREC_FIXUP_RF_FWD / _BWD: 12 or 6)
  static const int rf_fwd = env_int("LINREC_FIXUP_RF_FWD", 6) == 12 ? 12 : 6;
  static const int rf_bwd = env_int("LINREC_FIXUP_RF_BWD", 12) == 6 ? 6 : 12;
  const int rf = reverse ? rf_bwd : rf_fwd;
#define FIXRF(VV, RFV)                                                                                \
  LINREC_Q_SWITCH(q, if (reverse) linrec_dev::k_fixup<S, VV, Q_, true, RFV><<<grid, 256, 0, st>>>(    \
                         fa, cr, ncols, walk, exv, c_out, skip_if_deep);                  \
                     else linrec_dev::k_fixup<S, VV, Q_, false, RFV><<<grid, 256, 0, st>>>(           \
                         fa, cr, ncols, walk, exv, c_out, skip_if_deep));
#define FIX(VV)         \
  if (rf == 6) {        \
    FIXRF(VV, 6)        \
  } else {              \
    FIXRF(VV, 12)       \
  }
  if (vec_ok) {
    FIX(V)
  } else {
    FIX(1)
  }
#undef FIX
#undef FIXRF
  return cudaGetLastError();
}

template <class S>
cudaError_t launch_vseg_finalize(bool reverse, const S* lam, const S* vagg, int64_t nseg, int64_t tseg, S* carry,
                                 S* scale, S* agg_rank, S* dh0, int64_t W, cudaStream_t st, const Exchange* ex,
                                 const int* run_if_deep) {
  const Exchange exv = ex != nullptr ? *ex : Exchange{};
  constexpr int G = 16;
  const unsigned g = (unsigned)((W + 31) / 32);
  if (reverse)
    linrec_dev::k_vseg_finalize<S, true, G><<<g, 32 * G, 0, st>>>(lam, vagg, nseg, tseg, carry, scale, agg_rank, dh0, W, exv, run_if_deep);
  else
    linrec_dev::k_vseg_finalize<S, false, G><<<g, 32 * G, 0, st>>>(lam, vagg, nseg, tseg, carry, scale, agg_rank, dh0, W, exv, run_if_deep);
  return cudaGetLastError();
}

template <class S>
cudaError_t launch_compose(const S* aggs, int64_t first, int64_t last, int64_t step, const S* seed, S* out,
                           int64_t W, cudaStream_t st) {
  const int64_t blocks = (W + 255) / 256;
  linrec_dev::k_compose<S><<<(unsigned)(blocks < 1024 ? blocks : 1024), 256, 0, st>>>(aggs, first, last, step,
                                                                                      seed, out, W);
  return cudaGetLastError();
}

template <class S>
cudaError_t launch_decay_probe(const S* lam, int64_t T, int64_t W, int cpw, int64_t tseg, float thr, void* ctrl,
                               cudaStream_t st) {
  const unsigned ncols = (unsigned)((W + cpw - 1) / cpw);
  linrec_dev::k_decay_probe<S><<<ncols, 512, 0, st>>>(lam, T, W, cpw, tseg, thr,
                                                      reinterpret_cast<linrec_dev::Ctrl*>(ctrl));
  return cudaGetLastError();
}
template cudaError_t launch_decay_probe<float>(const float*, int64_t, int64_t, int, int64_t, float, void*,
                                               cudaStream_t);

template cudaError_t launch_fixup<float>(bool, const float*, const float*, const float*, const float*, const float*,
                                         const float*, const float*, const float*, float*, float*, int64_t, int64_t,
                                         int64_t, int64_t, int64_t, int64_t, bool, cudaStream_t, const Exchange*,
                                         float*, const float*, float*, const int*);
template cudaError_t launch_fixup<double>(bool, const double*, const double*, const double*, const double*,
                                          const double*, const double*, const double*, const double*, double*,
                                          double*,
                                          int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, bool, cudaStream_t,
                                          const Exchange*, double*, const double*, double*, const int*);
template cudaError_t launch_compose<float>(const float*, int64_t, int64_t, int64_t, const float*, float*,
                                           int64_t, cudaStream_t);
template cudaError_t launch_compose<double>(const double*, int64_t, int64_t, int64_t, const double*, double*,
                                            int64_t, cudaStream_t);
template cudaError_t launch_vseg_finalize<float>(bool, const float*, const float*, int64_t, int64_t, float*,
                                                 float*, float*, float*, int64_t, cudaStream_t, const Exchange*,
                                                 const int*);
template cudaError_t launch_vseg_finalize<double>(bool, const double*, const double*, int64_t, int64_t, double*,
                                                  double*, double*, double*, int64_t, cudaStream_t, const Exchange*,
                                                  const int*);

}  // namespace linrec_impl
