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

#include "chain_impl.cuh"

namespace linrec_dev {

// One CTA per (chain position, channel column); 8 warps; Q lanes across
// channels x G groups along time, RF rows per thread per pass; a tile of
// `rows` rows is covered in ceil(rows / (8*G*RF)) passes.  Chain positions
// run over nseg virtual segments of ntt tiles (tile p of segment s starts at
// row s*tseg + p*rows, or (ntt-1-p)*rows for the reverse scan).
template <class S, int VEC, int Q, bool REV>
__global__ void __launch_bounds__(256)
k_fixup(const S* __restrict__ lam, const S* __restrict__ hprev_row, const S* __restrict__ h,
        const S* __restrict__ lam_next, S* __restrict__ seg_prod, const S* __restrict__ carry,
        int64_t carry_stride, const S* __restrict__ scale, S* __restrict__ out0 /* fwd: h; bwd: dx */,
        S* __restrict__ out1 /* bwd: dlam */, int64_t T, int64_t W, int64_t rows, int64_t ncols, int64_t nseg,
        int64_t tseg, int64_t ntt, int64_t walk) {
  constexpr int NW = 8, RF = 12, G = 32 / Q, CPW = Q * VEC, NSEG = NW * G, PR = NSEG * RF;  // PR = a TMA tile
  using IO = VecIO<S, VEC>;
  __shared__ S s_wp[NW][CPW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % Q, g = lane / Q;
  const int64_t col = blockIdx.x % ncols;
  // walk == 0: one CTA per chain position.  walk > 0 (no `scale`): CTA k of
  // (segment, column) visits positions k, k+walk, ... and stops at the first
  // whose entering correction is zero in every channel -- exact, because the
  // products are applied oldest first (bit-identical whatever the look-back
  // depth), so a zero product stays zero further down the chain.
  int64_t vseg, p_in;
  if (walk > 0) {
    vseg = (blockIdx.x / ncols) / walk;
    p_in = (blockIdx.x / ncols) % walk;
  } else {
    vseg = (blockIdx.x / ncols) / ntt;
    p_in = (blockIdx.x / ncols) % ntt;
  }
  for (; p_in < ntt; p_in += (walk > 0 ? walk : ntt)) {
  const int64_t pos = vseg * ntt + p_in;
  const int64_t tile_row = vseg * tseg + (REV ? ntt - 1 - p_in : p_in) * rows;
  const int64_t ch = col * CPW + (int64_t)q * VEC;
  const bool valid = ch < W;
  // carry entering the tile: exclusive product * segment carry
  S e[VEC];
  bool nz = false;
#pragma unroll
  for (int v = 0; v < VEC; ++v) e[v] = S(0);
  if (valid) {
    const S* sp = seg_prod + pos * W + ch;
    const S* cr = carry + vseg * carry_stride + ch;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      e[v] = mul_(sp[v], cr[v]);
      nz = nz || e[v] != S(0);
    }
  }
  nz = __syncthreads_or(nz) != 0;  // every thread has read seg_prod past this point
  if (scale != nullptr && valid && warp == 0 && g == 0) {  // virtual -> segment-relative products
    S* sp = seg_prod + pos * W + ch;
    const S* sc = scale + vseg * W + ch;
#pragma unroll
    for (int v = 0; v < VEC; ++v) sp[v] = mul_(sp[v], sc[v]);
  }
  if (!nz) return;

  const int64_t t_lo = tile_row;
  const int64_t seg_end = (vseg + 1) * tseg < T ? (vseg + 1) * tseg : T;
  const int64_t t_hi = (t_lo + rows < seg_end ? t_lo + rows : seg_end);
  const int64_t npass = (rows + PR - 1) / PR;
  for (int64_t ps = 0; ps < npass; ++ps) {
    // rows of this pass, in processing order
    const int64_t pbase = REV ? t_lo + rows - (ps + 1) * PR : t_lo + ps * PR;
    const int seg = warp * G + g;
    S m[RF][VEC];
#pragma unroll
    for (int i = 0; i < RF; ++i) {
      // processing index within the pass: REV walks rows downward
      const int64_t t = REV ? pbase + (PR - 1 - (seg * RF + i)) : pbase + seg * RF + i;
      const bool in = valid && t >= t_lo && t < t_hi;
#pragma unroll
      for (int v = 0; v < VEC; ++v) m[i][v] = S(1);
      if (in) {
        if (!REV) {
          IO::load_cg(lam + t * W + ch, m[i]);
        } else if (t + 1 >= T) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) m[i][v] = lam_next != nullptr ? lam_next[ch + v] : S(0);
        } else if (nseg > 1 && (t + 1) % tseg == 0) {
          // end of a virtual segment: mu = 1 (m already 1)
        } else {
          IO::load_cg(lam + (t + 1) * W + ch, m[i]);
        }
      }
    }
    // segment product, inclusive scan across the warp's groups, then warps
    S A[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) A[v] = m[0][v];
#pragma unroll
    for (int i = 1; i < RF; ++i)
#pragma unroll
      for (int v = 0; v < VEC; ++v) A[v] = mul_(m[i][v], A[v]);
#pragma unroll
    for (int off = 1; off < G; off <<= 1)
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const S ap = __shfl_up_sync(0xffffffffu, A[v], off * Q);
        if (g >= off) A[v] = mul_(A[v], ap);
      }
    S Ae[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      Ae[v] = S(1);
      if (G > 1) {
        const S ap = __shfl_up_sync(0xffffffffu, A[v], Q);
        if (g > 0) Ae[v] = ap;
      }
    }
    __syncthreads();
    if (g == G - 1) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) s_wp[warp][q * VEC + v] = A[v];
    }
    __syncthreads();
    S ecur[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) ecur[v] = e[v];
    for (int w = 0; w < warp; ++w)
#pragma unroll
      for (int v = 0; v < VEC; ++v) ecur[v] = mul_(s_wp[w][q * VEC + v], ecur[v]);
#pragma unroll
    for (int v = 0; v < VEC; ++v) ecur[v] = mul_(Ae[v], ecur[v]);
    // apply
#pragma unroll
    for (int i = 0; i < RF; ++i) {
      const int64_t t = REV ? pbase + (PR - 1 - (seg * RF + i)) : pbase + seg * RF + i;
#pragma unroll
      for (int v = 0; v < VEC; ++v) ecur[v] = mul_(m[i][v], ecur[v]);
      if (valid && t >= t_lo && t < t_hi) {
        S o[VEC];
        IO::load_cg(out0 + t * W + ch, o);
#pragma unroll
        for (int v = 0; v < VEC; ++v) o[v] = o[v] + ecur[v];
        IO::store_cg(out0 + t * W + ch, o);
        if (REV && out1 != nullptr) {
          S hp[VEC], d[VEC];
          if (t >= 1) IO::load_cg(h + (t - 1) * W + ch, hp);
          else {
#pragma unroll
            for (int v = 0; v < VEC; ++v) hp[v] = hprev_row != nullptr ? hprev_row[ch + v] : S(0);
          }
          IO::load_cg(out1 + t * W + ch, d);
#pragma unroll
          for (int v = 0; v < VEC; ++v) d[v] = fma_(hp[v], ecur[v], d[v]);
          IO::store_cg(out1 + t * W + ch, d);
        }
      }
    }
    // carry into the next pass = e * product of this whole pass
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      S tot = S(1);
      for (int w = 0; w < NW; ++w) tot = mul_(s_wp[w][q * VEC + v], tot);
      e[v] = mul_(tot, e[v]);
    }
  }
  __syncthreads();  // s_wp is reused by the next position
  }
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

// Virtual-segment finalisation.
// forward: carry[s] = state entering segment s (0 for s = 0, whose chain was
//   seeded), scale[s] = decay product of the segments before s, agg_rank =
//   (product over all, final state).
// reverse: carry[s] = lam_E * G_E entering segment s from above (0 for the
//   last), scale[s] = product of the A' of the segments after s, agg_rank =
//   (A', B') of the whole range, dh0 = lam_0 * G_0 (the range's start).
// vagg[s] = (P_incl, c_incl) of segment s's chains.
// Block = 32 channels x G segment groups: each group composes its contiguous
// range of segments (processing order), the groups' composites are folded in
// group order, and each group re-walks its range from its incoming state --
// a fixed association (deterministic), sequential depth 2*nseg/G + G instead
// of nseg (C4: 256 segments, 49 -> a few us).
template <class S, bool REV>
__device__ __forceinline__ void vseg_pair(const S* __restrict__ lam, const S* __restrict__ vagg, int64_t nseg,
                                          int64_t tseg, int64_t W, int64_t i, int64_t j, S& A, S& B) {
  const int64_t s = REV ? nseg - 1 - i : i;
  A = vagg[s * 2 * W + j];
  B = vagg[s * 2 * W + W + j];
  if (REV) {
    const S l0 = lam[(s * tseg) * W + j];
    A = mul_(l0, A);
    B = mul_(l0, B);
  }
}

template <class S, bool REV, int G>
__global__ void __launch_bounds__(32 * G)
k_vseg_finalize(const S* __restrict__ lam, const S* __restrict__ vagg, int64_t nseg, int64_t tseg,
                S* __restrict__ carry, S* __restrict__ scale, S* __restrict__ agg_rank, S* __restrict__ dh0,
                int64_t W) {
  __shared__ S sA[G][32], sB[G][32];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const bool ok = j < W;
  const int64_t per = (nseg + G - 1) / G;
  const int64_t i0 = (int64_t)g * per, i1 = i0 + per < nseg ? i0 + per : nseg;
  // phase 1: composite (A, B) of this group's segments, oldest first
  S Ac = S(1), Bc = S(0);
  if (ok) {
#pragma unroll 4
    for (int64_t i = i0; i < i1; ++i) {
      S A, B;
      vseg_pair<S, REV>(lam, vagg, nseg, tseg, W, i, j, A, B);
      Bc = fma_(A, Bc, B);
      Ac = mul_(A, Ac);
    }
  }
  sA[g][lane] = Ac;
  sB[g][lane] = Bc;
  __syncthreads();
  // phase 2: state and product entering this group (groups folded in order)
  S c = S(0), pc = S(1);
  for (int q = 0; q < g; ++q) {
    c = fma_(sA[q][lane], c, sB[q][lane]);
    pc = mul_(sA[q][lane], pc);
  }
  if (!ok) return;
  // phase 3: re-walk, writing each segment's incoming state / product
#pragma unroll 4
  for (int64_t i = i0; i < i1; ++i) {
    const int64_t s = REV ? nseg - 1 - i : i;
    if (carry != nullptr) carry[s * W + j] = c;
    if (scale != nullptr) scale[s * W + j] = pc;
    S A, B;
    vseg_pair<S, REV>(lam, vagg, nseg, tseg, W, i, j, A, B);
    c = fma_(A, c, B);
    pc = mul_(A, pc);
  }
  if (i1 == nseg && i0 < i1) {  // the group holding the last segment reports the whole range
    if (agg_rank != nullptr) {
      agg_rank[j] = pc;
      agg_rank[W + j] = c;
    }
    if (dh0 != nullptr) dh0[j] = c;
  }
}

}  // namespace linrec_dev

namespace linrec_impl {

template <class S>
cudaError_t launch_fixup(bool reverse, const S* lam, const S* hprev_row, const S* h, const S* lam_next,
                         S* seg_prod, const S* carry, int64_t carry_stride, const S* scale, S* out0, S* out1,
                         int64_t T, int64_t W, int64_t rows, int64_t nseg, int64_t tseg, int64_t ntt,
                         bool vec_ok, cudaStream_t st) {
  constexpr int V = Tuning<S>::VEC;
  const int64_t nvec = vec_ok ? (W + V - 1) / V : W;
  const int q = pick_q(nvec);
  const int cpw = q * (vec_ok ? V : 1);
  const int64_t ncols = (W + cpw - 1) / cpw;
  // the walk needs seg_prod untouched after the check: only without `scale`
  const int64_t walk = scale == nullptr ? (ntt < 8 ? ntt : 8) : 0;
  const dim3 grid((unsigned)(ncols * nseg * (walk > 0 ? walk : ntt)));
#define FIX(VV)                                                                                       \
  LINREC_Q_SWITCH(q, if (reverse) linrec_dev::k_fixup<S, VV, Q_, true><<<grid, 256, 0, st>>>(         \
                         lam, hprev_row, h, lam_next, seg_prod, carry, carry_stride, scale, out0, out1, T, \
                         W, rows, ncols, nseg, tseg, ntt, walk);                                            \
                     else linrec_dev::k_fixup<S, VV, Q_, false><<<grid, 256, 0, st>>>(                \
                         lam, hprev_row, h, lam_next, seg_prod, carry, carry_stride, scale, out0, out1, T, \
                         W, rows, ncols, nseg, tseg, ntt, walk));
  if (vec_ok) {
    FIX(V)
  } else {
    FIX(1)
  }
#undef FIX
  return cudaGetLastError();
}

template <class S>
cudaError_t launch_vseg_finalize(bool reverse, const S* lam, const S* vagg, int64_t nseg, int64_t tseg, S* carry,
                                 S* scale, S* agg_rank, S* dh0, int64_t W, cudaStream_t st) {
  constexpr int G = 16;
  const unsigned g = (unsigned)((W + 31) / 32);
  if (reverse)
    linrec_dev::k_vseg_finalize<S, true, G><<<g, 32 * G, 0, st>>>(lam, vagg, nseg, tseg, carry, scale, agg_rank, dh0, W);
  else
    linrec_dev::k_vseg_finalize<S, false, G><<<g, 32 * G, 0, st>>>(lam, vagg, nseg, tseg, carry, scale, agg_rank, dh0, W);
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

template cudaError_t launch_fixup<float>(bool, const float*, const float*, const float*, const float*, float*,
                                         const float*, int64_t, const float*, float*, float*, int64_t, int64_t,
                                         int64_t, int64_t, int64_t, int64_t, bool, cudaStream_t);
template cudaError_t launch_fixup<double>(bool, const double*, const double*, const double*, const double*,
                                          double*, const double*, int64_t, const double*, double*, double*,
                                          int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, bool, cudaStream_t);
template cudaError_t launch_compose<float>(const float*, int64_t, int64_t, int64_t, const float*, float*,
                                           int64_t, cudaStream_t);
template cudaError_t launch_compose<double>(const double*, int64_t, int64_t, int64_t, const double*, double*,
                                            int64_t, cudaStream_t);
template cudaError_t launch_vseg_finalize<float>(bool, const float*, const float*, int64_t, int64_t, float*,
                                                 float*, float*, float*, int64_t, cudaStream_t);
template cudaError_t launch_vseg_finalize<double>(bool, const double*, const double*, int64_t, int64_t, double*,
                                                  double*, double*, double*, int64_t, cudaStream_t);

}  // namespace linrec_impl
