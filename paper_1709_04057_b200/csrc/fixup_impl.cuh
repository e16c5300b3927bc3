// Device building blocks of the virtual-segment / sequence-segment stitch
// (the kernels of segment.cu):
//
//   vseg_fold      carries entering each virtual segment from the segments'
//                  aggregates (blocked three-phase fold, fixed association)
//   fixup_position add the decaying contribution P_t * e of a segment's
//                  incoming carry to one tile (chain position)
//   fixup_chain    the positions of one (segment, column) chain that need it:
//                  the entering corrections are checked 8 positions per round
//                  and the non-zero ones form a prefix (a zero correction
//                  stays exactly zero further down the chain), so the walk
//                  stops at the first zero without touching the rest
//
// All run on a team of 8 warps (256 threads) synchronising through a policy
// class (CtaSync: the whole CTA).  A fused variant -- the stitch as the tail
// of the persistent TMA scan behind grid barriers, on named barriers -- was
// measured slower at C4 (one 8-warp team per SM against two resident fix-up
// CTAs) and is not built.
#pragma once

#include <cstdint>

#include "scan_chained.cuh"

namespace linrec_dev {

struct CtaSync {
  static __device__ __forceinline__ void sync() { __syncthreads(); }
  static __device__ __forceinline__ bool sync_or(bool p) { return __syncthreads_or(p) != 0; }
};

template <class S>
struct FixupArgs {
  const S* lam;
  const S* hprev_row;  // bwd: h row before the range (h0 / the previous rank's last row)
  const S* h;
  const S* lam_next;   // bwd: decay of the row after the range
  const S* seg_prod;   // exclusive decay product entering each chain position [nseg*ntt][W]
  S* out0;             // fwd: h; bwd: dx
  S* out1;             // bwd: dlam (nullable)
  int64_t T, W, rows, nseg, tseg, ntt;
};

// Entering correction of chain position p_in of (vseg, column ch): the
// position's product times the carry -- with `scale` (the product from the
// range start to the virtual segment's start, one row per segment) first
// multiplied in, exactly as a rescaled product would have been rounded.
template <class S, int VEC>
__device__ __forceinline__ bool entering(const FixupArgs<S>& f, int64_t vseg, int64_t p_in, int64_t ch,
                                         const S* __restrict__ carry, const S* __restrict__ scale, S (&e)[VEC]) {
  bool nz = false;
  const S* sp = f.seg_prod + (vseg * f.ntt + p_in) * f.W + ch;
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    S p = sp[v];
    if (scale != nullptr) p = mul_(p, scale[vseg * f.W + ch + v]);
    e[v] = mul_(p, carry[ch + v]);
    nz = nz || e[v] != S(0);
  }
  return nz;
}

// One tile (chain position p_in of virtual segment vseg, channel column col)
// of the stitch.  carry[ch] is the carry entering the segment (fwd: state;
// bwd: lam_E * G_E from above); scale as in entering().
template <class S, int VEC, int Q, bool REV, class Sync>
__device__ __forceinline__ void fixup_position(const FixupArgs<S>& f, int64_t vseg, int64_t col, int64_t p_in,
                                               const S* __restrict__ carry, const S* __restrict__ scale,
                                               S (*s_wp)[Q * VEC]) {
  constexpr int NW = 8, RF = 12, G = 32 / Q, CPW = Q * VEC, NSEG = NW * G, PR = NSEG * RF;  // PR = a TMA tile
  using IO = VecIO<S, VEC>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % Q, g = lane / Q;
  const int64_t W = f.W, T = f.T, rows = f.rows;
  const int64_t tile_row = vseg * f.tseg + (REV ? f.ntt - 1 - p_in : p_in) * rows;
  const int64_t ch = col * CPW + (int64_t)q * VEC;
  const bool valid = ch < W;
  S e[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) e[v] = S(0);
  if (valid) entering<S, VEC>(f, vseg, p_in, ch, carry, scale, e);

  const int64_t t_lo = tile_row;
  const int64_t seg_end = (vseg + 1) * f.tseg < T ? (vseg + 1) * f.tseg : T;
  const int64_t t_hi = (t_lo + rows < seg_end ? t_lo + rows : seg_end);
  const int64_t npass = (rows + PR - 1) / PR;
  for (int64_t ps = 0; ps < npass; ++ps) {
    const int64_t pbase = REV ? t_lo + rows - (ps + 1) * PR : t_lo + ps * PR;
    const int seg = warp * G + g;
    S m[RF][VEC], o[RF][VEC];
#pragma unroll
    for (int i = 0; i < RF; ++i) {
      const int64_t t = REV ? pbase + (PR - 1 - (seg * RF + i)) : pbase + seg * RF + i;
      const bool in = valid && t >= t_lo && t < t_hi;
#pragma unroll
      for (int v = 0; v < VEC; ++v) m[i][v] = S(1);
      if (in) IO::load_cg(f.out0 + t * W + ch, o[i]);  // in flight with the decays
      if (in) {
        if (!REV) {
          IO::load_cg(f.lam + t * W + ch, m[i]);
        } else if (t + 1 >= T) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) m[i][v] = f.lam_next != nullptr ? f.lam_next[ch + v] : S(0);
        } else if (f.nseg > 1 && (t + 1) % f.tseg == 0) {
          // end of a virtual segment: mu = 1 (m already 1)
        } else {
          IO::load_cg(f.lam + (t + 1) * W + ch, m[i]);
        }
      }
    }
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
    Sync::sync();
    if (g == G - 1) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) s_wp[warp][q * VEC + v] = A[v];
    }
    Sync::sync();
    S ecur[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) ecur[v] = e[v];
    for (int w = 0; w < warp; ++w)
#pragma unroll
      for (int v = 0; v < VEC; ++v) ecur[v] = mul_(s_wp[w][q * VEC + v], ecur[v]);
#pragma unroll
    for (int v = 0; v < VEC; ++v) ecur[v] = mul_(Ae[v], ecur[v]);
#pragma unroll
    for (int i = 0; i < RF; ++i) {
      const int64_t t = REV ? pbase + (PR - 1 - (seg * RF + i)) : pbase + seg * RF + i;
#pragma unroll
      for (int v = 0; v < VEC; ++v) ecur[v] = mul_(m[i][v], ecur[v]);
      if (valid && t >= t_lo && t < t_hi) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) o[i][v] = o[i][v] + ecur[v];
        IO::store_cg(f.out0 + t * W + ch, o[i]);
        if (REV && f.out1 != nullptr) {
          S hp[VEC], d[VEC];
          if (t >= 1) IO::load_cg(f.h + (t - 1) * W + ch, hp);
          else {
#pragma unroll
            for (int v = 0; v < VEC; ++v) hp[v] = f.hprev_row != nullptr ? f.hprev_row[ch + v] : S(0);
          }
          IO::load_cg(f.out1 + t * W + ch, d);
#pragma unroll
          for (int v = 0; v < VEC; ++v) d[v] = fma_(hp[v], ecur[v], d[v]);
          IO::store_cg(f.out1 + t * W + ch, d);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      S tot = S(1);
      for (int w = 0; w < NW; ++w) tot = mul_(s_wp[w][q * VEC + v], tot);
      e[v] = mul_(tot, e[v]);
    }
  }
  Sync::sync();  // s_wp is reused by the next position
}

// Fix-up of chain (vseg, col) by walker j of J: rounds of 8 positions, warp w
// checking position base + w; walker j then fixes the positions p = j mod J
// of the non-zero prefix.  s_flag: 8 ints of shared memory.
template <class S, int VEC, int Q, bool REV, class Sync>
__device__ __forceinline__ void fixup_chain(const FixupArgs<S>& f, int64_t vseg, int64_t col, int j, int J,
                                            const S* __restrict__ carry, const S* __restrict__ scale,
                                            S (*s_wp)[Q * VEC], int* s_flag) {
  constexpr int NW = 8, CPW = Q * VEC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ch = col * CPW + (int64_t)(lane % Q) * VEC;
  // positions holding rows < T: the last virtual segment is usually short,
  // and its tiles past T (decay 1, nothing to fix) would keep the walk going
  const int64_t seg_rows = (vseg + 1) * f.tseg < f.T ? f.tseg : f.T - vseg * f.tseg;
  const int64_t nreal = seg_rows > 0 ? (seg_rows + f.rows - 1) / f.rows : 0;
  const int64_t p_lo = REV ? f.ntt - nreal : 0, p_hi = REV ? f.ntt : nreal;
  for (int64_t base = p_lo; base < p_hi; base += NW) {
    const int64_t p = base + warp;
    bool nz = false;
    if (p < p_hi && ch < f.W) {
      S e[VEC];
      nz = entering<S, VEC>(f, vseg, p, ch, carry, scale, e);
    }
    nz = __any_sync(0xffffffffu, nz);
    if (lane == 0) s_flag[warp] = nz ? 1 : 0;
    Sync::sync();
    int n = 0;
    while (n < NW && s_flag[n]) ++n;
    Sync::sync();  // flags read before the next round rewrites them
    for (int k = 0; k < n; ++k)
      if ((base + k - p_lo) % J == j) fixup_position<S, VEC, Q, REV, Sync>(f, vseg, col, base + k, carry, scale, s_wp);
    if (n < NW) return;
  }
}

// Virtual-segment finalisation for one 32-channel chunk, on a team of 32*G
// threads (lane = channel, group = a contiguous range of segments).
// forward: carry[s] = state entering segment s (0 for s = 0, whose chain was
//   seeded), scale[s] = decay product of the segments before s, agg_rank =
//   (product over all, final state).
// reverse: carry[s] = lam_E * G_E entering segment s from above (0 for the
//   last), scale[s] = product of the A' of the segments after s, agg_rank =
//   (A', B') of the whole range, dh0 = lam_0 * G_0 (the range's start).
// vagg[s] = (P_incl, c_incl) of segment s's chains.  Fixed association:
// deterministic.
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

template <class S, bool REV, int G, class Sync>
__device__ __forceinline__ void vseg_fold(const S* __restrict__ lam, const S* __restrict__ vagg, int64_t nseg,
                                          int64_t tseg, S* __restrict__ carry, S* __restrict__ scale,
                                          S* __restrict__ agg_rank, S* __restrict__ dh0, int64_t W, int64_t chunk,
                                          S (*sA)[32], S (*sB)[32]) {
  constexpr int PMAX = 32;  // pairs a group keeps in registers (one load round for both passes)
  const int lane = threadIdx.x & 31, g = (threadIdx.x >> 5) % G;
  const int64_t j = chunk * 32 + lane;
  const bool ok = j < W;
  const int64_t per = (nseg + G - 1) / G;
  const int64_t i0 = (int64_t)g * per, i1 = i0 + per < nseg ? i0 + per : nseg;
  const bool regs = per <= PMAX;
  S rA[PMAX], rB[PMAX];
  S Ac = S(1), Bc = S(0);
  if (ok && regs) {
#pragma unroll
    for (int k = 0; k < PMAX; ++k)
      if (i0 + k < i1) vseg_pair<S, REV>(lam, vagg, nseg, tseg, W, i0 + k, j, rA[k], rB[k]);
#pragma unroll
    for (int k = 0; k < PMAX; ++k)
      if (i0 + k < i1) {
        Bc = fma_(rA[k], Bc, rB[k]);
        Ac = mul_(rA[k], Ac);
      }
  } else if (ok) {
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
  Sync::sync();
  S c = S(0), pc = S(1);
  for (int qq = 0; qq < g; ++qq) {
    c = fma_(sA[qq][lane], c, sB[qq][lane]);
    pc = mul_(sA[qq][lane], pc);
  }
  if (ok) {
    if (regs) {
#pragma unroll
      for (int k = 0; k < PMAX; ++k)
        if (i0 + k < i1) {
          const int64_t s = REV ? nseg - 1 - (i0 + k) : i0 + k;
          if (carry != nullptr) carry[s * W + j] = c;
          if (scale != nullptr) scale[s * W + j] = pc;
          c = fma_(rA[k], c, rB[k]);
          pc = mul_(rA[k], pc);
        }
    } else {
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
    }
    if (i1 == nseg && i0 < i1) {  // the group holding the last segment reports the whole range
      if (agg_rank != nullptr) {
        agg_rank[j] = pc;
        agg_rank[W + j] = c;
      }
      if (dh0 != nullptr) dh0[j] = c;
    }
  }
  Sync::sync();  // sA / sB reusable
}

}  // namespace linrec_dev
