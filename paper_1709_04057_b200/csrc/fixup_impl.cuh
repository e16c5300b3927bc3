// Device building blocks of the virtual-segment / sequence-segment stitch
// (the kernels of segment.cu):
//
//   vseg_fold      carries entering each virtual segment from the segments'
//                  aggregates (blocked three-phase fold, fixed association)
//   fixup_position add the decaying contribution P_t * e of a segment's
//                  incoming carry to one tile (chain position)
//   fixup_chain    the positions of one (segment, column) chain that need it:
//                  the non-zero entering corrections form a prefix (a zero
//                  correction stays exactly zero further down the chain), so
//                  the walk stops at the first zero without touching the rest
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
  S* dh0 = nullptr;    // bwd: dh0 += lam_0 * (correction of G_0) (when the fix-up owns the fold)
};

// The carry entering each virtual segment: its own (the fold of the earlier
// virtual segments of the range, rows[vseg]) plus the range's incoming carry
// cin carried to it (scale[vseg] = the decay product from the range start to
// the virtual segment).  Any pointer may be null (no such term).
template <class S>
struct Carries {
  const S* rows;   // [nseg][W]
  const S* scale;  // [nseg][W]
  const S* cin;    // [W]
  // instead of rows: the segments' aggregates [nseg][2][W] (P_incl, c_incl),
  // folded by each fix-up CTA for its own segment (fold_carry) into `own`
  const S* vagg = nullptr;
  const S* own = nullptr;        // its carry, indexed by channel (shared memory: generic loads)
  const S* own_scale = nullptr;  // with cin: the decay product from the range start to the segment
};

// Entering correction of chain position p_in of (vseg, channels ch..): the
// position's product times the segment's carry.
template <class S, int VEC>
__device__ __forceinline__ bool entering(const FixupArgs<S>& f, int64_t vseg, int64_t p_in, int64_t ch,
                                         const Carries<S>& cr, S (&e)[VEC]) {
  using IO = VecIO<S, VEC>;
  S p[VEC], c[VEC], sc[VEC], ci[VEC];
  IO::load_cg(f.seg_prod + (vseg * f.ntt + p_in) * f.W + ch, p);
  if (cr.own != nullptr) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) c[v] = cr.own[ch + v];
  } else if (cr.rows != nullptr) {
    IO::load_cg(cr.rows + vseg * f.W + ch, c);
  }
  if (cr.cin != nullptr) {  // cin / own_scale may live in shared memory: generic loads
    if (cr.own_scale != nullptr) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) sc[v] = cr.own_scale[ch + v];
    } else {
      IO::load_cg(cr.scale + vseg * f.W + ch, sc);
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) ci[v] = cr.cin[ch + v];
  }
  bool nz = false;
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    if (cr.rows == nullptr && cr.own == nullptr) c[v] = S(0);
    if (cr.cin != nullptr) c[v] = fma_(sc[v], ci[v], c[v]);
    e[v] = mul_(p[v], c[v]);
    nz = nz || e[v] != S(0);
  }
  return nz;
}

// One tile (chain position p_in of virtual segment vseg, channel column col)
// of the stitch; cr gives the carry entering the segment (fwd: state; bwd:
// lam_E * G_E from above).  The tile's rows are
// loaded together with its entering correction and, for p_next >= 0, the
// correction entering p_next (*more: non-zero in this thread's channels);
// returns false (nothing stored) when this position's correction is zero in
// every channel of the tile.
template <class S, int VEC, int Q, bool REV, class Sync, int RF = 12>
__device__ __forceinline__ bool fixup_position(const FixupArgs<S>& f, int64_t vseg, int64_t col, int64_t p_in,
                                               const Carries<S>& cr, S (*s_wp)[Q * VEC], int64_t p_next = -1,
                                               bool* more = nullptr) {
  // RF rows per thread: PR = NSEG * RF rows per pass (12: one 96-row tile per
  // pass; 6: two passes at half the registers, two CTAs per SM)
  constexpr int NW = 8, G = 32 / Q, CPW = Q * VEC, NSEG = NW * G, PR = NSEG * RF;
  using IO = VecIO<S, VEC>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % Q, g = lane / Q;
  const int seg = warp * G + g;
  const int64_t W = f.W, T = f.T, rows = f.rows;
  const int64_t t_lo = vseg * f.tseg + (REV ? f.ntt - 1 - p_in : p_in) * rows;
  const int64_t ch = col * CPW + (int64_t)q * VEC;
  const bool valid = ch < W;
  S e[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) e[v] = S(0);

  // the virtual segment's last row + 1 (its top, where the backward decay
  // mu = lam_{t+1} is replaced by 1 -- or by lam_next at T)
  const int64_t seg_top = (vseg + 1) * f.tseg < T ? (vseg + 1) * f.tseg : T;
  const int64_t t_hi = t_lo + rows < seg_top ? t_lo + rows : seg_top;
  const int64_t npass = (rows + PR - 1) / PR;
  const bool dl = REV && f.out1 != nullptr;
  for (int64_t ps = 0; ps < npass; ++ps) {
    // this thread's rows: t = t0 + i (forward) / t0 - i (backward), i < RF,
    // those in [t_lo, t_hi) being i in [ilo, ihi)
    const int64_t pbase = REV ? t_lo + rows - (ps + 1) * PR : t_lo + ps * PR;
    const int64_t t0 = REV ? pbase + PR - 1 - seg * RF : pbase + seg * RF;
    int ilo, ihi;
    if (!REV) {
      ilo = (int)(t_lo - t0 > 0 ? t_lo - t0 : 0);
      ihi = (int)(t_hi - t0 < RF ? t_hi - t0 : RF);
    } else {
      ilo = (int)(t0 - t_hi + 1 > 0 ? t0 - t_hi + 1 : 0);
      ihi = (int)(t0 - t_lo + 1 < RF ? t0 - t_lo + 1 : RF);
    }
    if (!valid) ihi = 0;
    const int64_t step = REV ? -W : W;
    const S* lam_p = f.lam + (t0 + (REV ? 1 : 0)) * W + ch;  // the decay applied at row t0
    S* out_p = f.out0 + t0 * W + ch;
    const int itop = REV ? (int)(t0 - (seg_top - 1)) : -1;  // i of the segment's top row
    // backward with dlam: dx and h_{t-1} are loaded in the same round as the
    // decays (one load round per position: the fix-up of a deep walk -- decays
    // near 1 -- is a streaming pass, bounded by the bytes each SM has in flight)
    S* d_p = REV ? f.out1 + t0 * W + ch : nullptr;
    const S* h_p = REV ? f.h + (t0 - 1) * W + ch : nullptr;
    const int izero = (int)t0;  // i of row 0 (h_{-1} = hprev_row)
    S m[RF][VEC], o[RF][VEC], hq[REV ? RF : 1][VEC];
#pragma unroll
    for (int i = 0; i < RF; ++i) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) m[i][v] = S(1);
      if (i >= ilo && i < ihi) {
        IO::load_cg(out_p + i * step, o[i]);  // in flight with the decays
        if constexpr (REV) {
          if (dl) {
            if (i != izero) {
              IO::load_cg(h_p + i * step, hq[i]);
            } else {
#pragma unroll
              for (int v = 0; v < VEC; ++v) hq[i][v] = f.hprev_row != nullptr ? f.hprev_row[ch + v] : S(0);
            }
          }
        }
        if (!REV || i != itop) {
          IO::load_cg(lam_p + i * step, m[i]);
        } else if (seg_top == T) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) m[i][v] = f.lam_next != nullptr ? f.lam_next[ch + v] : S(0);
        }  // else the top of an inner virtual segment: mu = 1
      }
    }
    if (ps == 0 && valid) {  // issued behind the tile's loads: one load round
      entering<S, VEC>(f, vseg, p_in, ch, cr, e);
      if (p_next >= 0) {
        S en[VEC];
        *more = entering<S, VEC>(f, vseg, p_next, ch, cr, en);
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
    bool nzl = false;
#pragma unroll
    for (int v = 0; v < VEC; ++v) nzl = nzl || e[v] != S(0);
    if (!Sync::sync_or(nzl)) return false;  // uniform: the rest of the walk is zero too
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
    // m[i] <- the correction of row i
#pragma unroll
    for (int i = 0; i < RF; ++i)
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        ecur[v] = mul_(m[i][v], ecur[v]);
        m[i][v] = ecur[v];
      }
    if (REV && f.dh0 != nullptr && t0 < RF && (int)t0 >= ilo && (int)t0 < ihi) {  // this thread holds row 0
      S l0[VEC], d[VEC];
      IO::load_cg(f.lam + ch, l0);
      IO::load_cg(f.dh0 + ch, d);
#pragma unroll
      for (int i = 0; i < RF; ++i)
        if (i == (int)t0)
#pragma unroll
          for (int v = 0; v < VEC; ++v) d[v] = fma_(l0[v], m[i][v], d[v]);
      IO::store_cg(f.dh0 + ch, d);
    }
    if (!dl) {
#pragma unroll
      for (int i = 0; i < RF; ++i)
        if (i >= ilo && i < ihi) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) o[i][v] = o[i][v] + m[i][v];
          IO::store_cg(out_p + i * step, o[i]);
        }
    } else if constexpr (REV) {
      // backward with dlam: dlam is recomputed from the corrected dx as the
      // scan computes it (dlam_t = h_{t-1} * g_t), so the old dlam is not read
#pragma unroll
      for (int i = 0; i < RF; ++i)
        if (i >= ilo && i < ihi) {
          S d[VEC];
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            o[i][v] = o[i][v] + m[i][v];
            d[v] = mul_(hq[i][v], o[i][v]);
          }
          IO::store_cg(out_p + i * step, o[i]);
          IO::store_cg(d_p + i * step, d);
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
  return true;
}

// The carry entering virtual segment vseg for this thread's channels: the
// fold of the aggregates of the segments before it (forward: 0 .. vseg-1;
// backward, from the top: nseg-1 .. vseg+1 with each pair scaled by the
// decay at its segment's first row, as vseg_pair), c = A c + B from 0.  The
// 8*G walkers of the team fold contiguous groups, combined in walker order
// through shared memory s_a / s_b [8*G][CPW] (fixed association).
template <class S, int VEC, int Q, bool REV, class Sync>
__device__ __forceinline__ void fold_carry(const FixupArgs<S>& f, const S* __restrict__ vagg, int64_t vseg,
                                           int64_t col, S* s_a, S* s_b, S (&carry)[VEC], S (&scale)[VEC]) {
  constexpr int G = 32 / Q, CPW = Q * VEC, NWK = 8 * G;
  using IO = VecIO<S, VEC>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % Q, k = warp * G + lane / Q;
  const int64_t ch = col * CPW + (int64_t)q * VEC;
  const bool valid = ch < f.W;
  const int64_t n = REV ? f.nseg - 1 - vseg : vseg;  // segments to fold
  const int64_t per = (n + NWK - 1) / NWK;
  const int64_t i0 = k * per, i1 = i0 + per < n ? i0 + per : n;
  S A[VEC], B[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { A[v] = S(1); B[v] = S(0); }
  constexpr int FOLD_UNROLL = REV ? 4 : 8;  // backward pairs carry a third load (the decay)
  if (valid)
#pragma unroll FOLD_UNROLL
    for (int64_t i = i0; i < i1; ++i) {  // unrolled: the pairs' loads are in flight together
      const int64_t sg = REV ? f.nseg - 1 - i : i;
      S a[VEC], b[VEC];
      IO::load_cg(vagg + sg * 2 * f.W + ch, a);
      IO::load_cg(vagg + sg * 2 * f.W + f.W + ch, b);
      if (REV) {
        S l0[VEC];
        IO::load_cg(f.lam + (sg * f.tseg) * f.W + ch, l0);
#pragma unroll
        for (int v = 0; v < VEC; ++v) { a[v] = mul_(l0[v], a[v]); b[v] = mul_(l0[v], b[v]); }
      }
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        B[v] = fma_(a[v], B[v], b[v]);
        A[v] = mul_(a[v], A[v]);
      }
    }
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    s_a[k * CPW + q * VEC + v] = A[v];
    s_b[k * CPW + q * VEC + v] = B[v];
  }
  Sync::sync();
#pragma unroll
  for (int v = 0; v < VEC; ++v) { carry[v] = S(0); scale[v] = S(1); }
  for (int w = 0; w < NWK; ++w)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      carry[v] = fma_(s_a[w * CPW + q * VEC + v], carry[v], s_b[w * CPW + q * VEC + v]);
      scale[v] = mul_(s_a[w * CPW + q * VEC + v], scale[v]);
    }
  Sync::sync();  // s_a / s_b reusable
}

// Fix-up of chain (vseg, col) by walker j of J: positions p_lo + j, + J, ...
// in order, each tile loaded together with the entering correction of the
// walker's next position (one load round per position); the walk stops at
// the first position whose correction is zero in every channel.
template <class S, int VEC, int Q, bool REV, class Sync, int RF = 12>
__device__ __forceinline__ void fixup_chain(const FixupArgs<S>& f, int64_t vseg, int64_t col, int j, int J,
                                            const Carries<S>& cr, S (*s_wp)[Q * VEC]) {
  // positions holding rows < T: the last virtual segment is usually short,
  // and its tiles past T (decay 1, nothing to fix) would keep the walk going
  const int64_t seg_rows = (vseg + 1) * f.tseg < f.T ? f.tseg : f.T - vseg * f.tseg;
  const int64_t nreal = seg_rows > 0 ? (seg_rows + f.rows - 1) / f.rows : 0;
  const int64_t p_lo = REV ? f.ntt - nreal : 0, p_hi = REV ? f.ntt : nreal;
  for (int64_t p = p_lo + j; p < p_hi; p += J) {
    bool more = false;
    if (!fixup_position<S, VEC, Q, REV, Sync, RF>(f, vseg, col, p, cr, s_wp, p + J < p_hi ? p + J : -1, &more))
      return;
    if (!Sync::sync_or(more)) return;
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
