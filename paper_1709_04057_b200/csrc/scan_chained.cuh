// Single-pass chained scans (forward and reverse-time backward) for sm_100a.
//
// Replaces the reference's three-phase chunked scan (recurrence.hpp:193-245:
// phase 1 chunk_summary, phase 2 sequential stitch, phase 3 seeded re-scan)
// and its reversed-copy backward (recurrence.hpp:283-348) with ONE pass over
// HBM: every element of the inputs is read once and every output written
// once (fp32: 12 B/element forward, 20 B/element backward).
//
// Decomposition.  The [T][W] tensor is cut into tiles of L rows x CPW
// channels.  Channels are independent (recurrence.hpp:109), so each of the
// ncols = ceil(W/CPW) channel columns is its own chain of T/L tiles.
//   * A thread owns VEC adjacent channels (128-bit vector) and R consecutive
//     rows, held in registers: it loads them once, reduces them to an affine
//     pair (A = prod lam, B = zero-seeded result) -- the reference's
//     chunk_summary (recurrence.hpp:114-131) at register granularity.
//   * Lanes are split Q across channels x G = 32/Q along time; the G row
//     segments of a warp are combined with __shfl_up_sync, the NW warps of
//     the CTA through shared memory.  Pair algebra: applying (A1,B1) then
//     (A2,B2) is (A2*A1, A2*B1 + B2).
//   * Tiles obtain their position from an atomic ticket (launch order), so
//     every predecessor of a tile is resident or retired: the look-back
//     always makes progress.  A coordinator warp (warp NW, holding no tile
//     data) publishes the tile aggregate, looks
//     back over up to 32 predecessors per round (one flag per lane, one
//     ballot), finds the nearest predecessor whose inclusive carry is
//     published, and APPLIES the intermediate aggregates to that carry oldest
//     first.  Because inclusive carries are defined by sequential
//     application, the carry each tile obtains is bit-identical whichever
//     predecessor the look-back stopped at: the scan is deterministic run to
//     run although the look-back is decoupled.
//   * The tile's registers are then re-scanned from the carry (the
//     reference's phase 3, recurrence.hpp:232-237) and written back with
//     streaming 128-bit stores.
// The backward runs the same machinery in reverse time on
// G_t = lam_{t+1} G_{t+1} + dh_t with mu_t = lam_{t+1} read through a
// one-row shift (no reversed copies, cf. recurrence.hpp:305-318) and fuses
// dx = G, dlam = h_{t-1} G, dh0 = lam_1 G_1 (recurrence.hpp:331-346) into the
// re-scan.
#pragma once

#include "launch.h"
#include "linrec_device.cuh"

namespace linrec_dev {

template <class S, int VEC, int Q, int R, int NW>
struct ChainCfg {
  static constexpr int G = 32 / Q;          // lane groups along time per warp
  static constexpr int CPW = Q * VEC;       // channels per column (tile width)
  static constexpr int NSEG = NW * G;       // row segments per tile
  static constexpr int L = NSEG * R;        // rows per tile
  static constexpr int THREADS = (NW + 1) * 32;  // + coordinator warp
  // carry record: two halves of REC 8-byte slots each (fp32: tagged words,
  // fp64: values), padded to 128-byte lines
  static constexpr int REC = ((CPW * 8 + 127) / 128) * 128 / 8;
};

// Workspace view of one chained launch (see capi.cpp for the layout).
struct ChainWs {
  Ctrl* ctrl;
  uint32_t* flags;   // [ntiles]
  void* agg;         // [ntiles][2][REC] tile aggregates (A, B)
  void* inc;         // [ntiles][2][REC] inclusive carries (P, c)
};

template <class S>
struct ChainArgs {
  // forward: a = lam, b = x, out0 = h
  // backward: a = lam, b = dh, c = h, out0 = dx, out1 = dlam, out2 = dh0
  const S* a;
  const S* b;
  const S* c;
  const S* seed;      // fwd: h0 (nullable); bwd: g_next (nullable)
  const S* aux;       // bwd: h0 (nullable) ; fwd: unused
  const S* lam_next;  // bwd: decay of the row after the segment (nullable)
  S* out0;
  S* out1;
  S* out2;
  // segment outputs (sequence sharding): exclusive decay product of every
  // chain position [ntt][W] and the chain's final (P_incl, c_incl) [2][W]
  S* seg_prod;
  S* agg_out;
  int64_t T;
  int64_t W;
  int64_t ncols;
  int64_t ntt;        // tiles along time per chain (per virtual segment)
  int64_t nseg;       // virtual T-segments scanned as independent chains (>= 1)
  int64_t tseg;       // rows per virtual segment (a multiple of the tile rows)
  // sequence-sharded TMA scans at W <= 256 (fp32): the CTA that retires last
  // folds the segments' aggregates (agg_out) into the rank aggregate
  // rank_agg [2][W] (backward: also dh0 = out2) and publishes it to the
  // consumers' mailboxes (ex) -- no separate fold launch before the exchange
  int tail_fold;
  S* rank_agg;
  linrec_impl::Exchange ex;
  // decay-adaptive stitch (TMA kernels): mode word (nullable; 1 = deep),
  // role (1 = reduce-only pass: runs only when deep, stores no outputs;
  // 2 = the unsplit twin of a wide scan, one chain per column: runs only when
  // deep; 3 = the split scan whose twin exists: runs only when not deep), and
  // the carries entering the virtual segments [nseg][W] a deep scan seeds
  // its chains with (no fix-up follows)
  const int* mode;
  int role;
  const S* seed_rows;
};

// Does a launch of this role sit out the current decay mode (decay-adaptive
// stitch, capi.cpp)?  Role 0 always runs.
__device__ __forceinline__ bool role_skips(int role, bool deep) {
  return ((role == 1 || role == 2) && !deep) || (role == 3 && deep);
}

// Position of ticket k: chain = (virtual segment, channel column), tiles in
// ticket order along the chain (so the look-back predecessor is k - nchains).
// 32-bit arithmetic: tickets < 2^31 and T < 2^31 are enforced by the host.
struct ChainPos {
  int nchains, chain, pos, col, seg;
};
template <class S>
__device__ __forceinline__ ChainPos chain_pos(const ChainArgs<S>& a, int64_t k) {
  ChainPos p;
  p.nchains = (int)(a.ncols * a.nseg);
  const unsigned kk = (unsigned)k, nc = (unsigned)p.nchains;
  p.pos = (int)(kk / nc);
  p.chain = (int)(kk - (unsigned)p.pos * nc);
  p.seg = (int)((unsigned)p.chain / (unsigned)a.ncols);
  p.col = p.chain - p.seg * (int)a.ncols;
  return p;
}
// first row of the tile at chain position pos; REV walks each segment from
// its last tile to its first
template <bool REV, class S>
__device__ __forceinline__ int tile_row0(const ChainArgs<S>& a, const ChainPos& p, int L) {
  return p.seg * (int)a.tseg + (REV ? (int)a.ntt - 1 - p.pos : p.pos) * L;
}
// Row after which the reverse scan's decay is 1 (the end of a non-final
// virtual segment: that link is applied by the carry fold), or INT_MAX.
template <class S>
__device__ __forceinline__ int vseg_end(const ChainArgs<S>& a, const ChainPos& p) {
  return (a.nseg > 1 && p.seg < a.nseg - 1) ? (p.seg + 1) * (int)a.tseg : 0x7fffffff;
}
// decay linking row t to row t+1 in the reverse scan (mu_t = lam_{t+1}):
// 2 = end of the sequence (lam_next, or 0), 1 = end of a virtual segment (1),
// 0 = lam[t+1]
__device__ __forceinline__ int mu_kind(int t, int T, int seg_end) {
  return t + 1 >= T ? 2 : (t + 1 == seg_end ? 1 : 0);
}

// ---------------------------------------------------------------------------
// Decoupled look-back, split in two so the tile's data warps can start their
// re-scan before the tile's inclusive carry is published:
//   Lookback<S,...>::exclusive()  -> exclusive carry (c = state entering the
//                                    tile, P = decay product from the chain
//                                    start) on lanes < Q; publishes the tile
//                                    aggregate when it has to wait;
//   Lookback<S,...>::publish()    -> inclusive carry of the tile.
// Carries are APPLIED oldest first to the nearest published inclusive value,
// so every tile obtains bit-identical carries whichever predecessor its look-
// back stopped at (deterministic scan).
//
// fp32: every record element is one self-validating 64-bit word
// (value << 32 | epoch << 2 | state) written and read with relaxed gpu-scope
// 128-bit vector accesses (each 64-bit element is single-copy atomic), so no
// memory fences and no separate flag are needed; each lane walks back over
// its own channels.  (A warp-wide flag window was measured slower on B200:
// the per-lane word probe is one round trip shorter on the common path.)  fp64 values do not fit beside a tag, so the fp64 path
// keeps value records + one release/acquire flag per tile.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_words2(uint64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_words2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_word(uint64_t* p, uint64_t a) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
}
__device__ __forceinline__ uint64_t ld_word(const uint64_t* p) {
  uint64_t a;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(a) : "l"(p) : "memory");
  return a;
}

template <int VEC>
__device__ __forceinline__ void store_words(uint64_t* p, const float (&v)[VEC], uint32_t tag) {
  uint64_t w[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) w[i] = ((uint64_t)__float_as_uint(v[i]) << 32) | tag;
  if constexpr (VEC % 2 == 0) {
#pragma unroll
    for (int i = 0; i < VEC; i += 2) st_words2(p + i, w[i], w[i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) st_word(p + i, w[i]);
  }
}

// Loads VEC words; returns true when every tag equals `tag`.
template <int VEC>
__device__ __forceinline__ bool load_words(const uint64_t* p, float (&v)[VEC], uint32_t tag) {
  uint64_t w[VEC];
  if constexpr (VEC % 2 == 0) {
#pragma unroll
    for (int i = 0; i < VEC; i += 2) ld_words2(p + i, w[i], w[i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) w[i] = ld_word(p + i);
  }
  bool ok = true;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    ok = ok && (uint32_t)w[i] == tag;
    v[i] = __uint_as_float((uint32_t)(w[i] >> 32));
  }
  return ok;
}

template <class S, int VEC, int Q, int REC>
struct Lookback;

// fp32: self-validating words.
template <int VEC, int Q, int REC>
struct Lookback<float, VEC, Q, REC> {
  // agg record k: words [k*2*REC, +CPW) = A, [k*2*REC + REC, +CPW) = B
  // inc record k: words [k*2*REC, +CPW) = c, [k*2*REC + REC, +CPW) = P
  static __device__ __forceinline__ void exclusive(const ChainWs& ws, uint32_t epoch, int64_t k,
                                                   int64_t pos, int64_t col, int64_t ncols,
                                                   const float (&TA)[VEC], const float (&TB)[VEC],
                                                   float (&c)[VEC], float (&P)[VEC], bool valid,
                                                   bool WANT_P) {
    const int lane = threadIdx.x & 31;
    if (pos == 0 || !(lane < Q && valid)) return;
    uint64_t* agg = reinterpret_cast<uint64_t*>(ws.agg);
    const uint64_t* inc = reinterpret_cast<const uint64_t*>(ws.inc);
    const int off = lane * VEC;
    const uint32_t tinc = (epoch << 2) | kFlagInc, tagg = (epoch << 2) | kFlagAgg;
    // fast path (one round trip): the predecessor's inclusive carry
    int64_t j = pos - 1;
    const uint64_t* r0 = inc + (j * ncols + col) * 2 * REC + off;
    if (load_words<VEC>(r0, c, tinc) && (!WANT_P || load_words<VEC>(r0 + REC, P, tinc))) return;
    // publish our aggregate so successors need not wait for our carry
    uint64_t* ra = agg + k * 2 * REC + off;
    store_words<VEC>(ra, TA, tagg);
    store_words<VEC>(ra + REC, TB, tagg);
    // walk back: inclusive carry of j, or step over j once its aggregate is
    // visible
    SpinGuard guard;
    for (;;) {
      guard.tick();
      const uint64_t* ri = inc + (j * ncols + col) * 2 * REC + off;
      if (load_words<VEC>(ri, c, tinc) && (!WANT_P || load_words<VEC>(ri + REC, P, tinc))) break;
      const uint64_t* rg = agg + (j * ncols + col) * 2 * REC + off;
      float a[VEC], b[VEC];
      if (load_words<VEC>(rg, a, tagg) & load_words<VEC>(rg + REC, b, tagg)) --j;
    }
    // apply the aggregates of j+1 .. pos-1, oldest first (all visible now),
    // four positions' loads in flight per round
#pragma unroll 1
    for (int64_t i = j + 1; i < pos; i += 4) {
      float a[4][VEC], b[4][VEC];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u < pos) {
          const uint64_t* rg = agg + ((i + u) * ncols + col) * 2 * REC + off;
          load_words<VEC>(rg, a[u], tagg);
          load_words<VEC>(rg + REC, b[u], tagg);
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u < pos)
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            c[v] = fma_(a[u][v], c[v], b[u][v]);
            if (WANT_P) P[v] = mul_(a[u][v], P[v]);
          }
    }
  }

  static __device__ __forceinline__ void publish(const ChainWs& ws, uint32_t epoch, int64_t k,
                                                 const float (&TA)[VEC], const float (&TB)[VEC],
                                                 const float (&c)[VEC], const float (&P)[VEC],
                                                 bool valid, bool WANT_P) {
    publish_words(ws, epoch, k, TA, TB, c, P, valid, WANT_P);
  }

  static __device__ __forceinline__ void publish_words(const ChainWs& ws, uint32_t epoch, int64_t k,
                                                       const float (&TA)[VEC], const float (&TB)[VEC],
                                                       const float (&c)[VEC], const float (&P)[VEC],
                                                       bool valid, bool WANT_P) {
    const int lane = threadIdx.x & 31;
    if (!(lane < Q && valid)) return;
    uint64_t* inc = reinterpret_cast<uint64_t*>(ws.inc);
    const uint32_t tinc = (epoch << 2) | kFlagInc;
    float ci[VEC], Pi[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      ci[v] = fma_(TA[v], c[v], TB[v]);
      Pi[v] = mul_(TA[v], P[v]);
    }
    uint64_t* r = inc + k * 2 * REC + lane * VEC;
    if (WANT_P) store_words<VEC>(r + REC, Pi, tinc);
    store_words<VEC>(r, ci, tinc);
  }

};

// fp64: value records + per-tile release/acquire flag.
template <int VEC, int Q, int REC>
struct Lookback<double, VEC, Q, REC> {
  using S = double;
  using IO = VecIO<S, VEC>;
  static __device__ __forceinline__ void exclusive(const ChainWs& ws, uint32_t epoch, int64_t k,
                                                   int64_t pos, int64_t col, int64_t ncols,
                                                   const S (&TA)[VEC], const S (&TB)[VEC],
                                                   S (&c)[VEC], S (&P)[VEC], bool valid,
                                                   bool /*want_p: fp64 records always carry P*/) {
    if (pos == 0) return;
    const int lane = threadIdx.x & 31;
    S* agg = reinterpret_cast<S*>(ws.agg);
    S* inc = reinterpret_cast<S*>(ws.inc);
    const bool owner = lane < Q && valid;
    const int off = lane * VEC;
    if (owner) {
      S* rec = agg + k * 2 * REC + off;
      IO::store_cg(rec, TA);
      IO::store_cg(rec + REC, TB);
      fence_acq_rel_gpu();
    }
    __syncwarp();
    if (lane == 0) st_release_gpu(&ws.flags[k], (epoch << 2) | kFlagAgg);
    int64_t jhi = pos - 1, jinc = 0;
    for (;;) {
      const int64_t jj = jhi - lane;
      bool is_inc = false;
      if (jj >= 0) {
        const uint32_t* fp = &ws.flags[jj * ncols + col];
        uint32_t f = ld_acquire_gpu(fp);
        SpinGuard guard;
        while ((f >> 2) != epoch) {
          guard.tick();
          f = ld_acquire_gpu(fp);
        }
        is_inc = (f & 3u) == kFlagInc;
      }
      const unsigned m = __ballot_sync(0xffffffffu, is_inc);
      if (m) {
        jinc = jhi - (__ffs(m) - 1);
        break;
      }
      jhi -= 32;
    }
    if (owner) {
      const S* rec = inc + (jinc * ncols + col) * 2 * REC + off;
      IO::load_cg(rec, c);
      IO::load_cg(rec + REC, P);
#pragma unroll 1
      for (int64_t j = jinc + 1; j < pos; ++j) {
        S a1[VEC], b1[VEC];
        const S* r = agg + (j * ncols + col) * 2 * REC + off;
        IO::load_cg(r, a1);
        IO::load_cg(r + REC, b1);
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          c[v] = fma_(a1[v], c[v], b1[v]);
          P[v] = mul_(a1[v], P[v]);
        }
      }
    }
  }

  static __device__ __forceinline__ void publish(const ChainWs& ws, uint32_t epoch, int64_t k,
                                                 const S (&TA)[VEC], const S (&TB)[VEC],
                                                 const S (&c)[VEC], const S (&P)[VEC], bool valid,
                                                 bool /*want_p*/) {
    const int lane = threadIdx.x & 31;
    S* inc = reinterpret_cast<S*>(ws.inc);
    if (lane < Q && valid) {
      S ci[VEC], Pi[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        ci[v] = fma_(TA[v], c[v], TB[v]);
        Pi[v] = mul_(TA[v], P[v]);
      }
      S* rec = inc + k * 2 * REC + lane * VEC;
      IO::store_cg(rec, ci);
      IO::store_cg(rec + REC, Pi);
      fence_acq_rel_gpu();
    }
    __syncwarp();
    if (lane == 0) st_release_gpu(&ws.flags[k], (epoch << 2) | kFlagInc);
  }
};

// Segment outputs of the coordinator (no-ops unless the launch asked for them):
// the tile's exclusive decay product per channel, and for the last tile of a
// chain the chain's inclusive (P, c).
template <class S, int VEC, int Q>
__device__ __forceinline__ void write_segment_outputs(const ChainArgs<S>& a, const ChainPos& cp, int64_t ch,
                                                      bool valid, const S (&TA)[VEC],
                                                      const S (&TB)[VEC], const S (&c)[VEC],
                                                      const S (&P)[VEC]) {
  const int lane = threadIdx.x & 31;
  if (!(lane < Q && valid)) return;
  if (a.seg_prod != nullptr) {
    S* sp = a.seg_prod + (cp.seg * a.ntt + cp.pos) * a.W + ch;
#pragma unroll
    for (int v = 0; v < VEC; ++v) sp[v] = P[v];
  }
  if (a.agg_out != nullptr && cp.pos == a.ntt - 1) {
    S* ag = a.agg_out + cp.seg * 2 * a.W + ch;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      ag[v] = mul_(TA[v], P[v]);
      ag[a.W + v] = fma_(TA[v], c[v], TB[v]);
    }
  }
}

// Named barriers between the NW data warps and the coordinator warp.
__device__ __forceinline__ void bar_arrive(int id, int n) {
  __threadfence_block();
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void chain_ticket(const ChainWs& ws, unsigned long long* s_k,
                                             uint32_t* s_epoch) {
  if (threadIdx.x == 0) {
    *s_epoch = __ldcg(&ws.ctrl->epoch);
    *s_k = atomicAdd(&ws.ctrl->ticket, 1ull);
  }
}

// Called by the coordinator warp once the CTA no longer needs the control
// block; the CTA that retires last resets the ticket and advances the epoch
// for the next launch on this workspace.  Returns (on lane 0) whether this
// CTA retired last.
__device__ __forceinline__ bool chain_retire(const ChainWs& ws, uint32_t epoch) {
  bool last = false;
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    const unsigned long long r = atomicAdd(&ws.ctrl->retired, 1ull);
    if (r == (unsigned long long)gridDim.x - 1ull) {
      ws.ctrl->ticket = 0ull;
      ws.ctrl->retired = 0ull;
      ws.ctrl->epoch = next_epoch(epoch);
      __threadfence();
      last = true;
    }
  }
  return last;
}

// ---------------------------------------------------------------------------
// Coordinator warp (warp NW of the CTA): waits for the data warps' segment
// totals, folds them into the tile aggregate, runs the look-back and hands the
// tile's exclusive carry to the data warps through shared memory.  Keeping the
// look-back in its own warp keeps its registers out of the data warps, whose
// register file holds the tile.
// ---------------------------------------------------------------------------
template <class S, int VEC, int Q, int NW, int CPW, int REC, bool REV>
__device__ __forceinline__ void chain_coordinator(const ChainArgs<S>& a, const ChainWs& ws,
                                                  uint32_t epoch, int64_t k, const ChainPos& cp,
                                                  S (*s_wa)[CPW], S (*s_wb)[CPW], S* s_c) {
  constexpr int NT = (NW + 1) * 32;
  const int lane = threadIdx.x & 31;
  const int64_t ch = cp.col * CPW + (int64_t)lane * VEC;
  const bool valid = lane < Q && ch < a.W;
  bar_sync(1, NT);  // segment totals are in shared memory
  S TA[VEC], TB[VEC], c[VEC], P[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { TA[v] = S(1); TB[v] = S(0); c[v] = S(0); P[v] = S(1); }
  if (lane < Q) {
    constexpr int w0 = REV ? NW - 1 : 0;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      TA[v] = s_wa[w0][lane * VEC + v];
      TB[v] = s_wb[w0][lane * VEC + v];
    }
#pragma unroll
    for (int i = 1; i < NW; ++i) {
      const int w = REV ? NW - 1 - i : i;
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        TB[v] = fma_(s_wa[w][lane * VEC + v], TB[v], s_wb[w][lane * VEC + v]);
        TA[v] = mul_(s_wa[w][lane * VEC + v], TA[v]);
      }
    }
    if (cp.pos == 0 && cp.seg == (REV ? a.nseg - 1 : 0) && a.seed != nullptr && valid) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) c[v] = a.seed[ch + v];
    }
  }
  const bool want_p = a.seg_prod != nullptr || a.agg_out != nullptr;
  Lookback<S, VEC, Q, REC>::exclusive(ws, epoch, k, cp.pos, cp.chain, cp.nchains, TA, TB, c, P, valid,
                                      want_p);
  if (lane < Q) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) s_c[lane * VEC + v] = c[v];
  }
  bar_arrive(2, NT);  // carry is in shared memory: the data warps re-scan now
  Lookback<S, VEC, Q, REC>::publish(ws, epoch, k, TA, TB, c, P, valid, want_p);
  write_segment_outputs<S, VEC, Q>(a, cp, ch, valid, TA, TB, c, P);
  chain_retire(ws, epoch);
}

// ---------------------------------------------------------------------------
// Forward: h_t = lam_t h_{t-1} + x_t, seeded with h0 (or 0).
// ---------------------------------------------------------------------------
template <class S, int VEC, int Q, int R, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 2)
k_chain_fwd(const ChainArgs<S> a, const ChainWs ws) {
  using Cfg = ChainCfg<S, VEC, Q, R, NW>;
  using IO = VecIO<S, VEC>;
  constexpr int G = Cfg::G, CPW = Cfg::CPW, L = Cfg::L;
  constexpr int NT = (NW + 1) * 32;
  __shared__ S s_wa[NW][CPW];
  __shared__ S s_wb[NW][CPW];
  __shared__ S s_c[CPW];
  __shared__ unsigned long long s_k;
  __shared__ uint32_t s_epoch;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  chain_ticket(ws, &s_k, &s_epoch);
  __syncthreads();
  const int64_t k = (int64_t)s_k;
  const uint32_t epoch = s_epoch;
  const ChainPos cp = chain_pos(a, k);

  if (warp == NW) {
    chain_coordinator<S, VEC, Q, NW, CPW, Cfg::REC, false>(a, ws, epoch, k, cp, s_wa, s_wb, s_c);
    return;
  }

  const int q = lane % Q, g = lane / Q;
  const int64_t ch = cp.col * CPW + (int64_t)q * VEC;
  const bool valid = ch < a.W;
  const int t0 = tile_row0<false>(a, cp, L) + (warp * G + g) * R;
  const int Ti = (int)a.T;
  const int64_t W = a.W;

  S l[R][VEC], xv[R][VEC];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int t = t0 + i;
    if (valid && t < Ti) {
      IO::load_stream(a.a + t * W + ch, l[i]);
      IO::load_stream(a.b + t * W + ch, xv[i]);
    } else {
#pragma unroll
      for (int v = 0; v < VEC; ++v) { l[i][v] = S(1); xv[i][v] = S(0); }
    }
  }

  // segment aggregate (chunk_summary at register granularity)
  S A[VEC], B[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { A[v] = l[0][v]; B[v] = xv[0][v]; }
#pragma unroll
  for (int i = 1; i < R; ++i)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      B[v] = fma_(l[i][v], B[v], xv[i][v]);
      A[v] = mul_(l[i][v], A[v]);
    }

  // inclusive scan over the G row segments of the warp
#pragma unroll
  for (int off = 1; off < G; off <<= 1) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const S ap = __shfl_up_sync(0xffffffffu, A[v], off * Q);
      const S bp = __shfl_up_sync(0xffffffffu, B[v], off * Q);
      if (g >= off) {
        B[v] = fma_(A[v], bp, B[v]);
        A[v] = mul_(A[v], ap);
      }
    }
  }
  S Ae[VEC], Be[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    Ae[v] = S(1);
    Be[v] = S(0);
    if (G > 1) {
      const S ap = __shfl_up_sync(0xffffffffu, A[v], Q);
      const S bp = __shfl_up_sync(0xffffffffu, B[v], Q);
      if (g > 0) { Ae[v] = ap; Be[v] = bp; }
    }
  }
  if (g == G - 1) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      s_wa[warp][q * VEC + v] = A[v];
      s_wb[warp][q * VEC + v] = B[v];
    }
  }
  bar_arrive(1, NT);
  bar_sync(2, NT);

  // seed of this thread's rows: carry, then earlier warps, then earlier groups
  S cs[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) cs[v] = s_c[q * VEC + v];
  for (int w = 0; w < warp; ++w)
#pragma unroll
    for (int v = 0; v < VEC; ++v)
      cs[v] = fma_(s_wa[w][q * VEC + v], cs[v], s_wb[w][q * VEC + v]);
#pragma unroll
  for (int v = 0; v < VEC; ++v) cs[v] = fma_(Ae[v], cs[v], Be[v]);

#pragma unroll
  for (int i = 0; i < R; ++i) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) cs[v] = fma_(l[i][v], cs[v], xv[i][v]);
    const int t = t0 + i;
    if (valid && t < Ti) IO::store_stream(a.out0 + t * W + ch, cs);
  }
}

// ---------------------------------------------------------------------------
// Backward: G_t = mu_t G_{t+1} + dh_t, mu_t = lam_{t+1} (lam_next for the
// last row, 0 at the true end), processed from the last tile to the first.
// dx_t = G_t, dlam_t = h_{t-1} G_t (h0 for t = 0), dh0 = lam_0 G_0.
// ---------------------------------------------------------------------------
template <class S, int VEC, int Q, int R, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 2)
k_chain_bwd(const ChainArgs<S> a, const ChainWs ws) {
  using Cfg = ChainCfg<S, VEC, Q, R, NW>;
  using IO = VecIO<S, VEC>;
  constexpr int G = Cfg::G, CPW = Cfg::CPW, L = Cfg::L;
  constexpr int NT = (NW + 1) * 32;
  __shared__ S s_wa[NW][CPW];
  __shared__ S s_wb[NW][CPW];
  __shared__ S s_c[CPW];
  __shared__ unsigned long long s_k;
  __shared__ uint32_t s_epoch;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  chain_ticket(ws, &s_k, &s_epoch);
  __syncthreads();
  const int64_t k = (int64_t)s_k;
  const uint32_t epoch = s_epoch;
  const ChainPos cp = chain_pos(a, k);

  if (warp == NW) {
    chain_coordinator<S, VEC, Q, NW, CPW, Cfg::REC, true>(a, ws, epoch, k, cp, s_wa, s_wb, s_c);
    return;
  }

  const int q = lane % Q, g = lane / Q;
  const int64_t ch = cp.col * CPW + (int64_t)q * VEC;
  const bool valid = ch < a.W;
  const int t0 = tile_row0<true>(a, cp, L) + (warp * G + g) * R;
  const int Ti = (int)a.T, se = vseg_end(a, cp);
  const int64_t W = a.W, T = a.T;

  S mu[R][VEC], dh[R][VEC], hp[R][VEC];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int t = t0 + i;
    if (valid && t < Ti) {
      const int mk = mu_kind(t, Ti, se);
      if (mk == 0) {
        IO::load_stream(a.a + (t + 1) * W + ch, mu[i]);
      } else if (mk == 1) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) mu[i][v] = S(1);
      } else if (a.lam_next != nullptr) {
        IO::load_cg(a.lam_next + ch, mu[i]);
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) mu[i][v] = S(0);
      }
      IO::load_stream(a.b + t * W + ch, dh[i]);
      if (t >= 1) {
        IO::load_stream(a.c + (t - 1) * W + ch, hp[i]);
      } else if (a.aux != nullptr) {
        IO::load_cg(a.aux + ch, hp[i]);
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) hp[i][v] = S(0);
      }
    } else {
#pragma unroll
      for (int v = 0; v < VEC; ++v) { mu[i][v] = S(1); dh[i][v] = S(0); hp[i][v] = S(0); }
    }
  }

  // segment aggregate, latest row first
  S A[VEC], B[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { A[v] = mu[R - 1][v]; B[v] = dh[R - 1][v]; }
#pragma unroll
  for (int i = R - 2; i >= 0; --i)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      B[v] = fma_(mu[i][v], B[v], dh[i][v]);
      A[v] = mul_(mu[i][v], A[v]);
    }

  // inclusive scan over the warp's row segments in reverse time
#pragma unroll
  for (int off = 1; off < G; off <<= 1) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const S ap = __shfl_down_sync(0xffffffffu, A[v], off * Q);
      const S bp = __shfl_down_sync(0xffffffffu, B[v], off * Q);
      if (g + off < G) {
        B[v] = fma_(A[v], bp, B[v]);
        A[v] = mul_(A[v], ap);
      }
    }
  }
  S Ae[VEC], Be[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    Ae[v] = S(1);
    Be[v] = S(0);
    if (G > 1) {
      const S ap = __shfl_down_sync(0xffffffffu, A[v], Q);
      const S bp = __shfl_down_sync(0xffffffffu, B[v], Q);
      if (g < G - 1) { Ae[v] = ap; Be[v] = bp; }
    }
  }
  if (g == 0) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      s_wa[warp][q * VEC + v] = A[v];
      s_wb[warp][q * VEC + v] = B[v];
    }
  }
  bar_arrive(1, NT);
  bar_sync(2, NT);

  S cs[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) cs[v] = s_c[q * VEC + v];
  for (int w = NW - 1; w > warp; --w)
#pragma unroll
    for (int v = 0; v < VEC; ++v)
      cs[v] = fma_(s_wa[w][q * VEC + v], cs[v], s_wb[w][q * VEC + v]);
#pragma unroll
  for (int v = 0; v < VEC; ++v) cs[v] = fma_(Ae[v], cs[v], Be[v]);

#pragma unroll
  for (int i = R - 1; i >= 0; --i) {
    S dl[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      cs[v] = fma_(mu[i][v], cs[v], dh[i][v]);
      dl[v] = mul_(hp[i][v], cs[v]);
    }
    const int t = t0 + i;
    if (valid && t < Ti) {
      IO::store_stream(a.out0 + t * W + ch, cs);
      if (a.out1 != nullptr) IO::store_stream(a.out1 + t * W + ch, dl);
      if (t == 0 && a.out2 != nullptr) {
        S l0[VEC], d0[VEC];
        IO::load_cg(a.a + ch, l0);
#pragma unroll
        for (int v = 0; v < VEC; ++v) d0[v] = mul_(l0[v], cs[v]);
        IO::store_cg(a.out2 + ch, d0);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Serial per-channel kernels: ScanMode::Serial on the GPU.  One thread per
// VEC channels walks the whole sequence with the reference's exact operation
// order (scan_span, recurrence.hpp:101-112; reversed scan + assembly,
// :309-346), so the result is bit-identical to the reference's serial scan.
// U rows of loads are kept in flight per thread.
// ---------------------------------------------------------------------------
template <class S, int VEC, int U>
__global__ void __launch_bounds__(128)
k_serial_fwd(const S* __restrict__ lam, const S* __restrict__ x, const S* __restrict__ h0,
             S* __restrict__ h, int64_t T, int64_t W) {
  using IO = VecIO<S, VEC>;
  const int64_t ch = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC;
  if (ch >= W) return;
  S c[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) c[v] = h0 ? h0[ch + v] : S(0);
  for (int64_t t0 = 0; t0 < T; t0 += U) {
    S l[U][VEC], xv[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (t0 + u < T) {
        IO::load_stream(lam + (t0 + u) * W + ch, l[u]);
        IO::load_stream(x + (t0 + u) * W + ch, xv[u]);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (t0 + u < T) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) c[v] = fma_(l[u][v], c[v], xv[u][v]);
        IO::store_stream(h + (t0 + u) * W + ch, c);
      }
  }
}

template <class S, int VEC, int U>
__global__ void __launch_bounds__(128)
k_serial_bwd(const S* __restrict__ lam, const S* __restrict__ h0, const S* __restrict__ h,
             const S* __restrict__ dh, const S* __restrict__ lam_next,
             const S* __restrict__ g_next, S* __restrict__ dlam, S* __restrict__ dx,
             S* __restrict__ dh0, int64_t T, int64_t W) {
  using IO = VecIO<S, VEC>;
  const int64_t ch = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC;
  if (ch >= W) return;
  S G[VEC], mu_last[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    G[v] = g_next ? g_next[ch + v] : S(0);
    mu_last[v] = lam_next ? lam_next[ch + v] : S(0);
  }
  for (int64_t t1 = T - 1; t1 >= 0; t1 -= U) {
    S mu[U][VEC], d[U][VEC], hp[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = t1 - u;
      if (t >= 0) {
        if (t + 1 < T) IO::load_stream(lam + (t + 1) * W + ch, mu[u]);
        else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) mu[u][v] = mu_last[v];
        }
        IO::load_stream(dh + t * W + ch, d[u]);
        if (t >= 1) IO::load_stream(h + (t - 1) * W + ch, hp[u]);
        else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) hp[u][v] = h0 ? h0[ch + v] : S(0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = t1 - u;
      if (t >= 0) {
        S dl[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          G[v] = fma_(mu[u][v], G[v], d[u][v]);
          dl[v] = mul_(hp[u][v], G[v]);
        }
        IO::store_stream(dx + t * W + ch, G);
        if (dlam != nullptr) IO::store_stream(dlam + t * W + ch, dl);
      }
    }
  }
  if (dh0) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) dh0[ch + v] = mul_(lam[ch + v], G[v]);
  }
}

}  // namespace linrec_dev
