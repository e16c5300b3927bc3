// Persistent, warp-specialised chained scans fed by TMA (sm_100a).
//
// Same algorithm and bit-for-bit the same arithmetic order as the register
// kernels of scan_chained.cuh (so the look-back stays deterministic), but the
// memory system is kept busy continuously:
//
//   warp NW+1  producer     takes the next chunk ticket, issues one 2-D
//                           cp.async.bulk.tensor per input array into a
//                           STAGES-deep shared-memory ring (mbarrier
//                           complete_tx), zero-filling rows/channels outside
//                           the tensor;
//   warps 0..NW-1 consumers copy their R rows x VEC channels of the staged tile
//                           into registers, release the ring slot at once,
//                           reduce them to an affine pair, publish warp
//                           totals, wait for the tile's carry and re-scan,
//                           storing results with 128-bit streaming stores;
//   warp NW    coordinator  folds the warp totals into the tile aggregate and
//                           runs the decoupled look-back (chain_lookback).
//
// One CTA (or two) per SM loops over tiles until the ticket counter passes the
// tile count, so up to STAGES tiles per CTA are in flight while earlier tiles
// wait for their carries: the look-back latency is hidden behind TMA traffic.
#pragma once

#include <type_traits>

#include "p2p_impl.cuh"
#include "scan_chained.cuh"
#include "tma_util.cuh"

namespace linrec_dev {

// Largest divisor of L that fits a TMA box dimension (<= 256).
constexpr int box_rows_for(int L) {
  for (int b = L < 256 ? L : 256; b > 1; --b)
    if (L % b == 0) return b;
  return 1;
}

template <class S, int VEC, int Q, int R, int NW, int STAGES, int NARR>
struct TmaCfg {
  static constexpr int kVEC = VEC, kQ = Q, kR = R, kNW = NW, kSTAGES = STAGES, kNARR = NARR;
  static constexpr int G = 32 / Q;
  static constexpr int CPW = Q * VEC;
  static constexpr int NSEG = NW * G;
  static constexpr int L = NSEG * R;
  static constexpr int BOX_ROWS = box_rows_for(L);
  static constexpr int NBOX = L / BOX_ROWS;
  static_assert(L % BOX_ROWS == 0, "tile rows must be a multiple of the TMA box");
  static constexpr int ARR_BYTES = ((L * CPW * (int)sizeof(S) + 127) / 128) * 128;
  static constexpr int STAGE_BYTES = NARR * ARR_BYTES;
  static constexpr int TX_BYTES = NARR * L * CPW * (int)sizeof(S);
  static constexpr int OFF_TOT = STAGES * STAGE_BYTES;  // [2][2][NW][CPW]
  static constexpr int OFF_CARRY = OFF_TOT + 2 * 2 * NW * CPW * (int)sizeof(S);  // [2][CPW]
  static constexpr int OFF_META = ((OFF_CARRY + 2 * CPW * (int)sizeof(S)) + 15) / 16 * 16;
  static constexpr int OFF_BAR = OFF_META + STAGES * 8;
  static constexpr int SMEM = OFF_BAR + (2 * STAGES + 4) * 8;
  static constexpr int THREADS = (NW + 2) * 32;
  static constexpr int REC = ChainCfg<S, VEC, Q, R, NW>::REC;
};

template <class Cfg, class S>
struct TmaSmem {
  unsigned char* base;
  __device__ S* arr(int stage, int a) const {
    return reinterpret_cast<S*>(base + stage * Cfg::STAGE_BYTES + a * Cfg::ARR_BYTES);
  }
  __device__ S* tot_a(int slot) const {
    return reinterpret_cast<S*>(base + Cfg::OFF_TOT) + slot * 2 * Cfg::kNW * Cfg::CPW;
  }
  __device__ S* tot_b(int slot) const { return tot_a(slot) + Cfg::kNW * Cfg::CPW; }
  __device__ S* carry(int slot) const {
    return reinterpret_cast<S*>(base + Cfg::OFF_CARRY) + slot * Cfg::CPW;
  }
  __device__ long long* meta() const { return reinterpret_cast<long long*>(base + Cfg::OFF_META); }
  __device__ uint64_t* full(int s) const { return reinterpret_cast<uint64_t*>(base + Cfg::OFF_BAR) + s; }
  __device__ uint64_t* empty(int s) const {
    return reinterpret_cast<uint64_t*>(base + Cfg::OFF_BAR) + Cfg::kSTAGES + s;
  }
  __device__ uint64_t* aggr(int slot) const {
    return reinterpret_cast<uint64_t*>(base + Cfg::OFF_BAR) + 2 * Cfg::kSTAGES + slot;
  }
  __device__ uint64_t* carry_bar(int slot) const {
    return reinterpret_cast<uint64_t*>(base + Cfg::OFF_BAR) + 2 * Cfg::kSTAGES + 2 + slot;
  }
};

// Barrier setup shared by both directions.
template <class Cfg, class SM>
__device__ __forceinline__ void tma_init_barriers(const SM& sm) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::kSTAGES; ++s) {
      mbar_init(sm.full(s), 1);
      mbar_init(sm.empty(s), (Cfg::kNW + 1) * 32);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(sm.aggr(i), Cfg::kNW * 32);
      mbar_init(sm.carry_bar(i), 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
}

// Coordinator warp loop (both directions).
template <class Cfg, class S, bool REV, class SM>
__device__ __forceinline__ bool tma_coordinator(const SM& sm, const ChainArgs<S>& a, const ChainWs& ws,
                                                uint32_t epoch, bool deep) {
  constexpr int VEC = Cfg::kVEC, Q = Cfg::kQ, NW = Cfg::kNW, CPW = Cfg::CPW, STAGES = Cfg::kSTAGES;
  const int lane = threadIdx.x & 31;
  for (int n = 0;; ++n) {
    const int s = n % STAGES;
    mbar_wait(sm.full(s), (n / STAGES) & 1);
    const long long k = sm.meta()[s];
    mbar_arrive(sm.empty(s));
    if (k < 0) break;
    const int slot = n & 1;
    mbar_wait(sm.aggr(slot), (n >> 1) & 1);
    const ChainPos cp = chain_pos(a, k);
    const int64_t ch = cp.col * CPW + (int64_t)lane * VEC;
    const bool valid = lane < Q && ch < a.W;
    S TA[VEC], TB[VEC], c[VEC], P[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) { TA[v] = S(1); TB[v] = S(0); c[v] = S(0); P[v] = S(1); }
    if (lane < Q) {
      const S* ta = sm.tot_a(slot);
      const S* tb = sm.tot_b(slot);
      constexpr int w0 = REV ? NW - 1 : 0;
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        TA[v] = ta[w0 * CPW + lane * VEC + v];
        TB[v] = tb[w0 * CPW + lane * VEC + v];
      }
#pragma unroll
      for (int i = 1; i < NW; ++i) {
        const int w = REV ? NW - 1 - i : i;
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          TB[v] = fma_(ta[w * CPW + lane * VEC + v], TB[v], tb[w * CPW + lane * VEC + v]);
          TA[v] = mul_(ta[w * CPW + lane * VEC + v], TA[v]);
        }
      }
      if (cp.pos == 0 && cp.seg == (REV ? a.nseg - 1 : 0) && a.seed != nullptr && valid) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) c[v] = a.seed[ch + v];
      } else if (deep && cp.pos == 0 && a.seed_rows != nullptr && valid) {
        // decay-adaptive stitch, deep mode: the true carry entering this
        // virtual segment (reduce pass + fold), so no fix-up follows
#pragma unroll
        for (int v = 0; v < VEC; ++v) c[v] = a.seed_rows[cp.seg * a.W + ch + v];
      }
    }
    // the reduce-only pass (role 1) stores nothing: its consumers need no
    // carry, so they are released as soon as this tile's totals are read and
    // run ahead at load speed while the look-back below resolves the chain
    // (its aggregate, agg_out, is what the pass is for).  The slot's totals
    // are not overwritten early: the consumers' next use of this slot waits
    // for this release.
    const bool early = a.role == 1;
    if (early) {
      __syncwarp();
      mbar_arrive(sm.carry_bar(slot));
    }
    const bool want_p = a.seg_prod != nullptr || a.agg_out != nullptr;
    Lookback<S, VEC, Q, Cfg::REC>::exclusive(ws, epoch, k, cp.pos, cp.chain, cp.nchains, TA, TB, c, P, valid,
                                             want_p);
    if (lane < Q && !early) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) sm.carry(slot)[lane * VEC + v] = c[v];
    }
    if (!early) mbar_arrive(sm.carry_bar(slot));  // consumers re-scan while the carry is published
    Lookback<S, VEC, Q, Cfg::REC>::publish(ws, epoch, k, TA, TB, c, P, valid, want_p);
    write_segment_outputs<S, VEC, Q>(a, cp, ch, valid, TA, TB, c, P);
  }
  return chain_retire(ws, epoch);
}

// Tail of a sequence-sharded launch (ChainArgs::tail_fold), run by the whole
// CTA that retired last: the rank aggregate (P, c) of the virtual segments'
// aggregates -- each 128-channel block as float4 lanes, the warps folding
// contiguous segment groups combined in order (backward: pairs scaled by the
// decay at each segment's first row, dh0 = c) -- then stored into every
// consumer's mailbox and their flags released.  scratch: 2 x warps x 128
// floats of shared memory.
template <bool REV>
__device__ __forceinline__ void tail_fold_publish(const ChainArgs<float>& a, float* scratch) {
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5, ngr = blockDim.x >> 5;
  float* sA = scratch;
  float* sB = scratch + ngr * 128;
  const int64_t W = a.W, nseg = a.nseg;
  const int64_t per = (nseg + ngr - 1) / ngr;
  const int64_t i0 = g * per, i1 = i0 + per < nseg ? i0 + per : nseg;
  for (int64_t c0 = 0; c0 < W; c0 += 128) {
    const int64_t ch = c0 + 4 * lane;
    const bool valid = ch < W;
    float A[4] = {1.f, 1.f, 1.f, 1.f}, B[4] = {0.f, 0.f, 0.f, 0.f};
    if (valid)
#pragma unroll 8
      for (int64_t i = i0; i < i1; ++i) {  // pairs in flight together
        const int64_t sg = REV ? nseg - 1 - i : i;
        const float4 av = __ldcg(reinterpret_cast<const float4*>(a.agg_out + sg * 2 * W + ch));
        const float4 bv = __ldcg(reinterpret_cast<const float4*>(a.agg_out + sg * 2 * W + W + ch));
        float x[4] = {av.x, av.y, av.z, av.w}, y[4] = {bv.x, bv.y, bv.z, bv.w};
        if (REV) {
          const float4 l0 = __ldcg(reinterpret_cast<const float4*>(a.a + (sg * a.tseg) * W + ch));
          const float l[4] = {l0.x, l0.y, l0.z, l0.w};
#pragma unroll
          for (int v = 0; v < 4; ++v) { x[v] = mul_(l[v], x[v]); y[v] = mul_(l[v], y[v]); }
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          B[v] = fma_(x[v], B[v], y[v]);
          A[v] = mul_(x[v], A[v]);
        }
      }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      sA[g * 128 + 4 * lane + v] = A[v];
      sB[g * 128 + 4 * lane + v] = B[v];
    }
    __syncthreads();
    if (g == 0 && valid) {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        float c = 0.f, pc = 1.f;
        for (int w = 0; w < ngr; ++w) {
          c = fma_(sA[w * 128 + 4 * lane + v], c, sB[w * 128 + 4 * lane + v]);
          pc = mul_(sA[w * 128 + 4 * lane + v], pc);
        }
        a.rank_agg[ch + v] = pc;
        a.rank_agg[W + ch + v] = c;
        if (REV && a.out2 != nullptr) a.out2[ch + v] = c;
      }
    }
    __syncthreads();
  }
  if (!a.ex.has_consumers()) return;
  const p2p::MboxLayout L = p2p::layout(a.ex);
  void* own = a.ex.mboxes[a.ex.rank];
  for (int q = a.ex.q0; q < a.ex.q1; ++q) {
    if (q == a.ex.rank) continue;
    if (threadIdx.x == 0) p2p::wait_geq(L.ack(own, a.ex.dir, q), a.ex.epoch - 1);  // q read the previous epoch
    __syncthreads();
    float* dst = L.slot(a.ex.mboxes[q], a.ex.dir, a.ex.rank);
    for (int64_t j = threadIdx.x; j < W; j += blockDim.x) {
      dst[j] = a.ex.zero_a ? 0.f : a.rank_agg[j];
      dst[W + j] = a.rank_agg[W + j];
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = a.ex.q0; q < a.ex.q1; ++q)
      if (q != a.ex.rank) p2p::st_release_sys(L.flag(a.ex.mboxes[q], a.ex.dir, a.ex.rank), a.ex.epoch);
}

// Common end of the TMA kernels with a tail fold: every warp arrives here;
// only the CTA that retired last (s_last, set by its coordinator) continues.
template <class S, bool REV>
__device__ __forceinline__ void tma_tail(const ChainArgs<S>& a, const int* s_last, unsigned char* scratch) {
  __syncthreads();
  if (!*s_last) return;
  __threadfence();  // the other CTAs' aggregates (they fenced before retiring)
  if constexpr (std::is_same<S, float>::value) tail_fold_publish<REV>(a, reinterpret_cast<float*>(scratch));
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
template <class S, int VEC, int Q, int R, int NW, int STAGES>
__global__ void __launch_bounds__((NW + 2) * 32, 1)
k_tma_fwd(const __grid_constant__ CUtensorMap map_lam, const __grid_constant__ CUtensorMap map_x,
          const ChainArgs<S> a, const ChainWs ws, const long long ntiles) {
  using Cfg = TmaCfg<S, VEC, Q, R, NW, STAGES, 2>;
  using IO = VecIO<S, VEC>;
  constexpr int G = Cfg::G, CPW = Cfg::CPW, L = Cfg::L;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const TmaSmem<Cfg, S> sm{smem_raw};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // decay-adaptive stitch: the reduce-only pass runs only in deep mode
  const bool deep = a.mode != nullptr && __ldcg(a.mode) != 0;
  if (role_skips(a.role, deep)) return;
  tma_init_barriers<Cfg>(sm);
  const uint32_t epoch = __ldcg(&ws.ctrl->epoch);
  __shared__ int s_last;  // tail fold: this CTA retired last

  if (warp == NW + 1) {  // ---------------- producer
    if (lane == 0) {
      prefetch_tmap(&map_lam);
      prefetch_tmap(&map_x);
      const uint64_t pol = policy_evict_first(), pol_keep = policy_evict_last();
      for (int n = 0;; ++n) {
        const int s = n % STAGES;
        if (n >= STAGES) mbar_wait(sm.empty(s), ((n / STAGES) + 1) & 1);
        const long long k = (long long)atomicAdd(&ws.ctrl->ticket, 1ull);
        if (k >= ntiles) {
          sm.meta()[s] = -1;
          mbar_arrive(sm.full(s));
          break;
        }
        sm.meta()[s] = k;
        const ChainPos cp = chain_pos(a, (int64_t)k);
        const int c0 = (int)(cp.col * CPW);
        const int r0 = (int)tile_row0<false>(a, cp, L);
        const bool keep = a.seg_prod != nullptr && cp.pos < kKeepPositions;  // revisited by the fix-up
        mbar_arrive_expect_tx(sm.full(s), Cfg::TX_BYTES);
#pragma unroll
        for (int b = 0; b < Cfg::NBOX; ++b) {
          tma_load_2d(sm.arr(s, 0) + b * Cfg::BOX_ROWS * CPW, &map_lam, c0, r0 + b * Cfg::BOX_ROWS, sm.full(s),
                      keep ? pol_keep : pol);
          tma_load_2d(sm.arr(s, 1) + b * Cfg::BOX_ROWS * CPW, &map_x, c0, r0 + b * Cfg::BOX_ROWS, sm.full(s), pol);
        }
      }
    }
  } else if (warp == NW) {  // ---------------- coordinator
    const bool last = tma_coordinator<Cfg, S, false>(sm, a, ws, epoch, deep);
    if (lane == 0) s_last = last ? 1 : 0;
  } else {

  // ---------------------------------- consumers
  const uint64_t pol_keep = policy_evict_last();
  const int q = lane % Q, g = lane / Q;
  const int seg = warp * G + g;
  const int64_t W = a.W;
  for (int n = 0;; ++n) {
    const int s = n % STAGES;
    mbar_wait(sm.full(s), (n / STAGES) & 1);
    const long long k = sm.meta()[s];
    if (k < 0) break;
    const ChainPos cp = chain_pos(a, (int64_t)k);
    const bool keep = a.seg_prod != nullptr && cp.pos < kKeepPositions;
    const int64_t ch = cp.col * CPW + (int64_t)q * VEC;
    const bool valid = ch < W;
    const int t0 = tile_row0<false>(a, cp, L) + seg * R;
    const int Ti = (int)a.T;
    S l[R][VEC], xv[R][VEC];
    const S* sl = sm.arr(s, 0) + seg * R * CPW + q * VEC;
    const S* sx = sm.arr(s, 1) + seg * R * CPW + q * VEC;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (t0 + i < Ti) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) { l[i][v] = sl[i * CPW + v]; xv[i][v] = sx[i * CPW + v]; }
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) { l[i][v] = S(1); xv[i][v] = S(0); }
      }
    }
    mbar_arrive(sm.empty(s));  // tile is in registers: the ring slot can refill

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
    const int slot = n & 1;
    S* ta = sm.tot_a(slot);
    S* tb = sm.tot_b(slot);
    if (g == G - 1) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        ta[warp * CPW + q * VEC + v] = A[v];
        tb[warp * CPW + q * VEC + v] = B[v];
      }
    }
    mbar_arrive(sm.aggr(slot));
    mbar_wait(sm.carry_bar(slot), (n >> 1) & 1);

    S cs[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) cs[v] = sm.carry(slot)[q * VEC + v];
    for (int w = 0; w < warp; ++w)
#pragma unroll
      for (int v = 0; v < VEC; ++v) cs[v] = fma_(ta[w * CPW + q * VEC + v], cs[v], tb[w * CPW + q * VEC + v]);
#pragma unroll
    for (int v = 0; v < VEC; ++v) cs[v] = fma_(Ae[v], cs[v], Be[v]);
#pragma unroll
    for (int i = 0; i < R; ++i) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) cs[v] = fma_(l[i][v], cs[v], xv[i][v]);
      const int t = t0 + i;
      if (valid && t < Ti && a.out0 != nullptr) {  // (reduce-only pass: no outputs)
        if (keep) IO::store_hint(a.out0 + t * W + ch, cs, pol_keep);
        else IO::store_stream(a.out0 + t * W + ch, cs);
      }
    }
  }
  }  // consumers
  // one barrier site for every role (the tail fold's __syncthreads)
  if (a.tail_fold) tma_tail<S, false>(a, &s_last, smem_raw);
}

// ---------------------------------------------------------------------------
// backward (reverse time): arrays mu = lam shifted +1 row, dh, h shifted -1 row
// ---------------------------------------------------------------------------
// GATED: a fourth staged array g (map_gate) multiplies the adjoint as it is
// copied out of shared memory -- the scan runs on dh * g, so a gated layer
// output h = g * c needs no separate dc = dh * g pass (GILR-LSTM / QRNN).
template <class S, int VEC, int Q, int R, int NW, int STAGES, bool GATED = false>
__global__ void __launch_bounds__((NW + 2) * 32, 1)
k_tma_bwd(const __grid_constant__ CUtensorMap map_lam, const __grid_constant__ CUtensorMap map_dh,
          const __grid_constant__ CUtensorMap map_h, const __grid_constant__ CUtensorMap map_gate,
          const ChainArgs<S> a, const ChainWs ws, const long long ntiles) {
  using Cfg = TmaCfg<S, VEC, Q, R, NW, STAGES, GATED ? 4 : 3>;
  using IO = VecIO<S, VEC>;
  constexpr int G = Cfg::G, CPW = Cfg::CPW, L = Cfg::L;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const TmaSmem<Cfg, S> sm{smem_raw};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // decay-adaptive stitch: the reduce-only pass runs only in deep mode
  const bool deep = a.mode != nullptr && __ldcg(a.mode) != 0;
  if (role_skips(a.role, deep)) return;
  tma_init_barriers<Cfg>(sm);
  const uint32_t epoch = __ldcg(&ws.ctrl->epoch);
  __shared__ int s_last;  // tail fold: this CTA retired last

  if (warp == NW + 1) {  // ---------------- producer
    if (lane == 0) {
      prefetch_tmap(&map_lam);
      prefetch_tmap(&map_dh);
      prefetch_tmap(&map_h);
      if (GATED) prefetch_tmap(&map_gate);
      const uint64_t pol = policy_evict_first(), pol_keep = policy_evict_last();
      for (int n = 0;; ++n) {
        const int s = n % STAGES;
        if (n >= STAGES) mbar_wait(sm.empty(s), ((n / STAGES) + 1) & 1);
        const long long k = (long long)atomicAdd(&ws.ctrl->ticket, 1ull);
        if (k >= ntiles) {
          sm.meta()[s] = -1;
          mbar_arrive(sm.full(s));
          break;
        }
        sm.meta()[s] = k;
        const ChainPos cp = chain_pos(a, (int64_t)k);
        const int c0 = (int)(cp.col * CPW);
        const int r0 = (int)tile_row0<true>(a, cp, L);
        const bool keep = a.seg_prod != nullptr && cp.pos < kKeepPositions;  // revisited by the fix-up
        // the reduce-only pass (role 1) needs mu and the adjoint, not h: it
        // stages 8 B/el instead of 12 (the h box is not loaded)
        const bool need_h = a.role != 1;
        mbar_arrive_expect_tx(sm.full(s), need_h ? Cfg::TX_BYTES : Cfg::TX_BYTES / Cfg::kNARR * (Cfg::kNARR - 1));
#pragma unroll
        for (int b = 0; b < Cfg::NBOX; ++b) {
          const int rb = r0 + b * Cfg::BOX_ROWS;
          tma_load_2d(sm.arr(s, 0) + b * Cfg::BOX_ROWS * CPW, &map_lam, c0, rb + 1, sm.full(s),
                      keep ? pol_keep : pol);
          tma_load_2d(sm.arr(s, 1) + b * Cfg::BOX_ROWS * CPW, &map_dh, c0, rb, sm.full(s), pol);
          if (need_h)
            tma_load_2d(sm.arr(s, 2) + b * Cfg::BOX_ROWS * CPW, &map_h, c0, rb - 1, sm.full(s),
                        keep ? pol_keep : pol);
          if (GATED) tma_load_2d(sm.arr(s, GATED ? 3 : 0) + b * Cfg::BOX_ROWS * CPW, &map_gate, c0, rb, sm.full(s), pol);
        }
      }
    }
  } else if (warp == NW) {  // ---------------- coordinator
    const bool last = tma_coordinator<Cfg, S, true>(sm, a, ws, epoch, deep);
    if (lane == 0) s_last = last ? 1 : 0;
  } else {

  // ---------------------------------- consumers
  const uint64_t pol_keep = policy_evict_last();
  const int q = lane % Q, g = lane / Q;
  const int seg = warp * G + g;
  const int64_t W = a.W, T = a.T;
  for (int n = 0;; ++n) {
    const int s = n % STAGES;
    mbar_wait(sm.full(s), (n / STAGES) & 1);
    const long long k = sm.meta()[s];
    if (k < 0) break;
    const ChainPos cp = chain_pos(a, (int64_t)k);
    const bool keep = a.seg_prod != nullptr && cp.pos < kKeepPositions;
    const int64_t ch = cp.col * CPW + (int64_t)q * VEC;
    const bool valid = ch < W;
    const int t0 = tile_row0<true>(a, cp, L) + seg * R;
    const int Ti = (int)a.T, se = vseg_end(a, cp);
    S mu[R][VEC], dh[R][VEC], hp[R][VEC];
    const S* smu = sm.arr(s, 0) + seg * R * CPW + q * VEC;
    const S* sdh = sm.arr(s, 1) + seg * R * CPW + q * VEC;
    const S* shp = sm.arr(s, 2) + seg * R * CPW + q * VEC;
    const S* sg = sm.arr(s, GATED ? 3 : 0) + seg * R * CPW + q * VEC;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int t = t0 + i;
      if (t < Ti) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          mu[i][v] = smu[i * CPW + v];
          dh[i][v] = GATED ? sdh[i * CPW + v] * sg[i * CPW + v] : sdh[i * CPW + v];
          hp[i][v] = shp[i * CPW + v];
        }
        const int mk = mu_kind(t, Ti, se);
        if (mk == 2) {  // zero-filled past the end; the segment form supplies lam_next
#pragma unroll
          for (int v = 0; v < VEC; ++v) mu[i][v] = (a.lam_next != nullptr && valid) ? a.lam_next[ch + v] : S(0);
        } else if (mk == 1) {  // end of a virtual segment: linked by the carry fold
#pragma unroll
          for (int v = 0; v < VEC; ++v) mu[i][v] = S(1);
        }
        if (t == 0) {  // zero-filled row -1 -> h0
#pragma unroll
          for (int v = 0; v < VEC; ++v) hp[i][v] = (a.aux != nullptr && valid) ? a.aux[ch + v] : S(0);
        }
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) { mu[i][v] = S(1); dh[i][v] = S(0); hp[i][v] = S(0); }
      }
    }
    mbar_arrive(sm.empty(s));

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
    const int slot = n & 1;
    S* ta = sm.tot_a(slot);
    S* tb = sm.tot_b(slot);
    if (g == 0) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        ta[warp * CPW + q * VEC + v] = A[v];
        tb[warp * CPW + q * VEC + v] = B[v];
      }
    }
    mbar_arrive(sm.aggr(slot));
    mbar_wait(sm.carry_bar(slot), (n >> 1) & 1);

    S cs[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) cs[v] = sm.carry(slot)[q * VEC + v];
    for (int w = NW - 1; w > warp; --w)
#pragma unroll
      for (int v = 0; v < VEC; ++v) cs[v] = fma_(ta[w * CPW + q * VEC + v], cs[v], tb[w * CPW + q * VEC + v]);
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
      if (valid && t < Ti && a.out0 != nullptr) {  // (reduce-only pass: no outputs)
        if (keep) {
          IO::store_hint(a.out0 + t * W + ch, cs, pol_keep);
          if (a.out1 != nullptr) IO::store_hint(a.out1 + t * W + ch, dl, pol_keep);
        } else {
          IO::store_stream(a.out0 + t * W + ch, cs);
          if (a.out1 != nullptr) IO::store_stream(a.out1 + t * W + ch, dl);
        }
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
  }  // consumers
  // one barrier site for every role (the tail fold's __syncthreads)
  if (a.tail_fold) tma_tail<S, true>(a, &s_last, smem_raw);
}

}  // namespace linrec_dev
