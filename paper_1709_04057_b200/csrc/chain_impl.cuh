// Runtime dispatch of the chained-scan templates (included once per
// dtype/direction translation unit so nvcc compiles them in parallel).
#pragma once

#include <cstdlib>

#include "launch.h"
#include "scan_chained.cuh"

namespace linrec_impl {

template <class S>
struct Tuning;
// forward: 2 arrays in registers (lam, x); backward: 3 (mu, dh, h_{t-1})
template <>
struct Tuning<float> {
  static constexpr int VEC = 4, FWD_R = 6, FWD_NW = 8, BWD_R = 4, BWD_NW = 8;
};
template <>
struct Tuning<double> {
  static constexpr int VEC = 2, FWD_R = 6, FWD_NW = 8, BWD_R = 4, BWD_NW = 8;
};

inline int pick_q(int64_t nvec) {
  int q = 1;
  while (q < 32 && q < nvec) q <<= 1;
  return q;
}

// Virtual T-segments: few channel columns make each look-back chain long and
// serial; splitting T into independent chains (stitched afterwards by a carry
// fold + fix-up, segment.cu) restores parallelism.  Aim for >= 64 chains
// (LINREC_CHAINS overrides for tuning), keeping >= 8 tiles per segment.
// Independent look-back chains wanted per launch (columns x virtual
// segments).  Measured on B200 (scripts/tune.py sweeps of 64-512 chains over
// W = 16 ... 8192): the forward scan is best at ~256 chains
// (C2 0.90 -> 0.96 of peak; W = 2048 0.78 -> 0.84; C4 / W = 16 within 1-2 %
// of their best), the backward -- 20 B/el per tile, so the look-back is
// already hidden -- at 64.  LINREC_CHAINS / LINREC_CHAINS_FWD /
// LINREC_CHAINS_BWD override.
inline bool chains_overridden() {
  static const bool any = std::getenv("LINREC_CHAINS") || std::getenv("LINREC_CHAINS_FWD") ||
                          std::getenv("LINREC_CHAINS_BWD");
  return any;
}

inline int64_t chain_target(bool forward) {
  static const long env_all = [] { const char* e = std::getenv("LINREC_CHAINS"); return e ? std::atol(e) : 0L; }();
  static const long env_fwd = [] { const char* e = std::getenv("LINREC_CHAINS_FWD"); return e ? std::atol(e) : 0L; }();
  static const long env_bwd = [] { const char* e = std::getenv("LINREC_CHAINS_BWD"); return e ? std::atol(e) : 0L; }();
  const long env = forward ? env_fwd : env_bwd;
  if (env > 0) return env;
  if (env_all > 0) return env_all;
  return forward ? 256 : 64;
}

// Chains shorter than this many tiles stay whole: below it the stitch (fold
// + fix-up launches) costs more than the look-back latency it removes
// (scripts/dev/split_sweep.py at W = 256 with the batched look-back apply:
// 64 tiles 29.1 us forward whole / 33.2 split, 86 tiles 31.7 / 34.3,
// 107 tiles 36.4 / 35.8, 128 tiles 39.5 / 36.5).
constexpr int64_t kMinSplitTiles = 96;

inline void choose_segments(ChainPlan& p, int64_t T, bool forward) {
  const int64_t ntt_total = (T + p.rows - 1) / p.rows;
  const int64_t target = chain_target(forward);
  int64_t nseg = (target + p.ncols - 1) / p.ncols;
  if (nseg > ntt_total / 8) nseg = ntt_total / 8;
  if (ntt_total < kMinSplitTiles && !chains_overridden()) nseg = 1;
  if (nseg < 1) nseg = 1;
  const int64_t per = (ntt_total + nseg - 1) / nseg;
  p.ntt = per;
  p.tseg = per * p.rows;
  p.nseg = (T + p.tseg - 1) / p.tseg;
  p.ntiles = p.ncols * p.nseg * p.ntt;
}

// Extra workspace of a virtually segmented launch: vagg [nseg][2][W] and the
// internal seg_prod [nseg*ntt][W] (capi.cpp::vseg_ptrs).
template <class S>
size_t vseg_bytes(const ChainPlan& p, int64_t W) {
  if (p.nseg <= 1) return 0;
  // vagg [nseg][2][W], seg_prod [nseg*ntt][W], carry [nseg][W] (adaptive stitch)
  return sizeof(S) * (size_t)W * (size_t)(3 * p.nseg + p.nseg * p.ntt) + 1024;
}

template <class S, int VEC, int Q, int R, int NW>
void fill_plan(ChainPlan& p, int64_t T, int64_t W, bool forward) {
  using Cfg = linrec_dev::ChainCfg<S, VEC, Q, R, NW>;
  p.vec = VEC; p.q = Q; p.r = R; p.nw = NW;
  p.cpw = Cfg::CPW; p.rows = Cfg::L; p.rec = Cfg::REC;
  p.ncols = (W + Cfg::CPW - 1) / Cfg::CPW;
  choose_segments(p, T, forward);
  p.flags_bytes = ((size_t)p.ntiles * 4 + 255) / 256 * 256;
  p.rec_bytes = (size_t)p.ntiles * 2 * Cfg::REC * 8;
  p.ws_bytes = 256 + p.flags_bytes + 2 * p.rec_bytes + vseg_bytes<S>(p, W);
}

#define LINREC_Q_SWITCH(QV, ...)                            \
  switch (QV) {                                             \
    case 1: { constexpr int Q_ = 1; __VA_ARGS__; } break;   \
    case 2: { constexpr int Q_ = 2; __VA_ARGS__; } break;   \
    case 4: { constexpr int Q_ = 4; __VA_ARGS__; } break;   \
    case 8: { constexpr int Q_ = 8; __VA_ARGS__; } break;   \
    case 16: { constexpr int Q_ = 16; __VA_ARGS__; } break; \
    default: { constexpr int Q_ = 32; __VA_ARGS__; } break; \
  }

inline linrec_dev::ChainWs to_dev(const ChainPtrs& w) {
  linrec_dev::ChainWs d;
  d.ctrl = reinterpret_cast<linrec_dev::Ctrl*>(w.ctrl);
  d.flags = reinterpret_cast<uint32_t*>(w.flags);
  d.agg = w.agg;
  d.inc = w.inc;
  return d;
}

template <class S, bool FWD>
ChainPlan plan_chain_dir(int64_t T, int64_t W, bool vec_ok) {
  using Tn = Tuning<S>;
  constexpr int R = FWD ? Tn::FWD_R : Tn::BWD_R;
  constexpr int NW = FWD ? Tn::FWD_NW : Tn::BWD_NW;
  ChainPlan p;
  if (vec_ok) {
    const int q = pick_q((W + Tn::VEC - 1) / Tn::VEC);
    LINREC_Q_SWITCH(q, fill_plan<S, Tn::VEC, Q_, R, NW>(p, T, W, FWD));
  } else {
    const int q = pick_q(W);
    LINREC_Q_SWITCH(q, fill_plan<S, 1, Q_, R, NW>(p, T, W, FWD));
  }
  return p;
}

}  // namespace linrec_impl
