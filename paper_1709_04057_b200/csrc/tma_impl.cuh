// Host-side planning and launch of the TMA-fed persistent scans.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "chain_impl.cuh"
#include "scan_tma.cuh"

namespace linrec_impl {

// (rows per thread, ring stages, consumer warps) of one TMA configuration.
struct TmaChoice {
  int r, stages, nw;
};

// Default configuration per dtype / direction / lane split (tuned on B200 at
// the C2 workload, profiles/); LINREC_TMA_FWD / LINREC_TMA_BWD ("R,STAGES,NW")
// override it for tuning runs when that triple is instantiated.
inline TmaChoice tma_choice(bool f64, bool fwd, int q) {
  TmaChoice c = fwd ? TmaChoice{12, 2, 8} : TmaChoice{12, 1, 8};
  if (f64) c = fwd ? TmaChoice{4, 3, 8} : TmaChoice{4, 2, 8};
  if (!f64) {
    const char* e = std::getenv(fwd ? "LINREC_TMA_FWD" : "LINREC_TMA_BWD");
    int r = 0, s = 0, nw = 8;
    if (e && std::sscanf(e, "%d,%d,%d", &r, &s, &nw) >= 2) c = TmaChoice{r, s, nw};
  }
  return c;
}

// Lanes across channels for the TMA kernels: as wide as W allows (128-bit
// vectors, up to 32 lanes); chain parallelism for narrow W comes from virtual
// T-segments (choose_segments).  LINREC_NARROW_COLUMNS=1 restores the older
// "at least 8 channel columns" rule for comparison.
inline int pick_q_tma(int64_t nvec) {
  if (const char* e = std::getenv("LINREC_NARROW_COLUMNS")) {
    if (std::atoi(e) > 0) {
      int q = pick_q(nvec);
      while (q > 4 && (nvec + q - 1) / q < 8) q >>= 1;
      return q;
    }
  }
  return pick_q(nvec);
}

inline int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

template <class Kern>
int tma_grid(Kern kern, int threads, int smem, long long ntiles) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  long long g = (long long)occ * sm_count();
  if (g > ntiles) g = ntiles;
  return (int)(g < 1 ? 1 : g);
}

template <class S, int VEC, int Q, int R, int NW, int STAGES, int NARR, class Kern>
void fill_tma_plan(ChainPlan& p, int64_t T, int64_t W, Kern kern) {
  using Cfg = linrec_dev::TmaCfg<S, VEC, Q, R, NW, STAGES, NARR>;
  p.kind = 1;
  p.vec = VEC; p.q = Q; p.r = R; p.nw = NW; p.stages = STAGES;
  p.cpw = Cfg::CPW; p.rows = Cfg::L; p.rec = Cfg::REC;
  p.box_cols = Cfg::CPW; p.box_rows = Cfg::BOX_ROWS;
  p.ncols = (W + Cfg::CPW - 1) / Cfg::CPW;
  choose_segments(p, T, NARR == 2);  // forward kernels stage 2 arrays, backward 3
  p.flags_bytes = ((size_t)p.ntiles * 4 + 255) / 256 * 256;
  p.rec_bytes = (size_t)p.ntiles * 2 * Cfg::REC * 8;
  p.ws_bytes = 256 + p.flags_bytes + 2 * p.rec_bytes + vseg_bytes<S>(p, W);
  p.threads = Cfg::THREADS;
  p.smem = Cfg::SMEM;
  p.grid = tma_grid(kern, Cfg::THREADS, Cfg::SMEM, p.ntiles);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
inline cudaError_t make_tmap_2d(CUtensorMap* map, const void* ptr, bool f64, int64_t W, int64_t T,
                                int box_cols, int box_rows) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<Fn>(f);
  }();
  if (!fn) return cudaErrorNotSupported;
  const size_t es = f64 ? 8 : 4;
  const cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)T};
  const cuuint64_t strides[1] = {(cuuint64_t)(W * es)};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                        const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <class S>
linrec_dev::ChainArgs<S> fwd_args(const ChainPlan& p, const FwdCall<S>& c) {
  linrec_dev::ChainArgs<S> a{};
  a.a = c.lam;
  a.b = c.x;
  a.seed = c.h0;
  a.out0 = c.h;
  a.seg_prod = c.seg_prod;
  a.agg_out = c.agg_out;
  a.T = c.T;
  a.W = c.W;
  a.ncols = p.ncols;
  a.ntt = p.ntt;
  a.nseg = p.nseg;
  a.tseg = p.tseg;
  a.tail_fold = c.rank_agg != nullptr ? 1 : 0;
  a.rank_agg = c.rank_agg;
  a.ex = c.ex;
  a.mode = c.mode;
  a.role = c.role;
  a.seed_rows = c.seed_rows;
  return a;
}

template <class S>
linrec_dev::ChainArgs<S> bwd_args(const ChainPlan& p, const BwdCall<S>& c) {
  linrec_dev::ChainArgs<S> a{};
  a.a = c.lam;
  a.b = c.dh;
  a.c = c.h;
  a.seed = c.g_next;
  a.aux = c.h0;
  a.lam_next = c.lam_next;
  a.out0 = c.dx;
  a.out1 = c.dlam;
  a.out2 = c.dh0;
  a.seg_prod = c.seg_prod;
  a.agg_out = c.agg_out;
  a.T = c.T;
  a.W = c.W;
  a.ncols = p.ncols;
  a.ntt = p.ntt;
  a.nseg = p.nseg;
  a.tseg = p.tseg;
  a.tail_fold = c.rank_agg != nullptr ? 1 : 0;
  a.rank_agg = c.rank_agg;
  a.ex = c.ex;
  a.mode = c.mode;
  a.role = c.role;
  a.seed_rows = c.seed_rows;
  return a;
}

// Instantiation tables: (Q, R, STAGES, NW) compiled for each direction; the
// first Q=32 rows are the defaults, the others tuning candidates.
#define LINREC_TMA_FWD_TABLE(X)                                                     \
  X(32, 12, 2, 8) X(32, 8, 2, 8) X(32, 16, 1, 8) X(32, 12, 1, 8) X(32, 10, 2, 8)       \
  X(16, 12, 2, 8) X(8, 12, 2, 8) X(4, 12, 2, 8) X(16, 8, 2, 8) X(8, 8, 2, 8) X(4, 8, 2, 8)
#define LINREC_TMA_BWD_TABLE(X)                                                     \
  X(32, 12, 1, 8) X(32, 8, 2, 8) X(32, 10, 1, 8) X(32, 16, 1, 8)                       \
  X(16, 12, 1, 8) X(8, 12, 1, 8) X(4, 12, 1, 8) X(16, 8, 2, 8) X(8, 8, 2, 8) X(4, 8, 2, 8)
#define LINREC_TMA_F64_FWD_TABLE(X) X(32, 4, 3, 8) X(16, 4, 3, 8) X(8, 4, 3, 8) X(4, 4, 3, 8)
#define LINREC_TMA_F64_BWD_TABLE(X) X(32, 4, 2, 8) X(16, 4, 2, 8) X(8, 4, 2, 8) X(4, 4, 2, 8)

}  // namespace linrec_impl
