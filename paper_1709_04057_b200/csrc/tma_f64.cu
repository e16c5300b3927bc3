// TMA-fed persistent scans, double (see scan_tma.cuh).
#include "tma_impl.cuh"

namespace linrec_impl {

#define FWD64(Q, R, ST, NW) linrec_dev::k_tma_fwd<double, 2, Q, R, NW, ST>
#define BWD64(Q, R, ST, NW) linrec_dev::k_tma_bwd<double, 2, Q, R, NW, ST>

template <>
cudaError_t launch_tma_fwd<double>(const ChainPlan& p, const FwdCall<double>& c, const ChainPtrs& w,
                                   cudaStream_t st) {
  CUtensorMap ml, mx;
  cudaError_t e;
  if ((e = make_tmap_2d(&ml, c.lam, true, c.W, c.T, p.box_cols, p.box_rows)) != cudaSuccess) return e;
  if ((e = make_tmap_2d(&mx, c.x, true, c.W, c.T, p.box_cols, p.box_rows)) != cudaSuccess) return e;
  const auto a = fwd_args<double>(p, c);
  const auto d = to_dev(w);
#define X(Q, R, ST, NW)                                                            \
  if (p.q == Q && p.r == R && p.stages == ST && p.nw == NW) {                                \
    FWD64(Q, R, ST, NW)<<<p.grid, p.threads, p.smem, st>>>(ml, mx, a, d, p.ntiles); \
    return cudaGetLastError();                                                 \
  }
  LINREC_TMA_F64_FWD_TABLE(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

template <>
cudaError_t launch_tma_bwd<double>(const ChainPlan& p, const BwdCall<double>& c, const ChainPtrs& w,
                                   cudaStream_t st) {
  CUtensorMap ml, md, mh;
  cudaError_t e;
  if ((e = make_tmap_2d(&ml, c.lam, true, c.W, c.T, p.box_cols, p.box_rows)) != cudaSuccess) return e;
  if ((e = make_tmap_2d(&md, c.dh, true, c.W, c.T, p.box_cols, p.box_rows)) != cudaSuccess) return e;
  if ((e = make_tmap_2d(&mh, c.h, true, c.W, c.T, p.box_cols, p.box_rows)) != cudaSuccess) return e;
  const auto a = bwd_args<double>(p, c);
  const auto d = to_dev(w);
#define X(Q, R, ST, NW)                                                                \
  if (p.q == Q && p.r == R && p.stages == ST && p.nw == NW) {                                    \
    BWD64(Q, R, ST, NW)<<<p.grid, p.threads, p.smem, st>>>(ml, md, mh, md, a, d, p.ntiles); \
    return cudaGetLastError();                                                     \
  }
  LINREC_TMA_F64_BWD_TABLE(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

template <>
bool plan_tma<double>(bool forward, int64_t T, int64_t W, ChainPlan* p) {
  const int q = pick_q_tma(W / 2);
  if (q < 4) return false;
  const TmaChoice ch = tma_choice(true, forward, q);
  if (forward) {
#define X(Q, R, ST, NW)                                                                  \
    if (q == Q && ch.r == R && ch.stages == ST && ch.nw == NW) {                                    \
      fill_tma_plan<double, 2, Q, R, NW, ST, 2>(*p, T, W, FWD64(Q, R, ST, NW));           \
      return true;                                                                   \
    }
    LINREC_TMA_F64_FWD_TABLE(X)
#undef X
  } else {
#define X(Q, R, ST, NW)                                                                  \
    if (q == Q && ch.r == R && ch.stages == ST && ch.nw == NW) {                                    \
      fill_tma_plan<double, 2, Q, R, NW, ST, 3>(*p, T, W, BWD64(Q, R, ST, NW));           \
      return true;                                                                   \
    }
    LINREC_TMA_F64_BWD_TABLE(X)
#undef X
  }
  return false;
}

}  // namespace linrec_impl
