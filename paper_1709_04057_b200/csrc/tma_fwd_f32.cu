// TMA-fed persistent forward scan, float (see scan_tma.cuh).
#include "tma_impl.cuh"

namespace linrec_impl {

#define FWD_KERN(Q, R, ST, NW) linrec_dev::k_tma_fwd<float, 4, Q, R, NW, ST>

template <>
cudaError_t launch_tma_fwd<float>(const ChainPlan& p, const FwdCall<float>& c, const ChainPtrs& w,
                                  cudaStream_t st) {
  CUtensorMap ml, mx;
  cudaError_t e;
  if ((e = make_tmap_2d(&ml, c.lam, false, c.W, c.T, p.box_cols, p.box_rows)) != cudaSuccess) return e;
  if ((e = make_tmap_2d(&mx, c.x, false, c.W, c.T, p.box_cols, p.box_rows)) != cudaSuccess) return e;
  const auto a = fwd_args<float>(p, c);
  const auto d = to_dev(w);
#define X(Q, R, ST, NW)                                                              \
  if (p.q == Q && p.r == R && p.stages == ST && p.nw == NW) {                                  \
    FWD_KERN(Q, R, ST, NW)<<<p.grid, p.threads, p.smem, st>>>(ml, mx, a, d, p.ntiles); \
    return cudaGetLastError();                                                   \
  }
  LINREC_TMA_FWD_TABLE(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

// forward planning for float lives here (the kernel pointers are needed for
// the occupancy query); the backward planning is in tma_bwd_f32.cu.
bool plan_tma_fwd_f32(int64_t T, int64_t W, ChainPlan* p) {
  const int q = pick_q_tma(W / 4);
  if (q < 4) return false;
  const TmaChoice ch = tma_choice(false, true, q);
#define X(Q, R, ST, NW)                                                                  \
  if (q == Q && ch.r == R && ch.stages == ST && ch.nw == NW) {                                      \
    fill_tma_plan<float, 4, Q, R, NW, ST, 2>(*p, T, W, FWD_KERN(Q, R, ST, NW));           \
    return true;                                                                     \
  }
  LINREC_TMA_FWD_TABLE(X)
#undef X
  return false;
}

}  // namespace linrec_impl
