// TMA-fed persistent backward scan, float (see scan_tma.cuh).
#include "tma_impl.cuh"

namespace linrec_impl {

#define BWD_KERN(Q, R, ST, NW) linrec_dev::k_tma_bwd<float, 4, Q, R, NW, ST>

template <>
cudaError_t launch_tma_bwd<float>(const ChainPlan& p, const BwdCall<float>& c, const ChainPtrs& w,
                                  cudaStream_t st) {
  CUtensorMap ml, md, mh;
  cudaError_t e;
  if ((e = make_tmap_2d(&ml, c.lam, false, c.W, c.T, p.box_cols, p.box_rows)) != cudaSuccess) return e;
  if ((e = make_tmap_2d(&md, c.dh, false, c.W, c.T, p.box_cols, p.box_rows)) != cudaSuccess) return e;
  if ((e = make_tmap_2d(&mh, c.h, false, c.W, c.T, p.box_cols, p.box_rows)) != cudaSuccess) return e;
  const auto a = bwd_args<float>(p, c);
  const auto d = to_dev(w);
  if (c.gate != nullptr) {  // gated adjoint: the default configuration only (capi falls back otherwise)
    using GCfg = linrec_dev::TmaCfg<float, 4, 32, 12, 8, 1, 4>;
    auto kern = linrec_dev::k_tma_bwd<float, 4, 32, 12, 8, 1, true>;
    if (!(p.q == 32 && p.r == 12 && p.stages == 1 && p.nw == 8)) return cudaErrorNotSupported;
    const cudaError_t attr = func_attr_once(reinterpret_cast<const void*>(kern),
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, GCfg::SMEM);
    if (attr != cudaSuccess) return attr;
    CUtensorMap mg;
    if ((e = make_tmap_2d(&mg, c.gate, false, c.W, c.T, p.box_cols, p.box_rows)) != cudaSuccess) return e;
    kern<<<p.grid, p.threads, GCfg::SMEM, st>>>(ml, md, mh, mg, a, d, p.ntiles);
    return cudaGetLastError();
  }
#define X(Q, R, ST, NW)                                                                  \
  if (p.q == Q && p.r == R && p.stages == ST && p.nw == NW) {                                      \
    BWD_KERN(Q, R, ST, NW)<<<p.grid, p.threads, p.smem, st>>>(ml, md, mh, md, a, d, p.ntiles); \
    return cudaGetLastError();                                                       \
  }
  LINREC_TMA_BWD_TABLE(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

bool plan_tma_fwd_f32(int64_t T, int64_t W, ChainPlan* p);

template <>
bool plan_tma<float>(bool forward, int64_t T, int64_t W, ChainPlan* p) {
  if (forward) return plan_tma_fwd_f32(T, W, p);
  const int q = pick_q_tma(W / 4);
  if (q < 4) return false;
  const TmaChoice ch = tma_choice(false, false, q);
#define X(Q, R, ST, NW)                                                                  \
  if (q == Q && ch.r == R && ch.stages == ST && ch.nw == NW) {                                      \
    fill_tma_plan<float, 4, Q, R, NW, ST, 3>(*p, T, W, BWD_KERN(Q, R, ST, NW));           \
    return true;                                                                     \
  }
  LINREC_TMA_BWD_TABLE(X)
#undef X
  return false;
}

}  // namespace linrec_impl
