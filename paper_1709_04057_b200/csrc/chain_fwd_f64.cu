// Chained forward scan, double instantiations (see scan_chained.cuh).
#include "chain_impl.cuh"

namespace linrec_impl {

template <>
cudaError_t launch_chain_fwd<double>(const ChainPlan& p, const FwdCall<double>& c,
                                  const ChainPtrs& w, cudaStream_t st) {
  using S = double;
  using Tn = Tuning<S>;
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
  const linrec_dev::ChainWs d = to_dev(w);
  const dim3 grid((unsigned)p.ntiles), block((Tn::FWD_NW + 1) * 32);
  if (p.vec == Tn::VEC) {
    LINREC_Q_SWITCH(p.q, linrec_dev::k_chain_fwd<S, Tn::VEC, Q_, Tn::FWD_R, Tn::FWD_NW><<<grid, block, 0, st>>>(a, d));
  } else {
    LINREC_Q_SWITCH(p.q, linrec_dev::k_chain_fwd<S, 1, Q_, Tn::FWD_R, Tn::FWD_NW><<<grid, block, 0, st>>>(a, d));
  }
  return cudaGetLastError();
}

}  // namespace linrec_impl
