// Chained reverse-time backward scan, float instantiations (see scan_chained.cuh).
#include "chain_impl.cuh"

namespace linrec_impl {

template <>
cudaError_t launch_chain_bwd<float>(const ChainPlan& p, const BwdCall<float>& c,
                                  const ChainPtrs& w, cudaStream_t st) {
  using S = float;
  using Tn = Tuning<S>;
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
  const linrec_dev::ChainWs d = to_dev(w);
  const dim3 grid((unsigned)p.ntiles), block((Tn::BWD_NW + 1) * 32);
  if (p.vec == Tn::VEC) {
    LINREC_Q_SWITCH(p.q, linrec_dev::k_chain_bwd<S, Tn::VEC, Q_, Tn::BWD_R, Tn::BWD_NW><<<grid, block, 0, st>>>(a, d));
  } else {
    LINREC_Q_SWITCH(p.q, linrec_dev::k_chain_bwd<S, 1, Q_, Tn::BWD_R, Tn::BWD_NW><<<grid, block, 0, st>>>(a, d));
  }
  return cudaGetLastError();
}

}  // namespace linrec_impl
